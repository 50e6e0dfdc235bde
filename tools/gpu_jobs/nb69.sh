# 4 TMEM accumulator buffers (persistent BMM / conv), compiled on the box (fresh source hash)
mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 300 python tools/timing_modes.py batchmatmul:960,128,64,128 128,64,64,6,1,1 128,64,128,3,1,1 128,64,64,8,1,1 > gpurun_out/nb69_modes.txt 2>&1
timeout 300 python tools/timing_modes.py conv2d:32,64,56,56,64,3,3,1,1 128,64,64,4,1,1,8,14 256,64,64,4,1,1,8,8 >> gpurun_out/nb69_modes.txt 2>&1
timeout 300 python tools/timing_modes.py matmul:1024,1024,1024 128,64,128,4,1,1 >> gpurun_out/nb69_modes.txt 2>&1
grep TF gpurun_out/nb69_modes.txt
timeout 600 python tools/ablate.py batchmatmul:960,128,64,128@128,64,64,8,1,1 > gpurun_out/nb69_ablate.txt 2>&1; cat gpurun_out/nb69_ablate.txt
