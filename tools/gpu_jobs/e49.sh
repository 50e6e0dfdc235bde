mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/e49_pytest.txt 2>&1; tail -3 gpurun_out/e49_pytest.txt
timeout 300 python tools/timing_modes.py matmul:1024,1024,1024 128,64,128,4,1,1 128,128,128,3,1,1 > gpurun_out/e49_modes.txt 2>&1
timeout 300 python tools/timing_modes.py batchmatmul:960,128,64,128 128,64,128,3,1,1 128,64,64,6,1,1 >> gpurun_out/e49_modes.txt 2>&1
timeout 300 python tools/timing_modes.py conv2d:32,64,56,56,64,3,3,1,1 256,64,64,4,1,1,4,4 256,64,64,4,1,1,8,8 >> gpurun_out/e49_modes.txt 2>&1
timeout 300 python tools/timing_modes.py matmul:4096,4096,4096 256,256,64,6,1,1,1,1,1,2 256,128,128,4,1,1,1,1,1,2 >> gpurun_out/e49_modes.txt 2>&1
grep TF gpurun_out/e49_modes.txt
