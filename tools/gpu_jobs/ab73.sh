mkdir -p gpurun_out
timeout 900 python tools/ablate.py batchmatmul:960,128,64,128@128,64,64,6,1,1 conv2d:32,64,56,56,64,3,3,1,1@128,64,64,4,1,1,4,14 matmul:1024,1024,1024@128,64,128,4,1,1 > gpurun_out/ab73.txt 2>&1; cat gpurun_out/ab73.txt
