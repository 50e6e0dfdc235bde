mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider > gpurun_out/e15_pytest.txt 2>&1; tail -3 gpurun_out/e15_pytest.txt
timeout 600 python tools/ablate.py conv2d:32,64,56,56,64,3,3,1,1@128,64,64,6,1,1,8,8 batchmatmul:960,128,64,128@128,64,64,8,1,1 matmul:1024,1024,1024@128,64,128,3,1,1 > gpurun_out/e15_ablate.txt 2>&1; cat gpurun_out/e15_ablate.txt
