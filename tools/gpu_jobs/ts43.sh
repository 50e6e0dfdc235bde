mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider > gpurun_out/t43_pytest.txt 2>&1; tail -3 gpurun_out/t43_pytest.txt
timeout 300 python tools/timing_modes.py matmul:1024,1024,1024 128,64,128,4,1,1 128,128,64,4,2,1 128,128,128,3,2,1 128,128,64,6,2,1 128,128,128,2,2,1 128,256,64,3,2,1 128,128,64,4,4,1 > gpurun_out/t43_modes.txt 2>&1; cat gpurun_out/t43_modes.txt
