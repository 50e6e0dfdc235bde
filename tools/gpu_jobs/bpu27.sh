mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider > gpurun_out/u27_pytest.txt 2>&1; tail -3 gpurun_out/u27_pytest.txt
timeout 300 python tools/timing_modes.py batchmatmul:960,128,64,128 128,64,128,3,1,1 128,64,128,2,1,1,1,1,1,1,0,0,2 128,64,64,4,1,1,1,1,1,1,0,0,2 128,64,64,2,1,1,1,1,1,1,0,0,4 128,64,32,4,1,1,1,1,1,1,0,0,4 128,64,32,3,1,1,1,1,1,1,0,0,4 > gpurun_out/u27_modes.txt 2>&1; cat gpurun_out/u27_modes.txt
