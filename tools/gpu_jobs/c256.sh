mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "conv" > gpurun_out/c24_pytest.txt 2>&1; tail -3 gpurun_out/c24_pytest.txt
timeout 300 python tools/timing_modes.py conv2d:32,64,56,56,64,3,3,1,1 128,64,64,4,1,1,8,8,1,1,0,1 256,64,64,4,1,1,8,8 256,64,64,3,1,1,8,8,1,1,0,1 256,64,64,5,1,1,8,8 256,64,64,3,1,1,8,4,1,1,0,1 256,64,64,3,1,1,4,8,1,1,0,1 > gpurun_out/c24_modes.txt 2>&1; cat gpurun_out/c24_modes.txt
