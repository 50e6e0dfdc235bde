mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "conv" > gpurun_out/r21_pytest.txt 2>&1; tail -3 gpurun_out/r21_pytest.txt
timeout 300 python tools/timing_modes.py conv2d:32,64,56,56,64,3,3,1,1 128,64,64,6,1,1,8,8 128,64,64,4,1,1,8,8,1,1,0,1 128,64,64,3,1,1,8,8,1,1,0,1 128,64,64,4,1,1,4,8,1,1,0,1 128,64,64,4,1,1,8,4,1,1,0,1 128,64,64,4,1,1,2,8,1,1,0,1 > gpurun_out/r21_modes.txt 2>&1; cat gpurun_out/r21_modes.txt
timeout 600 python tools/ablate.py conv2d:32,64,56,56,64,3,3,1,1@128,64,64,4,1,1,8,8,1,1,0,1 > gpurun_out/r21_ablate.txt 2>&1; cat gpurun_out/r21_ablate.txt
