mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "halo or conv2d_parity" > gpurun_out/halo63_pytest.txt 2>&1; tail -15 gpurun_out/halo63_pytest.txt
C=conv2d:32,64,56,56,64,3,3,1,1
timeout 300 python tools/timing_modes.py $C 256,64,64,4,1,1,8,8 128,64,64,4,1,1,8,14 128,64,64,4,1,1,8,14,1,1,0,1 256,64,64,3,1,1,8,14 256,64,64,3,1,1,8,14,1,1,0,1 128,64,64,6,1,1,8,14,1,1,0,1 256,64,64,4,1,1,4,14,1,1,0,1 > gpurun_out/halo63_modes.txt 2>&1; cat gpurun_out/halo63_modes.txt
