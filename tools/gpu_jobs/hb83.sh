mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "conv2d" > gpurun_out/hb83_pytest.txt 2>&1; tail -3 gpurun_out/hb83_pytest.txt
C=conv2d:32,64,56,56,64,3,3,1,1
timeout 300 python tools/timing_modes.py $C 128,64,64,4,1,1,4,14 128,64,64,4,1,1,8,14 256,64,64,3,1,1,8,14 256,64,64,4,1,1,8,8 2>&1 | grep TF
timeout 120 python tools/trace_units.py $C 128,64,64,4,1,1,4,14
