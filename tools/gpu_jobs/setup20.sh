mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider > gpurun_out/s20_pytest.txt 2>&1; tail -3 gpurun_out/s20_pytest.txt
timeout 300 python tools/timing_modes.py matmul:1024,1024,1024 128,64,128,3,1,1 128,64,128,4,1,1 256,64,128,4,1,1,1,1,1,2 256,64,128,3,1,1,1,1,1,2 256,128,128,3,1,1,1,1,1,2 > gpurun_out/s20_modes.txt 2>&1; cat gpurun_out/s20_modes.txt
timeout 120 python tools/trace_kernel.py matmul:1024,1024,1024 256,64,128,4,1,1,1,1,1,2 4 > gpurun_out/s20_trace.txt 2>&1; tail -9 gpurun_out/s20_trace.txt
timeout 120 python tools/trace_kernel.py matmul:1024,1024,1024 128,64,128,3,1,1 4 >> gpurun_out/s20_trace.txt 2>&1; tail -7 gpurun_out/s20_trace.txt
