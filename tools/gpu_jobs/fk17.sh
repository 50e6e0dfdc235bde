mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider > gpurun_out/f17_pytest.txt 2>&1; tail -3 gpurun_out/f17_pytest.txt
timeout 300 python tools/timing_modes.py matmul:1024,1024,1024 128,64,128,3,1,1 128,64,128,4,1,1 128,64,256,2,1,1 128,128,128,3,1,1 256,64,128,4,1,1,1,1,1,2 256,128,128,3,1,1,1,1,1,2 > gpurun_out/f17_modes.txt 2>&1
timeout 300 python tools/timing_modes.py batchmatmul:960,128,64,128 128,64,64,8,1,1 128,64,128,4,1,1 >> gpurun_out/f17_modes.txt 2>&1
timeout 300 python tools/timing_modes.py matmul:4096,4096,4096 256,256,64,6,1,1,1,1,1,2 256,256,128,3,1,1,1,1,1,2 >> gpurun_out/f17_modes.txt 2>&1
cat gpurun_out/f17_modes.txt
timeout 120 python tools/trace_kernel.py matmul:1024,1024,1024 128,64,128,3,1,1 4 > gpurun_out/f17_trace.txt 2>&1; grep -E "mainloop|first stage|steady" gpurun_out/f17_trace.txt
