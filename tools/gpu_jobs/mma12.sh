mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 300 python tools/timing_modes.py matmul:1024,1024,1024 128,64,128,3,1,1 128,64,128,4,1,1 128,64,64,6,1,1 128,128,128,3,1,1 256,64,128,4,1,1,1,1,1,2 256,64,64,8,1,1,1,1,1,2 256,64,64,10,1,1,1,1,1,2 256,128,64,6,1,1,1,1,1,2 > gpurun_out/m12_modes.txt 2>&1
cat gpurun_out/m12_modes.txt
timeout 120 python tools/trace_kernel.py matmul:1024,1024,1024 128,64,128,3,1,1 4 > gpurun_out/m12_trace.txt 2>&1; cat gpurun_out/m12_trace.txt
