mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
M=matmul:1024,1024,1024
timeout 300 python tools/timing_modes.py $M 128,64,128,4,1,1 128,64,64,2,1,1 128,64,64,3,1,1 128,64,64,4,1,1 128,64,32,6,1,1 128,64,128,2,1,1 128,32,128,3,1,1 128,32,64,4,1,1 > gpurun_out/co50_modes.txt 2>&1; cat gpurun_out/co50_modes.txt
timeout 120 python tools/trace_kernel.py $M 128,64,64,3,1,1 4 > gpurun_out/co50_trace.txt 2>&1; tail -7 gpurun_out/co50_trace.txt
timeout 120 python tools/trace_kernel.py $M 128,64,128,4,1,1 4 >> gpurun_out/co50_trace.txt 2>&1; tail -7 gpurun_out/co50_trace.txt
