mkdir -p gpurun_out
S="python tools/sweep.py matmul:1024,1024,1024"
timeout 900 $S --grid "128;32,64,96,128;256;1,2,3;1;1;1;1;1;1" > gpurun_out/s7_bk256.txt 2>&1; head -12 gpurun_out/s7_bk256.txt
timeout 900 $S --grid "256;64,128;256;1,2,3;1;1;1;1;1;2" > gpurun_out/s7_pair256.txt 2>&1; head -8 gpurun_out/s7_pair256.txt
timeout 120 python tools/trace_kernel.py matmul:1024,1024,1024 128,64,256,2,1,1 4 > gpurun_out/s7_trace.txt 2>&1; cat gpurun_out/s7_trace.txt
