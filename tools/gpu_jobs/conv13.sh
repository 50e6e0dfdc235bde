mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
C=conv2d:32,64,56,56,64,3,3,1,1
timeout 300 python tools/trace_kernel.py $C 128,64,64,6,1,1,8,8 2 > gpurun_out/c13_trace_conv.txt 2>&1; cat gpurun_out/c13_trace_conv.txt
timeout 300 python tools/trace_kernel.py batchmatmul:960,128,64,128 128,64,64,8,1,1 2 > gpurun_out/c13_trace_bmm.txt 2>&1; cat gpurun_out/c13_trace_bmm.txt
timeout 600 python tools/sweep.py $C --grid "128;64,32;64,32;4,6,8;1;1;8,4,2;8,4" > gpurun_out/c13_sweep_conv.txt 2>&1; head -15 gpurun_out/c13_sweep_conv.txt
timeout 600 python tools/sweep.py batchmatmul:960,128,64,128 --grid "128;64,32;64,128;4,6,8;1;1;1;1" > gpurun_out/c13_sweep_bmm.txt 2>&1; head -10 gpurun_out/c13_sweep_bmm.txt
