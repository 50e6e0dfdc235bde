mkdir -p gpurun_out
B=batchmatmul:960,128,64,128
C=conv2d:32,64,56,56,64,3,3,1,1
timeout 120 python tools/trace_units.py $B 128,64,64,6,1,1 > gpurun_out/ut79.txt 2>&1
OPEVO_ABLATE_FLAG=-DOPEVO_ABLATE=7 timeout 120 python tools/trace_units.py $B 128,64,64,6,1,1 >> gpurun_out/ut79.txt 2>&1
timeout 120 python tools/trace_units.py $C 128,64,64,4,1,1,4,14 >> gpurun_out/ut79.txt 2>&1
OPEVO_ABLATE_FLAG=-DOPEVO_ABLATE=7 timeout 120 python tools/trace_units.py $C 128,64,64,4,1,1,4,14 >> gpurun_out/ut79.txt 2>&1
cat gpurun_out/ut79.txt
