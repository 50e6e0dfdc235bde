mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 300 python tools/gen_breakdown.py matmul:1024,1024,1024 60 > gpurun_out/gb58.txt 2>&1; cat gpurun_out/gb58.txt
OPEVO_PROFILE_BATCH=1 timeout 300 python tools/gen_breakdown.py matmul:1024,1024,1024 30 > gpurun_out/gb58_c.txt 2>&1; tail -12 gpurun_out/gb58_c.txt
