mkdir -p gpurun_out
for r in 1 2; do
(cd ab_old && timeout 300 python tools/timing_modes.py matmul:1024,1024,1024 128,64,128,4,1,1 128,64,128,3,1,1 2>&1 | sed 's/^/OLD /')
timeout 300 python tools/timing_modes.py matmul:1024,1024,1024 128,64,128,4,1,1 128,64,128,3,1,1 2>&1 | sed 's/^/NEW /'
done
