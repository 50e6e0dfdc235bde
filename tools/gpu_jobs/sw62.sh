mkdir -p gpurun_out
[ -x tools/bin/swizzle_probe ] || nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/swizzle_probe tools/swizzle_probe.cu
timeout 120 tools/bin/swizzle_probe > gpurun_out/sw62.txt 2>&1; cat gpurun_out/sw62.txt
