# microbenchmarks + phase trace + bench trial log
mkdir -p gpurun_out
timeout 120 ./tools/bin/microbench > gpurun_out/microbench.txt 2>&1
timeout 120 python tools/trace_kernel.py matmul:1024,1024,1024 128,64,128,3,1,1 > gpurun_out/trace_128x64.txt 2>&1
timeout 120 python tools/trace_kernel.py matmul:1024,1024,1024 128,128,128,3,1,1 > gpurun_out/trace_128x128.txt 2>&1
timeout 120 python tools/trace_kernel.py matmul:1024,1024,1024 256,128,128,4,1,1,1,1,1,2 > gpurun_out/trace_pair256x128.txt 2>&1
timeout 600 python bench.py --no-cpu --no-e2e --log gpurun_out/bench_log.jsonl > gpurun_out/bench_p2.json 2>&1
cat gpurun_out/microbench.txt gpurun_out/trace_*.txt
