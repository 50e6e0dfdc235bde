mkdir -p gpurun_out/cmp_mm1024 gpurun_out/cmp_mm4096
timeout 1500 python -m paper_2006_05664_b200 compare --operator matmul:1024,1024,1024 --seeds 0,1,2 --budget 300 --out gpurun_out/cmp_mm1024 > gpurun_out/cmp_mm1024/stdout.txt 2>&1
cat gpurun_out/cmp_mm1024/stdout.txt
timeout 1500 python -m paper_2006_05664_b200 compare --operator matmul:4096,4096,4096 --seeds 0,1 --budget 200 --out gpurun_out/cmp_mm4096 > gpurun_out/cmp_mm4096/stdout.txt 2>&1
cat gpurun_out/cmp_mm4096/stdout.txt
