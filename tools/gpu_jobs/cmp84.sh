# the paper's comparison on the final pipeline: conv (halo lines now in the space) and 1024^3
mkdir -p gpurun_out/cmp_conv gpurun_out/cmp_mm1024_final
timeout 1500 python -m paper_2006_05664_b200 compare --operator conv2d:32,64,56,56,64,3,3,1,1 --seeds 0,1,2 --budget 300 --out gpurun_out/cmp_conv > gpurun_out/cmp_conv/stdout.txt 2>&1
cat gpurun_out/cmp_conv/stdout.txt
timeout 1500 python -m paper_2006_05664_b200 compare --operator matmul:1024,1024,1024 --seeds 0,1,2 --budget 300 --out gpurun_out/cmp_mm1024_final > gpurun_out/cmp_mm1024_final/stdout.txt 2>&1
cat gpurun_out/cmp_mm1024_final/stdout.txt
