# multi-GPU evidence on one GPU: projected 1/2/4/8 scaling (trial sharding replayed per rank) and a
# 2-rank torchrun of bench.py with the gloo test backend (both ranks share the one GPU)
mkdir -p gpurun_out/sc77
make -s -C paper_2006_05664_b200/csrc
timeout 900 python tools/scaling_projection.py matmul:1024,1024,1024 40 > gpurun_out/sc77/projection_mm1024.txt 2>&1; grep "N=" gpurun_out/sc77/projection_mm1024.txt
timeout 900 python tools/scaling_projection.py matmul:4096,4096,4096 20 > gpurun_out/sc77/projection_mm4096.txt 2>&1; grep "N=" gpurun_out/sc77/projection_mm4096.txt
OPEVO_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu > gpurun_out/sc77/bench_n2_gloo_shared_gpu.json 2> gpurun_out/sc77/n2_err.txt; tail -c 400 gpurun_out/sc77/bench_n2_gloo_shared_gpu.json
