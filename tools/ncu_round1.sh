set -x
export OPEVO_LINEINFO=1
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/prof_mm1024_best python tools/profile_kernel.py matmul:1024,1024,1024 128,64,256,2,1,1 > gpurun_out/ncu_full_1024.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/prof_mm4096_best python tools/profile_kernel.py matmul:4096,4096,4096 256,256,64,3,1,1 > gpurun_out/ncu_full_4096.log 2>&1
unset OPEVO_LINEINFO
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
python - <<'PY' > gpurun_out/cublas_1024.txt 2>&1
import torch
a = torch.randn(1024, 1024, device="cuda", dtype=torch.bfloat16)
b = torch.randn(1024, 1024, device="cuda", dtype=torch.bfloat16)
for _ in range(20): torch.matmul(a, b.t())
torch.cuda.synchronize()
PY
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__cluster_dim_x,launch__block_size,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv -s 10 -c 3 python -c "
import torch
a = torch.randn(1024, 1024, device='cuda', dtype=torch.bfloat16)
b = torch.randn(1024, 1024, device='cuda', dtype=torch.bfloat16)
for _ in range(20): torch.matmul(a, b.t())
torch.cuda.synchronize()
" > gpurun_out/ncu_cublas_1024.csv 2>&1
ls -la gpurun_out
