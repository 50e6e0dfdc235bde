mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
export OPEVO_LINEINFO=1
NCU=/usr/local/cuda/bin/ncu
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/n11_mm1024_128x64 python tools/profile_kernel.py matmul:1024,1024,1024 128,64,128,3,1,1 > gpurun_out/n11_a.log 2>&1
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/n11_mm1024_pair256x64 python tools/profile_kernel.py matmul:1024,1024,1024 256,64,128,4,1,1,1,1,1,2 > gpurun_out/n11_b.log 2>&1
timeout 300 $NCU --set full --clock-control none -k regex:nvjet -s 10 -c 1 -o gpurun_out/n11_cublas1024 python -c "
import torch
a = torch.randn(1024, 1024, device='cuda', dtype=torch.bfloat16)
b = torch.randn(1024, 1024, device='cuda', dtype=torch.bfloat16)
for _ in range(20): torch.matmul(a, b.t())
torch.cuda.synchronize()
" > gpurun_out/n11_c.log 2>&1
unset OPEVO_LINEINFO
timeout 600 python tools/profile_bench.py matmul:1024,1024,1024 40 > gpurun_out/n11_profile_bench.txt 2>&1
head -40 gpurun_out/n11_profile_bench.txt
ls -la gpurun_out/ | grep n11
