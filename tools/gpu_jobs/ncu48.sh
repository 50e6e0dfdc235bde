# round1_c ncu evidence: launch list of a short bench (shares) + full captures of the best kernels
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
export OPEVO_LINEINFO=1
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/c_mm1024 python tools/profile_kernel.py matmul:1024,1024,1024 128,64,128,4,1,1 > /dev/null 2>&1
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/c_mm4096 python tools/profile_kernel.py matmul:4096,4096,4096 256,256,64,6,1,1,1,1,1,2 > /dev/null 2>&1
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/c_conv python tools/profile_kernel.py conv2d:32,64,56,56,64,3,3,1,1 256,64,64,4,1,1,4,4 > /dev/null 2>&1
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/c_bmm python tools/profile_kernel.py batchmatmul:960,128,64,128 128,64,128,3,1,1 > /dev/null 2>&1
unset OPEVO_LINEINFO
OPEVO_NO_POOL=1 timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file gpurun_out/c_launches.csv python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu > gpurun_out/c_bench_under_ncu.log 2>&1
ls -la gpurun_out | grep " c_"
