# tf32x3 evidence: ncu full capture of the best MM1 fp32 instance, GPU suite, bench lines
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
make -s -C paper_2006_05664_b200/csrc
timeout 1200 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/f55_pytest.txt 2>&1; tail -3 gpurun_out/f55_pytest.txt
OPEVO_LINEINFO=1 timeout 300 $NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/f55_x3_mm1 python tools/profile_kernel.py matmul:512,1024,1024 128,64,64,2,2 5 --tf32x3 > gpurun_out/f55_x3_prof.txt 2>&1; tail -2 gpurun_out/f55_x3_prof.txt
timeout 600 python bench.py --op matmul:512,1024,1024 --dtype tf32x3 > gpurun_out/f55_bench_tf32x3.json 2> gpurun_out/f55_bench_tf32x3.err; tail -c 300 gpurun_out/f55_bench_tf32x3.json
timeout 600 python bench.py > gpurun_out/f55_bench.json 2> gpurun_out/f55_bench.err; tail -c 600 gpurun_out/f55_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/f55_bench_ref.json 2> gpurun_out/f55_bench_ref.err; tail -c 600 gpurun_out/f55_bench_ref.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f55_smoke.txt 2>&1; tail -2 gpurun_out/f55_smoke.txt
