mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 1200 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/x3_52_pytest.txt 2>&1; tail -3 gpurun_out/x3_52_pytest.txt
timeout 600 python bench.py --op matmul:512,1024,1024 --dtype tf32x3 --no-cpu > gpurun_out/x3_52_bench_tf32x3.json 2> gpurun_out/x3_52_bench_tf32x3.err; tail -c 1500 gpurun_out/x3_52_bench_tf32x3.json
timeout 900 python bench.py --op matmul:512,1024,1024 --dtype f32 --no-cpu --no-e2e > gpurun_out/x3_52_bench_f32.json 2> gpurun_out/x3_52_bench_f32.err; tail -c 600 gpurun_out/x3_52_bench_f32.json
timeout 600 python bench.py > gpurun_out/x3_52_bench_default.json 2> gpurun_out/x3_52_bench_default.err; tail -c 600 gpurun_out/x3_52_bench_default.json
