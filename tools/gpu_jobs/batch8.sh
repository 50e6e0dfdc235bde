mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/b8_pytest_gpu.txt 2>&1; tail -5 gpurun_out/b8_pytest_gpu.txt
timeout 600 python bench.py --no-cpu > gpurun_out/b8_bench.json 2> gpurun_out/b8_bench.err; cat gpurun_out/b8_bench.json; tail -3 gpurun_out/b8_bench.err
