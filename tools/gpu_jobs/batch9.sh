mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 300 python tools/trial_cost.py matmul:1024,1024,1024 40 > gpurun_out/b9_trial_cost.txt 2>&1; cat gpurun_out/b9_trial_cost.txt
timeout 900 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider -k "batch or timing or scheduler or smoke or log_replay" > gpurun_out/b9_pytest_gpu.txt 2>&1; tail -3 gpurun_out/b9_pytest_gpu.txt
timeout 600 python bench.py --no-cpu > gpurun_out/b9_bench.json 2> gpurun_out/b9_bench.err; cat gpurun_out/b9_bench.json; tail -3 gpurun_out/b9_bench.err
