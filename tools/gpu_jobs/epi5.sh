mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/e5_pytest_gpu.txt 2>&1; tail -5 gpurun_out/e5_pytest_gpu.txt
timeout 300 python tools/trial_cost.py matmul:1024,1024,1024 40 > gpurun_out/e5_trial_cost.txt 2>&1; cat gpurun_out/e5_trial_cost.txt
S="python tools/sweep.py matmul:1024,1024,1024"
timeout 600 $S --grid "128;64,128;64,128;2,3,4,6;1;1;1;1;1;1" > gpurun_out/e5_sw_single.txt 2>&1; head -12 gpurun_out/e5_sw_single.txt
timeout 600 $S --grid "256;64,128;64,128;3,4,6;1;1;1;1;1;2" > gpurun_out/e5_sw_pair.txt 2>&1; head -8 gpurun_out/e5_sw_pair.txt
timeout 120 python tools/trace_kernel.py matmul:1024,1024,1024 128,64,128,3,1,1 4 > gpurun_out/e5_trace.txt 2>&1; cat gpurun_out/e5_trace.txt
timeout 600 python bench.py --no-cpu > gpurun_out/e5_bench.json 2> gpurun_out/e5_bench.err; cat gpurun_out/e5_bench.json
