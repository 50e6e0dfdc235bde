mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 300 python tools/timing_modes.py matmul:1024,1024,1024 128,64,128,3,1,1 128,64,128,4,1,1 128,128,128,3,1,1 256,64,128,4,1,1,1,1,1,2 > gpurun_out/m6_modes.txt 2>&1
timeout 300 python tools/timing_modes.py matmul:4096,4096,4096 256,256,64,6,1,1,1,1,1,2 >> gpurun_out/m6_modes.txt 2>&1
cat gpurun_out/m6_modes.txt
timeout 300 python tools/trial_cost.py matmul:1024,1024,1024 40 > gpurun_out/m6_trial_cost.txt 2>&1; cat gpurun_out/m6_trial_cost.txt
timeout 900 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/m6_pytest_gpu.txt 2>&1; tail -3 gpurun_out/m6_pytest_gpu.txt
