mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 300 python tools/trial_cost.py matmul:1024,1024,1024 40 > gpurun_out/trial_cost.txt 2>&1
timeout 300 python tools/trial_cost.py matmul:1024,1024,1024 40 >> gpurun_out/trial_cost.txt 2>&1
cat gpurun_out/trial_cost.txt
