# two epilogue groups (alternate units) vs one: correctness on the persistent shapes, then timing
mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
OPEVO_EPI_GROUPS=2 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "matmul_parity or batchmatmul_parity or conv2d" > gpurun_out/e2_72_pytest.txt 2>&1; tail -3 gpurun_out/e2_72_pytest.txt
for g in 1 2; do
echo "== epilogue groups $g"
OPEVO_EPI_GROUPS=$g timeout 300 python tools/timing_modes.py batchmatmul:960,128,64,128 128,64,64,6,1,1 128,64,128,3,1,1 128,64,64,8,1,1 2>&1 | grep TF
OPEVO_EPI_GROUPS=$g timeout 300 python tools/timing_modes.py conv2d:32,64,56,56,64,3,3,1,1 128,64,64,4,1,1,4,14 128,64,64,4,1,1,8,14 256,64,64,4,1,1,8,8 2>&1 | grep TF
OPEVO_EPI_GROUPS=$g timeout 300 python tools/timing_modes.py matmul:4096,4096,4096 128,256,64,4,1,1 128,128,64,6,1,1 2>&1 | grep "^(" 
OPEVO_EPI_GROUPS=$g timeout 300 python tools/timing_modes.py matmul:1024,1024,1024 128,64,128,4,1,1 2>&1 | grep "^("
done
