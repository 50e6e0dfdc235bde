mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "batchmatmul or bmm or batched or tf32x3" > gpurun_out/bf80_pytest.txt 2>&1; tail -3 gpurun_out/bf80_pytest.txt
timeout 300 python tools/timing_modes.py batchmatmul:960,128,64,128 128,64,64,6,1,1 128,64,128,3,1,1 128,64,64,8,1,1 128,64,128,4,1,1 2>&1 | grep TF
timeout 120 python tools/trace_units.py batchmatmul:960,128,64,128 128,64,64,6,1,1
