mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "tf32x3" > gpurun_out/x3_51_pytest.txt 2>&1; tail -15 gpurun_out/x3_51_pytest.txt
M=matmul:512,1024,1024
timeout 300 python tools/x3_probe.py $M 128,64,32,4 128,128,32,3 128,64,32,4,2 128,64,32,3,4 128,32,32,4 128,32,32,4,2 128,64,16,6,2 256,64,32,2 --simt 2,8,4,2,16,2,8,2 1,16,4,1,16,4,4,4 > gpurun_out/x3_51_probe.txt 2>&1; cat gpurun_out/x3_51_probe.txt
OPEVO_EXTRA_FLAGS=-DOPEVO_X3_HW_TRUNC=1 timeout 300 python tools/x3_probe.py $M 128,64,32,4 > gpurun_out/x3_51_hwtrunc.txt 2>&1; cat gpurun_out/x3_51_hwtrunc.txt
