mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "tf32x3" > gpurun_out/x3_53_pytest.txt 2>&1; tail -3 gpurun_out/x3_53_pytest.txt
M=matmul:512,1024,1024
timeout 300 python tools/x3_probe.py $M 128,64,32,4 128,64,64,2,2 128,64,32,4,2 128,128,32,3,4 128,128,64,1,4 128,256,16,3,4 256,128,16,4 > gpurun_out/x3_53_probe.txt 2>&1; cat gpurun_out/x3_53_probe.txt
