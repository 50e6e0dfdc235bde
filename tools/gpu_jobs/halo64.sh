mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "halo or conv2d_parity" > gpurun_out/halo64_pytest.txt 2>&1; tail -3 gpurun_out/halo64_pytest.txt
C=conv2d:32,64,56,56,64,3,3,1,1
timeout 600 python tools/ablate.py $C@128,64,64,4,1,1,8,14 $C@128,64,64,4,1,1,8,14,1,1,0,1 $C@256,64,64,4,1,1,8,8 > gpurun_out/halo64_ablate.txt 2>&1; cat gpurun_out/halo64_ablate.txt
timeout 120 python tools/trace_kernel.py $C 128,64,64,4,1,1,8,14,1,1,0,1 1 > gpurun_out/halo64_trace.txt 2>&1; cat gpurun_out/halo64_trace.txt
timeout 120 python tools/trace_kernel.py $C 128,64,64,4,1,1,8,14 1 >> gpurun_out/halo64_trace.txt 2>&1; tail -18 gpurun_out/halo64_trace.txt
