mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
for kn in 128,64,64,3,1,1 128,64,64,4,1,1 128,64,128,3,1,1; do
timeout 120 python tools/trace_kernel.py matmul:1024,1024,1024 $kn 4 >> gpurun_out/c10_trace.txt 2>&1
done
cat gpurun_out/c10_trace.txt
timeout 600 python bench.py --no-cpu > gpurun_out/c10_bench.json 2> gpurun_out/c10_bench.err; cat gpurun_out/c10_bench.json
