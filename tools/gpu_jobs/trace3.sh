mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
for kn in 128,64,128,3,1,1 128,128,128,3,1,1 256,128,128,4,2,1,1,1,1,2 128,128,128,3,2,1 256,64,128,4,1,1,1,1,1,2; do
  timeout 120 python tools/trace_kernel.py matmul:1024,1024,1024 $kn 4 >> gpurun_out/trace3.txt 2>&1
done
cat gpurun_out/trace3.txt
