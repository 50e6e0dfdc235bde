# 1024^3 landscape: CTA pairs x split-K, single-CTA split-K, multicast; ablations
mkdir -p gpurun_out
S="python tools/sweep.py matmul:1024,1024,1024"
timeout 600 $S --grid "256;128,64,256;64,128;2,3,4,6;1,2,4;1;1;1;1;2" > gpurun_out/sw_pair.txt 2>&1
timeout 600 $S --grid "128;128,64,256;64,128;2,3,4,6;1,2,4,8;1;1;1;1;1" > gpurun_out/sw_single.txt 2>&1
timeout 300 $S --grid "128;64,128;64,128;3,4;1,2;2,4;1;1;1;1" > gpurun_out/sw_mc.txt 2>&1
timeout 600 python tools/ablate.py matmul:1024,1024,1024@128,64,128,3,1,1 matmul:1024,1024,1024@256,128,64,4,2,1,1,1,1,2 matmul:1024,1024,1024@128,128,128,3,2,1 > gpurun_out/ablate.txt 2>&1
tail -n 12 gpurun_out/sw_*.txt
cat gpurun_out/ablate.txt
