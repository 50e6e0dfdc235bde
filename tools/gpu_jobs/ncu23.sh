mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 300 /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/n23_conv python tools/profile_kernel.py conv2d:32,64,56,56,64,3,3,1,1 128,64,64,4,1,1,8,8,1,1,0,1 > gpurun_out/n23.log 2>&1
ls -la gpurun_out/n23*
