mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for spec in "gemm_split_global matmul:256,512,1024 128,64,64,2,16,1" "gemm_sw32 matmul:256,480,512 128,48,16,8,1,1" "conv_split_taps conv2d:8,64,16,16,64,3,3,1,1 128,64,32,6,3,1,2,8"; do
  set -- $spec
  for tool in memcheck synccheck; do
    timeout 600 $CS --tool $tool --error-exitcode 9 python tools/profile_kernel.py $2 $3 1 > gpurun_out/sanitize/$1_$tool.log 2>&1
    echo "$1 $tool exit=$? $(grep -E 'ERROR SUMMARY' gpurun_out/sanitize/$1_$tool.log | tail -1)"
  done
done
