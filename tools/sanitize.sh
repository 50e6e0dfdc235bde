#!/bin/bash
# compute-sanitizer (memcheck, synccheck) over one instance of every kernel
# variant on small operators; one process per instance. Usage: bash tools/sanitize.sh OUTDIR
OUT=${1:-gpurun_out/sanitize}
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name op knobs [--tf32x3]
  for tool in memcheck synccheck; do
    timeout 600 $CS --tool $tool --error-exitcode 9 python tools/profile_kernel.py $2 $3 1 $4 > $OUT/$1_$tool.log 2>&1
    echo "$1 $tool exit=$? $(grep -E 'ERROR SUMMARY' $OUT/$1_$tool.log | tail -1)"
  done
}
run gemm_single        matmul:256,512,512            128,64,128,3,1,1
run gemm_256rows       matmul:256,512,512            256,128,64,3,1,1
run gemm_pair          matmul:512,512,512            256,64,128,4,1,1,1,1,1,2
run gemm_multicast     matmul:256,512,512            128,64,64,4,1,2
run gemm_split_dsmem   matmul:256,512,512            128,64,64,4,2,1
run gemm_split_global  matmul:256,512,1024           128,64,64,2,16,1
run gemm_split_tma2    matmul:256,512,1024           128,128,64,4,2,1
run gemm_split_tma4    matmul:256,512,1024           128,64,64,4,4,1
run gemm_persistent    matmul:2048,2048,256          128,64,64,4,1,1
run gemm_sw32          matmul:256,480,512            128,48,16,8,1,1
run bmm_bpu4           batchmatmul:8,128,64,128      128,64,64,2,1,1,1,1,1,1,0,0,4
run conv_128           conv2d:4,64,16,16,64,3,3,1,1  128,64,64,4,1,1,8,8
run conv_256_resident  conv2d:4,64,16,16,64,3,3,1,1  256,64,64,3,1,1,8,8,1,1,0,1
run conv_split_taps    conv2d:8,64,16,16,64,3,3,1,1  128,64,32,6,3,1,2,8
run x3_single          matmul:256,512,512            128,64,32,4                   --tf32x3
run x3_split_dsmem     matmul:256,512,512            128,64,32,3,2                 --tf32x3
run x3_256rows         matmul:256,512,512            256,64,16,3                   --tf32x3
run x3_persistent      matmul:2048,2048,256          128,64,32,3                   --tf32x3
run x3_bmm             batchmatmul:8,128,64,128      128,64,32,3                   --tf32x3
run conv_halo          conv2d:4,64,28,28,64,3,3,1,1  128,64,64,4,1,1,4,14
run conv_halo_resident conv2d:4,64,28,28,64,3,3,1,1  256,64,64,3,1,1,4,14,1,1,0,1
run bmm_nbuf4          batchmatmul:64,128,64,128     128,64,64,4,1,1
