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
# round 2: conv widening (stride 4 + Cin padded to 16, padded lines, tap split with lines, CTA pairs),
# the rotating-copy timing and the per-block compare ride along in every run
run conv_c1_stride4_lines  conv2d:8,3,227,227,64,11,11,4,0   256,64,16,8,1,1,11,11,1,1,0,0,1,16
run conv_c1_lines_split    conv2d:8,3,227,227,64,11,11,4,0   256,64,16,8,11,1,11,5,1,1,0,0,1,16
run conv_c2_lines          conv2d:8,64,27,27,192,5,5,1,2     256,16,32,2,1,1,9,9,1,1,0,0,1,16
run conv_c2_lines_split    conv2d:8,64,27,27,192,5,5,1,2     256,192,32,6,5,1,9,3,1,1,0,0,1,16
run conv_pair              conv2d:4,64,56,56,64,3,3,1,1      256,16,16,3,1,1,8,8,1,2,0,0,1,0
run conv_pair_split        conv2d:4,64,56,56,64,3,3,1,1      256,64,16,2,3,1,8,8,1,2,0,0,1,0
run conv_pair_halo         conv2d:4,64,56,56,64,3,3,1,1      256,32,64,6,1,1,4,14,1,2,0,0,1,0
run conv_pair_lines_split  conv2d:4,64,56,56,64,3,3,1,1      256,32,16,6,9,1,8,7,1,2,0,0,1,16
run conv_lines_resident    conv2d:4,64,56,56,64,3,3,1,1      256,64,64,3,1,1,8,28,1,1,0,1,1,32
# late round 2: 512-row halo CTA pairs, one weight box per filter row, 32-column epilogue staging with two
# CTAs (pairs) per SM (pair)
run conv_pair512_halo      conv2d:8,64,56,56,64,3,3,1,1      512,64,64,3,1,1,4,14,1,2,0,0,1,0
run conv_pair512_halo_2st  conv2d:4,64,56,56,64,3,3,1,1      512,64,64,2,1,1,8,14,1,2,0,0,1,0
run conv_pair_halo_narrow  conv2d:8,64,56,56,64,3,3,1,1      256,64,64,3,1,1,2,14,1,2,0,0,1,0
run conv_halo_narrow       conv2d:8,64,28,28,64,3,3,1,1      128,64,64,2,1,1,1,14,1,1,0,0,1,0
run gemm_narrow_2cta       matmul:1024,1024,1024             256,64,64,2,1,1,1,1,1,1,0,0,1,0
run gemm_pair_narrow       matmul:1024,1024,1024             256,64,64,4,1,1,1,1,1,2,0,0,1,0
