mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for spec in "gemm_split_tma2 matmul:256,512,1024 128,128,64,4,2,1" "gemm_split_tma4 matmul:256,512,1024 128,64,64,4,4,1"; do
  set -- $spec
  for tool in memcheck synccheck; do
    timeout 600 $CS --tool $tool --error-exitcode 9 python tools/profile_kernel.py $2 $3 1 > gpurun_out/sanitize/$1_$tool.log 2>&1
    echo "$1 $tool exit=$? $(grep -E 'ERROR SUMMARY' gpurun_out/sanitize/$1_$tool.log | tail -1)"
  done
done
for i in 1 2; do
timeout 600 python bench.py --no-cpu > gpurun_out/s46_bench$i.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/s46_bench$i.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],2), round(d['best_tflops'],1), round(d['roofline']['achieved'],1), round(d['e2e']['value']), d['best_knobs'])"
done
