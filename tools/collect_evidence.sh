#!/bin/bash
# One GPU call that refreshes the round's evidence under gpurun_out/.
set -x
TAG=${1:-r01}
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
tail -3 gpurun_out/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 600 python bench.py --log gpurun_out/${TAG}_bench_trials.jsonl > gpurun_out/${TAG}_bench_n1.json 2> gpurun_out/${TAG}_bench_n1.err
for op in matmul:4096,4096,4096 batchmatmul:960,128,64,128 conv2d:32,64,56,56,64,3,3,1,1 matmul:512,1024,1024; do
  name=$(echo $op | tr ':,' '__')
  timeout 600 python bench.py --op $op --steps 30 --no-cpu > gpurun_out/${TAG}_bench_${name}.json 2> gpurun_out/${TAG}_bench_${name}.err
done
timeout 300 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2>&1
# launch list of a short bench (cold, serialised: compare shares, not absolutes)
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu --reps 5 > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
export OPEVO_LINEINFO=1
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/${TAG}_prof_mm1024 python tools/profile_kernel.py matmul:1024,1024,1024 $2 > /dev/null 2>&1
timeout 300 $NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/${TAG}_prof_mm4096 python tools/profile_kernel.py matmul:4096,4096,4096 $3 > /dev/null 2>&1
ls -la gpurun_out | tail -30
