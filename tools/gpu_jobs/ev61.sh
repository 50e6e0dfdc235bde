# evidence refresh: default bench x3 (with CPU baselines), reference arm, other operators
mkdir -p gpurun_out/ev61
make -s -C paper_2006_05664_b200/csrc
for i in 1 2 3; do
timeout 600 python bench.py > gpurun_out/ev61/bench_n1_run$i.json 2> gpurun_out/ev61/err$i.txt; python -c "import json;d=json.loads(open('gpurun_out/ev61/bench_n1_run$i.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],2), round(d['best_tflops'],1), round(d['roofline']['achieved'],1), round(d['e2e']['value']), d['gpu_launches'], d['clocks'])"
done
timeout 600 python bench.py --impl reference > gpurun_out/ev61/bench_reference.json 2> gpurun_out/ev61/err_ref.txt; tail -c 300 gpurun_out/ev61/bench_reference.json
for op in batchmatmul:960,128,64,128 conv2d:32,64,56,56,64,3,3,1,1 matmul:4096,4096,4096 matmul:512,1024,1024; do
n=$(echo $op | tr ':,' '__')
timeout 900 python bench.py --op $op --no-cpu > gpurun_out/ev61/bench_$n.json 2> gpurun_out/ev61/err_$n.txt; python -c "import json;d=json.loads(open('gpurun_out/ev61/bench_$n.json').read().strip().splitlines()[-1]);print('$op', round(d['value']), round(d['best_tflops'],1), d.get('best_tflops_cold_l2'), round(d['roofline']['achieved'],1), d['roofline']['unit'], round(d['roofline']['frac'],3))"
done
timeout 600 python bench.py --op matmul:512,1024,1024 --dtype tf32x3 > gpurun_out/ev61/bench_mm1_tf32x3.json 2> gpurun_out/ev61/err_x3.txt; python -c "import json;d=json.loads(open('gpurun_out/ev61/bench_mm1_tf32x3.json').read().strip().splitlines()[-1]);print('tf32x3', round(d['value']), round(d['best_tflops'],1), round(d['roofline']['achieved'],1), round(d['roofline']['frac'],3), d['cpu_baseline']['operator'])"
