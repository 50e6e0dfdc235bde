# full evidence refresh: GPU tests, smoke, bench lines for every BASELINE operator, reference arm
mkdir -p gpurun_out
T=r27
timeout 900 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.txt 2>&1; tail -3 gpurun_out/${T}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1; tail -1 gpurun_out/${T}_smoke.txt
timeout 600 python bench.py --log gpurun_out/${T}_bench_trials.jsonl > gpurun_out/${T}_bench_n1.json 2> gpurun_out/${T}_bench_n1.err; cat gpurun_out/${T}_bench_n1.json
for op in matmul:4096,4096,4096 batchmatmul:960,128,64,128 conv2d:32,64,56,56,64,3,3,1,1 matmul:512,1024,1024; do
  name=$(echo $op | tr ':,' '__')
  timeout 600 python bench.py --op $op --steps 60 --no-cpu > gpurun_out/${T}_bench_${name}.json 2> gpurun_out/${T}_bench_${name}.err
  python -c "import json;d=json.loads(open('gpurun_out/${T}_bench_${name}.json').read().strip().splitlines()[-1]);print('$op', round(d['value']), 'trials/s best', round(d['best_tflops'],1), d['best_knobs'], 'retimed', round(d['roofline']['achieved'],1))"
done
timeout 600 python bench.py --op matmul:512,1024,1024 --dtype f32 --steps 60 --no-cpu > gpurun_out/${T}_bench_mm1_f32.json 2> gpurun_out/${T}_bench_mm1_f32.err; tail -c 600 gpurun_out/${T}_bench_mm1_f32.json
timeout 300 python bench.py --impl reference > gpurun_out/${T}_bench_reference.json 2>&1; tail -c 300 gpurun_out/${T}_bench_reference.json
