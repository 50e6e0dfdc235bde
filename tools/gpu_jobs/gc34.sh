mkdir -p gpurun_out
for t in stream graph stream graph stream graph; do
timeout 600 python bench.py --no-cpu --no-e2e --timing $t > gpurun_out/g34_$t.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/g34_$t.json').read().strip().splitlines()[-1]);print('$t', round(d['value']), round(d['ms_per_step'],2), round(d['best_tflops'],1), round(d['roofline']['achieved'],1))"
done
