mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do
timeout 600 python bench.py --no-cpu --no-e2e --log gpurun_out/r47_log$i.jsonl > gpurun_out/r47_bench$i.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r47_bench$i.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['best_tflops'],1), round(d['roofline']['achieved'],1), d['trials_to_95pct'], d['best_knobs'])"
done
