# search reliability: the default bench (1024^3, 504 trials) for seeds 0..7
mkdir -p gpurun_out/seeds85
for s in 0 1 2 3 4 5 6 7; do
timeout 600 python bench.py --seed $s --no-cpu --no-e2e > gpurun_out/seeds85/bench_seed$s.json 2> gpurun_out/seeds85/err$s.txt
python -c "import json;d=json.loads(open('gpurun_out/seeds85/bench_seed$s.json').read().strip().splitlines()[-1]);print('seed $s', round(d['value']), round(d['best_tflops'],1), d['trials_to_95pct'], d['best_knobs'][:5])"
done
