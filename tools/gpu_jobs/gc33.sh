mkdir -p gpurun_out
for i in 1 2 3; do
OPEVO_NO_CLOCKS=1 OPEVO_PROFILE_BATCH=1 timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/g33_bench$i.json 2> gpurun_out/g33_err$i.txt; python -c "import json;d=json.loads(open('gpurun_out/g33_bench$i.json').read().strip().splitlines()[-1]);print('noclk', d['value'], d['ms_per_step'])"
done
for i in 1 2 3; do
timeout 600 python bench.py --no-cpu --no-e2e --steps 200 > gpurun_out/g33_long$i.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/g33_long$i.json').read().strip().splitlines()[-1]);print('long', d['value'], d['ms_per_step'], d['clocks'])"
done
