mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
for i in 1 2 3; do
OPEVO_PROFILE_BATCH=1 timeout 600 python bench.py --no-cpu --no-e2e --log gpurun_out/g30_log$i.jsonl > gpurun_out/g30_bench$i.json 2> gpurun_out/g30_err$i.txt; python -c "import json;d=json.loads(open('gpurun_out/g30_bench$i.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['best_tflops'], d['gpu_launches'])"
done
