mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
for i in 1 2; do
timeout 600 python bench.py --op matmul:512,1024,1024 --dtype tf32x3 --no-cpu --log gpurun_out/x3_56_log$i.jsonl > gpurun_out/x3_56_bench$i.json 2> gpurun_out/x3_56_err$i.txt; python -c "import json;d=json.loads(open('gpurun_out/x3_56_bench$i.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],2), round(d['best_tflops'],1), d['gpu_launches'])"
done
OPEVO_PROFILE_BATCH=1 timeout 600 python bench.py --op matmul:512,1024,1024 --dtype tf32x3 --no-cpu --no-e2e --steps 20 > gpurun_out/x3_56_prof.json 2> gpurun_out/x3_56_prof.txt; tail -30 gpurun_out/x3_56_prof.txt
