mkdir -p gpurun_out
for i in 1 2 3; do
timeout 600 python bench.py --no-cpu > gpurun_out/p39_bench$i.json 2>gpurun_out/p39_err$i.txt; python -c "import json;d=json.loads(open('gpurun_out/p39_bench$i.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],2), round(d['best_tflops'],1), round(d['roofline']['achieved'],1), round(d['e2e']['value']), d['gpu_launches'])"
done
tail -3 gpurun_out/p39_err1.txt
timeout 900 python tools/scaling_projection.py matmul:1024,1024,1024 40 > gpurun_out/p39_scaling_mm1024.txt 2>&1; grep "N=" gpurun_out/p39_scaling_mm1024.txt
