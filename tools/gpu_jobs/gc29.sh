mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/g29_pytest.txt 2>&1; tail -2 gpurun_out/g29_pytest.txt
for i in 1 2; do
timeout 600 python bench.py --no-cpu --log gpurun_out/g29_log$i.jsonl > gpurun_out/g29_bench$i.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/g29_bench$i.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['best_tflops'], d['e2e']['value'], d['gpu_launches'])"
done
timeout 900 python tools/scaling_projection.py matmul:1024,1024,1024 40 > gpurun_out/g29_scaling_mm1024.txt 2>&1; grep "N=" gpurun_out/g29_scaling_mm1024.txt
timeout 900 python tools/scaling_projection.py matmul:4096,4096,4096 20 > gpurun_out/g29_scaling_mm4096.txt 2>&1; grep "N=" gpurun_out/g29_scaling_mm4096.txt
