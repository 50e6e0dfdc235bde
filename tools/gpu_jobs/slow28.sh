mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 900 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/w28_pytest.txt 2>&1; tail -3 gpurun_out/w28_pytest.txt
timeout 900 python tools/scaling_projection.py matmul:1024,1024,1024 40 > gpurun_out/w28_scaling_mm1024.txt 2>&1; grep "N=" gpurun_out/w28_scaling_mm1024.txt
timeout 900 python tools/scaling_projection.py matmul:4096,4096,4096 20 > gpurun_out/w28_scaling_mm4096.txt 2>&1; grep "N=" gpurun_out/w28_scaling_mm4096.txt
timeout 600 python bench.py --no-cpu > gpurun_out/w28_bench.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/w28_bench.json').read().strip().splitlines()[-1]);print(d['value'], d['best_tflops'], d['e2e']['value'], d['gpu_launches'])"
timeout 600 python bench.py --op matmul:4096,4096,4096 --no-cpu > gpurun_out/w28_bench4096.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/w28_bench4096.json').read().strip().splitlines()[-1]);print(d['value'], d['best_tflops'], d['e2e']['value'], d['gpu_launches'])"
