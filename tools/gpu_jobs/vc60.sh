mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
timeout 1200 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/vc60_pytest.txt 2>&1; tail -3 gpurun_out/vc60_pytest.txt
timeout 300 python tools/gen_breakdown.py matmul:1024,1024,1024 60 > gpurun_out/vc60_gb.txt 2>&1; cat gpurun_out/vc60_gb.txt
for i in 1 2; do
timeout 600 python bench.py --no-cpu > gpurun_out/vc60_bench$i.json 2> gpurun_out/vc60_err$i.txt; python -c "import json;d=json.loads(open('gpurun_out/vc60_bench$i.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],2), round(d['best_tflops'],1), round(d['roofline']['achieved'],1), round(d['e2e']['value']), d['gpu_launches'])"
done
