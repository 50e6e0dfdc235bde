mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
for i in 1 2 3; do
OPEVO_PROFILE_BATCH=1 timeout 600 python bench.py --no-cpu > gpurun_out/g32_bench$i.json 2> gpurun_out/g32_err$i.txt; python -c "import json;d=json.loads(open('gpurun_out/g32_bench$i.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['best_tflops'], d['e2e']['value'], d['clocks'])"
done
timeout 900 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/g32_pytest.txt 2>&1; tail -2 gpurun_out/g32_pytest.txt
