# final tree check: GPU suite, smoke, default bench (cache rebuilt for the final kernel source)
mkdir -p gpurun_out/fin82
make -s -C paper_2006_05664_b200/csrc
timeout 1200 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/fin82/pytest.txt 2>&1; tail -2 gpurun_out/fin82/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin82/smoke.txt 2>&1; tail -1 gpurun_out/fin82/smoke.txt
timeout 600 python bench.py > gpurun_out/fin82/bench_n1.json 2> gpurun_out/fin82/err.txt; python -c "import json;d=json.loads(open('gpurun_out/fin82/bench_n1.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['best_tflops'],1), round(d['roofline']['achieved'],1), d['roofline']['traffic'], round(d['e2e']['value']), d['gpu_launches'], d['clocks'])"
