mkdir -p gpurun_out/f68
make -s -C paper_2006_05664_b200/csrc
timeout 1200 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/f68/pytest.txt 2>&1; tail -3 gpurun_out/f68/pytest.txt
for op in conv2d:32,64,56,56,64,3,3,1,1; do
n=$(echo $op | tr ':,' '__')
timeout 900 python bench.py --op $op > gpurun_out/f68/bench_$n.json 2> gpurun_out/f68/err_$n.txt; python -c "import json;d=json.loads(open('gpurun_out/f68/bench_$n.json').read().strip().splitlines()[-1]);print('$op', round(d['value']), round(d['best_tflops'],1), d.get('best_tflops_cold_l2'), round(d['roofline']['achieved'],1), round(d['roofline']['frac'],3), d['best_knobs'])"
done
timeout 600 python bench.py > gpurun_out/f68/bench_n1.json 2> gpurun_out/f68/err_n1.txt; python -c "import json;d=json.loads(open('gpurun_out/f68/bench_n1.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['best_tflops'],1), round(d['roofline']['achieved'],1), round(d['e2e']['value']), d['gpu_launches'])"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f68/smoke.txt 2>&1; tail -1 gpurun_out/f68/smoke.txt
