# final round-1 evidence: GPU suite, sanitizers, all bench lines, ncu (conv halo best + launch list), smoke
mkdir -p gpurun_out/fin71
make -s -C paper_2006_05664_b200/csrc
NCU=/usr/local/cuda/bin/ncu
timeout 1200 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/fin71/pytest.txt 2>&1; tail -2 gpurun_out/fin71/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin71/smoke.txt 2>&1; tail -1 gpurun_out/fin71/smoke.txt
for i in 1 2 3; do
timeout 600 python bench.py > gpurun_out/fin71/bench_n1_run$i.json 2> gpurun_out/fin71/err$i.txt; python -c "import json;d=json.loads(open('gpurun_out/fin71/bench_n1_run$i.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['best_tflops'],1), round(d['roofline']['achieved'],1), round(d['e2e']['value']), d['gpu_launches'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
timeout 600 python bench.py --impl reference > gpurun_out/fin71/bench_reference.json 2> gpurun_out/fin71/err_ref.txt
for op in batchmatmul:960,128,64,128 conv2d:32,64,56,56,64,3,3,1,1 matmul:4096,4096,4096 matmul:512,1024,1024; do
n=$(echo $op | tr ':,' '__')
timeout 900 python bench.py --op $op --no-cpu > gpurun_out/fin71/bench_$n.json 2> gpurun_out/fin71/err_$n.txt; python -c "import json;d=json.loads(open('gpurun_out/fin71/bench_$n.json').read().strip().splitlines()[-1]);print('$op', round(d['value']), round(d['best_tflops'],1), round(d['roofline']['achieved'],1), d['roofline']['unit'], round(d['roofline']['frac'],3), d['best_knobs'])"
done
timeout 600 python bench.py --op matmul:512,1024,1024 --dtype tf32x3 --no-cpu > gpurun_out/fin71/bench_mm1_tf32x3.json 2> gpurun_out/fin71/err_x3.txt; python -c "import json;d=json.loads(open('gpurun_out/fin71/bench_mm1_tf32x3.json').read().strip().splitlines()[-1]);print('tf32x3', round(d['value']), round(d['best_tflops'],1), round(d['roofline']['achieved'],1), round(d['roofline']['frac'],3), d['best_knobs'])"
bash tools/sanitize.sh gpurun_out/fin71/san > gpurun_out/fin71/sanitizer.txt 2>&1; grep -c "0 errors" gpurun_out/fin71/sanitizer.txt; grep -v "0 errors" gpurun_out/fin71/sanitizer.txt | head
OPEVO_LINEINFO=1 timeout 300 $NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/fin71/conv_halo python tools/profile_kernel.py conv2d:32,64,56,56,64,3,3,1,1 128,64,64,4,1,1,4,14 > /dev/null 2>&1
OPEVO_LINEINFO=1 timeout 300 $NCU --set full --clock-control none --import-source on -k regex:opevo_gemm -s 5 -c 1 -o gpurun_out/fin71/bmm python tools/profile_kernel.py batchmatmul:960,128,64,128 128,64,64,6,1,1 > /dev/null 2>&1
OPEVO_NO_POOL=1 OPEVO_TIME_BUDGET_MS=0 timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file gpurun_out/fin71/launches.csv python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu --timing graph > gpurun_out/fin71/bench_under_ncu.log 2>&1
ls gpurun_out/fin71 | head -40
