mkdir -p gpurun_out/clk86
for i in 1 2 3; do
timeout 600 python bench.py --no-cpu > gpurun_out/clk86/b$i.json 2> gpurun_out/clk86/e$i.txt; python -c "import json;d=json.loads(open('gpurun_out/clk86/b$i.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['best_tflops'],1), round(d['e2e']['value']), d['clocks'])"
done
