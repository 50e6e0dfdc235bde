# cold kernel cache: every instance the search reaches is NVRTC-compiled on the host pool during the run
mkdir -p gpurun_out/cold87
mv paper_2006_05664_b200/kernel_cache /tmp/kernel_cache_moved
mkdir -p paper_2006_05664_b200/kernel_cache
timeout 1200 python bench.py --no-preload --no-cpu --no-e2e > gpurun_out/cold87/bench_cold_cache.json 2> gpurun_out/cold87/err.txt
python -c "import json;d=json.loads(open('gpurun_out/cold87/bench_cold_cache.json').read().strip().splitlines()[-1]);print(round(d['value'],1), round(d['best_tflops'],1), d['ms_per_step'], d['gpu_launches'])"
ls paper_2006_05664_b200/kernel_cache | wc -l
rm -rf paper_2006_05664_b200/kernel_cache; mv /tmp/kernel_cache_moved paper_2006_05664_b200/kernel_cache
