mkdir -p gpurun_out
for f in "" "-DOPEVO_NO_WATCHDOG"; do
echo "== extra flags: '$f'"
for ab in 0 7; do
OPEVO_EXTRA_FLAGS="$f -DOPEVO_ABLATE=$ab" timeout 300 python tools/timing_modes.py batchmatmul:960,128,64,128 128,64,64,6,1,1 2>&1 | grep "^(" | sed "s/^/ablate=$ab /"
OPEVO_EXTRA_FLAGS="$f -DOPEVO_ABLATE=$ab" timeout 300 python tools/timing_modes.py conv2d:32,64,56,56,64,3,3,1,1 128,64,64,4,1,1,4,14 2>&1 | grep "^(" | sed "s/^/ablate=$ab /"
done
done
