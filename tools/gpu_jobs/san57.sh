mkdir -p gpurun_out
make -s -C paper_2006_05664_b200/csrc
bash tools/sanitize.sh gpurun_out/san57 > gpurun_out/san57_summary.txt 2>&1; cat gpurun_out/san57_summary.txt
