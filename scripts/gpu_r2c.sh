# round-2: GPU tests after the fp32-range fix; C5 per-query counters; C5 DTW DP ncu capture
python -m pytest tests -m gpu -x -q > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2c_pytest.log
python scripts/diag_counters.py 5 dtw > gpurun_out/r2c_counters_c5dtw.txt 2>&1; echo "diag rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --legs none"
$CMD > gpurun_out/r2c_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:dtw4_kernel -s 3 -c 1 -o gpurun_out/r2c_dtw4_c5 $CMD > gpurun_out/r2c_ncu.log 2>&1; echo "ncu rc=$?"
