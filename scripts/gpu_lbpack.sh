# packed LB terms: parity on the LB paths, then the DTW configs
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "lb or knn" > gpurun_out/lp_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/lp_tests.log
for c in 2 3 4 5; do
  st=10; [ $c -ge 4 ] && st=3
  timeout 600 python bench.py --config $c --metric dtw --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/lp_c${c}.log 2>&1
  echo "c$c $(python scripts/summarize_bench.py gpurun_out/lp_c${c}.log 2>/dev/null | cut -c24-150)"
done
