# G = 4 DTW fast path: parity of every variant, then A/B against G = 2 on the DTW configs
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fast_path_variants" > gpurun_out/g4_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/g4_tests.log
for v in "2,8" "4,8"; do for c in 2 3 5; do
  st=10; [ $c -ge 4 ] && st=3
  TSW_DTW4=$v timeout 600 python bench.py --config $c --metric dtw --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/g4_${v}_c${c}.log 2>&1
  echo "G,WL=$v c$c $(python scripts/summarize_bench.py gpurun_out/g4_${v}_c${c}.log 2>/dev/null | cut -c24-150)"
done; done
