# same-box A/B of two builds of the library (TSW_LIB=$ALT vs the in-tree one), DTW configs
ALT=${ALT:-build_var/libtswarp_b200_nopf.so}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "dtw or knn" 2>&1 | tail -1
for rep in 1 2; do for lib in $ALT ""; do for c in 2 3 5; do
  st=10; [ $c -ge 4 ] && st=3
  TSW_LIB=$lib timeout 600 python bench.py --config $c --metric dtw --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  echo "rep$rep lib=${lib:-current} c$c $(python scripts/summarize_bench.py gpurun_out/ab.log 2>/dev/null | cut -c24-150)"
done; done; done
