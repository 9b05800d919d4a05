ALT=build_var/lib_base.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -x -k "dtw or knn or config" 2>&1 | tail -1
for rep in 1 2; do for lib in $ALT ""; do for cm in "2 dtw" "3 dtw" "5 dtw"; do set -- $cm
  st=10; [ $1 -ge 5 ] && st=3
  TSW_LIB=$lib timeout 600 python bench.py --config $1 --metric $2 --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  echo "rep$rep lib=${lib:-current} c$1 $2 $(python scripts/summarize_bench.py gpurun_out/ab.log 2>/dev/null | cut -c28-150)"
done; done; done
