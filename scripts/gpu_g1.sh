for v in "2,8" "1,16"; do for c in 2 3; do
  TSW_DTW4=$v timeout 600 python bench.py --config $c --metric dtw --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g_${v}_c${c}.log 2>&1
  echo "G,WL=$v c$c $(python scripts/summarize_bench.py gpurun_out/g_${v}_c${c}.log 2>/dev/null | cut -c24-150)"
done; done
