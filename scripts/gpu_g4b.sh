for rep in 1 2; do for v in "" "4,8"; do for c in 3 5; do
  st=10; [ $c -ge 4 ] && st=3
  TSW_DTW4=$v timeout 600 python bench.py --config $c --metric dtw --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/g4b.log 2>&1
  echo "rep$rep G,WL=${v:-default} c$c $(python scripts/summarize_bench.py gpurun_out/g4b.log 2>/dev/null | cut -c24-150)"
done; done; done
