# seed sample size / probe count sweep on the DTW configs (A/B only)
for v in "2048 8" "1024 8" "4096 8" "2048 4" "2048 16"; do set -- $v
  for c in 2 3; do
    TSW_SAMPLE=$1 TSW_PROBE=$2 timeout 600 python bench.py --config $c --metric dtw --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sw_${1}_${2}_c${c}.log 2>&1
    echo "S=$1 P=$2 c$c $(python scripts/summarize_bench.py gpurun_out/sw_${1}_${2}_c${c}.log 2>/dev/null | cut -c24-150)"
  done
done
