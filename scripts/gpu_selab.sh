for cm in "3 dk" "3 dtw" "4 dk" "1 dk" "2 dtw"; do set -- $cm
  timeout 600 python bench.py --config $1 --metric $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sel.log 2>&1
  echo "c$1 $2 $(python scripts/summarize_bench.py gpurun_out/sel.log 2>/dev/null | cut -c24-150)"
done
