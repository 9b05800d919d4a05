timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_sub.py -q -m gpu -x 2>&1 | tail -1
for cm in "1 dk" "2 dtw" "4 dk" "4 dtw" "5 dk" "5 dtw" "3 dk"; do set -- $cm
  st=10; [ $1 -ge 4 ] && st=3
  timeout 600 python bench.py --config $1 --metric $2 --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/sel.log 2>&1
  echo "c$1 $2 $(python scripts/summarize_bench.py gpurun_out/sel.log 2>/dev/null | cut -c24-150)"
done
