timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -x -k "knn or config" 2>&1 | tail -1
for cm in "3 dk" "3 dtw" "1 dk"; do set -- $cm
  timeout 600 python bench.py --config $1 --metric $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ubc.log 2>&1
  echo "c$1 $2 $(python scripts/summarize_bench.py gpurun_out/ubc.log 2>/dev/null | cut -c24-150)"
done
