timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -x -k "dk or knn or config" 2>&1 | tail -1
for c in 1 3 4 5; do
  st=10; [ $c -ge 5 ] && st=3
  timeout 600 python bench.py --config $c --metric dk --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/dkp.log 2>&1
  echo "c$c $(python scripts/summarize_bench.py gpurun_out/dkp.log 2>/dev/null | cut -c24-150)"
done
