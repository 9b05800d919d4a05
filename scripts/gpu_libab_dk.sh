ALT=${ALT:-build_var/lib_base.so}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -x -k "dk" 2>&1 | tail -1
for rep in 1 2; do for lib in $ALT ""; do for c in 3 4; do
  TSW_LIB=$lib timeout 600 python bench.py --config $c --metric dk --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  echo "rep$rep lib=${lib:-current} c$c $(python scripts/summarize_bench.py gpurun_out/ab.log 2>/dev/null | cut -c24-150)"
done; done; done
