# DTW fast-path A/B: parity tests, then config benches for the given variants ("c:variant" items)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -x > gpurun_out/q_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/q_tests.log
for cv in "$@"; do
  c=${cv%%:*}; v=${cv#*:}
  unset TSW_DTW_GENERIC TSW_DTW4
  [ $v = generic ] && export TSW_DTW_GENERIC=1
  [ $v != generic ] && [ $v != auto ] && export TSW_DTW4=$v
  timeout 300 python bench.py --config $c --metric dtw --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v_c${c}_${v}.log 2>&1; echo "c$c $v rc=$?"
  python scripts/summarize_bench.py gpurun_out/v_c${c}_${v}.log 2>/dev/null | head -2
done
