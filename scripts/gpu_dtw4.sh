# DTW A/B: parity tests, then config benches for "config:variant[:lib]" items
# (variant: auto | generic | G,WL ; lib: optional alternative build directory with libtswarp_b200.so)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -x > gpurun_out/q_tests.log 2>&1; echo "tests rc=$?"
tail -1 gpurun_out/q_tests.log
for cv in "$@"; do
  IFS=: read c v lib <<< "$cv"
  unset TSW_DTW_GENERIC TSW_DTW4 TSW_LIB
  [ "$v" = generic ] && export TSW_DTW_GENERIC=1
  [ "$v" != generic ] && [ "$v" != auto ] && export TSW_DTW4=$v
  [ -n "$lib" ] && export TSW_LIB=$PWD/$lib/libtswarp_b200.so
  tag=c${c}_${v}${lib:+_$lib}
  timeout 300 python bench.py --config $c --metric dtw --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v_$tag.log 2>&1; echo "$tag rc=$?"
  python scripts/summarize_bench.py gpurun_out/v_$tag.log 2>/dev/null | head -2
done
