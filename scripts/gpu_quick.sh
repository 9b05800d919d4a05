# quick iteration loop: parity tests, then DTW benches of the headline configs (no CPU baseline)
set -o pipefail
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -x > gpurun_out/q_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/q_tests.log
for c in 2 3 4 5; do
  timeout 600 python bench.py --config $c --metric dtw --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q_c${c}.log 2>&1; echo "c$c rc=$?"
  python scripts/summarize_bench.py gpurun_out/q_c${c}.log 2>/dev/null | head -3
done
