# DK iteration loop: every DK parity test, then the DK bench lines (no CPU baseline)
set -o pipefail
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sub.py tests/test_gpu_stress.py tests/test_gpu_configs.py -q -m gpu -x -k "dk or DK or knn or sub or config" > gpurun_out/dk_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/dk_tests.log
for c in 1 3 4 5; do
  timeout 600 python bench.py --config $c --metric dk --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dk_c${c}.log 2>&1; echo "c$c rc=$?"
  python scripts/summarize_bench.py gpurun_out/dk_c${c}.log 2>/dev/null | head -3
done
for c in 3 5; do
  timeout 600 python bench.py --config $c --metric dk_sub --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/dksub_c${c}.log 2>&1; echo "c$c sub rc=$?"
  python scripts/summarize_bench.py gpurun_out/dksub_c${c}.log 2>/dev/null | head -3
done
