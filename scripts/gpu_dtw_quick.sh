# DTW parity + benches of the DTW configs
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -x -k "dtw or knn or config or lb" > gpurun_out/dq_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/dq_tests.log
for c in 2 3 5; do
  timeout 600 python bench.py --config $c --metric dtw --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/dq_c${c}.log 2>&1; echo "c$c rc=$?"
  python scripts/summarize_bench.py gpurun_out/dq_c${c}.log 2>/dev/null | head -3
done
