# shared-memory envelope K2 (lb_env_kernel): parity, then A/B against the L1 path on the DTW benches
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_stress.py -q -m gpu -x > gpurun_out/lbenv_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/lbenv_tests.log
for e in 1 0; do for c in 2 3; do
  TSW_LB_ENV=$e timeout 600 python bench.py --config $c --metric dtw --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/lbenv${e}_c${c}.log 2>&1; echo "env$e c$c rc=$?"
  python scripts/summarize_bench.py gpurun_out/lbenv${e}_c${c}.log 2>/dev/null | head -3
done; done
