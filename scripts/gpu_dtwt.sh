# large-d DTW path: parity, then the config-4 DTW bench
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -x -k "tiled or large or config4 or dtw_all or knn_random" > gpurun_out/dt_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/dt_tests.log
timeout 600 python bench.py --config 4 --metric dtw --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/dt_c4.log 2>&1; echo "c4 rc=$?"
python scripts/summarize_bench.py gpurun_out/dt_c4.log 2>/dev/null | head -3
