timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2p_pytest.log
bash scripts/gpu_bench_all.sh r2p
python scripts/summarize_bench.py "gpurun_out/r2p_bench_c*.log"
