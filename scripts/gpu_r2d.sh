# round-2: GPU tests (fp32 range incl. +inf DTW semantics, long series / spill mode, concurrency)
python -m pytest tests -m gpu -x -q > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2d_pytest.log
