python -m pytest tests -m gpu -x -q > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2e_pytest.log
