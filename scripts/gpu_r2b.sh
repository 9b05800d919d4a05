# round-2: GPU tests (all-query reference pins, device counters, fp32-range inputs) + bench
python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2b_pytest.log
timeout 1200 python bench.py --steps 10 --warmup 3 --out gpurun_out/r2b_bench.jsonl > gpurun_out/r2b_bench.log 2>&1; echo "bench rc=$?"
