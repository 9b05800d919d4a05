# round-2 first GPU call: GPU tests + the new default bench line (C5 DTW + DK leg)
python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"
timeout 1200 python bench.py --steps 10 --warmup 3 --out gpurun_out/r2a_bench.jsonl > gpurun_out/r2a_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2a_ref.log 2>&1; echo "ref rc=$?"
nproc; tail -3 gpurun_out/r2a_pytest.log
