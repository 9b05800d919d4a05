# full evidence pass: GPU tests, smoke, every bench line, the reference arm, ncu captures
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1; echo "smoke rc=$?"
bash scripts/gpu_bench_all.sh
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.log 2>&1; echo "ref rc=$?"
bash scripts/gpu_profile_bench.sh
