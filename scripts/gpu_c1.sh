for i in 1 2; do
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c1_$i.log 2>&1
python scripts/summarize_bench.py gpurun_out/c1_$i.log | cut -c1-200
done
timeout 600 python bench.py --config 3 --metric dk_sub --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c3s.log 2>&1
python scripts/summarize_bench.py gpurun_out/c3s.log | cut -c1-200
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sub.py -q -m gpu -x -k "dk" 2>&1 | tail -1
