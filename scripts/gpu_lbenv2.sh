for ch in 8 32; do for c in 2 3; do
  TSW_LB_CHUNK=$ch timeout 600 python bench.py --config $c --metric dtw --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/lbch${ch}_c${c}.log 2>&1; echo "chunk$ch c$c rc=$?"
  python scripts/summarize_bench.py gpurun_out/lbch${ch}_c${c}.log 2>/dev/null | head -3
done; done
