# A/B of the DK rows-per-lane choice at the small-L configs
for r in 2 4; do for c in 1 3; do
  TSW_DK_RPL=$r timeout 600 python bench.py --config $c --metric dk --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/rpl${r}_c${c}.log 2>&1; echo "rpl$r c$c rc=$?"
  python scripts/summarize_bench.py gpurun_out/rpl${r}_c${c}.log 2>/dev/null | head -3
done; done
