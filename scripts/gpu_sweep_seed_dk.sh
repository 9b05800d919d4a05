# seed sample size sweep on the DK configs (same box)
for rep in 1 2; do for S in 2048 1024 512; do for c in 1 3 4 5; do
  st=10; [ $c -ge 5 ] && st=3
  TSW_SAMPLE=$S timeout 600 python bench.py --config $c --metric dk --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/swdk.log 2>&1
  echo "rep$rep S=$S c$c $(python scripts/summarize_bench.py gpurun_out/swdk.log 2>/dev/null | cut -c24-140)"
done; done; done
