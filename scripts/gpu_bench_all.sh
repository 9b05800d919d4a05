# bench every config (DTW and DK where the config runs both) + the subsequence-DK workloads;
# JSON lines into gpurun_out/
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo "c2 rc=$?"
python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; echo "c1 rc=$?"
for c in 3 4 5; do for m in dtw dk; do
  timeout 900 python bench.py --config $c --metric $m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c${c}_$m.log 2>&1; echo "c$c $m rc=$?"
done; done
for c in 3 5; do
  timeout 900 python bench.py --config $c --metric dk_sub --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c${c}_dk_sub.log 2>&1; echo "c$c dk_sub rc=$?"
done
