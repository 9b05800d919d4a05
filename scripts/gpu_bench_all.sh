# bench every config (DTW line + DK leg where the config runs both; C1 is DK only) with the
# host-core CPU baseline, plus the subsequence-DK workloads; JSON lines into gpurun_out/
TAG=${1:-r2}
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c5.log 2>&1; echo "c5 rc=$?"
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c1.log 2>&1; echo "c1 rc=$?"
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c2.log 2>&1; echo "c2 rc=$?"
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c3.log 2>&1; echo "c3 rc=$?"
timeout 1200 python bench.py --config 4 --steps 4 --warmup 3 > gpurun_out/${TAG}_bench_c4.log 2>&1; echo "c4 rc=$?"
for c in 3 5; do
  timeout 900 python bench.py --config $c --metric dk_sub --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/${TAG}_bench_c${c}_dk_sub.log 2>&1; echo "c$c dk_sub rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_reference_c5.log 2>&1; echo "ref c5 rc=$?"
