# round-1 GPU session: bench all configs, then launch list + full captures (each ncu only
# after the identical plain command exited 0 in this same call).
set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo "c2 rc=$?"
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "c$c rc=$?"; done
timeout 600 python bench.py --config 3 --metric dk --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c3dk.log 2>&1; echo "c3dk rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:dtw_dp_kernel -s 2 -c 1 -o gpurun_out/prof_dtw_c2 $CMD > gpurun_out/ncu_full.log 2>&1
$CMD > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:lb_ub_kernel -s 2 -c 1 -o gpurun_out/prof_lb_c2 $CMD > gpurun_out/ncu_full_lb.log 2>&1
echo done
