CMD="python bench.py --config 3 --metric dk --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/l3_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3dk.csv $CMD > gpurun_out/l3.log 2>&1; echo "rc $?"
