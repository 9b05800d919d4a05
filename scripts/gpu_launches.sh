# ncu launch list (gpu__time_duration per kernel) of one short bench run, after a plain run
CFG=${1:-2}; MET=${2:-dtw}
CMD="python bench.py --config $CFG --metric $MET --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/l_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c${CFG}_${MET}.csv $CMD > gpurun_out/l_ncu.log 2>&1; echo "launches $?"
