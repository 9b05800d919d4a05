# ncu: C5 launch list + full captures of lb12 and dtw4 (each after a clean plain run)
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --legs none"
$CMD > gpurun_out/r2m_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2m_launches.csv $CMD > gpurun_out/r2m_l.log 2>&1; echo "launches $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lb12_compact -s 2 -c 1 -f -o gpurun_out/r2m_lb12 $CMD > gpurun_out/r2m_f1.log 2>&1; echo "lb12 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dtw4_kernel -s 4 -c 1 -f -o gpurun_out/r2m_dtw4 $CMD > gpurun_out/r2m_f2.log 2>&1; echo "dtw4 $?"
