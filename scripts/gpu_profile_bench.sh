# ncu evidence for the default bench workload (config 2) and the DK DP (config 5); each ncu run
# follows a successful plain run of the identical command in this call.
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/prof_l.log 2>&1; echo "launches $?"
$CMD > gpurun_out/prof_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:dtw4_kernel -s 1 -c 1 -f -o gpurun_out/prof_dtw_dp_c2 $CMD > gpurun_out/prof_f1.log 2>&1; echo "dtw full $?"
$CMD > gpurun_out/prof_plain3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"lb_(env|compact)_kernel" -s 0 -c 1 -f -o gpurun_out/prof_lb_c2 $CMD > gpurun_out/prof_f2.log 2>&1; echo "lb full $?"
C5K="python bench.py --config 5 --metric dk --steps 1 --warmup 3 --no-cpu-baseline"
$C5K > gpurun_out/prof_plain4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:dk_dp_kernel -s 1 -c 1 -f -o gpurun_out/prof_dk_dp_c5 $C5K > gpurun_out/prof_f3.log 2>&1; echo "dk full $?"
C5T="python bench.py --config 5 --metric dtw --steps 1 --warmup 3 --no-cpu-baseline"
$C5T > gpurun_out/prof_plain5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:lb12_compact_kernel -s 0 -c 1 -f -o gpurun_out/prof_lb12_c5 $C5T > gpurun_out/prof_f4.log 2>&1; echo "lb12 full $?"
C4T="python bench.py --config 4 --metric dtw --steps 1 --warmup 3 --no-cpu-baseline"
$C4T > gpurun_out/prof_plain6.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:dtwt_kernel -s 1 -c 1 -f -o gpurun_out/prof_dtwt_c4 $C4T > gpurun_out/prof_f5.log 2>&1; echo "dtwt full $?"
C3S="python bench.py --config 3 --metric dk_sub --steps 1 --warmup 3 --no-cpu-baseline"
$C3S > gpurun_out/prof_plain7.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:dk_dp_kernel -s 1 -c 1 -f -o gpurun_out/prof_dk_sub_c3 $C3S > gpurun_out/prof_f6.log 2>&1; echo "dk sub full $?"
