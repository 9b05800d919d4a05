C5T="python bench.py --config 5 --metric dtw --steps 1 --warmup 3 --no-cpu-baseline"
$C5T > gpurun_out/p_c5dtw_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:dtw4_kernel -s 3 -c 1 -f -o gpurun_out/prof_dtw_dp_c5 $C5T > gpurun_out/p_c5dtw.log 2>&1; echo "c5 dtw dp full $?"
