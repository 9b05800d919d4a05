C3K="python bench.py --config 3 --metric dk --steps 1 --warmup 3 --no-cpu-baseline"
$C3K > gpurun_out/p_c3dk_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:dk_dp_kernel -s 1 -c 1 -f -o gpurun_out/prof_dk_dp_c3 $C3K > gpurun_out/p_c3dk.log 2>&1; echo "c3 dk full $?"
