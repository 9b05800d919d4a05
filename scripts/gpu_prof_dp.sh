# profile the main DP launches (probe launch is index 0 of each execute, main is index 1)
C2="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
C4="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline"
C3K="python bench.py --config 3 --metric dk --steps 1 --warmup 1 --no-cpu-baseline"
$C2 > gpurun_out/b2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:dtw_dp_kernel -s 1 -c 1 -o gpurun_out/prof_dtw_main_c2 $C2 > gpurun_out/ncu1.log 2>&1; echo "c2 $?"
$C4 > gpurun_out/b4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:dtw_dp_kernel -s 1 -c 1 -o gpurun_out/prof_dtw_main_c4 $C4 > gpurun_out/ncu2.log 2>&1; echo "c4 $?"
$C3K > gpurun_out/b3k.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:dk_dp_kernel -s 1 -c 1 -o gpurun_out/prof_dk_main_c3 $C3K > gpurun_out/ncu3.log 2>&1; echo "c3dk $?"
