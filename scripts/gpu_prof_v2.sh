# bench config 3 (previous timeout) + main-DP ncu captures for configs 2 (DTW) / 4 (DTW) / 5 (DK)
timeout 300 python bench.py --config 3 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c3_dtw.log 2>&1; echo "c3 rc=$?"
C2="python scripts/diag_config.py 2 dtw 64"
C4="python scripts/diag_config.py 4 dtw 8"
C5K="python scripts/diag_config.py 5 dk 4"
timeout 300 $C2 > gpurun_out/d2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:dtw_dp_kernel -s 3 -c 1 -o gpurun_out/prof2_dtw_c2 $C2 > gpurun_out/n1.log 2>&1; echo "p2 $?"
timeout 300 $C4 > gpurun_out/d4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:dtw_dp_kernel -s 3 -c 1 -o gpurun_out/prof2_dtw_c4 $C4 > gpurun_out/n2.log 2>&1; echo "p4 $?"
timeout 300 $C5K > gpurun_out/d5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:dk_dp_kernel -s 3 -c 1 -o gpurun_out/prof2_dk_c5 $C5K > gpurun_out/n3.log 2>&1; echo "p5 $?"
