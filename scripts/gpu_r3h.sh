timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/r3h_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3h_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/gpu_bench_all.sh r3h
python scripts/summarize_bench.py "gpurun_out/r3h_bench_c*.log"
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --legs none"
$CMD > gpurun_out/r3h_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3h_launches.csv $CMD > gpurun_out/r3h_l.log 2>&1; echo "launches $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lb12_compact -s 2 -c 1 -f -o gpurun_out/r3h_lb12 $CMD > gpurun_out/r3h_f1.log 2>&1; echo "lb12 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dtw4_kernel -s 5 -c 1 -f -o gpurun_out/r3h_dtw4 $CMD > gpurun_out/r3h_f2.log 2>&1; echo "dtw4 $?"
CMD5K="python bench.py --metric dk --steps 2 --warmup 1 --no-cpu-baseline --legs none"
$CMD5K > gpurun_out/r3h_plaink.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:dk_dp_kernel -s 3 -c 1 -f -o gpurun_out/r3h_dk $CMD5K > gpurun_out/r3h_f3.log 2>&1; echo "dk $?"
