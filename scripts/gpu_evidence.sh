# Round evidence on one B200.  Usage: bash scripts/gpu_evidence.sh TAG [all|quick|ncu-lb|ncu-dtw|ncu-dk]
#   all (default): GPU tests, smoke, every config benched (with CPU baselines), the C5 launch list
#   quick        : the same with the C5 bench only
#   ncu-*        : one full ncu capture (a report of the DP kernel is ~50 MB and gpurun_out/
#                  carries 64 MiB per call: one capture per gpurun call, summarised and deleted)
TAG=${1:-r2}; MODE=${2:-all}
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --legs none"
CMDK="python bench.py --metric dk --steps 2 --warmup 1 --no-cpu-baseline --legs none"
case $MODE in
ncu-lb) $CMD > gpurun_out/${TAG}_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:lb12_compact -s 2 -c 1 -f -o gpurun_out/${TAG}_lb12 $CMD > gpurun_out/${TAG}_f1.log 2>&1; echo "lb12 $?";;
ncu-dtw) $CMD > gpurun_out/${TAG}_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:dtw4_kernel -s 5 -c 1 -f -o gpurun_out/${TAG}_dtw4 $CMD > gpurun_out/${TAG}_f2.log 2>&1; echo "dtw4 $?";;
ncu-dk) $CMDK > gpurun_out/${TAG}_plaink.log 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:dk_dp_kernel -s 3 -c 1 -f -o gpurun_out/${TAG}_dk $CMDK > gpurun_out/${TAG}_f3.log 2>&1; echo "dk $?";;
*)
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
if [ "$MODE" = all ]; then bash scripts/gpu_bench_all.sh ${TAG}; else
  timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c5.log 2>&1; echo "c5 rc=$?"; fi
python scripts/summarize_bench.py "gpurun_out/${TAG}_bench_c*.log"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_l.log 2>&1; echo "launches $?"
;;
esac
