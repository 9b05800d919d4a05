CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --legs none"
$CMD > gpurun_out/r2n_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:dtw4_kernel -s 5 -c 1 -f -o gpurun_out/r2n_dtw4 $CMD > gpurun_out/r2n_f.log 2>&1; echo "dtw4 $?"
ncu -i gpurun_out/r2n_dtw4.ncu-rep --page raw --csv 2>/dev/null | python -c "import csv,sys; r=list(csv.reader(sys.stdin)); h=r[0]; print([ (h[i], x[i]) for x in r[2:] for i in range(len(h)) if h[i] in ('launch__grid_size','gpu__time_duration.sum')])"
