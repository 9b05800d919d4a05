# ncu capture of the C2 DTW fast-path main launch for the given variants
for v in "$@"; do
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
  TSW_DTW4=$v $CMD > gpurun_out/p_plain_$v.log 2>&1 && \
  TSW_DTW4=$v ncu --set full --clock-control none --import-source on -k regex:dtw4_kernel -s 1 -c 1 -o gpurun_out/prof_dtw4_c2_$v -f $CMD > gpurun_out/p_ncu_$v.log 2>&1; echo "ncu $v $?"
done
