# ncu --set full capture of one launch of kernel regex $1 (skip $2 launches) in bench config $3 metric $4
K=$1; SKIP=${2:-0}; CFG=${3:-2}; MET=${4:-dtw}; TAG=${5:-$K}
CMD="python bench.py --config $CFG --metric $MET --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/pk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -f -o gpurun_out/prof_$TAG $CMD > gpurun_out/pk_ncu.log 2>&1; echo "ncu $K $?"
