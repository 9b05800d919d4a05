# Same-box A/B of library builds / env switches:
#   bash scripts/ab.sh "cfg:metric ..." REPS "label=ENV=VAL,ENV=VAL" "label2=" ...
# e.g. bash scripts/ab.sh "2:dtw 5:dtw" 2 "base=TSW_LIB=build_var/base/libtswarp_b200.so" "cur="
CASES=$1; REPS=$2; shift 2
for rep in $(seq 1 $REPS); do for v in "$@"; do for cm in $CASES; do
  label=${v%%=*}; envs=${v#*=}; c=${cm%%:*}; m=${cm##*:}; st=10; [ "$c" -ge 4 ] && st=4
  env $(echo $envs | tr ',' ' ') timeout 600 python bench.py --config $c --metric $m --legs none --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/ab_run.log 2>&1
  echo "rep$rep $label c$c $m $(python scripts/summarize_bench.py gpurun_out/ab_run.log 2>&1 | head -1 | cut -c28-250)"
done; done; done
