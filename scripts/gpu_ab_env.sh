# A/B an environment variable over bench configs: items "config:metric:VAR=value" (VAR=value optional)
for it in "$@"; do
  IFS=: read c m kv <<< "$it"
  tag=c${c}_${m}${kv:+_$kv}
  env $kv timeout 900 python bench.py --config $c --metric $m --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$tag.log 2>&1; echo "$tag rc=$?"
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{t}.log").read().strip().splitlines()[-1])
    print(t, round(d["ms_per_step"], 3), d["dp_pairs_per_step"], {k: round(v, 3) for k, v in d["phases_ms"].items()})
except Exception as e:
    print(t, "unreadable", e)
PY
done
