"""Summarise bench JSON lines (gpurun_out/bench_*.log) into a compact table."""
import glob
import json
import sys

rows = []
for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench_*.log")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f"{f}: unreadable ({e})")
        continue
    c = d["config"]
    ph = d["phases_ms"]
    rdp, rlb = d["roofline_dp"], d["roofline_lb"]
    print(f"{f.split('/')[-1]:22s} cfg{c['config_id']} {c['metric']:3s} q/s={d['value']:10.1f} "
          f"ms/step={d['ms_per_step']:8.3f} e2e={d['e2e']['value']:10.1f} "
          f"bound={ph['ms_bound']:.3f} sel={ph['ms_select']:.3f} probe={ph['ms_probe_dp']:.3f} "
          f"dp={ph['ms_dp']:.3f} | GCUPS={rdp['gcups'] or 0:7.1f} fp64frac={rdp['frac'] or 0:.3f} "
          f"LB GB/s={rlb['achieved'] or 0:7.1f} pairs={d['dp_pairs_per_step']:.0f} "
          f"cpu={d.get('cpu_baseline', {}).get('value')} clk={d['clocks'].get('sm_mhz')}")
    for m, lg in d.get("legs", {}).items():
        print(f"{'  leg ' + m:22s} q/s={lg['value']:10.1f} ms/step={lg['ms_per_step']:8.3f} "
              f"e2e={lg['e2e']['value']:10.1f} dp={lg['phases_ms']['ms_dp']:.3f} "
              f"fp64frac={lg['roofline_dp']['frac'] or 0:.3f} cpu={lg.get('cpu_baseline', {}).get('value')}")
