"""CPU: bench.py's reference arm (the reference's own CPU implementation of the path) runs
here and prints the driver's JSON contract."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.5"], cwd=ROOT,
                         capture_output=True, text=True, timeout=600, check=True).stdout
    line = json.loads(out.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "queries/s"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert line["config"]["workload"].startswith("config1")


def test_reference_arm_maps_only_oracle_libraries():
    """The reference arm must not load the product library (it makes its inputs with the
    generator built into oracle/_build)."""
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.3"], cwd=ROOT,
                         capture_output=True, text=True, timeout=600, check=True).stdout
    line = json.loads(out.strip().splitlines()[-1])
    libs = line["native_libraries"]
    assert libs and all(p.startswith("oracle/") for p in libs), libs
    assert "execution" not in line["config"]


def test_oracle_generator_matches_product_generator():
    sys.path.insert(0, ROOT)
    import numpy as np

    import oracle
    import paper_1811_11076_b200 as t

    for cfg in (1, 2, 3):
        for part in (0, 1):
            assert oracle.synth_shape(cfg, part) == t.synth_shape(cfg, part)
            if cfg == 3 and part == 0:
                continue  # 50k x 256 x 2: the shape check is enough for the big one
            a, la = oracle.synth(cfg, part)
            b, lb = t.synth(cfg, part)
            assert np.array_equal(a, b) and np.array_equal(la, lb)
