"""CPU: bench.py's reference arm runs here (the oracle port on the host) and
prints one JSON line with the driver's keys; the GPU arm's line is checked
in profiles/r01/bench_*.json (written by the same code on a B200)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C1", "--steps", "1",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d) and d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0


def test_committed_gpu_bench_lines_have_the_contract_keys():
    for name in ("bench_c2.json", "bench_C4b.json", "bench_C5.json"):
        d = json.loads(open(os.path.join(ROOT, "profiles", "r01", name)).read().strip().splitlines()[-1])
        assert KEYS <= set(d)
        for k in ("gpu_launches", "roofline", "clocks"):
            assert k in d
        roof = d["roofline"]
        assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(roof)
        assert 0 < roof["frac"] < 1
        assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
