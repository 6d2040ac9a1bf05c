#!/bin/bash
# r2: smoke + parity suite + A/B bench (stream kernel vs register-prefetch kernels)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout -s KILL 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for cfg in C2 C4b; do
  timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $cfg > gpurun_out/b_new_$cfg.json 2> gpurun_out/b_new_$cfg.err; echo "new $cfg rc=$?"
  SH_STREAM=0 timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $cfg > gpurun_out/b_old_$cfg.json 2>gpurun_out/b_old_$cfg.err; echo "old $cfg rc=$?"
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/b_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        r=d["roofline"]; print(f, d["ms_per_step"], r["per_round_gbs"][:5], r["kernel_ms_by_kind"])
    except Exception as e: print(f, "ERR", e)
PY
