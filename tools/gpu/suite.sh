#!/bin/bash
# full GPU suite + bench lines (default C2, C5 strong on 1 GPU, C2 sharded at N=1, C4b)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
for a in "C2" "C4b" "C5"; do
  timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $a > gpurun_out/b_$a.json 2> gpurun_out/b_$a.err; echo "$a rc=$?"
done
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --sharded --config C2 > gpurun_out/b_C2sh.json 2> gpurun_out/b_C2sh.err; echo "C2sh rc=$?"
python - <<'PY'
import json
for c in ("C2", "C4b", "C5", "C2sh"):
    try:
        d = json.loads(open(f"gpurun_out/b_{c}.json").read().strip().splitlines()[-1]); r = d["roofline"]
        print(c, d["ms_per_step"], "value", d["value"], "e2e", d["e2e"]["value"], "frac", r["frac"], r["per_round_gbs"][:6], r["kernel_ms_by_kind"], "clocks", d["clocks"])
    except Exception as e:
        print(c, "ERR", e, open(f"gpurun_out/b_{c}.err").read()[-1500:])
PY
