#!/bin/bash
# usage: bash tools/gpu/ab.sh <cfgs> [prof-tag kind n kregex skip count]
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for cfg in $1; do
  timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $cfg > gpurun_out/b_$cfg.json 2> gpurun_out/b_$cfg.err; echo "$cfg rc=$?"
done
python - "$1" <<'PY'
import json,sys
for c in sys.argv[1].split():
    try:
        d=json.loads(open(f"gpurun_out/b_{c}.json").read().strip().splitlines()[-1]); r=d["roofline"]
        print(c, d["ms_per_step"], "frac", r["frac"], r["per_round_gbs"][:6], r["kernel_ms_by_kind"])
    except Exception as e: print(c, "ERR", e, open(f"gpurun_out/b_{c}.err").read()[-500:])
PY
if [ -n "$2" ]; then bash tools/gpu/prof.sh $2 $3 $4 $5 $6 $7; fi
