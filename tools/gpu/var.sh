#!/bin/bash
# usage: bash tools/gpu/var.sh "<cfgs>" "<variants>"   (variant "main" = the in-tree library)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in $2; do
  for cfg in $1; do
    if [ "$v" = main ]; then L=""; else L="$PWD/paper_1201_2936_b200/variants/$v.so"; fi
    SH_LIB=$L timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $cfg > gpurun_out/v_${v}_$cfg.json 2> gpurun_out/v_${v}_$cfg.err
    python - "$v" "$cfg" <<'PY'
import json,sys
v,c=sys.argv[1:3]
try:
    d=json.loads(open(f"gpurun_out/v_{v}_{c}.json").read().strip().splitlines()[-1]); r=d["roofline"]
    print(v, c, d["ms_per_step"], "frac", r["frac"], r["per_round_gbs"][:6], r["kernel_ms_by_kind"])
except Exception as e: print(v, c, "ERR", e, open(f"gpurun_out/v_{v}_{c}.err").read()[-800:])
PY
  done
done
