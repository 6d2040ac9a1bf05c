#!/bin/bash
# interleaved repetitions: bash tools/gpu/rep.sh "<cfgs>" "<variants>" <reps>
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for r in $(seq 1 $3); do
  for v in $2; do
    for cfg in $1; do
      if [ "$v" = main ]; then L=""; else L="$PWD/paper_1201_2936_b200/variants/$v.so"; fi
      SH_LIB=$L timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $cfg > gpurun_out/r_${v}_$cfg.json 2> /dev/null
      python -c "
import json
try:
    d=json.loads(open('gpurun_out/r_${v}_$cfg.json').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms_by_kind']
    print('REP $v $cfg', d['ms_per_step'], k.get('filter'), k.get('round'), k.get('book'))
except Exception as e: print('REP $v $cfg ERR', e)"
    done
  done
done
