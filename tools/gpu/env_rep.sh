#!/bin/bash
# interleaved repetitions over environment settings: bash tools/gpu/env_rep.sh "<cfgs>" "<tag=VAR=val ...>" <reps>
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for r in $(seq 1 $3); do
  for spec in $2; do
    tag=${spec%%=*}; kv=${spec#*=}
    for cfg in $1; do
      env $kv timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $cfg > gpurun_out/e_${tag}_$cfg.json 2> /dev/null
      python -c "
import json
try:
    d=json.loads(open('gpurun_out/e_${tag}_$cfg.json').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms_by_kind']
    print('REP $tag $cfg', d['ms_per_step'], k.get('round'), k.get('book'))
except Exception as e: print('REP $tag $cfg ERR', e)"
    done
  done
done
