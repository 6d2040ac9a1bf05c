#!/bin/bash
# k_tail variants: env settings x configs (bench ms/hull)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
run() {  # tag, config, env...
  local tag=$1 c=$2; shift 2
  env "$@" timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config $c > gpurun_out/tv_${c}_$tag.json 2> gpurun_out/tv_${c}_$tag.err
  python -c "
import json
try:
    d=json.loads(open('gpurun_out/tv_${c}_$tag.json').read().strip().splitlines()[-1]); print('$c $tag', d['ms_per_step'])
except Exception as e: print('$c $tag ERR', e, open('gpurun_out/tv_${c}_$tag.err').read()[-600:])"
}
for c in ${CONFIGS:-C1 C2 C4b}; do
  run notail $c SH_NO_TAIL=1
  run empty $c SH_TAIL_MAX_CHILDREN=0
  run tail $c X=1
  run occ2 $c SH_TAIL_OCC=2
  run live200k $c SH_TAIL_MAX_LIVE=200000
  run notail2 $c SH_NO_TAIL=1
done
