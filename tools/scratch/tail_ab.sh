#!/bin/bash
# k_tail A/B: parity subset, then bench lines with and without the tail kernel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "random or golden or full" > gpurun_out/tail_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/tail_pytest.log
for c in ${CONFIGS:-C1 C2 C3 C3n C4c C4b}; do
  for v in tail notail; do
    if [ $v = notail ]; then export SH_NO_TAIL=1; else unset SH_NO_TAIL; fi
    timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config $c > gpurun_out/ta_${c}_$v.json 2> gpurun_out/ta_${c}_$v.err
    python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/ta_${c}_$v.json').read().strip().splitlines()[-1]); print('$c $v', d['ms_per_step'], d['config'].get('rounds'), d['config'].get('hull'))
except Exception as e: print('$c $v ERR', e, open('gpurun_out/ta_${c}_$v.err').read()[-800:])"
  done
done
