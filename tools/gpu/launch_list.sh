#!/bin/bash
# ncu launch lists (device time, DRAM bytes, instructions per launch) of one
# measured hull: bash tools/gpu/launch_list.sh "<tag:kind:n> ..."
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for spec in $1; do
  IFS=: read tag kind n <<< "$spec"
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/ll_$tag.csv python tools/prof_run.py --kind $kind --n $n --reps 2 --hostloop 1 > gpurun_out/ll_$tag.log 2>&1
  echo "$tag rc=$?"
done
