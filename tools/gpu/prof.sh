#!/bin/bash
# usage: bash tools/gpu/prof.sh <tag> <kind> <n> <kernel-regex> <skip> <count> [extra env assignments]
# launch list (per-kernel device time + DRAM bytes) and one ncu --set full capture
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=$1; KIND=$2; N=$3; KRE=$4; SKIP=$5; CNT=$6
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_run.py --kind $KIND --n $N --reps 2 --hostloop 1 > gpurun_out/prof_run_$TAG.log 2>&1
echo "launches rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c $CNT -o gpurun_out/prof_$TAG python tools/prof_run.py --kind $KIND --n $N --reps 2 --hostloop 1 > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
