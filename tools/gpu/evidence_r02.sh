#!/bin/bash
# Round-2 evidence: launch lists (time + DRAM bytes per launch, host-loop
# hull), ncu --set full of the streaming round kernels, bench lines.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02; mkdir -p $O
for cfg in "unit-square 1000000 C1" "uniform-disk 100000000 C2" "on-circle 10000000 C3" "near-circle 10000000 C3n" "unit-cube 10000000 C4c" "uniform-ball 10000000 C4b" "uniform-ball 200000000 C5"; do
  set -- $cfg
  timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file $O/launches_$3.csv python tools/ncu_round.py $1 $2 > /dev/null 2>&1
  echo "launches $3 rc=$?"
done
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_stream -s 4 -c 2 -o $O/full_C2_stream python tools/prof_run.py --kind uniform-disk --n 100000000 --reps 2 --hostloop 1 > $O/full_C2.log 2>&1; echo "full C2 rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"k_stream|k_f_test|k_f_local|k_f_cert" -s 8 -c 5 -o $O/full_C4b python tools/prof_run.py --kind uniform-ball --n 10000000 --reps 2 --hostloop 1 > $O/full_C4b.log 2>&1; echo "full C4b rc=$?"
for a in C1 C2 C3 C3n C4c C4b C5; do
  timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --config $a > $O/bench_$a.json 2> $O/bench_$a.err; echo "bench $a rc=$?"
done
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --sharded --config C2 --no-cpu-baseline > $O/bench_C2_sharded.json 2> $O/bench_C2_sharded.err; echo "bench C2 sharded rc=$?"
timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 1 --config C2 > $O/bench_ref_C2.json 2> $O/bench_ref_C2.err; echo "ref rc=$?"
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > $O/gpu.txt
lscpu | head -20 > $O/host_cpu.txt
