# Round evidence: bench lines for every config, the reference arm, the ncu
# launch list of the C2 bench command and a full capture of the round kernels.
set -x
O=gpurun_out/ev
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/gpu.txt
lscpu | head -20 > $O/host_cpu.txt
timeout 400 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
for c in C1 C3 C3n C4c C4b; do timeout 400 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 400 python bench.py --config C4b --facets --no-cpu-baseline > $O/bench_C4b_facets.json 2> $O/bench_C4b_facets.err
timeout 600 python bench.py --config C5 --steps 5 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_round" -c 4 -o $O/round_c2 python tools/ncu_round.py > $O/ncu_full.log 2>&1
