mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ev/gpu.txt 2>&1
lscpu | head -20 > gpurun_out/ev/host_cpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1
timeout 900 python -m pytest tests -q -m gpu --timeout 300 --timeout_method thread -p no:cacheprovider > gpurun_out/ev/pytest_gpu.log 2>&1
timeout 300 python bench.py > gpurun_out/ev/bench_c2.json 2>gpurun_out/ev/bench_c2.err
timeout 300 python bench.py --impl reference > gpurun_out/ev/bench_ref.json 2>gpurun_out/ev/bench_ref.err
for c in C1 C3 C3n C4c C4b; do timeout 300 python bench.py --config $c --steps 5 > gpurun_out/ev/bench_$c.json 2>gpurun_out/ev/bench_$c.err; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev/launches_c2.csv python tools/prof_run.py --kind uniform-disk --n 100000000 --reps 2 --hostloop 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_round -s 13 -c 3 -o gpurun_out/ev/prof_round_c2 python tools/prof_run.py --kind uniform-disk --n 100000000 --reps 2 --hostloop 1 > /dev/null 2>&1
