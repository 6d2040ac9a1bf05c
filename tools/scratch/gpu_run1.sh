set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_run.py --kind uniform-disk --n 100000000 --reps 2 --hostloop 1 > gpurun_out/prof_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_round -s 13 -c 3 -o gpurun_out/prof_round_c2 python tools/prof_run.py --kind uniform-disk --n 100000000 --reps 2 --hostloop 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_c2.log | tail -2
