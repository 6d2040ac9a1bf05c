timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 600 python bench.py --config C3 --steps 5 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
bash tools/gpu_prof.sh c2v3 uniform-disk 100000000 k_round 13 3
tail -3 gpurun_out/pytest_gpu.log
