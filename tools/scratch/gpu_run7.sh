timeout 900 python -m pytest tests -q -m gpu --timeout 300 --timeout_method thread -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 300 python bench.py --config C3 --steps 5 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py --config C4b --steps 5 --no-cpu-baseline > gpurun_out/bench_c4b.log 2>&1
timeout 300 python bench.py --config C4c --steps 5 --no-cpu-baseline > gpurun_out/bench_c4c.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
