set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 10 > gpurun_out/bench_c2.log 2>&1
timeout 600 python bench.py --config C4b --steps 5 > gpurun_out/bench_c4b.log 2>&1
timeout 600 python bench.py --config C3 --steps 5 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
