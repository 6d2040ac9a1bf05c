timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 5 --sharded > gpurun_out/bench_sharded1.log 2>&1
timeout 600 python bench.py --steps 10 > gpurun_out/bench_c2.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
