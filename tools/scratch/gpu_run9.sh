timeout 600 python -m pytest tests/test_primitives.py -q -m gpu --timeout 300 --timeout_method thread -p no:cacheprovider > gpurun_out/pytest_prims.log 2>&1
