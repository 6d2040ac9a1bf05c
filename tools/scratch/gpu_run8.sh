timeout 200 python tools/filter_diag.py > gpurun_out/filter_diag.log 2>&1
timeout 400 python -m pytest tests -q -m gpu -k "3d or C4 or sharded" --timeout 300 --timeout_method thread -p no:cacheprovider -x > gpurun_out/pytest3d.log 2>&1
