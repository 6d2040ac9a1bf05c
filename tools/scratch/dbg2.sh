timeout 60 python tools/dbg_case.py uniform-ball-32-s1 > gpurun_out/dbg_graph.log 2>&1
echo "single rc=$?" >> gpurun_out/dbg_graph.log
timeout 120 python -m pytest tests/test_gpu_parity.py -k "golden_3d" -x -v -p no:cacheprovider > gpurun_out/dbg_golden3d.log 2>&1
echo "golden rc=$?" >> gpurun_out/dbg_golden3d.log
