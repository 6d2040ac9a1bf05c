cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
SH_LIB=$PWD/paper_1201_2936_b200/variants/ftrace.so python - > gpurun_out/ftrace_c4b.txt 2>&1 <<'PY'
import torch, paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate
d = tuple(torch.from_numpy(c).cuda() for c in generate("uniform-ball", 10_000_000, 0))
P.hull_indices_3d(d); torch.cuda.synchronize()
print("STATS", P.filter_stats())
PY
grep -c FT gpurun_out/ftrace_c4b.txt
for c in C4b C5; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['roofline']['kernel_ms_by_kind'])"; done
