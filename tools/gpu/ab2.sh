#!/bin/bash
# parity subset + A/B bench of the in-tree library against variants/<v>.so
# usage: bash tools/gpu/ab2.sh "<cfgs>" "<variants>" [pytest -k expr]
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
if [ -n "$3" ]; then
  timeout -s KILL 1200 python -m pytest tests -m gpu -x -q -k "$3" > gpurun_out/ab2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab2_pytest.log
fi
bash tools/gpu/var.sh "$1" "$2"
