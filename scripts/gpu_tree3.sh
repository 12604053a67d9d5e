#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tree.py -q > gpurun_out/pytest_t3.log 2>&1; echo "pytest rc=$?" > gpurun_out/tree3.txt
timeout 600 python scripts/tree_bench.py --steps 4 >> gpurun_out/tree3.txt 2>&1
