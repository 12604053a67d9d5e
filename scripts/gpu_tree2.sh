#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
: > gpurun_out/tree2.txt
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_t2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/tree2.txt
timeout 600 python scripts/tree_bench.py --steps 4 >> gpurun_out/tree2.txt 2>&1
timeout 300 python scripts/prof_layer.py --layers 4 --steps 16 >> gpurun_out/tree2.txt 2>&1
timeout 600 python scripts/decode_bench.py --tokens 64 >> gpurun_out/tree2.txt 2>&1
