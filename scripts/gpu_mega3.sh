#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
: > gpurun_out/mega3.txt
timeout 300 python scripts/prof_layer.py --layers 4 --steps 16 >> gpurun_out/mega3.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_tree.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_mega.log 2>&1; echo "pytest rc=$?" >> gpurun_out/mega3.txt
timeout 600 python scripts/decode_bench.py --tokens 64 >> gpurun_out/mega3.txt 2>&1
