#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/last_pytest.log 2>&1; echo "pytest rc=$?" > gpurun_out/last.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/last.txt 2>&1
timeout 300 python scripts/prof_layer.py --layers 4 --steps 16 >> gpurun_out/last.txt 2>&1
timeout 600 python scripts/decode_bench.py --tokens 64 >> gpurun_out/last.txt 2>&1
