#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/final2_pytest.log 2>&1; echo "pytest rc=$?" > gpurun_out/final2.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/final2.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final2_bench.json 2> gpurun_out/final2_bench.err; echo "bench rc=$?" >> gpurun_out/final2.txt
