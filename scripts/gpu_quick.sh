#!/usr/bin/env bash
# quick predictor timing: batch sweep + phase trace
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
: > gpurun_out/quick.txt
for B in 1024 148; do
  timeout 300 python bench.py --steps 20 --warmup 5 --batch $B --no-cpu-baseline --no-e2e --no-decode > gpurun_out/q_$B.json 2>gpurun_out/q_$B.err
  python3 -c "import json; d=json.load(open('gpurun_out/q_$B.json')); r=d['roofline']; print('B=$B', round(r['us_per_launch'],2), 'us', round(r['frac'],3), 'b1', round(d['batch1_us_per_eval'],2))" >> gpurun_out/quick.txt 2>&1
done
timeout 300 python scripts/trace_predictor.py >> gpurun_out/quick.txt 2>&1
B=148 timeout 300 python scripts/trace_predictor.py >> gpurun_out/quick.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_tree.py -q -x > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick.txt
