#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
: > gpurun_out/quick2.txt
for SM in 1 2 0; do
for B in 1024 4096; do
  SPX_PRED_STREAM=$SM timeout 300 python bench.py --steps 20 --warmup 5 --batch $B --no-cpu-baseline --no-e2e --no-decode > gpurun_out/q2_$B.json 2>gpurun_out/q2_$B.err
  python3 -c "import json; d=json.load(open('gpurun_out/q2_$B.json')); r=d['roofline']; print('stream=$SM B=$B', round(r['us_per_launch'],2), 'us', round(r['frac'],3), 'b1', round(d['batch1_us_per_eval'],2))" >> gpurun_out/quick2.txt 2>&1
done
done
SPX_PRED_STREAM=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_quick2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick2.txt
SPX_PRED_STREAM=2 B=1024 timeout 300 python scripts/trace_predictor.py >> gpurun_out/quick2.txt 2>&1
