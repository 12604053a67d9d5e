#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
: > gpurun_out/cps.txt
for C in 2 1; do for B in 1024 4096; do
  SPX_PRED_CTAS_PER_SM=$C timeout 300 python bench.py --steps 20 --warmup 5 --batch $B --no-cpu-baseline --no-e2e --no-decode > gpurun_out/c_$B.json 2>/dev/null
  python3 -c "import json; d=json.load(open('gpurun_out/c_$B.json')); r=d['roofline']; print('cps=$C B=$B', round(r['us_per_launch'],2), 'us', round(r['frac'],3), 'b1', round(d['batch1_us_per_eval'],2))" >> gpurun_out/cps.txt 2>&1
done; done
