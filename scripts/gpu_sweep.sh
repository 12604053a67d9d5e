#!/usr/bin/env bash
# quick perf sweep of predictor kernel variants (env-selected), device time only
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
: > gpurun_out/sweep.txt
for cfg in "4 -1" "4 0" "3 1" "3 0" "2 1"; do
  set -- $cfg
  SPX_PRED_TEAMS=$1 SPX_PRED_W1SMEM=$2 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/sweep_$1_$2.json 2>/dev/null
  python3 -c "import json,sys; d=json.load(open('gpurun_out/sweep_$1_$2.json')); print('teams=$1 w1smem=$2', round(d['roofline']['us_per_launch'],2), 'us', round(d['roofline']['frac'],3), 'b1', round(d['batch1_us_per_eval'],2))" >> gpurun_out/sweep.txt 2>&1
done
