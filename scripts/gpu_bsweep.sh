#!/usr/bin/env bash
# predictor launch time vs batch (ramp vs steady state), device time only
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
: > gpurun_out/bsweep.txt
for B in 148 296 592 1024 2048 4096 8192; do
  timeout 300 python bench.py --steps 20 --warmup 5 --batch $B --no-cpu-baseline --no-e2e > gpurun_out/bs_$B.json 2>/dev/null
  python3 -c "import json; d=json.load(open('gpurun_out/bs_$B.json')); r=d['roofline']; print('B=$B', round(r['us_per_launch'],2), 'us', round(r['frac'],3))" >> gpurun_out/bsweep.txt 2>&1
done
timeout 300 python scripts/trace_predictor.py > gpurun_out/trace_pred.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?" >> gpurun_out/bsweep.txt
