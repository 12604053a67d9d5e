#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
: > gpurun_out/knobs.txt
for PDL in 2 1 0; do
  SPX_PDL=$PDL timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-decode > gpurun_out/k.json 2>/dev/null
  python3 -c "import json; d=json.load(open('gpurun_out/k.json')); r=d['roofline']; print('pdl=$PDL', round(r['us_per_launch'],2), 'us', round(r['frac'],3))" >> gpurun_out/knobs.txt 2>&1
done
