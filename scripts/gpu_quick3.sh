#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
: > gpurun_out/quick3.txt
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -q > gpurun_out/pytest_q3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick3.txt
for B in 1024 4096; do
  timeout 300 python bench.py --steps 20 --warmup 5 --batch $B --no-cpu-baseline --no-e2e --no-decode > gpurun_out/q3_$B.json 2>/dev/null
  python3 -c "import json; d=json.load(open('gpurun_out/q3_$B.json')); r=d['roofline']; print('B=$B', round(r['us_per_launch'],2), 'us', round(r['frac'],3), 'b1', round(d['batch1_us_per_eval'],2))" >> gpurun_out/quick3.txt 2>&1
done
