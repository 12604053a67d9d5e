#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
: > gpurun_out/layer.txt
for TC in 1 0; do
  SPX_LAYER_TC=$TC timeout 300 python scripts/prof_layer.py --layers 4 --steps 16 >> gpurun_out/layer.txt 2>&1
  SPX_LAYER_TC=$TC timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/layer_tc$TC.csv python scripts/prof_layer.py --layers 2 --steps 2 > /dev/null 2>&1
  python scripts/summarize_launches.py gpurun_out/layer_tc$TC.csv | grep -E "gemv|attn" >> gpurun_out/layer.txt
done
