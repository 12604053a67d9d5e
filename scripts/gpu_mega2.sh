#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
: > gpurun_out/mega2.txt
for DBG in 0 1; do
  echo "dbg=$DBG" >> gpurun_out/mega2.txt
  SPX_MEGA_DBG=$DBG timeout 300 python scripts/prof_layer.py --layers 4 --steps 16 >> gpurun_out/mega2.txt 2>&1
done
