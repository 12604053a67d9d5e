#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
B=1024 ITERS=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:predictor_stream -s 4 -c 1 -o gpurun_out/prof_stream -f python scripts/prof_predictor.py > gpurun_out/prof_stream.log 2>&1
echo "rc=$?" >> gpurun_out/prof_stream.log
