#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:predictor_fast -s 2 -c 1 -o gpurun_out/prof_pred python scripts/prof_predictor.py > gpurun_out/prof_pred.log 2>&1
echo "rc=$?" >> gpurun_out/prof_pred.log
