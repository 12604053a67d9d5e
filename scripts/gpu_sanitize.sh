#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
for tool in racecheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python scripts/sanitize_smoke.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize.txt
  tail -n 3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize.txt
done
