#!/usr/bin/env bash
# One GPU session: tests, smoke, bench, launch list.  Outputs in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
python -c "import numpy; numpy.show_config()" > gpurun_out/numpy_config.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?" >> gpurun_out/status.txt
timeout 300 python -m pytest tests/test_numerics_port.py -q > gpurun_out/pytest_numerics_host.log 2>&1; echo "numerics_host rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo "ncu_list rc=$?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:predictor_fast -s 2 -c 1 -o gpurun_out/prof_pred python scripts/prof_predictor.py > gpurun_out/prof_pred.log 2>&1; echo "ncu_full rc=$?" >> gpurun_out/status.txt
