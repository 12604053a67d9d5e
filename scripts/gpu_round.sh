#!/usr/bin/env bash
# One GPU session: tests, smoke, bench, launch list, ncu captures.  Outputs in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
: > gpurun_out/status.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench_ref rc=$?" >> gpurun_out/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-decode > gpurun_out/ncu_bench.log 2>&1; echo "ncu_list rc=$?" >> gpurun_out/status.txt
B=1024 ITERS=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:predictor_stream -s 4 -c 1 -o gpurun_out/prof_pred -f python scripts/prof_predictor.py > gpurun_out/prof_pred.log 2>&1; echo "ncu_pred rc=$?" >> gpurun_out/status.txt
ncu -i gpurun_out/prof_pred.ncu-rep --page raw --csv > gpurun_out/prof_pred_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_pred.ncu-rep --page details --csv > gpurun_out/prof_pred_details.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:layer_mega -s 2 -c 1 -o /tmp/prof_layer -f python scripts/prof_layer.py --layers 2 --steps 2 > gpurun_out/prof_layer.log 2>&1; echo "ncu_layer rc=$?" >> gpurun_out/status.txt
ncu -i /tmp/prof_layer.ncu-rep --page raw --csv > gpurun_out/prof_layer_raw.csv 2>/dev/null
ncu -i /tmp/prof_layer.ncu-rep --page details --csv > gpurun_out/prof_layer_details.csv 2>/dev/null
ls -la gpurun_out >> gpurun_out/status.txt; du -sh gpurun_out >> gpurun_out/status.txt
