#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tree.py -q -x > gpurun_out/pytest_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/status3.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_all.log 2>&1; echo "gpu_all rc=$?" >> gpurun_out/status3.txt
timeout 600 python scripts/decode_bench.py --tokens 64 > gpurun_out/decode_7b.log 2>&1; echo "decode rc=$?" >> gpurun_out/status3.txt
timeout 600 python scripts/decode_bench.py --tokens 64 --thr 0.7 > gpurun_out/decode_7b_thr07.log 2>&1; echo "decode07 rc=$?" >> gpurun_out/status3.txt
timeout 600 python scripts/prof_layer.py --layers 4 --steps 16 > gpurun_out/layer_7b.log 2>&1; echo "layer rc=$?" >> gpurun_out/status3.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/layer_launches.csv python scripts/prof_layer.py --layers 2 --steps 2 > gpurun_out/layer_ncu.log 2>&1; echo "layer_ncu rc=$?" >> gpurun_out/status3.txt
