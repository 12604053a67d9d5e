#!/usr/bin/env bash
# Profiling session: full ncu capture of the fused predictor kernel, 7B decode
# tok/s through the device engine, decoder-layer timing.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:predictor_fast -s 2 -c 1 -o gpurun_out/prof_pred -f python scripts/prof_predictor.py > gpurun_out/prof_pred.log 2>&1; echo "ncu_pred rc=$?" >> gpurun_out/status2.txt
timeout 900 python scripts/decode_bench.py --tokens 64 > gpurun_out/decode_7b.log 2>&1; echo "decode rc=$?" >> gpurun_out/status2.txt
timeout 900 python scripts/decode_bench.py --tokens 64 --thr 0.7 > gpurun_out/decode_7b_thr07.log 2>&1; echo "decode07 rc=$?" >> gpurun_out/status2.txt
timeout 600 python scripts/prof_layer.py --layers 4 --steps 16 > gpurun_out/layer_7b.log 2>&1; echo "layer rc=$?" >> gpurun_out/status2.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/layer_launches.csv python scripts/prof_layer.py --layers 2 --steps 2 > gpurun_out/layer_ncu.log 2>&1; echo "layer_ncu rc=$?" >> gpurun_out/status2.txt
