#!/usr/bin/env bash
# One parameterised GPU session (run under gpurun).  Usage:
#   scripts/gpu.sh STAGE [STAGE ...]
# Stages (each bounded by its own timeout; outputs in gpurun_out/, status lines
# in gpurun_out/status.txt):
#   info        nvidia-smi clocks + lscpu
#   test        pytest -m gpu (all GPU tests)
#   test:PATH   pytest -m gpu on one file / node id (e.g. test:tests/test_gpu_stream.py)
#   smoke       __graft_entry__.smoke()
#   bench       bench.py --steps 20 --warmup 5  (N=1, every leg)
#   benchref    bench.py --impl reference --steps 3 --warmup 1
#   pred        bench.py predictor leg only (no cpu baseline, no e2e, no decode)
#   sweep       scripts/predictor_sweep.py over configs[4]
#   decode      scripts/decode_bench.py --tokens 64 (thr 0.5 and injected spec)
#   tree        scripts/tree_bench.py --steps 4
#   layer       scripts/prof_layer.py --layers 4 --steps 16
#   launches    ncu launch list of the predictor bench leg
#   ncupred     ncu --set full of one predictor_stream launch (B=1024)
#   ncugather   ncu --set full of one pipelined gather launch (B=1024)
#   ncuverify   ncu --set full of one verify launch (1 row, 7B head)
#   ncutree     ncu --set full of one tree-merged launch
#   nculayer    ncu --set full of one layer_mega launch
#   sanitize    compute-sanitizer memcheck/racecheck on scripts/sanitize_smoke.py
# Extra environment is passed through (e.g. SPX_PDL=1 scripts/gpu.sh pred).
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
ST=gpurun_out/status.txt
TAG=${TAG:-run}
note() { echo "$1 rc=$2" >> $ST; }
ncu_csv() { ncu -i "$1" --page raw --csv > "${1%.ncu-rep}_raw.csv" 2>/dev/null;
            ncu -i "$1" --page details --csv > "${1%.ncu-rep}_details.csv" 2>/dev/null; }
for stage in "$@"; do
  case "$stage" in
    info) nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/gpu.txt 2>&1
          lscpu > gpurun_out/lscpu.txt 2>&1; note info 0 ;;
    test) timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; note test $? ;;
    test:*) timeout 1200 python -m pytest "${stage#test:}" -q -m gpu > gpurun_out/${TAG}_pytest_part.log 2>&1; note "$stage" $? ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; note smoke $? ;;
    bench) timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; note bench $? ;;
    benchref) timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; note benchref $? ;;
    pred) timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-decode ${BENCH_ARGS:-} > gpurun_out/${TAG}_pred.json 2> gpurun_out/${TAG}_pred.err; note pred $? ;;
    sweep) timeout 1200 python scripts/predictor_sweep.py > gpurun_out/${TAG}_sweep.jsonl 2> gpurun_out/${TAG}_sweep.err; note sweep $? ;;
    decode) timeout 900 python scripts/decode_bench.py --tokens 64 > gpurun_out/${TAG}_decode.log 2>&1; note decode $?
            timeout 900 python scripts/decode_bench.py --tokens 32 --model 13b > gpurun_out/${TAG}_decode_13b.log 2>&1; note decode_13b $? ;;
    tree) timeout 900 python scripts/tree_bench.py --steps 4 > gpurun_out/${TAG}_tree.log 2>&1; note tree $? ;;
    layer) timeout 600 python scripts/prof_layer.py --layers 4 --steps 16 > gpurun_out/${TAG}_layer.log 2>&1; note layer $? ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-decode > gpurun_out/${TAG}_launches.log 2>&1; note launches $? ;;
    ncupred) B=1024 ITERS=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:predictor_stream -s 4 -c 1 -o gpurun_out/${TAG}_ncu_pred -f python scripts/prof_predictor.py > gpurun_out/${TAG}_ncu_pred.log 2>&1; note ncupred $?
             ncu_csv gpurun_out/${TAG}_ncu_pred.ncu-rep ;;
    ncugather) CHAIN=1 B=1024 ITERS=6 timeout 600 ncu --set full --clock-control none --import-source on -k regex:predictor_gather -s 6 -c 1 -o gpurun_out/${TAG}_ncu_gather -f python scripts/prof_predictor.py > gpurun_out/${TAG}_ncu_gather.log 2>&1; note ncugather $?
             ncu_csv gpurun_out/${TAG}_ncu_gather.ncu-rep ;;
    ncuverify) timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify -s 3 -c 1 -o gpurun_out/${TAG}_ncu_verify -f python scripts/prof_kernels.py verify > gpurun_out/${TAG}_ncu_verify.log 2>&1; note ncuverify $?
               ncu_csv gpurun_out/${TAG}_ncu_verify.ncu-rep ;;
    ncutree) timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_merged -s 3 -c 1 -o gpurun_out/${TAG}_ncu_tree -f python scripts/prof_kernels.py tree > gpurun_out/${TAG}_ncu_tree.log 2>&1; note ncutree $?
             ncu_csv gpurun_out/${TAG}_ncu_tree.ncu-rep ;;
    nculayer) timeout 600 ncu --set full --clock-control none -k regex:layer_mega -s 2 -c 1 -o gpurun_out/${TAG}_ncu_layer -f python scripts/prof_layer.py --layers 2 --steps 2 > gpurun_out/${TAG}_ncu_layer.log 2>&1; note nculayer $?
              ncu_csv gpurun_out/${TAG}_ncu_layer.ncu-rep; rm -f gpurun_out/${TAG}_ncu_layer.ncu-rep ;;
    sanitize) for tool in memcheck racecheck; do
                timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python scripts/sanitize_smoke.py > gpurun_out/${TAG}_sanitize_$tool.log 2>&1
                note "sanitize_$tool" $?; done ;;
    *) echo "unknown stage $stage" >> $ST ;;
  esac
done
du -sh gpurun_out >> $ST
