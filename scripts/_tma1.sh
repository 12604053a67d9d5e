cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
for E in 0 80; do SPX_TCL_MIN_OTILES_SPLIT=$E timeout 600 python scripts/tree_bench.py --steps 6 > gpurun_out/t27_tree_$E.log 2>&1; SPX_TCL_MIN_OTILES_SPLIT=$E timeout 600 python scripts/batch_sweep.py --batches 16,64,256 --steps 4 > gpurun_out/t27_sweep_$E.jsonl 2>&1; done
echo done >> gpurun_out/t27_status.txt
