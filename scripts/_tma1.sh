cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
for P in 1 0 1 0; do SPX_PDL_LAYERS=$P timeout 600 python scripts/tree_bench.py --steps 6 >> gpurun_out/t16_tree_pdl$P.log 2>&1; done
for P in 1 0; do SPX_PDL_LAYERS=$P timeout 600 python scripts/batch_sweep.py --batches 4,64,256 --steps 4 > gpurun_out/t16_sweep_pdl$P.jsonl 2>&1; done
echo done >> gpurun_out/t16_status.txt
