cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 600 python scripts/batch_sweep.py --batches 1,2,4,8,16,32,64,128,256 --steps 4 --profile gpurun_out/t9_kt > gpurun_out/t9_sweep.jsonl 2>&1; echo "sweep rc=$?" >> gpurun_out/t9_status.txt
SPX_TCL_MIN2=3 timeout 600 python scripts/batch_sweep.py --batches 16,64 --steps 4 --profile gpurun_out/t9_kt_min3 > gpurun_out/t9_sweep_min3.jsonl 2>&1; echo "sweep3 rc=$?" >> gpurun_out/t9_status.txt
timeout 600 python scripts/tree_bench.py --steps 4 --profile gpurun_out/t9_kt_tree.txt > gpurun_out/t9_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/t9_status.txt
