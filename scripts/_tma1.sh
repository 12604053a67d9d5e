cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 600 python scripts/batch_sweep.py --batches 64,256 --steps 2 --profile gpurun_out/t2_kt > gpurun_out/t2_sweep.jsonl 2>&1; echo "sweep rc=$?" >> gpurun_out/t2_status.txt
timeout 600 python scripts/tree_bench.py --steps 2 --profile gpurun_out/t2_kt_tree.txt > gpurun_out/t2_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/t2_status.txt
