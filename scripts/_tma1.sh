cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python scripts/batch_sweep.py --batches 1,2,4,8,16,32,64,128,256 --steps 6 > gpurun_out/f2_sweep.jsonl 2>&1; echo "sweep rc=$?" >> gpurun_out/f2_status.txt
TAG=f2 bash scripts/gpu.sh bench benchref
timeout 600 python scripts/tree_bench.py --steps 6 --profile gpurun_out/f2_kt_tree.txt > gpurun_out/f2_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/f2_status.txt
timeout 600 python scripts/batch_sweep.py --batches 64,256 --steps 4 --profile gpurun_out/f2_kt > /dev/null 2>&1; echo "prof rc=$?" >> gpurun_out/f2_status.txt
