cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
TAG=f4 bash scripts/gpu.sh test smoke bench
timeout 600 python scripts/tree_bench.py --steps 6 --profile gpurun_out/f4_kt_tree.txt > gpurun_out/f4_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/status.txt
