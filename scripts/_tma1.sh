cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_tree.py tests/test_gpu_batched.py -x > gpurun_out/t18_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t18_status.txt
timeout 600 python scripts/tree_bench.py --steps 6 > gpurun_out/t18_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/t18_status.txt
timeout 600 python scripts/prof_tree_host.py > gpurun_out/t18_tree_host.log 2>&1; echo "treehost rc=$?" >> gpurun_out/t18_status.txt
