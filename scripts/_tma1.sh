cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests -x > gpurun_out/t26_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t26_status.txt
timeout 600 python scripts/tree_bench.py --steps 6 --profile gpurun_out/t26_kt_tree.txt > gpurun_out/t26_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/t26_status.txt
