cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_engine.py tests/test_gpu_batched.py tests/test_gpu_tree.py -x > gpurun_out/t32_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t32_status.txt
timeout 600 python scripts/tree_bench.py --steps 6 > gpurun_out/t32_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/t32_status.txt
timeout 600 python scripts/batch_sweep.py --batches 4,16,64,256 --steps 4 > gpurun_out/t32_sweep.jsonl 2>&1; echo "sweep rc=$?" >> gpurun_out/t32_status.txt
SPX_TCL_FIXUP=0 timeout 600 python scripts/tree_bench.py --steps 6 > gpurun_out/t32_tree_nofix.log 2>&1; echo "tree0 rc=$?" >> gpurun_out/t32_status.txt
