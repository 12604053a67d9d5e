cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 600 python scripts/batch_sweep.py --batches 2,4,8,16 --steps 4 > gpurun_out/t10_sweep.jsonl 2>&1; echo "sweep rc=$?" >> gpurun_out/t10_status.txt
SPX_TCL_MIN_ROWS=16 timeout 600 python scripts/batch_sweep.py --batches 2,4,8 --steps 4 > gpurun_out/t10_sweep16.jsonl 2>&1; echo "sweep16 rc=$?" >> gpurun_out/t10_status.txt
timeout 600 python scripts/tree_bench.py --steps 4 --profile gpurun_out/t10_kt_tree.txt > gpurun_out/t10_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/t10_status.txt
timeout 900 python -m pytest -q -m gpu tests/test_gpu_engine.py tests/test_gpu_batched.py tests/test_gpu_tree.py -x > gpurun_out/t10_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t10_status.txt
