cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_engine.py tests/test_gpu_batched.py tests/test_gpu_tree.py -x > gpurun_out/t20_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t20_status.txt
timeout 600 python scripts/batch_sweep.py --batches 4,16,64,256 --steps 4 --profile gpurun_out/t20_kt > gpurun_out/t20_sweep.jsonl 2>&1; echo "sweep rc=$?" >> gpurun_out/t20_status.txt
timeout 600 python scripts/tree_bench.py --steps 6 --profile gpurun_out/t20_kt_tree.txt > gpurun_out/t20_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/t20_status.txt
