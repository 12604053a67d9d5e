cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_verify_tc.py -x > gpurun_out/t3_vtc.log 2>&1; echo "vtc rc=$?" >> gpurun_out/t3_status.txt
timeout 900 python -m pytest -q -m gpu tests/test_gpu_batched.py tests/test_gpu_tree.py tests/test_gpu_engine.py tests/test_gpu_parity.py -x > gpurun_out/t3_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t3_status.txt
timeout 600 python scripts/batch_sweep.py --batches 16,64,256 --steps 4 --profile gpurun_out/t3_kt > gpurun_out/t3_sweep.jsonl 2>&1; echo "sweep rc=$?" >> gpurun_out/t3_status.txt
timeout 600 python scripts/tree_bench.py --steps 4 --profile gpurun_out/t3_kt_tree.txt > gpurun_out/t3_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/t3_status.txt
