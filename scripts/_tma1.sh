cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_verify_tc.py -x > gpurun_out/t4_vtc.log 2>&1; echo "vtc rc=$?" >> gpurun_out/t4_status.txt
timeout 900 python -m pytest -q -m gpu tests/test_gpu_batched.py -x > gpurun_out/t4_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t4_status.txt
timeout 600 python scripts/batch_sweep.py --batches 1,16,64,256 --steps 4 --profile gpurun_out/t4_kt > gpurun_out/t4_sweep.jsonl 2>&1; echo "sweep rc=$?" >> gpurun_out/t4_status.txt
