cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_engine.py tests/test_gpu_batched.py tests/test_gpu_tree.py -x > gpurun_out/t34_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t34_status.txt
for N in 1 0; do SPX_TCL_N256=$N timeout 600 python scripts/batch_sweep.py --batches 128,256 --steps 4 > gpurun_out/t34_sweep_$N.jsonl 2>&1; done
echo done >> gpurun_out/t34_status.txt
