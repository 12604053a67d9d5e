cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_engine.py -k "reuse or topk" > gpurun_out/t33_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t33_status.txt
