cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_features_wide.py tests/test_gpu_verify_tc.py tests/test_gpu_tree.py -x > gpurun_out/t28_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t28_status.txt
