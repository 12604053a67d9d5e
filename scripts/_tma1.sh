cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests > gpurun_out/t30_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t30_status.txt
