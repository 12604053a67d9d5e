cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_features_wide.py tests/test_gpu_tree.py tests/test_gpu_batched.py -x > gpurun_out/t11_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t11_status.txt
timeout 600 python scripts/tree_bench.py --steps 4 --profile gpurun_out/t11_kt_tree.txt > gpurun_out/t11_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/t11_status.txt
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/t11_bench.json 2> gpurun_out/t11_bench.err; echo "bench rc=$?" >> gpurun_out/t11_status.txt
