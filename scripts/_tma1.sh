cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_engine.py tests/test_gpu_batched.py tests/test_gpu_tree.py -x > gpurun_out/t22_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t22_status.txt
timeout 600 python scripts/decode_bench.py --tokens 64 --profile gpurun_out/t22_kt_decode.txt > gpurun_out/t22_decode.log 2>&1; echo "decode rc=$?" >> gpurun_out/t22_status.txt
