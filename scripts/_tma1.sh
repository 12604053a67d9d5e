cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests -x > gpurun_out/t5_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t5_status.txt
timeout 600 python scripts/batch_sweep.py --batches 1,16,64,256 --steps 4 --profile gpurun_out/t5_kt > gpurun_out/t5_sweep.jsonl 2>&1; echo "sweep rc=$?" >> gpurun_out/t5_status.txt
timeout 600 python scripts/tree_bench.py --steps 4 --profile gpurun_out/t5_kt_tree.txt > gpurun_out/t5_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/t5_status.txt
timeout 600 python scripts/decode_bench.py --tokens 64 > gpurun_out/t5_decode.log 2>&1; echo "decode rc=$?" >> gpurun_out/t5_status.txt
