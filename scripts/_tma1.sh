cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_engine.py tests/test_gpu_batched.py tests/test_gpu_tree.py -x > gpurun_out/t24_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t24_status.txt
timeout 600 python scripts/batch_sweep.py --batches 4,16,64,256 --steps 4 > gpurun_out/t24_sweep.jsonl 2>&1; echo "sweep rc=$?" >> gpurun_out/t24_status.txt
timeout 600 python scripts/tree_bench.py --steps 6 > gpurun_out/t24_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/t24_status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tcl_|attn_fast128" -c 400 --csv --log-file gpurun_out/t24_tree_launches.csv python scripts/tree_bench.py --steps 1 > gpurun_out/t24_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/t24_status.txt
python scripts/summarize_launches.py gpurun_out/t24_tree_launches.csv > gpurun_out/t24_tree_launches.txt 2>&1
