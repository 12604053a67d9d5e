cd $GRAFT_REPO_ROOT; export PYTHONPATH=$PWD; mkdir -p gpurun_out
timeout 900 python scripts/batch_sweep.py --batches 1,2,4,8,16,32,64,128,256 --steps 6 > gpurun_out/f3_sweep.jsonl 2>&1; echo "sweep rc=$?" >> gpurun_out/f3_status.txt
TAG=f3 bash scripts/gpu.sh bench smoke
timeout 600 python scripts/tree_bench.py --steps 6 --profile gpurun_out/f3_kt_tree.txt > gpurun_out/f3_tree.log 2>&1; echo "tree rc=$?" >> gpurun_out/f3_status.txt
timeout 600 python scripts/batch_sweep.py --batches 64,256 --steps 4 --profile gpurun_out/f3_kt > /dev/null 2>&1; echo "prof rc=$?" >> gpurun_out/f3_status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"tcl_|attn_fast128|tcv_|verify|softmax_pick|tree_" -c 600 --csv --log-file gpurun_out/f3_tree_launches.csv python scripts/tree_bench.py --steps 1 > gpurun_out/f3_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/f3_status.txt
python scripts/summarize_launches.py gpurun_out/f3_tree_launches.csv > gpurun_out/f3_tree_launches.txt 2>&1
