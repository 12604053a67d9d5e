#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PYTHONPATH=$PWD:${PYTHONPATH:-}
mkdir -p gpurun_out
timeout 600 python -c "
import cProfile, pstats, sys
sys.argv=['x']
from paper_2504_08850_b200 import numerics
numerics.set_mode('fast')
import scripts.tree_bench as tb
import torch
m = None
pr = cProfile.Profile()
res = tb.run(steps=1)
pr.enable()
res = tb.run(steps=3)
pr.disable()
print(res)
pstats.Stats(pr).sort_stats('cumulative').print_stats(35)
" > gpurun_out/tprof.txt 2>&1
