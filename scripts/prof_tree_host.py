import cProfile, pstats, sys, os, io
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "scripts"))
import torch
import tree_bench
from paper_2504_08850_b200 import numerics
numerics.set_mode("fast")
pr = cProfile.Profile()
pr.enable()
r = tree_bench.run(steps=3)
pr.disable()
print(r["ms_per_step"])
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(35)
print(s.getvalue()[:9000])
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(20)
print(s.getvalue()[:6000])
