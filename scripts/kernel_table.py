"""Per-kernel device-time table of one callable (torch.profiler / CUPTI: every
kernel the process launches, graph nodes included, timed live -- not
serialised like ncu).  Used by batch_sweep.py / tree_bench.py --profile."""
from collections import defaultdict

import torch


def kernel_table(fn, path, top=40):
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    agg = defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            a = agg[ev.name.split("(")[0][:90]]
            a[0] += 1
            a[1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    tot = sum(a[1] for a in agg.values()) or 1.0
    with open(path, "w") as fh:
        fh.write(f"{'kernel':90s} {'n':>6s} {'mean_us':>9s} {'total_ms':>9s} {'share':>6s}\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
            fh.write(f"{k:90s} {n:6d} {t / n:9.2f} {t / 1e3:9.3f} {t / tot:6.1%}\n")
        fh.write(f"total kernel time {tot / 1e3:.3f} ms\n")
