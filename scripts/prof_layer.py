"""Decode-step decoder layers at Llama2-7B dims for ncu / timing: a short
prompt is prefilled, then `--steps` single-token steps run all layers.
Prints the device time per layer (CUDA events, PDL chained launches)."""
import argparse
import json

import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import numerics
from paper_2504_08850_b200.decode import DecodeState


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=11008)
    ap.add_argument("--heads", type=int, default=32)
    args = ap.parse_args()
    numerics.set_mode("fast")
    cfg = spx.ModelConfig(32000, args.d, args.layers, args.heads, args.ffn, 512, 5)
    m = spx.init_model(cfg, dtype="bf16")
    st = DecodeState(m)
    st.begin(list(range(1, 17)))
    for l in range(args.layers):
        st.launch_layer(l)
    g = torch.cuda.CUDAGraph()
    tok = torch.tensor([42], dtype=torch.int32, device="cuda")
    # one captured decode step (embed + all layers), replayed
    with torch.cuda.graph(g):
        st.embed_device(tok, 1)
        for l in range(args.layers):
            st.launch_layer(l)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    st.check()
    ms = e0.elapsed_time(e1) / args.steps
    lay_bytes = (4 * args.d * args.d + 2 * args.d * args.ffn) * 2
    us_layer = ms * 1e3 / args.layers
    try:
        import ctypes
        import numpy as np
        from paper_2504_08850_b200 import _native as N
        buf = np.zeros(64, np.uint64)
        N.lib().spx_debug_mega_trace(ctypes.c_void_p(buf.ctypes.data))
        names = ["start", "rowset", "qkv", "bar0", "attn", "bar1", "wo", "bar2", "ffn1", "bar3",
                 "ffn2", "end"]
        for c in range(2):
            t = buf[c * 16:c * 16 + 13].astype(np.int64)
            if t[0] and t[12]:
                print(f"mega CTA{c}: " + " ".join(f"{names[k]}={(t[k + 1] - t[k]) / 1e3:.2f}"
                                                  for k in range(12)) +
                      f" total={(t[12] - t[0]) / 1e3:.2f}us")
        a = buf[32:37].astype(np.int64)
        print(f"attn item0: start->scores {(a[0]-a[4])/1e3:.2f} scores->exp {(a[1]-a[0])/1e3:.2f} "
              f"exp->out {(a[2]-a[1])/1e3:.2f} nctx {a[3]}")
    except Exception as e:  # noqa: BLE001
        print("no mega trace:", e)
    print(json.dumps({"us_per_layer": us_layer, "GBps": lay_bytes / (us_layer * 1e-6) / 1e9,
                      "layer_MB": lay_bytes / 1e6}))


if __name__ == "__main__":
    main()
