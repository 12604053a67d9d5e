"""Build libspecexit_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2504_08850_b200.build [--force]

The library lands in paper_2504_08850_b200/_lib/ (git-ignored, but shipped to
the GPU box with the repo snapshot).  nvcc cross-compiles without a GPU.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIB_DIR, "libspecexit_b200.so")
SOURCES = ["spx_predictor.cu", "spx_pred_stream.cu", "spx_pred_split.cu", "spx_pred_team_bf16_a.cu", "spx_pred_team_bf16_b.cu",
           "spx_pred_team_bf16_c.cu", "spx_pred_team_bf16_w.cu", "spx_pred_team_f32.cu", "spx_verify.cu", "spx_sched.cu", "spx_tree.cu", "spx_tree_tc.cu", "spx_init.cu",
           "spx_layers.cu", "spx_engine.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "specexit_b200.h"))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def _obj_stale(src, obj):
    """An object is rebuilt when missing, older than its source, or older
    than any shared header (.cuh / include/*.h)."""
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    hdrs.append(os.path.join(HERE, "..", "include", "specexit_b200.h"))
    return any(os.path.getmtime(p) > t for p in [src] + hdrs if os.path.exists(p))


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    objs = []
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    procs = []
    for s in srcs:
        src = os.path.join(CSRC, s)
        obj = os.path.join(LIB_DIR, s.replace(".cu", ".o"))
        objs.append(obj)
        if not force and not _obj_stale(src, obj):
            continue
        cmd = [NVCC, *FLAGS, "-c", src, "-o", obj + ".tmp"]
        procs.append((s, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                               stderr=subprocess.STDOUT)))
    logs = []
    for s, obj, p in procs:
        out, _ = p.communicate()
        logs.append(out.decode())
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {s}:\n{out.decode()}")
        os.replace(obj + ".tmp", obj)
    if logs:
        with open(os.path.join(LIB_DIR, "ptxas.log"), "w") as fh:
            fh.write("\n".join(logs))
    tmp = LIB + ".tmp"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-o", tmp, *objs, "-lcudart"])
    os.replace(tmp, LIB)
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
