"""Build recipe for the oracle's native pieces (test infrastructure only).

* oracle/_lib/libspx_oracle.so  <- oracle/strict.c (our C restatement of the
  reference's strict kernels), gcc -O2 -ffp-contract=off.
* oracle/_ref/_ckern*.so         <- the REFERENCE's own Cython-generated C
  kernel, compiled from where it lies
  (/root/reference/pkg/src/specexit/kernels/_ckern.c) with the flags of the
  reference's setup.py:17-24 (-O3 -ffp-contract=off).  Only when
  /root/reference exists (this container); the built .so travels to the GPU
  box in the repo snapshot.  Outputs go only to oracle/_ref/ (git-ignored).
"""
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
REF_CKERN = "/root/reference/pkg/src/specexit/kernels/_ckern.c"


def build(force=False):
    out_dir = os.path.join(HERE, "_lib")
    os.makedirs(out_dir, exist_ok=True)
    so = os.path.join(out_dir, "libspx_oracle.so")
    src = os.path.join(HERE, "strict.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", so, src])
    build_ref(force)
    return so


def ref_so_path():
    suffix = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
    return os.path.join(HERE, "_ref", "specexit_ref_kernels", "_ckern" + suffix)


def build_ref(force=False):
    """Compile the reference's _ckern.c into oracle/_ref (if present here)."""
    if not os.path.exists(REF_CKERN):
        return None
    so = ref_so_path()
    if os.path.exists(so) and not force:
        return so
    import numpy as np
    os.makedirs(os.path.dirname(so), exist_ok=True)
    open(os.path.join(os.path.dirname(so), "__init__.py"), "a").close()
    inc = [sysconfig.get_paths()["include"], np.get_include()]
    cmd = ["gcc", "-O3", "-ffp-contract=off", "-fPIC", "-shared", "-w",
           "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION"]
    cmd += [f"-I{p}" for p in inc] + ["-o", so, REF_CKERN]
    subprocess.check_call(cmd)
    return so


def load_ref_kernels():
    """Import the compiled reference kernel module from oracle/_ref, or None."""
    so = ref_so_path()
    if not os.path.exists(so):
        return None
    import importlib.machinery
    import importlib.util
    loader = importlib.machinery.ExtensionFileLoader("_ckern", so)
    spec = importlib.util.spec_from_file_location("_ckern", so, loader=loader)
    mod = importlib.util.module_from_spec(spec)
    loader.exec_module(mod)
    return mod


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
    print(build_ref(force="--force" in sys.argv))
