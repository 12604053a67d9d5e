"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every entry point declared in include/specexit_b200.h (no compute calls)."""
import ctypes
import os
import re
import subprocess

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "specexit_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(spx_\w+)\s*\(", text, re.M)))


def test_header_declares_the_operator_set():
    syms = declared_symbols()
    for s in ("spx_predictor_eval", "spx_verify", "spx_sched_update", "spx_sched_active",
              "spx_tree_merged_logits", "spx_path_and", "spx_tree_gate", "spx_tree_node_eval",
              "spx_final_norm", "spx_extract_features",
              "spx_predictor_mlp", "spx_init_uniform", "spx_version"):
        assert s in syms, s


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2504_08850_b200 import _native
    lib = _native.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} not exported"
    assert b"sm_100a" in lib.spx_version()


def test_library_is_sm100a_code():
    from paper_2504_08850_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2504_08850_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\S+)", src, re.M), f
                assert "specexit_oracle" not in src, f
