"""The C-ABI library builds for sm_100a, loads, and exports every symbol
include/mis2.h declares (no compute calls: no GPU needed)."""
import ctypes
import os
import re
import subprocess

import paper_2204_02934_b200 as M
from paper_2204_02934_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "mis2.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(mis2[a-z_0-9]*)\s*\(", src, flags=re.M)))


def test_header_declares_expected():
    assert declared_functions() == sorted(M.EXPORTS)


def test_library_exports_every_symbol():
    L = M.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert b"sm_100a" in L.mis2_version()
    assert L.mis2_strerror(-6) == b"not converged within max_iters"


def test_built_for_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2204_02934_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.c" not in txt, f
