"""Measurement aid: build libmis2.so with extra nvcc flags (e.g. -DMIS2_WARPS=32)
into tools/ab/<name>/ for an A/B run through MIS2_LIB_PATH (same ABI).
usage: python tools/build_variant.py NAME FLAG [FLAG ...]"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_02934_b200 import build as B

name, extra = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "abv", name)  # shipped by gpurun; delete after use
os.makedirs(out, exist_ok=True)
inc = B.nccl_include()


def cc(src):
    obj = os.path.join(out, os.path.basename(src)[:-3] + ".o")
    subprocess.check_call([B.NVCC, *B.ARCH, *B.FLAGS, *extra, "-I", inc, "-c", "-o", obj, src])
    return obj


with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
    objs = list(ex.map(cc, B.sources()))
lib = os.path.join(out, "libmis2.so")
subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", lib, *objs, "-ldl"])
print(lib)
