"""Build an experimental variant of the library (extra nvcc flags) into its own .so (experiments only).

    python tools/build_variant.py OUT.so [-DFLAG ...]

Objects go to _build/variants/<name>/, so the product build is untouched.
"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_1404_0466_b200 import build as b  # noqa: E402

out = os.path.abspath(sys.argv[1])
extra = sys.argv[2:]
name = os.path.basename(out).replace(".so", "")
bdir = os.path.join(b.BUILD, "variants", name)
os.makedirs(bdir, exist_ok=True)
srcs = sorted(glob.glob(os.path.join(b.CSRC, "*.cu")))


def comp(src):
    obj = os.path.join(bdir, os.path.basename(src)[:-3] + ".o")
    subprocess.run([b.nvcc(), *b.ARCH, *b.NVCC_FLAGS, *extra, "-c", src, "-o", obj], check=True)
    return obj


with cf.ThreadPoolExecutor(len(srcs)) as pool:
    objs = list(pool.map(comp, srcs))
subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", out, *objs, "-lcudart_static", "-lrt", "-lpthread", "-ldl"],
               check=True)
print("built", out, extra)
