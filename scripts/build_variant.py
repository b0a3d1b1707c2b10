"""Build a variant of the C-ABI library with extra -D defines into gpu_ab/ (A/B runs
via ARMT_LIB_PATH). python scripts/build_variant.py NAME -DFOO=1 [-DBAR=2 ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2506_05229_b200 import _build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "gpu_ab", name)
os.makedirs(out_dir, exist_ok=True)
objs = []
for src in B.sources():
    obj = os.path.join(out_dir, os.path.basename(src)[:-3] + ".o")
    r = subprocess.run([B.NVCC, *B.FLAGS, *defs, "-c", src, "-o", obj], capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    objs.append(obj)
lib = os.path.join(ROOT, "gpu_ab", f"libarmt_{name}.so")
r = subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static", *objs,
                    "-o", lib], capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
for o in objs:
    os.remove(o)
print(lib)
