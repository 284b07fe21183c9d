"""Build a variant of libbvc_b200.so with extra nvcc defines for one source file, for A/B
runs on the GPU box (select it with BVC_LIB=...):
    python scripts/variant_lib.py NAME SOURCE.cu -DMACRO=VALUE ...
Output: paper_2302_11825_b200/_build/variants/NAME/libbvc_b200.so (git-ignored; travels with gpurun)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_11825_b200 import build as Bd  # noqa: E402

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
Bd.build()
out = os.path.join(Bd.OUT, "variants", name)
os.makedirs(out, exist_ok=True)
obj = os.path.join(out, src + ".o")
cmd = [Bd.NVCC, *Bd.ARCH, *Bd.FLAGS, *defs, "-c", os.path.join(Bd.CSRC, src), "-o", obj]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
objs = [obj if s == src else os.path.join(Bd.OUT, s + ".o") for s in Bd.SOURCES]
lib = os.path.join(out, "libbvc_b200.so")
r = subprocess.run([Bd.NVCC, *Bd.ARCH, "-shared", "-o", lib, *objs, "-cudart", "static", "-ldl"], capture_output=True,
                   text=True)
if r.returncode:
    sys.exit(r.stderr)
print(lib)
