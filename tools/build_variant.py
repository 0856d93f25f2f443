"""Build a diagnostic variant of libpsb200.so with extra -D flags (timing
experiments only; never the product): python tools/build_variant.py NAME -DFLAG ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2411_00688_b200"))
import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
obj_dir = os.path.join(ROOT, "build", "variant_" + name)
os.makedirs(obj_dir, exist_ok=True)
objs = []
for src in sorted(os.listdir(B.CSRC)):
    if not src.endswith(".cu"):
        continue
    o = os.path.join(obj_dir, src.replace(".cu", ".o"))
    subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", o],
                   check=True, capture_output=True)
    objs.append(o)
out = os.path.join(ROOT, "build", f"libpsb200_{name}.so")
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, "-lcudart"], check=True)
print(out)
