"""Build a variant of libvolpg_b200.so with extra nvcc defines for one-box A/B
runs:  python tools/build_variant.py NAME -DVPG_STORE_EVERY=3 ...
Load it with VPG_LIB_VARIANT=NAME (paper_2404_11894_b200/_native.py)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_11894_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(B.OUT_DIR, "variants", name)
os.makedirs(out_dir, exist_ok=True)
nvcc = B._nvcc()
objs = []
for src in B._sources():
    obj = os.path.join(out_dir, src.replace(".cu", ".o"))
    subprocess.run([nvcc, *B.ARCH, *B.COMMON, *B.PER_FILE.get(src, []), *defs, "-c",
                    os.path.join(B.CSRC, src), "-o", obj], check=True)
    objs.append(obj)
lib = os.path.join(B.OUT_DIR, "variants", f"libvolpg_b200_{name}.so")
subprocess.run([nvcc, *B.ARCH, "-shared", "-o", lib, *objs, "-Xcompiler", "-fPIC"], check=True)
print(lib)
