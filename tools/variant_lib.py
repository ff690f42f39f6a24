"""Build an A/B variant of the library: one source recompiled with extra -D flags, linked
with the in-tree objects into scratch/<name>.so (use it with SBG_LIB_PATH=...).

    python tools/variant_lib.py far_u2 cuda/assemble.cu -DFAR_FLAT_UNROLL=2
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_09204_b200 import build as B  # noqa: E402

name, src, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
os.makedirs(os.path.join(ROOT, "scratch"), exist_ok=True)
srcp = os.path.join(B.CSRC, src)
obj = os.path.join(ROOT, "scratch", name + ".o")
cmd = [B.NVCC] + B.COMMON + B.ARCH + flags + ["-c", srcp, "-o", obj]
subprocess.run(cmd, check=True)
rel = os.path.relpath(srcp, B.CSRC).replace(os.sep, "_") + ".o"
objs = [o for o in glob.glob(os.path.join(B.OUT_DIR, "obj", "*.o")) if os.path.basename(o) != rel] + [obj]
out = os.path.join(ROOT, "scratch", name + ".so")
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", out] + objs, check=True)
print(out)
