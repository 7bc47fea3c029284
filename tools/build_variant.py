"""Build an A/B variant of libfraclap_b200.so with extra nvcc flags (dev tool).

    python tools/build_variant.py OUT.so -DFOO=1 ...

Objects go to build/var_<name>/; the library is loaded by tools through
FL_LIB_OVERRIDE=OUT.so.  Only dst.cu is recompiled with the flags; the other
objects are taken from the main build.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1809_01971_b200 import build as B  # noqa: E402

out, flags = sys.argv[1], sys.argv[2:]
B.build()
name = os.path.splitext(os.path.basename(out))[0]
odir = os.path.join(ROOT, "build", "var_" + name)
os.makedirs(odir, exist_ok=True)
objs = []
for src in B.sources():
    base = os.path.basename(src).replace(".cu", ".o")
    if base == os.environ.get("VARIANT_OBJ", "dst.o"):
        obj = os.path.join(odir, base)
        cmd = [B._nvcc()] + B.ARCH + B.NVCC_FLAGS + flags + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stderr)
        objs.append(obj)
    else:
        objs.append(os.path.join(B.BUILD, base))
cmd = [B._nvcc()] + B.ARCH + ["-shared", "-o", out] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread",
                                                            "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
print(out)
