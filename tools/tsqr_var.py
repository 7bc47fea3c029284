"""TSQR timing for library variants: python tools/tsqr_var.py LIB... (dev tool)"""
import os, subprocess, sys
if len(sys.argv) > 2:
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, __file__, lib])
    sys.exit(0)
os.environ["FL_LIB_OVERRIDE"] = os.path.abspath(sys.argv[1])
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1809_01971_b200 import decomp
out = []
for k, m in [(127, 2039), (127, 8192), (127, 130000), (96, 30000), (64, 2048), (48, 1024)]:
    M = torch.randn((k, m), dtype=torch.float64, device="cuda")
    decomp.qr_r_wide([M]); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        decomp.qr_r_wide([M])
    b.record(); torch.cuda.synchronize()
    out.append("%dx%d %.3f" % (k, m, a.elapsed_time(b) / 20))
print(os.path.basename(sys.argv[1]), " | ".join(out), flush=True)
