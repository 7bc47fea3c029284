"""Per-source-line shared-memory wavefronts (actual vs ideal) from an ncu
source-page CSV (dev tool): python tools/smem_lines.py src.csv [top]."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr, cur, out = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and r and r[0].isdigit():
        try:
            w = float(r[hdr["L1 Wavefronts Shared"]] or 0)
            wi = float(r[hdr["L1 Wavefronts Shared Ideal"]] or 0)
            st = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, IndexError):
            continue
        if w:
            out.append((w, wi, st, cur, r[0], r[1].strip()[:90]))
T = sum(o[0] for o in out)
TI = sum(o[1] for o in out)
print("total shared wavefronts %.3e, ideal %.3e (%.2fx)" % (T, TI, T / max(TI, 1)))
for o in sorted(out, reverse=True)[:top]:
    print("  %5.1f%%  x%.2f  %s:%s  %s" % (100 * o[0] / T, o[0] / max(o[1], 1), o[3], o[4], o[5]))
