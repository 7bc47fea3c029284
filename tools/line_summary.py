"""Per-CUDA-source-line instruction and stall totals from `ncu --page source --print-source=cuda,sass --csv`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
cur_file = None; out = []
hdr = None
for r in rows:
    if r and r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        ix = {h: i for i, h in enumerate(hdr)}
        try:
            ins = float(r[ix["Instructions Executed"]]); st = float(r[ix["Warp Stall Sampling (All Samples)"]])
        except ValueError: continue
        out.append((ins, st, cur_file, r[0], r[1].strip()[:100]))
T = sum(o[0] for o in out); S = sum(o[1] for o in out)
print("by instructions:")
for o in sorted(out, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]: print(f"  {100*o[0]/T:5.1f}% ins {100*o[1]/S:5.1f}% stall  {o[2]}:{o[3]}  {o[4]}")
