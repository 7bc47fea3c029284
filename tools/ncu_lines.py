"""Per-source-line instruction and stall-sample attribution of an .ncu-rep (dev tool).
usage: python tools/ncu_lines.py REP [N]"""
import csv, collections, subprocess, sys, io, re
rep = sys.argv[1]; topn = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = collections.defaultdict(lambda: [0.0, 0.0, "", collections.Counter(), collections.Counter()])
f = None; cur = None; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if len(r) < 8 or hdr is None: continue
    if r[0] != "":
        cur = (f, r[0]); agg[cur][2] = r[1][:80]
    else:
        try:
            n = float(r[7]); st = float(r[4])
        except ValueError:
            continue
        agg[cur][0] += n; agg[cur][1] += st
        op = r[3].split(); o = op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "?")
        agg[cur][3][o.split(".")[0]] += n
        for k, v in zip(hdr, r):
            if k.startswith("stall_"):
                try: agg[cur][4][k] += float(v)
                except ValueError: pass
tot = sum(v[0] for v in agg.values()) or 1; st = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:topn]:
    print("%5.1f%% stall %5.1f%% inst %s:%s %s | %s | %s" % (100 * v[1] / st, 100 * v[0] / tot, k[0], k[1], v[2],
          dict(v[3].most_common(3)), dict((a, int(b)) for a, b in v[4].most_common(2))))
