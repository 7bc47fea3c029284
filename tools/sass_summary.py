"""Summarise an ncu --page source --print-source=sass CSV: stall totals, hot instructions, opcode mix."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def num(r, k):
    try: return float(r[ix[k]])
    except: return 0.0
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for r in data:
    for s in stalls: tot[s] += num(r, s)
S = sum(tot.values())
print("stall breakdown (all samples):")
for s, v in tot.most_common(10): print(f"  {s:28s} {100*v/S:5.1f}%")
ops = collections.Counter(); ops_inst = collections.Counter()
for r in data:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]] else "?"
    if op.startswith("@"): op = r[ix["Source"]].split()[1]
    ops[op.split(".")[0]] += num(r, "Instructions Executed")
T = sum(ops.values())
print("opcode mix (warp instructions executed):", int(T))
for o, v in ops.most_common(25): print(f"  {o:10s} {100*v/T:5.1f}%")
print("top stall instructions:")
data.sort(key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))
for r in data[:25]:
    print(f"  {num(r,'Warp Stall Sampling (All Samples)'):8.0f} {r[ix['Address']]} {r[ix['Source']][:90]}")
