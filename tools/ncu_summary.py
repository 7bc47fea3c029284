"""Text summary of an .ncu-rep (key SOL / memory / scheduler metrics, stalls, opcode mix)."""
import csv, io, subprocess, sys, collections

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__grid_size", "launch__block_size", "smsp__cycles_active.avg"]
lines = []
for v in vals:
    d = dict(zip(hdr, v))
    u = dict(zip(hdr, units))
    lines.append("== launch ==")
    for k in want:
        if k in d:
            lines.append("%-60s %s %s" % (k, d[k], u.get(k, "")))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    rd = float(d.get("dram__bytes_read.sum", "0").replace(",", "") or 0) * scale.get(u.get("dram__bytes_read.sum", "byte"), 1.0)
    wr = float(d.get("dram__bytes_write.sum", "0").replace(",", "") or 0) * scale.get(u.get("dram__bytes_write.sum", "byte"), 1.0)
    lines.append("%-60s %.6e bytes" % ("traffic (dram read + write)", rd + wr))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
if len(srows) > 2:
    h = srows[1]; ix = {k: i for i, k in enumerate(h)}
    stall = collections.Counter(); ops = collections.Counter()
    for r in srows[2:]:
        for k in h:
            if k.startswith("stall_") and "Not Issued" not in k:
                try: stall[k] += float(r[ix[k]]) if ix[k] < len(r) else 0.0
                except ValueError: pass
        op = r[ix["Source"]].split()
        if op:
            o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
            try: ops[o.split(".")[0]] += float(r[ix["Instructions Executed"]]) if ix["Instructions Executed"] < len(r) else 0.0
            except ValueError: pass
    S = sum(stall.values()) or 1; T = sum(ops.values()) or 1
    lines.append("== stall breakdown ==")
    lines += ["  %-28s %5.1f%%" % (k, 100 * v / S) for k, v in stall.most_common(10)]
    lines.append("== opcode mix (%d warp instructions) ==" % T)
    lines += ["  %-10s %5.1f%%" % (k, 100 * v / T) for k, v in ops.most_common(14)]
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:20]))
