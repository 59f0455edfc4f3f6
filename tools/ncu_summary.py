"""Summarise an ncu report: key throughput metrics, stall reasons, hot SASS."""
import csv, io, re, subprocess, sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum", "smsp__inst_executed.sum"]
for k in keys:
    if k in d:
        print(f"{k:70s} {d[k][1]:>18s} {d[k][0]}")
st = []
for h, (u, v) in d.items():
    m = re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", h)
    if m and not h.endswith("not_issued"):
        try:
            st.append((float(v), m.group(1)))
        except ValueError:
            pass
tot = sum(v for v, _ in st) or 1
print("stall samples:", ", ".join(f"{n} {100*v/tot:.1f}%" for v, n in sorted(st, reverse=True)[:10]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
h2 = r[1]; data = r[2:]
ia = h2.index("Source"); isamp = h2.index("Warp Stall Sampling (All Samples)"); iex = h2.index("Instructions Executed")
c = Counter(); n = Counter(); tot = 0
for row in data:
    toks = row[ia].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    c[op] += int(row[isamp]); n[op] += int(row[iex]); tot += int(row[isamp])
print("opcode   samples%   executed(warp-instr)")
for op, v in c.most_common(16):
    print(f"  {op:10s} {100*v/max(tot,1):5.1f}%  {n[op]}")

# per-opcode stall reasons
cols = [c for c in h2 if c.startswith("stall_") and "Not Issued" not in c]
agg = {}
for row in data:
    toks = row[ia].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    a = agg.setdefault(op, Counter())
    for cname in cols:
        try:
            a[cname] += int(row[h2.index(cname)])
        except ValueError:
            pass
print("per-opcode top stall reasons (samples):")
for op, v in c.most_common(10):
    top = ", ".join(f"{k[6:]}={n}" for k, n in agg[op].most_common(4))
    print(f"  {op:10s} {top}")
