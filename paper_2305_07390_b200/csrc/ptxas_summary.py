"""Summarise ptxas -v logs: demangled kernel, registers, spills."""
import glob, os, re, subprocess, sys

base = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.abspath(__file__)), "../../build/csrc")
recs = []
for log in sorted(glob.glob(os.path.join(base, "*.ptxas.log"))):
    cur = spill = None
    for line in open(log):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            spill = m.groups()
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            recs.append((cur, m.group(1), spill))
            cur = None
names = subprocess.run(["c++filt"], input="\n".join(r[0] for r in recs), capture_output=True, text=True).stdout.splitlines()
for (mangled, regs, sp), name in zip(recs, names):
    name = re.sub(r"\(ebisu::TmapSet.*$", "", name).replace("ebisu::", "")
    print(f"{name:75s} regs={regs:>4s} stack={sp[0]} spill={sp[1]}/{sp[2]}")
