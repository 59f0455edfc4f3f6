"""Summarise ptxas -v logs: kernel template args, registers, spills."""
import glob, re, sys, os
base = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "../../build/csrc")
for log in sorted(glob.glob(os.path.join(base, "*.ptxas.log"))):
    cur = None
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
            dm = re.search(r"k_stream2dINS_(\w+?)ILi(\d)ELi(\d)EEELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELb(\d)ELi(\d+)E", cur)
            name = cur if not dm else f"stream2d {dm.group(1)}<{dm.group(2)},{dm.group(3)}> T={dm.group(4)} C={dm.group(5)} exact={dm.group(8)} minb={dm.group(9)}"
            print(f"{name:60s} regs={m.group(1):>4s} stack={spill[0]} spill_st={spill[1]} spill_ld={spill[2]}")
            cur = None
