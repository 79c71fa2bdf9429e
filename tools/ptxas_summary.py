"""Summarise ptxas -v output (paper_2503_08935_b200/lib/ptxas.log): regs / spills per kernel."""
import re
import subprocess
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2503_08935_b200/lib/ptxas.log").read()
cur = None
info = {}
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        info[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        info[cur]["stack"], info[cur]["spill_st"], info[cur]["spill_ld"] = map(int, m.groups())
    m = re.search(r"Used (\d+) registers", line)
    if m:
        info[cur]["regs"] = int(m.group(1))
names = {}
try:
    out = subprocess.run(["c++filt"], input="\n".join(info), capture_output=True, text=True).stdout
    names = dict(zip(info, out.splitlines()))
except Exception:
    pass
for k, v in info.items():
    n = names.get(k, k)
    n = re.sub(r"\(anonymous namespace\)::", "", n)
    print(f"{v.get('regs', '?'):>4} regs  stack {v.get('stack', 0):>3}  spill {v.get('spill_st', 0):>4}/{v.get('spill_ld', 0):<4} {n[:110]}")
