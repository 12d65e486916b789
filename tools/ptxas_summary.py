"""Summarise ptxas -v output (paper_1407_7737_b200/build.log): registers,
stack and spills per kernel entry, demangled."""
import re
import subprocess
import sys
from pathlib import Path

log = Path(sys.argv[1] if len(sys.argv) > 1 else "paper_1407_7737_b200/build.log").read_text()
rows, cur = [], None
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\S+)' for", line)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and "stack" not in cur:
        cur["stack"], cur["st"], cur["ld"] = map(int, m.groups())
    m = re.search(r"Used (\d+) registers", line)
    if m and "regs" not in cur:
        cur["regs"] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(r["name"] for r in rows), capture_output=True,
                       text=True).stdout.splitlines()
only_spills = "--spills" in sys.argv
for r, n in zip(rows, names):
    if only_spills and not r.get("st"):
        continue
    n = n.replace("(rb::Args<double>)", "").replace("(rb::Args<float>)", "")
    print(f"{r.get('regs', 0):4d} regs {r.get('stack', 0):5d} B stack {r.get('st', 0):5d}/{r.get('ld', 0):5d} spill  {n}")
