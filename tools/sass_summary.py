"""Per-kernel SASS mnemonic counts of the built library (the evidence for
which pipes each kernel uses: DMMA = fp64 tensor-core MMA, UBLKCP = TMA bulk
copy, SYNCS = mbarrier, FFMA2/FADD2 = packed FP32, ...).
usage: python tools/sass_summary.py [lib] > profiles/r02/sass_summary.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1407_7737_b200/librobench_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["DMMA", "UTCMMA", "UTCHMMA", "LDTM", "UTMALDG", "UBLKCP", "UBLKPF", "SYNCS", "DFMA", "DMUL",
        "DADD", "FFMA2", "FADD2", "FMUL2", "FFMA", "FMUL", "FADD", "MUFU", "F2F", "LDG", "STG", "LDS",
        "STS", "LDL", "STL", "BAR", "SHFL", "CALL"]
funcs = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if cur and m:
        op = m.group(1)
        funcs[cur][op] += 1
        funcs[cur]["_total"] += 1
names = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.split("\n")
tot = collections.Counter()
print("kernel".ljust(58), "insts", *[k for k in KEYS])
for (mangled, cnt), name in zip(funcs.items(), names):
    name = re.sub(r"\(rb::.*", "", name.replace("void ", "").replace("rb::", ""))
    tot.update(cnt)
    print(name[:58].ljust(58), cnt["_total"], *[cnt.get(k, 0) for k in KEYS])
print("TOTAL".ljust(58), tot["_total"], *[tot.get(k, 0) for k in KEYS])
