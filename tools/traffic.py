"""DRAM traffic per launch of the bench's largest kernels (ncu metrics-only
pass at the bench size), written to profiles/r02/ncu_traffic.json for
bench.py's roofline "traffic".  Run under gpurun:
    python tools/traffic.py 32:single 33:single 32:double 33:double"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

out = {}
for spec in sys.argv[1:]:
    fn, prec = spec.split(":")
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:evaluate_kernel", "-s", "1", "-c", "1", "--csv",
           sys.executable, "tools/profile_one.py", "100", "10000000", fn, prec, "2"]
    txt = subprocess.run(cmd, capture_output=True, text=True).stdout
    vals = {}
    for r in csv.reader(io.StringIO(txt[txt.find('"ID"'):])):
        if len(r) > 14 and r[12] in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            unit, v = r[13], float(r[14].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6,
                     "msecond": 1e-3, "nsecond": 1e-9, "second": 1}.get(unit, 1)
            vals[r[12]] = v * scale
    if "dram__bytes_read.sum" in vals:
        out[f"{fn}/{prec}"] = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
        print(spec, vals)
path = Path("profiles/r02/ncu_traffic.json")
prev = json.loads(path.read_text()) if path.exists() else {}
prev.update(out)
path.write_text(json.dumps(prev, indent=1))
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/ncu_traffic_r02.json").write_text(json.dumps(prev, indent=1))
