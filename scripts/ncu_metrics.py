"""Extract the per-launch figures bench.py reports next to its roofline (DRAM bytes, tensor-pipe
activity) from `ncu --set full` captures into profiles/ncu_metrics.json:
    python scripts/ncu_metrics.py <key> <capture.ncu-rep> [<key> <capture.ncu-rep> ...]
key = "<kernel>/<config>", e.g. mvm_tc2_kernel/C3.  Existing keys not named are kept."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_metrics.json")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(m, k):
    v, u = m[k]
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 0.01}.get(u, 1)
    return x * scale


data = {}
if os.path.exists(OUT):
    with open(OUT) as f:
        data = json.load(f)
args = sys.argv[1:]
for key, rep in zip(args[0::2], args[1::2]):
    m = raw(rep)
    data[key] = {"dram_bytes": num(m, "dram__bytes_read.sum") + num(m, "dram__bytes_write.sum"),
                 "tensor_pipe_active": num(m, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                 "duration_us": num(m, "gpu__time_duration.sum") * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[
                     m["gpu__time_duration.sum"][1]],
                 "source": f"{os.path.relpath(rep, ROOT)} (ncu --set full --clock-control none)"}
    print(key, data[key])
with open(OUT, "w") as f:
    json.dump(data, f, indent=1, sort_keys=True)
