"""Per-kernel share of an `ncu --metrics gpu__time_duration.sum --csv` launch list.
    python scripts/launch_summary.py gpurun_out/launches_r01b.csv"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
iname, imet, ival, iunit = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[1:]:
    if r[imet] != "gpu__time_duration.sum":
        continue
    v = float(r[ival].replace(",", ""))
    v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[iunit], 1.0)
    name = re.sub(r"\(.*$", "", r[iname]).replace("void ", "").replace("ciq::", "").replace("<unnamed>::", "")
    name = name.replace("(int)", "")
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
print(f"{'kernel':44s} {'launches':>9s} {'total ms':>10s} {'share':>7s} {'avg us':>9s}")
for k, v in tot.most_common():
    print(f"{k[:44]:44s} {cnt[k]:9d} {v:10.2f} {100*v/s:6.1f}% {1000*v/cnt[k]:9.1f}")
print(f"{'total':44s} {sum(cnt.values()):9d} {s:10.2f}")
