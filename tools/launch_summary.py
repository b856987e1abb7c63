"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) from
the first k_gp_append on (the steady-state BO iterations of bench.py)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
names = [d["Kernel Name"] for d in data]
i0 = next(i for i, n in enumerate(names) if "k_gp_append" in n)
agg = collections.OrderedDict()
for d in data[i0:]:
    n = d["Kernel Name"].split("(")[0]
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}[d["Metric Unit"]]
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += float(d["Metric Value"]) * scale
tot = sum(a[1] for a in agg.values())
print(f"# {len(data)} launches total; steady-state region from the first k_gp_append ({len(data) - i0} launches)")
print(f"{'kernel':50s} launches   total_us    avg_us   share")
for n, a in agg.items():
    print(f"{n:50s} {a[0]:8d} {a[1]:10.1f} {a[1] / a[0]:9.2f} {a[1] / tot * 100:6.1f}%")
