"""Prints the per-kernel times of gpurun_out/rb_launch_<mode>.csv (tools/rb_launches.sh)."""
import csv
import sys

for m in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f"gpurun_out/rb_launch_{m}.csv")) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot = 0.0
    print("==", m)
    for r in rows[1:]:
        us = float(r[vi].replace(",", "")) / 1e3
        tot += us
        print(f"  {r[ki][:44]:44s} {us:9.1f} us")
    print(f"  {'total':44s} {tot:9.1f} us")
