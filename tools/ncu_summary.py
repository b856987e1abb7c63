"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list of
`bench.py --steps K`: per-kernel launches / time / share over the bench's
timed resident call (the launches between the 2nd and 3rd k_gp_truncate,
i.e. the second gtc_run_steps chunk incl. its posterior refresh)."""
import csv
import sys
from collections import OrderedDict


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}
    seq = [(r[ki], float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)) for r in data
           if r[mi] == "gpu__time_duration.sum"]
    cuts = [i for i, (k, _) in enumerate(seq) if k.startswith("k_gp_truncate")]
    lo, hi_ = cuts[1], cuts[2]
    region = seq[lo:hi_]
    agg = OrderedDict()
    for k, v in region:
        name = k.split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"# {len(seq)} launches total; summary over the timed resident call (launches {lo}..{hi_ - 1})")
    print(f"{'kernel':50s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>7s}")
    for k, (n, t) in agg.items():
        print(f"{k:50s} {n:8d} {t:10.1f} {t / n:9.2f} {100 * t / tot:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
