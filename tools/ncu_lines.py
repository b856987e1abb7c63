"""Warp-stall samples of one kernel aggregated per CUDA source line, from
`ncu -i REP --page source --csv --print-source cuda,sass`.  Diagnostic.

  ncu -i rep --page source --csv --print-source cuda,sass -k regex:NAME > x.csv
  python tools/ncu_lines.py x.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg, cur, fname = {}, None, ""
si = None
reasons = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        si = r.index("Warp Stall Sampling (All Samples)")
        reasons = [(i, h) for i, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if si is None or len(r) <= si:
        continue
    if r[0]:
        cur = (fname, r[0], r[1].strip()[:100])
        continue
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    e = agg.setdefault(cur, [0.0, {}])
    e[0] += v
    for i, h in reasons:
        try:
            x = float(r[i] or 0)
        except ValueError:
            continue
        if x:
            e[1][h] = e[1].get(h, 0) + x
tot = sum(v[0] for v in agg.values()) or 1
print("total samples", tot)
for k, (v, rs) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    main = ", ".join(f"{h[6:]} {100 * x / v:.0f}%" for h, x in sorted(rs.items(), key=lambda t: -t[1])[:3])
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]} {k[2]}  [{main}]")
