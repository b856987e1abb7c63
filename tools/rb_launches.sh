#!/bin/bash
# Per-kernel launch list of one C4-shape fit for each rebuild mode given
# (GTC_REBUILD=wide|pmma|widemma|dmma|stream), into gpurun_out/rb_launch_<mode>.csv
for m in "$@"; do
  GTC_REBUILD=$m timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/fit_timing.py 220 1 > gpurun_out/rb_launch_$m.csv 2>/dev/null
done
