"""Timeline of one resident C4 iteration from the %globaltimer marks of a
GTC_SEL_TRACE build (tools/build_trace.sh -> libgridtune_b200_trace.so):
selection phases per block, the last block's publish, the loop-mode append
and the pass start.  Diagnostic only.

  GRIDTUNE_B200_LIB=paper_2111_14991_b200/libgridtune_b200_trace.so python tools/select_trace.py [c4|c3]
"""
import ctypes as C
import json
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2111_14991_b200 as gt  # noqa: E402
from paper_2111_14991_b200 import _lib  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = bench.CONFIGS[cfg_name]
coords, ids, values = bench.make_workload(cfg)
n = 220
space = gt.Space(coords)
run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0), n_max=n)
pos = bench.prefix_positions(values, n - 1, bench.BASE_SEED)
y = values[pos]
run.fit(pos, y)
for p in pos:
    run.mark_visited(int(p))
af = gt.AcquisitionId(bench.CONFIG_AF[cfg["af"]])
cv = gt.ContextualVarianceState(float(np.mean(y[:20])), run.mean_variance())
run.set_values(values)
out = []
for rep in range(5):
    run.truncate_async(n - 1)
    recs = run.steps(af, 4, float(np.min(y)), gt.ExplorationConfig(), cv, hold=True)
    run.unmark_visited(recs[-1].position)
    marks = np.zeros((2048, 8), dtype=np.uint64)
    rc = _lib.load().gtc_debug_select_trace(marks.ctypes.data_as(_lib.U64P), 2048)
    if rc != 0:  # (not a GTC_SEL_TRACE build: the loop still runs, e.g. under ncu)
        continue
    blocks = marks[:2040]
    used = blocks[:, 0] > 0
    b = blocks[used].astype(np.int64)
    t0 = int(b[:, 7].min())
    rel = lambda v: round((int(v) - t0) / 1e3, 2)  # noqa: E731
    row = {
        "blocks": int(used.sum()),
        "select_start_first": 0.0, "select_start_last": rel(b[:, 0].max()),
        "setup_median": rel(np.median(b[:, 1])), "threshold_median": rel(np.median(b[:, 2])),
        "expand_median": rel(np.median(b[:, 3])), "expand_max": rel(b[:, 3].max()),
        "partials_max": rel(b[:, 5].max()),
        "entry_median": rel(np.median(b[:, 7])), "loaded_median": rel(np.median(b[:, 4])),
        "pass_end": rel(marks[2043, 1]),
        "last_block_entry": rel(marks[2042, 0]), "last_merged": rel(marks[2042, 1]),
        "publish_done": rel(marks[2042, 2]), "advance_done": rel(marks[2042, 3]),
        "append_start": rel(marks[2040, 0]), "append_prologue": rel(marks[2040, 1]),
        "append_column": rel(marks[2040, 2]), "pass_start": rel(marks[2041, 0]),
        "pass_staged_block0": rel(marks[2041, 1]), "pass_staged_last": rel(marks[2041, 2]),
    }
    out.append(row)
print(json.dumps({"config": cfg_name, "us_since_first_select_block": out}, indent=1))
