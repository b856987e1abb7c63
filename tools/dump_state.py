"""Dumps the C4 bench selection state (mu, var, visited, scalars) for
tools/sel_bench.cu.  Diagnostic only."""
import struct
import sys

import numpy as np

sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import paper_2111_14991_b200 as gt  # noqa: E402
from paper_2111_14991_b200 import synthetic  # noqa: E402

coords, ids, values = synthetic.random_rough([10] * 6, 20261017, 0.0)
space = gt.Space(coords)
run = gt.SurrogateRun(space, gt.MaternKernel(gt.MaternNu.three_halves, 1.5, 1.0), n_max=220)
rng = np.random.default_rng(20261017)
pos = rng.choice(len(values), 219, replace=False)
y = values[pos]
run.fit(pos, y)
for p in pos:
    run.mark_visited(int(p))
mu, var = run.predictions()
vis = np.zeros((len(mu) + 31) // 32, np.uint32)
for p in pos:
    vis[p >> 5] |= np.uint32(1 << (p & 31))
with open(sys.argv[1] if len(sys.argv) > 1 else "/tmp/gtc_state.bin", "wb") as f:
    f.write(struct.pack("<q", len(mu)))
    f.write(struct.pack("<5d", float(np.min(y)), float(np.mean(y)), float(np.std(y)), float(np.mean(y[:20])),
                        run.mean_variance()))
    f.write(mu.tobytes())
    f.write(var.tobytes())
    f.write(vis.tobytes())
