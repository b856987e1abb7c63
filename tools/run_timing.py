"""Per-run latency of gtc_run_bo_table on the C2 conv space (diagnostics):
resident single-AF loop vs the per-iteration gtc_observe loop, and the batch
throughput of single-AF runs with both."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2111_14991_b200 as gt  # noqa: E402

params, rs, invalid, minimum = bench.C2_SPACES["conv"]
es = gt.SearchSpace([gt.ParameterDef(k, v) for k, v in params], rs).enumerate()
values = bench.c2_values(es.n, invalid, minimum, 5)
for mode in ("1", "0"):
    os.environ["GTC_RESIDENT_LOOP"] = mode
    ts = []
    for r in range(6):
        cfg = gt.StrategyConfig(id=gt.StrategyId.bo_ei, seed=r, budget=220, n_init=20)
        t0 = time.perf_counter()
        gt.run_bo(es, es.ids, cfg, values=values)
        ts.append(time.perf_counter() - t0)
    print(f"resident={mode} single run ms: {[round(1e3 * t, 2) for t in ts]}")
    cfg = gt.StrategyConfig(id=gt.StrategyId.bo_ei, seed=1, budget=40, n_init=20)
    t0 = time.perf_counter()
    gt.run_bo(es, es.ids, cfg, values=values)
    print(f"  budget 40 (initial design incl. repairs + fit + ~few iterations): {1e3 * (time.perf_counter() - t0):.2f} ms")
for br in ("1", "0"):
    os.environ["GTC_RESIDENT_LOOP"] = "1"
    os.environ["GTC_BATCH_RESIDENT"] = br
    cfgs = [gt.StrategyConfig(id=gt.StrategyId.bo_ei, seed=r, budget=220, n_init=20) for r in range(128)]
    for threads in (4, 16, 32):
        t0 = time.perf_counter()
        gt.run_bo_batch(es, es.ids, cfgs, values, threads=threads)
        dt = time.perf_counter() - t0
        print(f"batch resident={br} threads={threads}: {len(cfgs) / dt:.1f} runs/s")
