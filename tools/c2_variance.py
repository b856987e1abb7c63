"""Diagnostics: run-to-run spread of the C2 sweep inside one process, by host
thread count and batch mode (observe groups vs resident loops)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2111_14991_b200 as gt  # noqa: E402

prepared = []
for name, (params, rs, invalid, minimum) in bench.C2_SPACES.items():
    es = gt.SearchSpace([gt.ParameterDef(k, v) for k, v in params], rs).enumerate()
    values = bench.c2_values(es.n, invalid, minimum, bench.BASE_SEED + len(name))
    cfgs = [gt.StrategyConfig(id=gt.StrategyId.bo_multi, seed=bench.BASE_SEED + r, budget=220, n_init=20)
            for r in range(35)]
    gt.run_bo_batch(es, es.ids, cfgs, values, threads=35)  # populate the space's run pool
    prepared.append((es, values, cfgs))
for mode in ("0", "1"):
    os.environ["GTC_BATCH_RESIDENT"] = mode
    for threads in (4, 8, 16, 35):
        ts = []
        for rep in range(4):
            t0 = time.perf_counter()
            for es, values, cfgs in prepared:
                gt.run_bo_batch(es, es.ids, cfgs, values, threads=threads)
            ts.append(time.perf_counter() - t0)
        print(f"resident={mode} threads={threads}: runs/s per rep {[round(70 / t, 1) for t in ts]}", flush=True)
