"""Diagnostics: where a C2 sweep's time goes -- budget 220 vs budget 45 (the
initial design + first iterations only), resident batch, 35 threads."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2111_14991_b200 as gt  # noqa: E402

os.environ["GTC_BATCH_RESIDENT"] = sys.argv[1] if len(sys.argv) > 1 else "1"
params, rs, invalid, minimum = bench.C2_SPACES["pnpoly"]
es = gt.SearchSpace([gt.ParameterDef(k, v) for k, v in params], rs).enumerate()
values = bench.c2_values(es.n, invalid, minimum, bench.BASE_SEED + 6)
for budget in (220, 45, 220, 45):
    cfgs = [gt.StrategyConfig(id=gt.StrategyId.bo_ei, seed=r, budget=budget, n_init=20) for r in range(140)]
    gt.run_bo_batch(es, es.ids, cfgs[:35], values, threads=35)
    t0 = time.perf_counter()
    gt.run_bo_batch(es, es.ids, cfgs, values, threads=35)
    dt = time.perf_counter() - t0
    print(f"resident={os.environ['GTC_BATCH_RESIDENT']} budget={budget}: {len(cfgs) / dt:.1f} runs/s "
          f"({1e3 * dt / len(cfgs) * 35:.2f} ms per run per thread)", flush=True)
