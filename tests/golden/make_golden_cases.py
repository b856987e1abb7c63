"""Golden trajectories of the UNMODIFIED reference run_bo (oracle/_ref/ref_tool
runbo_spec) on the BASELINE.json simulation-mode cases: C1 (GEMM space of
PAPER.md:319-333 with Kernel Tuner's restrictions, 17,956 configurations) and
C2 (convolution 9,400 / pnpoly 8,184 configurations with their invalid
fractions), values = bench.c2_values (seeded synthetic measurements; no cache
files exist).  Each case_<name>.npz holds the space spec, the values and the
reference trajectory (positions, values, lambdas, best, warnings).

Needs /root/reference (this container only); the outputs are committed.

  python tests/golden/make_golden_cases.py
"""
from __future__ import annotations

import json
import pathlib
import subprocess
import sys
import tempfile

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

TOOL = ROOT / "oracle" / "_ref" / "ref_tool"
SPACES = {"gemm": bench.GEMM, **bench.C2_SPACES}
# (case, space, strategy, budget, n_init, bo_seed)
CASES = [
    ("c1_gemm_ei", "gemm", "bo-ei", 220, 20, 20261017),
    ("c1_gemm_lcb", "gemm", "bo-lcb", 120, 20, 11),
    ("c2_conv_multi", "conv", "bo-multi", 220, 20, 20261018),
    ("c2_pnpoly_multi", "pnpoly", "bo-multi", 220, 20, 20261019),
    ("c2_conv_poi", "conv", "bo-poi", 150, 20, 7),
    ("c2_pnpoly_adv", "pnpoly", "bo-advanced-multi", 150, 20, 8),
]


def spec_of(space):
    params, rs, _, _ = SPACES[space]
    return {"params": [{"name": k, "kind": "numeric", "values": [float(x) for x in v]} for k, v in params],
            "restrictions": rs}


def main():
    for name, space, strat, budget, n_init, seed in CASES:
        spec = spec_of(space)
        with tempfile.TemporaryDirectory() as tmp:
            tmp = pathlib.Path(tmp)
            (tmp / "spec.json").write_text(json.dumps(spec))
            info = json.loads(subprocess.run([str(TOOL), "enumjson", str(tmp / "spec.json"), str(tmp / "sp")],
                                             check=True, capture_output=True, text=True).stdout)
            _, _, invalid, minimum = SPACES[space]
            values = bench.c2_values(info["n"], invalid, minimum, bench.BASE_SEED + len(space))
            values.astype("<f8").tofile(tmp / "values.f64")
            out = subprocess.run([str(TOOL), "runbo_spec", str(tmp / "spec.json"), str(tmp / "values.f64"), strat,
                                  str(budget), str(n_init), str(seed), str(tmp / "run")],
                                 check=True, capture_output=True, text=True).stdout
            res = json.loads(out.strip().splitlines()[-1])
            np.savez_compressed(
                HERE / f"case_{name}.npz", spec=json.dumps(spec), ids=np.load(tmp / "sp" / "ids.npy"), values=values,
                strategy=strat, budget=budget, n_init=n_init, seed=seed,
                traj_pos=np.load(tmp / "run" / "traj_pos.npy"), traj_val=np.load(tmp / "run" / "traj_val.npy"),
                traj_lambda=np.load(tmp / "run" / "traj_lambda.npy"), best=res["best"], warnings=res["warnings"],
                surrogate=res["surrogate"])
            print(name, res, flush=True)


if __name__ == "__main__":
    main()
