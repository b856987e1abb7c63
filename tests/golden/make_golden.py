"""Regenerates the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs oracle/_ref/ref_tool (the reference headers compiled against the in-repo
Eigen/GTest shims, see oracle/Makefile).  Needs /root/reference, so it only
runs in the build container; the resulting .npz files are committed.

  python tests/golden/make_golden.py
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
TOOL = ROOT / "oracle" / "_ref" / "ref_tool"

# (name, function, grid, space seed, invalid fraction, strategy, budget, n_init, bo seed)
TRAJECTORIES = [
    ("rr13_adv", "random-rough", "13x13", 17, "0.3", "bo-advanced-multi", 70, 12, 1),
    ("rr13_multi", "random-rough", "13x13", 17, "0.3", "bo-multi", 70, 12, 2),
    ("rr13_ei", "random-rough", "13x13", 17, "0.3", "bo-ei", 70, 12, 1),
    ("rr13_poi", "random-rough", "13x13", 17, "0.3", "bo-poi", 70, 12, 1),
    ("rr13_lcb", "random-rough", "13x13", 17, "0.3", "bo-lcb", 70, 12, 1),
    ("rr10_adv", "random-rough", "10x10", 41, "0.1", "bo-advanced-multi", 45, 10, 12),
    ("rr6x6_ei", "random-rough", "6x6", 3, "0", "bo-ei", 100, 8, 1),
    ("rr4d_ei", "random-rough", "8x8x6x5", 5, "0.2", "bo-ei", 120, 20, 7),
    ("rr4d_multi", "random-rough", "8x8x6x5", 5, "0.2", "bo-multi", 120, 20, 8),
    ("rosen_adv", "rosenbrock-disc", "30x30", 1, "-", "bo-advanced-multi", 80, 15, 3),
    ("rr3d_lcb", "random-rough", "12x12x12", 9, "0.385", "bo-lcb", 150, 20, 4),
]

# BASELINE.json configs[2] (C3): synthetic 100k-candidate space (6 params, ~30 %
# invalid), bo-lcb with contextual variance, budget 220, n_init 20.  Written
# without the space (1.6 MB): tests regenerate it with
# paper_2111_14991_b200.synthetic.random_rough, which is pinned bit-exact to
# the reference generator (space_c3.npz).
BIG_TRAJECTORIES = [
    ("c3_lcb", "random-rough", "10x10x10x10x5x2", 20261017, "0.3", "bo-lcb", 220, 20, 1),
]


def run(*args) -> dict:
    out = subprocess.run([str(TOOL), *map(str, args)], check=True, capture_output=True, text=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def load_dir(d: pathlib.Path) -> dict:
    return {p.stem: np.load(p) for p in sorted(d.glob("*.npy"))}


def main() -> None:
    if not TOOL.exists():
        sys.exit("oracle/_ref/ref_tool missing: run `make -C oracle ref` (needs /root/reference)")
    with tempfile.TemporaryDirectory() as tmp:
        tmp = pathlib.Path(tmp)
        # GpModel::fit/predict, 24 instances (n 1..40, d 1..6, all three nu)
        run("gp", 20261017, 24, tmp / "gp")
        np.savez_compressed(HERE / "gp_predict.npz", **load_dir(tmp / "gp"))
        # synthetic generator: random-rough 100k (C3 shape) + rosenbrock
        meta = run("space", "random-rough", "10x10x10x10x5x2", 20261017, "0.3", tmp / "c3")
        arrs = load_dir(tmp / "c3")
        np.savez_compressed(HERE / "space_c3.npz", ids=arrs["ids"], values=arrs["values"],
                            meta=np.array([meta["n"], meta["d"], meta["invalid"], meta["true_minimum"]]))
        # C1 GEMM space through the reference restriction parser
        meta = run("gemm", tmp / "gemm")
        arrs = load_dir(tmp / "gemm")
        np.savez_compressed(HERE / "space_gemm.npz", ids=arrs["ids"], coords=arrs["coords"],
                            meta=np.array([meta["n"], meta["d"], meta["cartesian"]]))
        # reference run_bo trajectories
        for name, fn, grid, sseed, inv, strat, budget, n_init, bseed in TRAJECTORIES:
            meta = run("runbo", fn, grid, sseed, inv, strat, budget, n_init, bseed, tmp / name)
            arrs = load_dir(tmp / name)
            np.savez_compressed(HERE / f"traj_{name}.npz", **arrs,
                                spec=np.array([fn, grid, str(sseed), inv, strat, str(budget), str(n_init), str(bseed)]),
                                best=np.array([meta["best"]]), warnings=np.array([meta["warnings"]]))
        for name, fn, grid, sseed, inv, strat, budget, n_init, bseed in BIG_TRAJECTORIES:
            meta = run("runbo", fn, grid, sseed, inv, strat, budget, n_init, bseed, tmp / name)
            arrs = load_dir(tmp / name)
            np.savez_compressed(HERE / f"trajbig_{name}.npz", traj_pos=arrs["traj_pos"], traj_val=arrs["traj_val"],
                                traj_lambda=arrs["traj_lambda"],
                                spec=np.array([fn, grid, str(sseed), inv, strat, str(budget), str(n_init), str(bseed)]),
                                best=np.array([meta["best"]]), warnings=np.array([meta["warnings"]]))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
