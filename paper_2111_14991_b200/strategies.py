"""run_bo / run_strategy (strategies.hpp:25-122,261-457 of the reference) over
the C ABI: the C++ host mirror (include/gridtune_b200/strategies.hpp) drives
the resident device surrogate; this module only marshals arguments."""
from __future__ import annotations

import math

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from ._lib import load
from .gp import ExplorationConfig, MaternNu, check
from .runtime import Space


class StrategyId(enum.IntEnum):
    bo_advanced_multi = 0
    bo_multi = 1
    bo_ei = 2
    bo_poi = 3
    bo_lcb = 4

    def __str__(self):
        return {0: "bo-advanced-multi", 1: "bo-multi", 2: "bo-ei", 3: "bo-poi", 4: "bo-lcb"}[int(self)]


def strategy_from_string(s: str) -> Optional[StrategyId]:
    for sid in StrategyId:
        if str(sid) == s:
            return sid
    return None


@dataclass
class StrategyConfig:
    id: StrategyId = StrategyId.bo_advanced_multi
    seed: int = 0
    budget: int = 220
    n_init: int = 20
    invalid_consumes_budget: bool = True
    nu: MaternNu = MaternNu.three_halves
    lengthscale: Optional[float] = None
    output_variance: float = 1.0
    noise: float = 1e-10
    jitter: float = 1e-6
    exploration: ExplorationConfig = field(default_factory=ExplorationConfig)
    discount: Optional[float] = None
    required_improvement: float = 0.1
    skip_threshold: int = 5
    lhs_restarts: int = 50

    def c(self) -> _lib.gtc_bo_config:
        return _lib.gtc_bo_config(
            int(self.id), int(self.seed) & 0xFFFFFFFFFFFFFFFF, int(self.budget), int(self.n_init),
            1 if self.invalid_consumes_budget else 0, int(self.nu),
            float(self.lengthscale) if self.lengthscale is not None else math.nan, float(self.output_variance),
            float(self.noise), float(self.jitter), int(self.exploration.mode), float(self.exploration.constant),
            float(self.discount) if self.discount is not None else math.nan, float(self.required_improvement),
            int(self.skip_threshold), int(self.lhs_restarts))


@dataclass
class TuningRun:
    positions: np.ndarray
    ids: np.ndarray
    values: np.ndarray      # NaN where invalid
    valid: np.ndarray
    best_so_far: np.ndarray
    lambdas: np.ndarray     # per BO iteration (the inspect hook's lambda)
    evaluations: int
    budget_consumed: int
    invalid_count: int
    surrogate_size: int
    best_value: float
    best_position: int
    n_warnings: int

    def best_at(self, evaluation_count: int) -> float:
        if len(self.positions) == 0 or evaluation_count == 0:
            return float("inf")
        return float(self.best_so_far[min(evaluation_count, len(self.positions)) - 1])


def run_bo(space: Space, ids, config: StrategyConfig, values=None,
           objective: Optional[Callable[[int, int], Optional[float]]] = None) -> TuningRun:
    """Runs one BO tuning run.  Either `values` (replay table over positions,
    NaN = runtime-invalid; the simulation mode) or `objective(position, id)`
    returning a float or None (invalid)."""
    ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64))
    if len(ids) != space.n:
        raise ValueError("ids must have one entry per position")
    cap = int(config.budget) + space.n + 1 if not config.invalid_consumes_budget else int(config.budget) + 1
    cap = min(cap, space.n + 1)
    recs = (_lib.gtc_bo_record * cap)()
    lams = np.zeros(cap)
    summ = _lib.gtc_bo_summary()
    cfg = config.c()
    lib = load()
    if values is not None:
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
        rc = lib.gtc_run_bo_table(space.handle, ids.ctypes.data_as(_lib.U64P), C.byref(cfg), _lib.dptr(v),
                                  recs, _lib.dptr(lams), cap, C.byref(summ))
    else:
        err = []

        def cb(ctx, pos, cid, out):
            try:
                r = objective(int(pos), int(cid))
            except Exception as e:  # noqa: BLE001
                err.append(e)
                return -1
            if r is None:
                return 0
            out[0] = float(r)
            return 1

        fn = _lib.OBJECTIVE_FN(cb)
        rc = lib.gtc_run_bo(space.handle, ids.ctypes.data_as(_lib.U64P), C.byref(cfg), fn, None, recs,
                            _lib.dptr(lams), cap, C.byref(summ))
        if err:
            raise err[0]
    check(rc)
    return _tuning_run(recs, lams, summ)


def _tuning_run(recs, lams, summ) -> TuningRun:
    n = summ.n_records
    arr = np.ctypeslib.as_array(recs)[:n]
    return TuningRun(
        positions=np.array([r["position"] for r in arr], dtype=np.int64) if n else np.zeros(0, np.int64),
        ids=np.array([r["id"] for r in arr], dtype=np.uint64) if n else np.zeros(0, np.uint64),
        values=np.array([r["value"] for r in arr]) if n else np.zeros(0),
        valid=np.array([bool(r["valid"]) for r in arr]) if n else np.zeros(0, bool),
        best_so_far=np.array([r["best_so_far"] for r in arr]) if n else np.zeros(0),
        lambdas=lams[:summ.n_lambdas].copy(),
        evaluations=summ.evaluations, budget_consumed=summ.budget_consumed,
        invalid_count=summ.invalid_count, surrogate_size=summ.surrogate_size,
        best_value=summ.best_value, best_position=summ.best_position, n_warnings=summ.n_warnings)


def run_bo_batch(space: Space, ids, configs, values, threads: int = 0) -> list:
    """Independent BO runs over one resident space and replay table, driven by
    a host thread pool on the device (run_experiment's worker model,
    experiment.hpp:313-358; gtc_run_bo_batch).  Returns one TuningRun per
    config, in order; raises the first failing run's error."""
    ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64))
    if len(ids) != space.n:
        raise ValueError("ids must have one entry per position")
    v = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    n = len(configs)
    cap = space.n + 1
    recs = (_lib.gtc_bo_record * (cap * max(n, 1)))()
    lams = np.zeros(cap * max(n, 1))
    summ = (_lib.gtc_bo_summary * max(n, 1))()
    cfgs = (_lib.gtc_bo_config * max(n, 1))(*[c.c() for c in configs])
    st = np.zeros(max(n, 1), dtype=np.int32)
    rc = load().gtc_run_bo_batch(space.handle, ids.ctypes.data_as(_lib.U64P), cfgs, n, _lib.dptr(v), int(threads),
                                 recs, _lib.dptr(lams), cap, summ, st.ctypes.data_as(C.POINTER(C.c_int32)))
    check(rc)
    rsize = C.sizeof(_lib.gtc_bo_record)
    out = []
    for i in range(n):
        sub = (_lib.gtc_bo_record * cap).from_address(C.addressof(recs) + i * cap * rsize)
        out.append(_tuning_run(sub, lams[i * cap:(i + 1) * cap], summ[i]))
    return out


run_strategy = run_bo
