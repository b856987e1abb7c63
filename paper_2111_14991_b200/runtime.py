"""Resident search space and BO-run handles (C ABI gtc_space / gtc_run).

`Space` keeps the normalised candidate coordinates in HBM
(EnumeratedSpace, search_space.hpp:216-245).  `SurrogateRun` owns one run's
surrogate state on the device — the Cholesky factor, V = L^-1 K* for every
candidate, the posterior and the visited mask — and exposes the hot path of
run_bo (strategies.hpp:298-449) as fit / append / mark_visited / select.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import load
from .gp import (AcquisitionId, ContextualVarianceState, ExplorationConfig, MaternKernel, check)


class Space:
    def __init__(self, coords, device: int = 0):
        c = np.ascontiguousarray(np.asarray(coords, dtype=np.float64))
        if c.ndim != 2:
            raise ValueError("coords must be n x d")
        self.n, self.d = c.shape
        self.device = device
        self.coords = c
        h = C.c_void_p()
        check(load().gtc_space_create(device, _lib.dptr(c), self.n, self.d, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def size(self) -> int:
        return self.n

    def nearest(self, points) -> np.ndarray:
        """Positions of the configurations nearest to `points` (m x d in
        [0,1]^d; lowest position on ties) -- the initial-sample snap of
        draw_initial_sample (sampling.hpp:98-117), on the device."""
        p = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, self.d))
        out = np.empty(len(p), dtype=np.int64)
        check(load().gtc_space_nearest(self._h, _lib.dptr(p), len(p), _lib.i64ptr(out)))
        return out

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            load().gtc_space_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class FitInfo:
    n: int
    rebuilt: bool
    y_mean: float
    y_std: float
    jitter: float

    @staticmethod
    def of(i: _lib.gtc_fit_info) -> "FitInfo":
        return FitInfo(i.n, bool(i.rebuilt), i.y_mean, i.y_std, i.jitter)


@dataclass
class Selection:
    position: tuple          # per AF slot (ei, poi, lcb); -1 when not requested
    score: tuple
    lambda_: float
    mean_variance: float
    best_std: float
    n_candidates: int
    cv_fallback: bool

    def pick(self, af: AcquisitionId) -> int:
        return int(self.position[int(af)])


class SurrogateRun:
    def __init__(self, space: Space, kernel: MaternKernel, noise: float = 1e-10,
                 jitter: float = 1e-6, n_max: int = 220):
        self.space = space
        cfg = _lib.gtc_model_config(kernel.c(), float(noise), float(jitter), int(n_max))
        h = C.c_void_p()
        check(load().gtc_run_create(space.handle, C.byref(cfg), C.byref(h)))
        self._h = h
        self.kernel = kernel
        self.n_max = n_max

    @property
    def handle(self):
        return self._h

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            load().gtc_run_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def fit(self, positions: Sequence[int], y_raw: Sequence[float]) -> FitInfo:
        p = np.ascontiguousarray(np.asarray(positions, dtype=np.int64))
        y = np.ascontiguousarray(np.asarray(y_raw, dtype=np.float64))
        info = _lib.gtc_fit_info()
        check(load().gtc_fit(self._h, _lib.i64ptr(p), _lib.dptr(y), len(y), C.byref(info)))
        return FitInfo.of(info)

    def append(self, position: int, y_raw: float) -> FitInfo:
        info = _lib.gtc_fit_info()
        check(load().gtc_append(self._h, int(position), float(y_raw), C.byref(info)))
        return FitInfo.of(info)

    def truncate(self, n: int) -> FitInfo:
        info = _lib.gtc_fit_info()
        check(load().gtc_truncate(self._h, int(n), C.byref(info)))
        return FitInfo.of(info)

    def mark_visited(self, position: int) -> None:
        check(load().gtc_mark_visited(self._h, int(position)))

    def unmark_visited(self, position: int) -> None:
        check(load().gtc_unmark_visited(self._h, int(position)))

    def unvisited_count(self) -> int:
        return int(load().gtc_unvisited_count(self._h))

    def mean_variance(self) -> float:
        out = C.c_double()
        cnt = C.c_int64()
        check(load().gtc_mean_variance(self._h, C.byref(out), C.byref(cnt)))
        return out.value

    def predictions(self):
        n = self.space.n
        mean = np.empty(n)
        var = np.empty(n)
        check(load().gtc_read_predictions(self._h, _lib.dptr(mean), _lib.dptr(var)))
        return mean, var

    @staticmethod
    def _args(afs, f_best_raw, exploration, cv_state, excluded):
        mask = 0
        for af in afs:
            mask |= 1 << int(af)
        a = _lib.gtc_select_args(mask, int(exploration.mode), float(exploration.constant),
                                 float(cv_state.initial_sample_mean),
                                 float(cv_state.initial_mean_variance), float(f_best_raw), None, 0)
        ex = None
        if excluded:
            ex = np.ascontiguousarray(np.asarray(excluded, dtype=np.int64))
            a.excluded = _lib.i64ptr(ex)
            a.n_excluded = len(ex)
        return a, ex

    @staticmethod
    def _selection(r) -> Selection:
        return Selection(tuple(r.position[:]), tuple(r.score[:]), r.lambda_, r.mean_variance, r.best_std,
                         r.n_candidates, bool(r.cv_fallback))

    def select(self, afs: Sequence[AcquisitionId], f_best_raw: float,
               exploration: ExplorationConfig = ExplorationConfig(),
               cv_state: ContextualVarianceState = ContextualVarianceState(),
               excluded: Optional[Sequence[int]] = None) -> Selection:
        a, _keep = self._args(afs, f_best_raw, exploration, cv_state, excluded)
        r = _lib.gtc_select_result()
        check(load().gtc_select(self._h, C.byref(a), C.byref(r)))
        return self._selection(r)

    def observe(self, position: int, y_raw: Optional[float], afs: Sequence[AcquisitionId] = (),
                f_best_raw: float = 0.0, exploration: ExplorationConfig = ExplorationConfig(),
                cv_state: ContextualVarianceState = ContextualVarianceState(),
                excluded: Optional[Sequence[int]] = None):
        """gtc_observe: mark visited, append when y_raw is not None, then the
        next selection (when afs is non-empty) with one host round trip.
        Returns (FitInfo, Selection or None)."""
        valid = y_raw is not None
        bufs = getattr(self, "_obs_bufs", None)  # result structs (and their refs) reused across calls
        if bufs is None:
            r0, i0 = _lib.gtc_select_result(), _lib.gtc_fit_info()
            bufs = self._obs_bufs = (r0, i0, load().gtc_observe, C.byref(r0), C.byref(i0))
        r, info, observe, r_ref, info_ref = bufs
        if afs:
            if excluded:
                a, _keep = self._args(afs, f_best_raw, exploration, cv_state, excluded)
                a_ref = C.byref(a)
            else:  # per-iteration calls: reuse the argument struct, only f_best changes
                key = (tuple(map(int, afs)), exploration.mode, exploration.constant,
                       cv_state.initial_sample_mean, cv_state.initial_mean_variance)
                cached = getattr(self, "_obs_args", None)
                if cached is None or cached[0] != key:
                    a = self._args(afs, f_best_raw, exploration, cv_state, None)[0]
                    cached = self._obs_args = (key, a, C.byref(a))
                a, a_ref = cached[1], cached[2]
                a.f_best_raw = float(f_best_raw)
            rc = observe(self._h, int(position), float(y_raw) if valid else 0.0, valid, a_ref, r_ref, info_ref)
            if rc:
                check(rc)
            return FitInfo(info.n, bool(info.rebuilt), info.y_mean, info.y_std, info.jitter), self._selection(r)
        check(observe(self._h, int(position), float(y_raw) if valid else 0.0, int(valid), None, r_ref, info_ref))
        return FitInfo.of(info), None

    def set_values(self, values) -> None:
        """Simulation-mode objective: values[pos] (NaN = runtime-invalid) on the device."""
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
        check(load().gtc_run_set_values(self._h, _lib.dptr(v), len(v)))

    def set_pdl(self, enable: bool) -> None:
        """gtc_run_set_pdl: programmatic dependent launch on (default) or off
        (then gtc_run_steps launches captured graphs of its iterations)."""
        check(load().gtc_run_set_pdl(self._h, 1 if enable else 0))

    def set_portfolio(self, mode: int, skip_threshold: int = 5, discount: float = 0.65,
                      required_improvement: float = 0.1) -> None:
        """gtc_run_set_portfolio: 0 single AF, 1 multi, 2 advanced multi (fresh state)."""
        c = _lib.gtc_portfolio_config(int(mode), int(skip_threshold), float(discount), float(required_improvement))
        check(load().gtc_run_set_portfolio(self._h, C.byref(c)))

    def steps(self, af: AcquisitionId, k: int, f_best_raw: float,
              exploration: ExplorationConfig = ExplorationConfig(),
              cv_state: ContextualVarianceState = ContextualVarianceState(), hold: bool = False,
              timing: bool = False):
        """gtc_run_steps: k resident BO iterations (select -> table lookup ->
        mark -> append + pass) with one host synchronisation.  Returns the
        step records (position, value, lambda_, valid, cv_fallback)."""
        a, _keep = self._args([af], f_best_raw, exploration, cv_state, None)
        recs = (_lib.gtc_step_record * max(1, int(k)))()
        done = C.c_int32()
        info = _lib.gtc_fit_info()
        flags = (_lib.GTC_STEPS_HOLD_N if hold else 0) | (_lib.GTC_STEPS_TIMING if timing else 0)
        check(load().gtc_run_steps(self._h, C.byref(a), int(k), flags, recs,
                                   C.byref(done), C.byref(info)))
        return recs[:done.value]

    def exact_rows(self) -> int:
        """Bordered rows that needed the exact forward substitution because
        the V-column pivot was below the exactness margin."""
        return int(load().gtc_run_exact_rows(self._h))

    def last_steps_ms(self) -> float:
        return float(load().gtc_last_steps_ms(self._h))

    def last_steps_phase_ms(self):
        """(selection + advance, append, pass) mean CUDA-event ms per step of
        the last gtc_run_steps(timing=True) chunk."""
        out = (C.c_double * 3)()
        check(load().gtc_last_steps_phase_ms(self._h, out))
        return tuple(out)

    def truncate_async(self, n: int) -> None:
        """Model back to its first n observations without a host round trip."""
        check(load().gtc_truncate(self._h, int(n), None))

    def last_pass_ms(self) -> float:
        return float(load().gtc_last_pass_ms(self._h))

    def last_step_ms(self) -> float:
        return float(load().gtc_last_step_ms(self._h))

    def last_phase_ms(self):
        """(append, pass, selection) CUDA-event ms of the last appending observe."""
        out = (C.c_double * 3)()
        check(load().gtc_last_phase_ms(self._h, out))
        return tuple(out)
