"""Candidate-axis sharding of one BO run over several GPUs (config C4).

Each rank holds a contiguous slice [offset, offset + n_local) of the global
candidate list; the GP is replicated (every rank applies the same
observations with explicit coordinates).  Per iteration:

  1. gtc_shard_observe  -> this shard's (sum, count) of the posterior variance
  2. exchange (sum, count), summed in rank order on every rank -> global mean
     variance, hence the same lambda everywhere (strategies.hpp:404-418)
  3. gtc_shard_select   -> this shard's best (score, position) per AF plus its
     first eligible position and whether that candidate's score is NaN
  4. exchange the 13-double records; `merge_shard_records` applies the
     reference's best_candidate rule (portfolio.hpp:32-61) globally.

Two latency-bound exchanges per iteration (16 B and 104 B per rank).  The
communicator is anything with `allgather(np.ndarray) -> list[np.ndarray]` in
rank order: `TorchComm` (torch.distributed, nccl or gloo) or the in-process
`ShardGroup` used to test the protocol on one device.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import load
from .gp import (AcquisitionId, ContextualVarianceState, Error, ExplorationConfig, MaternKernel, check)
from .runtime import FitInfo, Selection, Space, SurrogateRun

RECORD = 13  # doubles per shard record


@dataclass
class ShardRecord:
    best_position: tuple
    best_score: tuple
    first_eligible: int
    first_nan_mask: int
    n_candidates: int
    lambda_: float
    mean_variance: float
    best_std: float
    cv_fallback: bool

    def pack(self) -> np.ndarray:
        return np.array(list(self.best_position) + list(self.best_score) +
                        [self.first_eligible, self.first_nan_mask, self.n_candidates, self.lambda_,
                         self.mean_variance, self.best_std, float(self.cv_fallback)], dtype=np.float64)

    @staticmethod
    def unpack(a: np.ndarray) -> "ShardRecord":
        a = np.asarray(a, dtype=np.float64)
        return ShardRecord(tuple(int(x) for x in a[0:3]), tuple(float(x) for x in a[3:6]), int(a[6]), int(a[7]),
                           int(a[8]), float(a[9]), float(a[10]), float(a[11]), bool(a[12]))


def sum_in_rank_order(totals: Sequence[np.ndarray]):
    """Global (sum, count) of the per-shard variance totals, rank order."""
    s, c = 0.0, 0
    for t in totals:
        s += float(t[0])
        c += int(t[1])
    return s, c


def merge_shard_records(records: Sequence[ShardRecord], af_mask: int) -> Selection:
    """The reference's best_candidate over the union of the shards: the first
    eligible candidate (lowest global position) is taken unconditionally; if
    its score is NaN nothing beats it, otherwise the highest non-NaN score
    wins with the lowest position on ties (portfolio.hpp:32-61)."""
    live = [r for r in records if r.n_candidates > 0 and r.first_eligible >= 0]
    n_cand = sum(r.n_candidates for r in records)
    if not live:
        raise Error("acquisition: no candidates remaining")
    owner = min(live, key=lambda r: r.first_eligible)
    gfirst = owner.first_eligible
    pos = [-1, -1, -1]
    score = [0.0, 0.0, 0.0]
    for af in range(3):
        if not af_mask & (1 << af):
            continue
        if owner.first_nan_mask & (1 << af):
            pos[af], score[af] = gfirst, math.nan
            continue
        best = None
        for r in live:
            p, s = r.best_position[af], r.best_score[af]
            if p < 0:
                continue
            if best is None or s > best[0] or (s == best[0] and p < best[1]):
                best = (s, p)
        if best is None:  # every score NaN: the first candidate stands
            pos[af], score[af] = gfirst, math.nan
        else:
            score[af], pos[af] = best
    ref = records[0]
    return Selection(tuple(pos), tuple(score), ref.lambda_, ref.mean_variance, ref.best_std, int(n_cand),
                     ref.cv_fallback)


class Shard:
    """One rank's slice: a resident space of the slice + a replicated GP."""

    def __init__(self, coords_slice, offset: int, kernel: MaternKernel, noise: float = 1e-10,
                 jitter: float = 1e-6, n_max: int = 220, device: int = 0):
        self.offset = int(offset)
        self.space = Space(coords_slice, device=device)
        self.run = SurrogateRun(self.space, kernel, noise, jitter, n_max)
        self.n_local = self.space.n
        check(load().gtc_run_set_shard(self.run.handle, self.offset))

    def local(self, global_pos: int) -> int:
        p = int(global_pos) - self.offset
        return p if 0 <= p < self.n_local else -1

    def fit_points(self, X, y) -> FitInfo:
        X = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
        y = np.ascontiguousarray(np.asarray(y, dtype=np.float64))
        info = _lib.gtc_fit_info()
        check(load().gtc_fit_points(self.run.handle, _lib.dptr(X), _lib.dptr(y), len(y), C.byref(info)))
        return FitInfo.of(info)

    def mark_global(self, global_pos: int) -> None:
        p = self.local(global_pos)
        if p >= 0:
            self.run.mark_visited(p)

    def observe_local(self, x_new, global_pos: int, y: Optional[float]) -> np.ndarray:
        x = np.ascontiguousarray(np.asarray(x_new, dtype=np.float64))
        s, c = C.c_double(), C.c_int64()
        info = _lib.gtc_fit_info()
        check(load().gtc_shard_observe(self.run.handle, _lib.dptr(x), self.local(global_pos),
                                       float(y) if y is not None else 0.0, int(y is not None), C.byref(s),
                                       C.byref(c), C.byref(info)))
        return np.array([s.value, float(c.value)])

    def local_totals(self) -> np.ndarray:
        """(sum, count) of the current posterior variance over unvisited local candidates."""
        mv = C.c_double()
        cnt = C.c_int64()
        check(load().gtc_mean_variance(self.run.handle, C.byref(mv), C.byref(cnt)))
        return np.array([mv.value * cnt.value, float(cnt.value)])

    def select_local(self, afs, f_best_raw, exploration, cv_state, gsum, gcnt, excluded=None) -> ShardRecord:
        a, _keep = SurrogateRun._args(afs, f_best_raw, exploration, cv_state, excluded)
        r = _lib.gtc_shard_selection()
        check(load().gtc_shard_select(self.run.handle, C.byref(a), float(gsum), int(gcnt), C.byref(r)))
        return ShardRecord(tuple(r.best_position), tuple(r.best_score), int(r.first_eligible),
                           int(r.first_nan_mask), int(r.n_candidates), r.lambda_, r.mean_variance, r.best_std,
                           bool(r.cv_fallback))


def af_mask_of(afs) -> int:
    m = 0
    for af in afs:
        m |= 1 << int(af)
    return m


class ShardGroup:
    """All shards in one process (protocol tests on a single device)."""

    def __init__(self, shards: List[Shard]):
        self.shards = shards

    def mean_variance(self) -> float:
        s, c = sum_in_rank_order([sh.local_totals() for sh in self.shards])
        return s / c if c else 0.0

    def observe(self, x_new, global_pos, y, afs, f_best_raw, exploration=ExplorationConfig(),
                cv_state=ContextualVarianceState(), excluded=None) -> Selection:
        totals = [sh.observe_local(x_new, global_pos, y) for sh in self.shards]
        gsum, gcnt = sum_in_rank_order(totals)
        recs = [sh.select_local(afs, f_best_raw, exploration, cv_state, gsum, gcnt, excluded) for sh in self.shards]
        return merge_shard_records(recs, af_mask_of(afs))

    def select(self, afs, f_best_raw, exploration=ExplorationConfig(), cv_state=ContextualVarianceState(),
               excluded=None) -> Selection:
        gsum, gcnt = sum_in_rank_order([sh.local_totals() for sh in self.shards])
        recs = [sh.select_local(afs, f_best_raw, exploration, cv_state, gsum, gcnt, excluded) for sh in self.shards]
        return merge_shard_records(recs, af_mask_of(afs))


class TorchComm:
    """allgather over torch.distributed (nccl: CUDA tensors; gloo: CPU)."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world = dist.get_world_size()
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu"))

    def allgather(self, a: np.ndarray) -> List[np.ndarray]:
        t = self.torch.as_tensor(np.asarray(a, dtype=np.float64), device=self.device)
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t)
        return [o.cpu().numpy() for o in out]


class DistributedShard:
    """One shard per rank; the two per-iteration exchanges go through `comm`."""

    def __init__(self, shard: Shard, comm):
        self.shard, self.comm = shard, comm

    def mean_variance(self) -> float:
        s, c = sum_in_rank_order(self.comm.allgather(self.shard.local_totals()))
        return s / c if c else 0.0

    def _select(self, totals, afs, f_best_raw, exploration, cv_state, excluded) -> Selection:
        gsum, gcnt = sum_in_rank_order(self.comm.allgather(totals))
        rec = self.shard.select_local(afs, f_best_raw, exploration, cv_state, gsum, gcnt, excluded)
        recs = [ShardRecord.unpack(r) for r in self.comm.allgather(rec.pack())]
        return merge_shard_records(recs, af_mask_of(afs))

    def observe(self, x_new, global_pos, y, afs, f_best_raw, exploration=ExplorationConfig(),
                cv_state=ContextualVarianceState(), excluded=None) -> Selection:
        return self._select(self.shard.observe_local(x_new, global_pos, y), afs, f_best_raw, exploration,
                            cv_state, excluded)

    def select(self, afs, f_best_raw, exploration=ExplorationConfig(), cv_state=ContextualVarianceState(),
               excluded=None) -> Selection:
        return self._select(self.shard.local_totals(), afs, f_best_raw, exploration, cv_state, excluded)


def split_bounds(n: int, parts: int, rank: int):
    """Contiguous near-equal slices [lo, hi) of n candidates."""
    lo = (n * rank) // parts
    hi = (n * (rank + 1)) // parts
    return lo, hi


TILE = 256  # candidates per tile (gtc_internal.h kTile)


def split_tiles(n: int, parts: int, rank: int):
    """Contiguous slices [lo, hi) of n candidates on 256-candidate tile
    boundaries (gtc_run_attach_comm requires tile-aligned offsets: the
    per-tile fixed-point variance totals then sum to exactly the one-device
    total, so lambda and every pick are bit-identical)."""
    tiles = (n + TILE - 1) // TILE
    lo = min(n, TILE * ((tiles * rank) // parts))
    hi = min(n, TILE * ((tiles * (rank + 1)) // parts))
    return lo, hi


# ---------------------------------------------------------------------------
# Device-resident sharding (gtc_comm + gtc_run_attach_comm): the whole
# iteration -- local selection, all-gather of the shard records, merge, loop
# advance, bordered row, local pass, all-gather of the variance accumulators --
# is enqueued on the run's stream by gtc_run_steps; no host round trip.

class Comm:
    """A gtc_comm handle (NCCL rank or a member of an in-process group)."""

    def __init__(self, handle):
        self._h = handle

    @property
    def handle(self):
        return self._h

    @property
    def rank(self) -> int:
        return int(load().gtc_comm_rank(self._h))

    @property
    def size(self) -> int:
        return int(load().gtc_comm_size(self._h))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(load().gtc_comm_nccl_id(buf))
        return bytes(buf)

    @staticmethod
    def nccl(uid: bytes, rank: int, nranks: int, device: int) -> "Comm":
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        check(load().gtc_comm_create_nccl(buf, int(rank), int(nranks), int(device), C.byref(h)))
        return Comm(h)

    @staticmethod
    def local_group(nranks: int) -> List["Comm"]:
        hs = (C.c_void_p * int(nranks))()
        check(load().gtc_comm_create_local(int(nranks), hs))
        return [Comm(C.c_void_p(h)) for h in hs]

    def close(self):
        if self._h:
            load().gtc_comm_destroy(self._h)
            self._h = None


class ShardedRun:
    """One shard of a run whose candidate axis is split over devices/ranks:
    global candidates [offset, offset + len(coords_slice)), a replicated GP,
    and gtc_run_steps iterations with the exchanges on the device."""

    def __init__(self, coords_slice, offset: int, n_global: int, comm: Comm, kernel: MaternKernel,
                 noise: float = 1e-10, jitter: float = 1e-6, n_max: int = 220, device: int = 0):
        self.offset = int(offset)
        self.n_global = int(n_global)
        self.comm = comm
        self.space = Space(coords_slice, device=device)
        self.run = SurrogateRun(self.space, kernel, noise, jitter, n_max)
        self.n_local = self.space.n
        check(load().gtc_run_attach_comm(self.run.handle, comm.handle, self.offset, self.n_global))

    def local(self, global_pos: int) -> int:
        p = int(global_pos) - self.offset
        return p if 0 <= p < self.n_local else -1

    def fit_points(self, X, y) -> FitInfo:
        X = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
        y = np.ascontiguousarray(np.asarray(y, dtype=np.float64))
        info = _lib.gtc_fit_info()
        check(load().gtc_fit_points(self.run.handle, _lib.dptr(X), _lib.dptr(y), len(y), C.byref(info)))
        return FitInfo.of(info)

    def mark_global(self, global_pos: int) -> None:
        p = self.local(global_pos)
        if p >= 0:
            self.run.mark_visited(p)

    def unmark_global(self, global_pos: int) -> None:
        p = self.local(global_pos)
        if p >= 0:
            self.run.unmark_visited(p)

    def local_totals(self) -> np.ndarray:
        mv = C.c_double()
        cnt = C.c_int64()
        check(load().gtc_mean_variance(self.run.handle, C.byref(mv), C.byref(cnt)))
        return np.array([mv.value * cnt.value, float(cnt.value)])

    def set_values(self, values) -> None:
        """The GLOBAL replay table (every shard evaluates every pick)."""
        self.run.set_values(values)

    def steps(self, af, k, f_best_raw, exploration=ExplorationConfig(), cv_state=ContextualVarianceState(),
              hold=False, timing=False):
        return self.run.steps(af, k, f_best_raw, exploration, cv_state, hold=hold, timing=timing)

    def close(self):
        self.run.close()
        self.space.close()
