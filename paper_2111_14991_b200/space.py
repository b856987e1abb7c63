"""Search spaces with restrictions, enumerated on the device.

Mirror of the reference's ParameterDef / SearchSpace / EnumeratedSpace /
Restriction (parameter.hpp:62-125, search_space.hpp:23-245,
restriction.hpp:472-520) over the C ABI: the restriction text is parsed and
type-checked by the library (same grammar, messages and positions as the
reference), and the Cartesian grid is filtered, compacted and normalised by
sm_100a kernels (gtc_space_enumerate) into a resident `Space`.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import _lib
from ._lib import load
from .gp import check
from .runtime import Space


class ParamKind(enum.IntEnum):
    numeric = 0
    categorical = 1
    boolean = 2


def _kind_of(v) -> ParamKind:
    if isinstance(v, (bool, np.bool_)):
        return ParamKind.boolean
    if isinstance(v, str):
        return ParamKind.categorical
    return ParamKind.numeric


@dataclass
class ParameterDef:
    """parameter.hpp:62-125: a name and its ordered values (numbers, strings or
    booleans; the kind is that of the first value unless given)."""
    name: str
    values: Sequence
    kind: ParamKind = None

    def __post_init__(self):
        self.values = list(self.values)
        if self.kind is None:
            self.kind = _kind_of(self.values[0]) if self.values else ParamKind.numeric

    def size(self) -> int:
        return len(self.values)


class _Defs:
    """ctypes view of a parameter list (keeps the buffers alive)."""

    def __init__(self, params: Sequence[ParameterDef]):
        self.keep = []
        self.arr = (_lib.gtc_param_def * max(1, len(params)))()
        for i, p in enumerate(params):
            d = self.arr[i]
            name = p.name.encode()
            self.keep.append(name)
            d.name = name
            d.kind = int(p.kind)
            d.n_values = len(p.values)
            if p.kind == ParamKind.numeric:
                a = np.ascontiguousarray(np.asarray(p.values, dtype=np.float64))
                self.keep.append(a)
                d.numbers = _lib.dptr(a)
            elif p.kind == ParamKind.categorical:
                enc = [str(v).encode() for v in p.values]
                a = (C.c_char_p * max(1, len(enc)))(*enc)
                self.keep += [enc, a]
                d.strings = a
            else:
                a = np.ascontiguousarray(np.asarray([1 if v else 0 for v in p.values], dtype=np.uint8))
                self.keep.append(a)
                d.booleans = _lib.u8ptr(a)
        self.n = len(params)


def parse_restriction(text: str, params: Sequence[ParameterDef]) -> str:
    """Restriction::parse (restriction.hpp:479-486): raises ParseError with the
    reference's message and position; returns the source on success."""
    defs = _Defs(params)
    pos = C.c_int64(0)
    rc = load().gtc_restriction_validate(defs.arr, defs.n, text.encode(), C.byref(pos))
    check(rc, pos.value)
    return text


@dataclass
class SearchSpace:
    """SearchSpace(params, restriction_sources), search_space.hpp:35-44."""
    params: List[ParameterDef]
    restrictions: List[str] = field(default_factory=list)

    def cartesian_size(self) -> int:
        n = 1
        for p in self.params:
            n *= p.size()
        return n

    def dimension(self) -> int:
        return len(self.params)

    def enumerate(self, device: int = 0) -> "EnumeratedSpace":
        return EnumeratedSpace(self, device)


class EnumeratedSpace(Space):
    """EnumeratedSpace (search_space.hpp:216-245) built on the device: the
    valid configurations in canonical order (`ids`), their normalised
    coordinates (`coords`, rank / (k - 1)), resident for SurrogateRun."""

    def __init__(self, space: SearchSpace, device: int = 0):
        self.space = space
        defs = _Defs(space.params)
        srcs = [r.encode() for r in space.restrictions]
        arr = (C.c_char_p * max(1, len(srcs)))(*srcs)
        pos = C.c_int64(0)
        h = C.c_void_p()
        rc = load().gtc_space_enumerate(device, defs.arr, defs.n, arr, len(srcs), C.byref(pos), C.byref(h))
        check(rc, pos.value)
        self._h = h
        self.device = device
        self.n = int(load().gtc_space_size(h))
        self.d = space.dimension()
        self.ids = np.empty(self.n, dtype=np.uint64)
        check(load().gtc_space_ids(h, self.ids.ctypes.data_as(_lib.U64P)))
        ptr = load().gtc_space_coords(h)
        self.coords = np.ctypeslib.as_array(ptr, shape=(self.n, self.d)).copy()

    def cartesian_size(self) -> int:
        return int(load().gtc_space_cartesian_size(self._h))

    def position_of(self, index: int) -> int:
        """EnumeratedSpace::position_of: position of a canonical index (-1 if restricted)."""
        k = int(np.searchsorted(self.ids, np.uint64(index)))
        return k if k < self.n and int(self.ids[k]) == int(index) else -1
