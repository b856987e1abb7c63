"""Measurement caches: the reference's JSON format and a compact binary one.

Mirror of MeasurementCache (/root/reference/proj/include/gridtune/cache.hpp:
22-270): a fully measured search space -- definition + one measurement per
valid configuration keyed by canonical index -- replayed as the objective of
simulation-mode runs.  `load_json` / `save_json` read and write the
reference's JSON (same fields, FNV-1a checksum, validation and error texts);
`save_binary` / `load_binary` add the §8(f)#4 format: the same header as a
small JSON document followed by dense little-endian arrays in canonical order
(index u64, value f64 with NaN for invalid, reason u8) -- 17 bytes per entry
instead of ~100-200 bytes of JSON, read with one memory map.  Validation
(`validate`) enumerates the space on the device (gtc_space_enumerate) and
checks completeness against it.

  magic   8 bytes  b"GTCBIN\\x00\\x01"
  u64     header length H, then H bytes of UTF-8 JSON (schema_version,
          kernel_name, device_name, objective_unit, parameters, restrictions,
          true_minimum?, checksum, entries = N)
  u64[N]  canonical indices, ascending
  f64[N]  values (NaN: invalid)
  u8[N]   0 valid, 1 compile_error, 2 runtime_error, 3 restricted
"""
from __future__ import annotations

import json
import math
import pathlib
import struct
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .gp import Error
from .space import ParameterDef, ParamKind, SearchSpace, parse_restriction

SCHEMA_VERSION = 1  # cache.hpp:27
MAGIC = b"GTCBIN\x00\x01"
REASONS = ["", "compile_error", "runtime_error", "restricted"]  # measurement.hpp:12-21


class CacheError(Error):
    """gridtune::CacheError"""


@dataclass
class MeasurementCache:
    kernel_name: str
    params: List[ParameterDef]
    restrictions: List[str] = field(default_factory=list)
    ids: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))   # ascending canonical indices
    values: np.ndarray = field(default_factory=lambda: np.zeros(0))           # NaN where invalid
    reasons: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))  # 0 valid, else REASONS[k]
    device_name: str = "simulated"
    objective_unit: str = "ms"
    true_minimum: Optional[float] = None

    # ---- reference semantics --------------------------------------------
    def space(self) -> SearchSpace:
        return SearchSpace(self.params, list(self.restrictions))

    def invalid_count(self) -> int:
        return int(np.count_nonzero(self.reasons))

    def min_valid_value(self) -> float:
        v = self.values[self.reasons == 0]
        return float(v.min()) if len(v) else math.inf

    def checksum(self) -> int:
        """FNV-1a over the canonical entry serialisation (cache.hpp:55-70),
        computed by the native library (gtc_cache_checksum)."""
        from . import _lib
        ids = np.ascontiguousarray(self.ids, dtype=np.uint64)
        vals = np.ascontiguousarray(self.values, dtype=np.float64)
        rs = np.ascontiguousarray(self.reasons, dtype=np.uint8)
        return int(_lib.load().gtc_cache_checksum(ids.ctypes.data_as(_lib.U64P), _lib.dptr(vals),
                                                  _lib.u8ptr(rs), len(ids)))

    def validate(self, device: int = 0):
        """MeasurementCache::validate (cache.hpp:74-108), with the space
        enumerated on the device; returns the EnumeratedSpace."""
        from .gp import EmptySearchSpaceError
        try:
            es = self.space().enumerate(device)
        except EmptySearchSpaceError:
            raise CacheError(f"cache '{self.kernel_name}': restrictions exclude every configuration") from None
        if es.n != len(self.ids):
            raise CacheError(f"cache '{self.kernel_name}' has {len(self.ids)} entries but the space has "
                             f"{es.n} valid configurations")
        # the reference walks the valid configurations in ascending order and
        # reports the first one that is missing or has a non-positive value
        missing = np.setdiff1d(es.ids, self.ids)
        bad = self.ids[(self.reasons == 0) & ~(self.values > 0.0)]
        bad = bad[np.isin(bad, es.ids)]
        first_missing = int(missing[0]) if len(missing) else None
        first_bad = int(bad.min()) if len(bad) else None
        if first_missing is not None and (first_bad is None or first_missing < first_bad):
            raise CacheError(f"cache '{self.kernel_name}' is missing an entry for configuration {first_missing}")
        if first_bad is not None:
            raise CacheError(f"cache '{self.kernel_name}' entry {first_bad} has non-positive value")
        if self.true_minimum is not None and self.min_valid_value() != self.true_minimum:
            raise CacheError(f"cache '{self.kernel_name}' states minimum {self.true_minimum:.6f} but the entries' "
                             f"minimum is {self.min_valid_value():.6f}")
        return es

    def replay(self, device: int = 0):
        """(EnumeratedSpace, values by position) for simulation-mode runs
        (run_bo(space, space.ids, config, values=...)), cache.hpp:246-257."""
        es = self.validate(device)
        return es, np.where(self.reasons == 0, self.values, np.nan)

    # ---- JSON (reference format) -------------------------------------------
    def _header(self) -> dict:
        doc = {"schema_version": SCHEMA_VERSION, "kernel_name": self.kernel_name,
               "device_name": self.device_name, "objective_unit": self.objective_unit,
               "parameters": [{"name": p.name, "kind": p.kind.name, "values": list(p.values)} for p in self.params],
               "restrictions": list(self.restrictions)}
        if self.true_minimum is not None:
            doc["true_minimum"] = self.true_minimum
        doc["checksum"] = "fnv1a64:%016x" % self.checksum()
        return doc

    def save_json(self, path) -> None:
        doc = self._header()
        radices = [p.size() for p in self.params]
        entries = []
        for idx, v, r in zip(self.ids.tolist(), self.values.tolist(), self.reasons.tolist()):
            ranks, rest = [], idx
            for k in reversed(radices):
                ranks.append(rest % k)
                rest //= k
            cfg = [p.values[q] for p, q in zip(self.params, reversed(ranks))]
            e = {"index": idx, "config": cfg}
            if r == 0:
                e["value"] = v
            else:
                e["invalid"] = REASONS[r]
            entries.append(e)
        doc["entries"] = entries
        pathlib.Path(path).write_text(json.dumps(doc, indent=1) + "\n")

    def config_at(self, index: int) -> list:
        """The configuration tuple of a canonical index (mixed radix, first
        parameter most significant; SearchSpace::config_at, search_space.hpp:57-72)."""
        out, rest = [], int(index)
        for p in reversed(self.params):
            out.append(p.values[rest % p.size()])
            rest //= p.size()
        return out[::-1]

    @staticmethod
    def load_json(path, validate: bool = True) -> "MeasurementCache":
        """MeasurementCache::load (cache.hpp:156-241): header, restrictions
        parsed, entries in file order (unknown reason, embedded config tuple
        against its index, duplicates), stored checksum, then validate() --
        which enumerates the space on the device; validate=False skips only
        that last step (host-only tools and CPU tests)."""
        try:
            doc = json.loads(pathlib.Path(path).read_text())
        except OSError:
            raise CacheError(f"cannot open cache file '{path}'") from None
        except json.JSONDecodeError as e:
            raise CacheError(f"cache file '{path}' is not valid JSON: {e}") from None
        try:
            c = MeasurementCache._from_header(doc, path)
            ids, values, reasons, seen = [], [], [], set()
            for e in doc["entries"]:
                idx = int(e["index"])
                if "value" in e:
                    values.append(float(e["value"]))
                    reasons.append(0)
                else:
                    reason = e["invalid"]
                    if reason not in REASONS[1:]:
                        raise CacheError(f"unknown invalid reason '{reason}'")
                    values.append(math.nan)
                    reasons.append(REASONS.index(reason))
                if "config" in e:  # the embedded tuple must match the index
                    want = c.config_at(idx)
                    got = e["config"]
                    if len(got) != len(want):
                        raise CacheError(f"entry {idx} config tuple has wrong arity")
                    if any(not _same_value(g, w) for g, w in zip(got, want)):
                        raise CacheError(f"entry {idx} config tuple does not match its index")
                if idx in seen:
                    raise CacheError(f"duplicate entry for configuration {idx}")
                seen.add(idx)
                ids.append(idx)
        except KeyError as e:
            raise CacheError(f"cache file '{path}' is malformed: missing key {e}") from None
        order = np.argsort(np.array(ids, dtype=np.uint64), kind="stable")
        c.ids = np.array(ids, dtype=np.uint64)[order]
        c.values = np.array(values, dtype=np.float64)[order]
        c.reasons = np.array(reasons, dtype=np.uint8)[order]
        c._check_stored_checksum(doc, path)
        if validate:
            c.validate()
        return c

    @staticmethod
    def _from_header(doc: dict, path) -> "MeasurementCache":
        if doc.get("schema_version") != SCHEMA_VERSION:
            raise CacheError("unsupported cache schema version")
        params = []
        for jp in doc["parameters"]:
            if jp["kind"] not in ("numeric", "categorical", "boolean"):
                raise CacheError(f"unknown parameter kind '{jp['kind']}'")
            params.append(ParameterDef(jp["name"], jp["values"], ParamKind[jp["kind"]]))
        for text in doc.get("restrictions", []):  # SearchSpace construction parses them (host only)
            parse_restriction(text, params)
        return MeasurementCache(kernel_name=doc["kernel_name"], params=params,
                                restrictions=list(doc.get("restrictions", [])),
                                device_name=doc.get("device_name", "unknown"),
                                objective_unit=doc.get("objective_unit", "ms"),
                                true_minimum=doc.get("true_minimum"))

    def _check_stored_checksum(self, doc: dict, path) -> None:
        if "checksum" in doc and doc["checksum"] != "fnv1a64:%016x" % self.checksum():
            raise CacheError(f"cache file '{path}' checksum mismatch")

    # ---- binary ------------------------------------------------------------
    def save_binary(self, path) -> None:
        head = self._header()
        head["entries"] = int(len(self.ids))
        hb = json.dumps(head).encode()
        with open(path, "wb") as f:
            f.write(MAGIC)
            f.write(struct.pack("<Q", len(hb)))
            f.write(hb)
            f.write(np.ascontiguousarray(self.ids, dtype="<u8").tobytes())
            f.write(np.ascontiguousarray(self.values, dtype="<f8").tobytes())
            f.write(np.ascontiguousarray(self.reasons, dtype=np.uint8).tobytes())

    @staticmethod
    def load_binary(path, verify_checksum: bool = True, validate: bool = True) -> "MeasurementCache":
        """The binary format: same header and checks as load_json (ascending
        unique indices instead of per-entry tuples), then validate()."""
        try:
            raw = np.memmap(path, dtype=np.uint8, mode="r")
        except OSError:
            raise CacheError(f"cannot open cache file '{path}'") from None
        if raw.size < 16 or bytes(raw[:8]) != MAGIC:
            raise CacheError(f"cache file '{path}' is not a gridtune binary cache")
        hl = struct.unpack("<Q", bytes(raw[8:16]))[0]
        doc = json.loads(bytes(raw[16:16 + hl]).decode())
        c = MeasurementCache._from_header(doc, path)
        n = int(doc["entries"])
        o = 16 + hl
        if raw.size != o + 17 * n:
            raise CacheError(f"cache file '{path}' is truncated")
        c.ids = np.frombuffer(raw, dtype="<u8", count=n, offset=o).astype(np.uint64)
        c.values = np.frombuffer(raw, dtype="<f8", count=n, offset=o + 8 * n).astype(np.float64)
        c.reasons = np.frombuffer(raw, dtype=np.uint8, count=n, offset=o + 16 * n).copy()
        if n > 1 and not np.all(np.diff(c.ids.astype(np.int64)) > 0):
            raise CacheError(f"cache file '{path}' entries are not in ascending index order")
        if verify_checksum:
            c._check_stored_checksum(doc, path)
        if validate:
            c.validate()
        return c

    @staticmethod
    def load(path, validate: bool = True) -> "MeasurementCache":
        """Either format, by content."""
        with open(path, "rb") as f:
            head = f.read(8)
        if head == MAGIC:
            return MeasurementCache.load_binary(path, validate=validate)
        return MeasurementCache.load_json(path, validate=validate)


def _same_value(a, b) -> bool:
    """value_from_json(a) == b (parameter.hpp Value equality: same kind and value)."""
    if isinstance(b, bool) or isinstance(a, bool):
        return isinstance(a, bool) and isinstance(b, bool) and a == b
    if isinstance(b, str) or isinstance(a, str):
        return isinstance(a, str) and isinstance(b, str) and a == b
    return float(a) == float(b)
