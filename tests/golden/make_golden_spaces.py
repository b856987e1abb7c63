"""Golden fixtures of the search-space layer, written by the UNMODIFIED reference
(oracle/_ref/ref_tool: Restriction::parse / evaluate, SearchSpace,
EnumeratedSpace; restriction.hpp, search_space.hpp, parameter.hpp).

  restrictions.json   per restriction text over the reference test's tuning
                      parameters (test_restriction.cpp:11-21): the parse
                      outcome (message + position) or its truth value at every
                      Cartesian point; the reference KATs plus a seeded fuzz
                      set of well-formed and malformed expressions
  enum_<name>.npz     ids + coords of enumerated spaces (conv and pnpoly of
                      PAPER.md, categorical/boolean restrictions, IEEE edge
                      cases), with the spec
  enum_errors.json    SearchSpace construction errors (messages)

Needs /root/reference (this container only); the outputs are committed.

  python tests/golden/make_golden_spaces.py
"""
from __future__ import annotations

import json
import pathlib
import random
import subprocess
import sys
import tempfile

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parents[1]
TOOL = ROOT / "oracle" / "_ref" / "ref_tool"

TUNING = [  # test_restriction.cpp:11-21
    {"name": "block_size_x", "kind": "numeric", "values": [16.0, 32.0, 64.0]},
    {"name": "block_size_y", "kind": "numeric", "values": [1.0, 2.0, 4.0, 8.0]},
    {"name": "tile_size", "kind": "numeric", "values": [1.0, 2.0, 4.0]},
    {"name": "method", "kind": "categorical", "values": ["fast", "safe"]},
    {"name": "use_padding", "kind": "boolean", "values": [False, True]},
]

KATS = [  # test_restriction.cpp:23-123
    "block_size_x * block_size_y <= 1024", "tile_size >", "foo == 1", "method == 1",
    "block_size_x and tile_size", "not block_size_x", "use_padding < true", "block_size_x + method == 2",
    "block_size_x", "", "1 + 2 * 3 == 7", "(1 + 2) * 3 == 9",
    "use_padding or block_size_x == 16 and tile_size == 2", "not (use_padding == false)", "method != 'safe'",
    "method < 'g'", "block_size_x % 16 == 0", "block_size_x / block_size_y == 8", "tile_size / 2 == 0.5",
    "-tile_size < 0", "1e3 == 1000", "1 / (tile_size - tile_size) > 0", "tile_size % 0 == 0",
    "tile_size == 1.2.3", "tile_size == 'open", "tile_size = 1", "tile_size == bar",
    # more edges: NaN / inf comparisons, string orders, boolean equality, literals
    "0 / 0 != 0 / 0", "not (0 / 0 == 0 / 0)", "1 / 0 > 1e308", "-1 / 0 < -1e308", "-0 == 0",
    "tile_size % -3 == tile_size % 3", "-tile_size % 3 < 0", "block_size_x % 2.5 == 1.5",
    "method <= 'fast' and method >= 'fast'", "'a' < 'b'", "'b' > method", "method == method",
    "use_padding == use_padding", "use_padding != true", "True == true", "not not use_padding",
    "method > 'FAST'", "\"safe\" == method", "block_size_x - - tile_size > 17", ".5 * block_size_y >= 1",
    "2e-1 * 5 == 1", "block_size_x*block_size_y>=64", "1 < 2 < 3", "(method == 'fast') == use_padding",
    "use_padding == 1", "method", "and", "tile_size ! 1", "tile_size == 1 or", "((tile_size == 1)",
    "tile_size == 1)", "1e", "tile_size == 1 # x", "use_padding > false", "True", "false or True",
]

NUM = ["block_size_x", "block_size_y", "tile_size"]


def rand_num(rng, depth):
    r = rng.random()
    if depth <= 0 or r < 0.3:
        return rng.choice(NUM) if rng.random() < 0.6 else rng.choice(["0", "1", "2", "3", "16", "0.5", "1e2", "7"])
    if r < 0.4:
        return "-" + rand_num(rng, depth - 1)
    if r < 0.5:
        return "(" + rand_num(rng, depth - 1) + ")"
    op = rng.choice(["+", "-", "*", "/", "%"])
    return rand_num(rng, depth - 1) + f" {op} " + rand_num(rng, depth - 1)


def rand_bool(rng, depth):
    r = rng.random()
    if depth <= 0 or r < 0.35:
        c = rng.random()
        if c < 0.6:
            return rand_num(rng, 2) + " " + rng.choice(["==", "!=", "<", "<=", ">", ">="]) + " " + rand_num(rng, 2)
        if c < 0.8:
            lhs = rng.choice(["method", "'fast'", "'safe'", "'m'", "'fastest'"])
            rhs = rng.choice(["method", "'fast'", "'safe'", "'a'", "''"])
            return lhs + " " + rng.choice(["==", "!=", "<", "<=", ">", ">="]) + " " + rhs
        return rng.choice(["use_padding", "true", "false", "use_padding == true", "use_padding != use_padding"])
    if r < 0.5:
        return "not " + rand_bool(rng, depth - 1)
    if r < 0.6:
        return "(" + rand_bool(rng, depth - 1) + ")"
    return rand_bool(rng, depth - 1) + rng.choice([" and ", " or "]) + rand_bool(rng, depth - 1)


def fuzz(n, seed):
    rng = random.Random(seed)
    out = [rand_bool(rng, 4) for _ in range(n)]
    # malformed variants: drop / duplicate a token or a character
    bad = []
    for t in out[:60]:
        toks = t.split(" ")
        k = rng.randrange(len(toks))
        bad.append(" ".join(toks[:k] + toks[k + 1:]))
        c = rng.randrange(len(t))
        bad.append(t[:c] + t[c + 1:])
    return out + bad


SPACES = {
    # PAPER.md:373-380 (convolution) with the SURVEY.md §8(d) C2 restrictions
    "conv": {"params": [
        {"name": "filter_width", "kind": "numeric", "values": [15]},
        {"name": "filter_height", "kind": "numeric", "values": [15]},
        {"name": "block_size_x", "kind": "numeric", "values": [1, 2, 4, 8, 16, 32, 48, 64, 80, 96, 112, 128]},
        {"name": "block_size_y", "kind": "numeric", "values": [1, 2, 4, 8, 16, 32]},
        {"name": "tile_size_x", "kind": "numeric", "values": [1, 2, 3, 4, 5, 6, 7, 8]},
        {"name": "tile_size_y", "kind": "numeric", "values": [1, 2, 3, 4, 5, 6, 7, 8]},
        {"name": "use_padding", "kind": "numeric", "values": [0, 1]},
        {"name": "read_only", "kind": "numeric", "values": [0, 1]}],
        "restrictions": ["block_size_x*block_size_y>=64", "tile_size_x*tile_size_y<30"]},
    # PAPER.md:345-355 (pnpoly), no restrictions
    "pnpoly": {"params": [
        {"name": "block_size_x", "kind": "numeric", "values": list(range(32, 993, 32))},
        {"name": "tile_size", "kind": "numeric", "values": [1] + list(range(2, 21, 2))},
        {"name": "between_method", "kind": "numeric", "values": [0, 1, 2, 3]},
        {"name": "use_precomputed_slopes", "kind": "numeric", "values": [0, 1]},
        {"name": "use_method", "kind": "numeric", "values": [0, 1, 2]}],
        "restrictions": []},
    "typed": {"params": TUNING + [
        {"name": "layout", "kind": "categorical", "values": ["row", "col", "tiled", "Row"]},
        {"name": "unroll", "kind": "numeric", "values": [0, 1, 2, 4, 8]}],
        "restrictions": ["method == 'fast' or use_padding", "layout < 'tz' and layout != 'col'",
                         "unroll % 2 == 0 or unroll == 1", "not (use_padding == true and layout == method)",
                         "block_size_x / unroll != 8"]},
    "ieee": {"params": [
        {"name": "a", "kind": "numeric", "values": [-2.5, -1, 0, 0.1, 0.3, 1, 3, 1e300, -1e-300]},
        {"name": "b", "kind": "numeric", "values": [0, 0.1, 0.2, 3, -3, 7.5, 1e-300, 1e308]},
        {"name": "c", "kind": "numeric", "values": [1, 2, 3]}],
        "restrictions": ["a % b != 7 or a / b != 1 / 0", "(a + b) * c != 0.1 * c + 0.2 * c",
                         "not (a / b < 0 / 0)", "a * b * 1e10 < 1 / 0 or c == 2", "a % (b - b) != a % (b - b) or c > 1",
                         "-a % c >= -c"]},
}

ERRORS = {
    "empty": {"params": [{"name": "x", "kind": "numeric", "values": [1, 2]}], "restrictions": ["x > 5"]},
    "dup_param": {"params": [{"name": "x", "kind": "numeric", "values": [1]}, {"name": "x", "kind": "numeric", "values": [2]}]},
    "dup_value": {"params": [{"name": "x", "kind": "numeric", "values": [1, 2, 1]}]},
    "dup_zero": {"params": [{"name": "x", "kind": "numeric", "values": [-0.0, 1, 0]}]},
    "dup_bool": {"params": [{"name": "b", "kind": "boolean", "values": [True, True]}]},
    "dup_string": {"params": [{"name": "m", "kind": "categorical", "values": ["a", "b", "a"]}]},
    "bad_name": {"params": [{"name": "2x", "kind": "numeric", "values": [1]}]},
    "no_values": {"params": [{"name": "x", "kind": "numeric", "values": []}]},
    "parse_first": {"params": [{"name": "x", "kind": "numeric", "values": [1, 1]}], "restrictions": ["x >"]},
    "too_big": {"params": [{"name": f"p{i}", "kind": "numeric", "values": list(range(10))} for i in range(8)]},
}


def run(*args):
    out = subprocess.run([str(TOOL), *map(str, args)], check=True, capture_output=True, text=True)
    return [json.loads(line) for line in out.stdout.strip().splitlines()]


def main():
    if not TOOL.exists():
        sys.exit("oracle/_ref/ref_tool missing: run `make -C oracle ref` (needs /root/reference)")
    with tempfile.TemporaryDirectory() as tmp:
        tmp = pathlib.Path(tmp)
        spec = tmp / "restrict.json"
        texts = KATS + fuzz(240, 20261017)
        spec.write_text(json.dumps({"params": TUNING, "restrictions": texts}))
        rows = run("restrict", spec)
        (HERE / "restrictions.json").write_text(json.dumps({"params": TUNING, "cases": rows}, indent=0))
        for name, sp in SPACES.items():
            p = tmp / f"{name}.json"
            p.write_text(json.dumps(sp))
            meta = run("enumjson", p, tmp / name)[-1]
            assert "error" not in meta, (name, meta)
            ids = np.load(tmp / name / "ids.npy")
            coords = np.load(tmp / name / "coords.npy")
            np.savez_compressed(HERE / f"enum_{name}.npz", ids=ids, coords=coords,
                                spec=np.array(json.dumps(sp)), cartesian=np.array([meta["cartesian"]]))
        errs = {}
        for name, sp in ERRORS.items():
            p = tmp / f"err_{name}.json"
            p.write_text(json.dumps(sp))
            errs[name] = {"spec": sp, "result": run("enumjson", p, tmp / f"err_{name}")[-1]}
        (HERE / "enum_errors.json").write_text(json.dumps(errs, indent=1))
        # reference measurement caches (MeasurementCache::save, cache.hpp:117-160):
        # the spaces of traj_rr13_* and traj_rosen_adv, and a 4-D one with invalids
        run("cachegen", "random-rough", "13x13", 17, "0.3", HERE / "cache_rr13.json")
        run("cachegen", "rosenbrock-disc", "30x30", 1, "-", HERE / "cache_rosen.json")
        run("cachegen", "random-rough", "6x5x4x3", 5, "0.2", HERE / "cache_rr4d.json")
    print("search-space fixtures written to", HERE)


if __name__ == "__main__":
    main()
