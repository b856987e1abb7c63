"""How many 256-candidate tiles a per-tile (min mean, max/min variance) bound
leaves for exact scoring at the C4 bench state.  Diagnostic only."""
import struct
import sys

import numpy as np
from scipy.special import erfc

path = sys.argv[1] if len(sys.argv) > 1 else "/tmp/gtc_state.bin"
with open(path, "rb") as f:
    n = struct.unpack("<q", f.read(8))[0]
    best_raw, ymean, ystd, mu_s, var_s = struct.unpack("<5d", f.read(40))
    mu = np.frombuffer(f.read(8 * n))
    var = np.frombuffer(f.read(8 * n))
    vis = np.frombuffer(f.read(4 * ((n + 31) // 32)), dtype=np.uint32)
bits = np.unpackbits(vis.view(np.uint8), bitorder="little")[:n].astype(bool)
best = (best_raw - ymean) / ystd
mv = var[~bits].mean()
lam = max(mv * best_raw / mu_s / var_s, 0.0)
Phi = lambda z: 0.5 * erfc(-z / np.sqrt(2))
phi = lambda z: np.exp(-0.5 * z * z) / np.sqrt(2 * np.pi)


def ei(m, s):
    mm = best - lam - m
    z = mm / s
    return mm * Phi(z) + s * phi(z)


def pi(m, s):
    return Phi((best + lam - m) / s)


def lcb(m, s):
    return lam * s - m


sd = np.sqrt(var)
for tile in (256, 64, 32):
    nt = (n + tile - 1) // tile
    pad = nt * tile - n
    mup = np.concatenate([mu, np.full(pad, np.inf)]).reshape(nt, tile)
    vp = np.concatenate([var, np.full(pad, -np.inf)]).reshape(nt, tile)
    vq = np.concatenate([var, np.full(pad, np.inf)]).reshape(nt, tile)
    mmin, vmax, vmin = mup.min(1), vp.max(1), vq.min(1)
    elig = ~bits
    for name, fn in (("ei", ei), ("poi", pi), ("lcb", lcb)):
        s = np.where(elig, fn(mu, sd), -np.inf)
        T = s.max()
        if name == "poi":
            M = best + lam - mmin
            ub = np.where(M >= 0, Phi(M / np.sqrt(vmin)), Phi(M / np.sqrt(vmax)))
        else:
            ub = fn(mmin, np.sqrt(vmax))
        print(f"tile {tile:4d} {name:4s} T={T:.6g}  tiles surviving {np.sum(ub >= T)} of {nt}  (x{tile} = {np.sum(ub >= T) * tile} candidates)")
