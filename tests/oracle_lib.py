"""ctypes binding of the CPU oracle (oracle/gtoracle.c) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use the
oracle, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import pathlib
import subprocess

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
LIB = ROOT / "oracle" / "build" / "liboracle.so"
DP = C.POINTER(C.c_double)
I64P = C.POINTER(C.c_int64)
U8P = C.POINTER(C.c_uint8)

_lib = None


def load():
    global _lib
    if _lib is not None:
        return Oracle(_lib)
    if not LIB.exists() or LIB.stat().st_mtime < (ROOT / "oracle" / "gtoracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "oracle"], check=True)
    lib = C.CDLL(str(LIB))
    lib.gto_matern.restype = C.c_double
    lib.gto_matern.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double]
    lib.gto_gp_fit.restype = C.c_int
    lib.gto_gp_fit.argtypes = [C.c_int, C.c_double, C.c_double, DP, DP, C.c_int, C.c_int, C.c_double,
                               C.c_double, DP, DP, DP]
    lib.gto_gp_predict.restype = None
    lib.gto_gp_predict.argtypes = [C.c_int, C.c_double, C.c_double, DP, C.c_int, C.c_int, DP, DP, DP,
                                   C.c_int64, DP, DP]
    for f in ("gto_acq_pi", "gto_acq_ei"):
        getattr(lib, f).restype = C.c_double
        getattr(lib, f).argtypes = [C.c_double] * 4
    lib.gto_acq_lcb.restype = C.c_double
    lib.gto_acq_lcb.argtypes = [C.c_double] * 3
    lib.gto_cv_lambda.restype = C.c_int
    lib.gto_cv_lambda.argtypes = [C.c_double] * 4 + [DP]
    lib.gto_best_candidate.restype = C.c_int64
    lib.gto_best_candidate.argtypes = [C.c_int, DP, DP, C.c_int64, C.c_double, C.c_double, U8P, DP]
    lib.gto_mean.restype = C.c_double
    lib.gto_mean.argtypes = [DP, C.c_int64]
    _lib = lib
    return Oracle(lib)


def _d(a):
    return a.ctypes.data_as(DP)


class Oracle:
    def __init__(self, lib):
        self.lib = lib

    def matern(self, nu, l, s2, r):
        return self.lib.gto_matern(int(nu), l, s2, r)

    def fit(self, nu, l, s2, X, y, noise=1e-10, jitter=1e-6):
        X = np.ascontiguousarray(X, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        n = len(y)
        d = X.shape[1] if X.ndim == 2 and X.shape[1] else 1
        L = np.zeros(max(n, 1) * max(n, 1))
        alpha = np.zeros(max(n, 1))
        sc = np.zeros(3)
        rc = self.lib.gto_gp_fit(int(nu), l, s2, _d(X), _d(y), n, d, noise, jitter, _d(L), _d(alpha), _d(sc))
        return rc, dict(X=X, n=n, d=d, L=L, alpha=alpha, y_mean=sc[0], y_std=sc[1], jitter=sc[2],
                        nu=int(nu), l=l, s2=s2)

    def predict(self, model, Xs):
        Xs = np.ascontiguousarray(Xs, dtype=np.float64)
        m = Xs.shape[0]
        mean = np.zeros(m)
        var = np.zeros(m)
        self.lib.gto_gp_predict(model["nu"], model["l"], model["s2"], _d(model["X"]), model["n"],
                                model["d"], _d(model["L"]), _d(model["alpha"]), _d(Xs), m, _d(mean),
                                _d(var))
        return mean, var

    def pi(self, m, s, b, l):
        return self.lib.gto_acq_pi(m, s, b, l)

    def ei(self, m, s, b, l):
        return self.lib.gto_acq_ei(m, s, b, l)

    def lcb(self, m, s, l):
        return self.lib.gto_acq_lcb(m, s, l)

    def cv_lambda(self, mu_s, var_s, mv, fb):
        out = C.c_double(0.0)
        ok = self.lib.gto_cv_lambda(mu_s, var_s, mv, fb, C.byref(out))
        return out.value if ok else None

    def best_candidate(self, af, means, stds, best_std, lam, excluded=None):
        m = np.ascontiguousarray(means, dtype=np.float64)
        s = np.ascontiguousarray(stds, dtype=np.float64)
        ex = None if excluded is None else np.ascontiguousarray(excluded, dtype=np.uint8)
        score = C.c_double()
        p = self.lib.gto_best_candidate(int(af), _d(m), _d(s), len(m), best_std, lam,
                                        ex.ctypes.data_as(U8P) if ex is not None else None, C.byref(score))
        return int(p), score.value

    def mean(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        return self.lib.gto_mean(_d(v), len(v))
