"""Python mirror of the reference's GP / acquisition API over the C ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/gridtune/{gp,acquisition,portfolio,errors}.hpp so
that the parity tests read like the reference's own tests.  Every compute call
runs the sm_100a kernels in libgridtune_b200.so; nothing here computes on the
host except the scalar formulas the reference itself evaluates once per
iteration (contextual_variance_lambda, discounted_observation_score).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import load


# ---------------------------------------------------------------- errors.hpp:55-108
class Error(RuntimeError):
    """gridtune::Error"""


class ModelConditioningError(Error):
    """gridtune::ModelConditioningError (gp.hpp:123-127)"""


class ConfigError(Error):
    """gridtune::ConfigError"""


class SamplingError(Error):
    """gridtune::SamplingError"""


class DeviceError(Error):
    """CUDA failure (no device / launch error).  There is no CPU fallback."""


class ParseError(Error):
    """gridtune::ParseError (errors.hpp:17-26): restriction syntax / type error."""

    def __init__(self, msg: str, position: int = 0):
        super().__init__(msg)
        self.position = position


class EmptySearchSpaceError(Error):
    """gridtune::EmptySearchSpaceError (errors.hpp:29-32)."""


def check(rc: int, position: int = 0) -> None:
    if rc == _lib.GTC_OK:
        return
    msg = _lib.last_error()
    if rc == _lib.GTC_ERR_PARSE:
        raise ParseError(msg, position)
    if rc == _lib.GTC_ERR_EMPTY:
        raise EmptySearchSpaceError(msg)
    if rc == _lib.GTC_ERR_CONDITIONING:
        raise ModelConditioningError(msg)
    if rc == _lib.GTC_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == _lib.GTC_ERR_SAMPLING:
        raise SamplingError(msg)
    if rc in (_lib.GTC_ERR_CUDA, _lib.GTC_ERR_OOM):
        raise DeviceError(msg)
    raise Error(msg)


# ---------------------------------------------------------------- gp.hpp:12-56
class MaternNu(enum.IntEnum):
    half = 0
    three_halves = 1
    five_halves = 2


@dataclass(frozen=True)
class MaternKernel:
    """MaternKernel (gp.hpp:27-56); defaults nu=3/2, l=2.0, s2=1.0."""
    nu: MaternNu = MaternNu.three_halves
    lengthscale: float = 2.0
    output_variance: float = 1.0

    def __post_init__(self):
        if not (self.lengthscale > 0.0):
            raise Error("kernel lengthscale must be positive")
        if not (self.output_variance > 0.0):
            raise Error("kernel output variance must be positive")

    def c(self) -> _lib.gtc_kernel:
        return _lib.gtc_kernel(int(self.nu), float(self.lengthscale), float(self.output_variance))


@dataclass
class GpPrediction:
    """GpPrediction (gp.hpp:62-69): standardized mean/variance + scaling."""
    mean: np.ndarray
    variance: np.ndarray
    y_mean: float = 0.0
    y_std: float = 1.0

    def raw_mean(self, i: int) -> float:
        return self.y_mean + self.y_std * float(self.mean[i])


class GpModel:
    """GpModel (gp.hpp:74-203) with the factor resident on the GPU."""

    def __init__(self, handle, kernel: MaternKernel, n: int, d: int, info: _lib.gtc_fit_info,
                 noise: float, device: int):
        self._h = handle
        self._kernel = kernel
        self._n = n
        self._d = d
        self._noise = noise
        self._device = device
        self._y_mean = info.y_mean
        self._y_std = info.y_std
        self._jitter = info.jitter

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            try:
                load().gtc_gp_destroy(h)
            except Exception:
                pass

    @staticmethod
    def fit(kernel: MaternKernel, X, y_raw, noise: float = 1e-10, jitter: float = 1e-6,
            device: int = 0) -> "GpModel":
        """GpModel::fit (gp.hpp:81-135): standardisation, Gram on device,
        Cholesky with jitter doubling (<= 6), ModelConditioningError after."""
        X = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
        y = np.ascontiguousarray(np.asarray(y_raw, dtype=np.float64).reshape(-1))
        if X.ndim != 2:
            X = X.reshape(len(y), -1) if len(y) else X.reshape(0, 1)
        if X.shape[0] != y.shape[0]:
            raise Error("GP fit: observation count does not match input count")
        d = X.shape[1] if X.shape[1] > 0 else 1
        if X.shape[1] == 0:
            X = np.zeros((X.shape[0], 1))
        lib = load()
        h = C.c_void_p()
        info = _lib.gtc_fit_info()
        kc = kernel.c()
        check(lib.gtc_gp_fit(device, C.byref(kc), _lib.dptr(X), _lib.dptr(y), int(len(y)), int(d),
                             float(noise), float(jitter), C.byref(h), C.byref(info)))
        return GpModel(h, kernel, len(y), d, info, noise, device)

    @property
    def kernel(self) -> MaternKernel:
        return self._kernel

    def train_size(self) -> int:
        return self._n

    def y_mean(self) -> float:
        return self._y_mean

    def y_std(self) -> float:
        return self._y_std

    def noise(self) -> float:
        return self._noise

    def jitter(self) -> float:
        return self._jitter

    def standardize(self, y_raw: float) -> float:
        """gp.hpp:145"""
        return (y_raw - self._y_mean) / self._y_std

    def predict(self, Xstar) -> GpPrediction:
        """GpModel::predict (gp.hpp:150-168) on the device."""
        Xs = np.ascontiguousarray(np.asarray(Xstar, dtype=np.float64))
        if Xs.ndim == 1:
            Xs = Xs.reshape(1, -1)
        m = Xs.shape[0]
        mean = np.empty(m)
        var = np.empty(m)
        if m:
            check(load().gtc_gp_predict(self._h, _lib.dptr(Xs), m, _lib.dptr(mean), _lib.dptr(var)))
        return GpPrediction(mean, var, self._y_mean, self._y_std)


def mean_posterior_variance(prediction: GpPrediction) -> float:
    """gp.hpp:207-212"""
    if prediction.variance.size == 0:
        raise Error("mean_posterior_variance: empty candidate set")
    return float(np.sum(prediction.variance) / prediction.variance.size)


# ---------------------------------------------------------------- acquisition.hpp
class AcquisitionId(enum.IntEnum):
    ei = 0
    poi = 1
    lcb = 2


@dataclass
class ExplorationConfig:
    """acquisition.hpp:55-59"""
    class Mode(enum.IntEnum):
        constant = 0
        contextual_variance = 1

    mode: "ExplorationConfig.Mode" = Mode.contextual_variance
    constant: float = 0.01


@dataclass
class ContextualVarianceState:
    """acquisition.hpp:63-66"""
    initial_sample_mean: float = 0.0
    initial_mean_variance: float = 0.0


def contextual_variance_lambda(state: ContextualVarianceState, mean_variance: float,
                               f_best_raw: float) -> Optional[float]:
    """acquisition.hpp:73-83 (host scalar formula; the device computes the same
    expression inside the selection kernel)."""
    if not (f_best_raw > 0.0) or not (state.initial_sample_mean > 0.0) or \
            not (state.initial_mean_variance > 0.0):
        return None
    lam = (mean_variance * f_best_raw / state.initial_sample_mean) / state.initial_mean_variance
    return lam if lam > 0.0 else 0.0


def discounted_observation_score(history: Sequence[float], gamma: float) -> float:
    """acquisition.hpp:88-92"""
    score = 0.0
    for o in history:
        score = score * gamma + o
    return score


# ---------------------------------------------------------------- portfolio.hpp:20-61
@dataclass
class CandidateScores:
    ids: np.ndarray
    means: np.ndarray
    stds: np.ndarray
    best_std: float = 0.0
    lambda_: float = 0.0

    def size(self) -> int:
        return int(len(self.ids))


def best_candidate(af: AcquisitionId, c: CandidateScores, excluded=None, device: int = 0) -> int:
    """best_candidate (portfolio.hpp:32-61) as one device pass: masked argmax,
    lowest position on ties, first candidate taken unconditionally; raises
    Error('acquisition: no candidates remaining')."""
    m = np.ascontiguousarray(np.asarray(c.means, dtype=np.float64))
    s = np.ascontiguousarray(np.asarray(c.stds, dtype=np.float64))
    n = len(m)
    if n == 0:
        raise Error("acquisition: no candidates remaining")
    ex = None
    if excluded is not None:
        ex = np.ascontiguousarray(np.asarray(excluded, dtype=np.uint8))
    pos = C.c_int64(-1)
    score = C.c_double(0.0)
    check(load().gtc_best_candidate(device, int(af), _lib.dptr(m), _lib.dptr(s), n, float(c.best_std),
                                    float(c.lambda_), _lib.u8ptr(ex) if ex is not None else None,
                                    C.byref(pos), C.byref(score)))
    return int(pos.value)


def acquisition_scores(af: AcquisitionId, means, stds, best_std: float, lambda_: float,
                       device: int = 0) -> np.ndarray:
    """Per-candidate EI / PI / -LCB on the device (acquisition.hpp:25-42)."""
    m = np.ascontiguousarray(np.asarray(means, dtype=np.float64))
    s = np.ascontiguousarray(np.asarray(stds, dtype=np.float64))
    out = np.empty(len(m))
    check(load().gtc_acquisition_scores(device, int(af), _lib.dptr(m), _lib.dptr(s), len(m),
                                        float(best_std), float(lambda_), _lib.dptr(out)))
    return out
