"""gridtune-b200: B200-native (sm_100a) surrogate pass of the BO kernel tuner
of arXiv 2111.14991, behind the reference `gridtune` API.

The compute path is libgridtune_b200.so (CUDA, built in-tree); this package is
the Python mirror of the reference interface over its C ABI
(include/gridtune_cuda.h).
"""
from ._lib import LIB_PATH, load  # noqa: F401
from .gp import (AcquisitionId, CandidateScores, ConfigError, ContextualVarianceState,  # noqa: F401
                 DeviceError, EmptySearchSpaceError, Error, ExplorationConfig, GpModel, GpPrediction,
                 MaternKernel, MaternNu, ModelConditioningError, ParseError, SamplingError,
                 acquisition_scores, best_candidate,
                 contextual_variance_lambda, discounted_observation_score,
                 mean_posterior_variance)
from .runtime import FitInfo, Selection, Space, SurrogateRun  # noqa: F401
from .cache import CacheError, MeasurementCache  # noqa: F401
from .space import EnumeratedSpace, ParameterDef, ParamKind, SearchSpace, parse_restriction  # noqa: F401
from .strategies import (StrategyConfig, StrategyId, TuningRun, run_bo, run_bo_batch,  # noqa: F401
                         run_strategy, strategy_from_string)

__version__ = "0.1.0"
