"""B200-native implicit moment-tensor CP f+grad (arXiv 1911.03813), drop-in for ``momentcp``.

The hot path of the reference package -- function/gradient evaluation of a rank-r symmetric
CP model against the d-th empirical moment tensor of p observations, computed from the n x p
observation matrix without forming the n^d tensor, plus the one-time ||X||^2 constant and the
packed adapter handed to the quasi-Newton driver -- re-built as hand-written sm_100a CUDA
kernels behind a C ABI (include/momentcp_b200.h).  Names and signatures follow the reference
exports (pkg/src/momentcp/__init__.py:14-68) for that path.
"""

__version__ = "0.1.0"

from .dense import ObservationSet
from .implicit import (
    GramCache,
    SymKruskal,
    build_gram_cache,
    data_norm_sq,
    kruskal_norm_sq,
    model_data_inner,
    ttsv_batch,
)
from .io import ParseError, read_observations_binary, write_observations_binary
from .multidevice import MultiDeviceObservationSet
from .objective import FgResult, fg_implicit, sample_observations
from .optimize import (AdamConfig, FgCallback, OptConfig, RunReport, adam_minimize, lbfgs_minimize,
                       lbfgs_minimize_batched, multistart_lbfgs, pack, packed_fg_implicit,
                       packed_fg_implicit_batched, unpack)

__all__ = [
    "AdamConfig",
    "adam_minimize",
    "sample_observations",
    "FgCallback",
    "FgResult",
    "GramCache",
    "ObservationSet",
    "MultiDeviceObservationSet",
    "OptConfig",
    "RunReport",
    "ParseError",
    "SymKruskal",
    "build_gram_cache",
    "data_norm_sq",
    "fg_implicit",
    "kruskal_norm_sq",
    "model_data_inner",
    "lbfgs_minimize",
    "lbfgs_minimize_batched",
    "multistart_lbfgs",
    "pack",
    "read_observations_binary",
    "packed_fg_implicit",
    "packed_fg_implicit_batched",
    "ttsv_batch",
    "unpack",
    "write_observations_binary",
]
