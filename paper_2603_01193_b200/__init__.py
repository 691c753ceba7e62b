"""B200-native Walk-on-Spheres label estimator (hot path of arxiv 2603.01193).

Drop-in for the reference package ``spherewalk``'s estimator path:
``WalkConfig``, ``Problem``, ``walk_poisson_values``, ``walk_poisson``,
``walk_poisson_antithetic``, ``estimate``, ``PointEstimate``, and the
epoch-averaged ``EstimateCache`` of the training-label loop — backed by
hand-written sm_100a CUDA kernels in ``libwos_b200.so`` behind the C ABI of
``include/wos_b200.h``. There is no CPU fallback. ``artifacts`` writes the
reference CLI's solve / bench files (run stamp, CSV, summary) from GPU estimates.
"""

from . import artifacts
from .cache import CacheShapeError, EstimateCache, cache_update, export_csv
from .estimator import (PointEstimate, WelfordAccumulator, chan_merge, estimate, estimate_arrays,
                        estimate_tensors)
from .engine import UnsupportedProblemError
from .geometry import (
    BallDomain,
    BoxDomain,
    ExteriorQueryError,
    MeshDomain,
    PolarDomain,
    PolygonDomain,
    star_polygon,
)
from .walker import (
    MajorantViolationError,
    ScreenedProblem,
    walk_screened_delta,
    walk_screened_values,
    TERM_BOUNDARY,
    TERM_MAX_STEPS,
    Problem,
    TrajectoryResult,
    TrajectoryStream,
    WalkConfig,
    walk_poisson,
    walk_poisson_antithetic,
    walk_poisson_values,
)

__version__ = "0.1.0"

__all__ = [
    "BallDomain",
    "CacheShapeError",
    "EstimateCache",
    "BoxDomain",
    "ExteriorQueryError",
    "MajorantViolationError",
    "PointEstimate",
    "WelfordAccumulator",
    "MeshDomain",
    "PolarDomain",
    "PolygonDomain",
    "Problem",
    "ScreenedProblem",
    "TERM_BOUNDARY",
    "TERM_MAX_STEPS",
    "TrajectoryResult",
    "TrajectoryStream",
    "UnsupportedProblemError",
    "WalkConfig",
    "cache_update",
    "chan_merge",
    "estimate",
    "estimate_arrays",
    "estimate_tensors",
    "export_csv",
    "star_polygon",
    "walk_poisson",
    "walk_poisson_antithetic",
    "walk_poisson_values",
    "walk_screened_delta",
    "walk_screened_values",
]
