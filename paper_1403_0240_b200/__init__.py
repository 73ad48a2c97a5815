"""B200-native Region Competition hot path (arXiv 1403.0240).

Drop-in for the reference package ``rcseg``'s engine, energy and Sobolev
entry points (rcseg/__init__.py:5-19).  All compute runs in
``librcseg_b200.so`` (hand-written CUDA for sm_100a) through a C ABI
(include/rcb.h); importing this package without the built library raises.
"""

__version__ = "0.1.0"

from .energy import (DegenerateStatsError, EnergyConfig, EnergyModel, EnergyValue,  # noqa: E402
                     delta_internal, delta_internal_batch, evaluate_total)
from .grid import (Connectivity, RegionStats, StatsTable, count_components,  # noqa: E402
                   flood_fill_components)
from .contour import ContourState, StaleParticleError, scan_contour  # noqa: E402
from .optimizer import (IterationRecord, OptimizerConfig, RegionCompetition,  # noqa: E402
                        RunResult, initialize, run)
from .synth import (NoiseSpec, SceneSpec, desk_scene, generate, two_blob_scene,  # noqa: E402
                    two_sphere_scene)
from .sobolev import SobolevParams, detect_oscillation, kernel_eval, sobolev_filter  # noqa: E402
from . import imageio, report  # noqa: E402

__all__ = [
    "Connectivity", "EnergyConfig", "EnergyValue", "evaluate_total", "EnergyModel",
    "delta_internal", "delta_internal_batch", "DegenerateStatsError", "StatsTable",
    "OptimizerConfig", "RegionCompetition", "RunResult", "IterationRecord", "run",
    "SobolevParams", "kernel_eval", "sobolev_filter", "detect_oscillation",
    "ContourState", "StaleParticleError", "scan_contour", "imageio", "report", "__version__",
    "initialize", "SceneSpec", "NoiseSpec", "desk_scene", "generate", "two_blob_scene",
    "two_sphere_scene", "RegionStats", "flood_fill_components", "count_components",
]
