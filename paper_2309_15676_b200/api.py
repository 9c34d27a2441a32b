"""Host-side mirror of the reference `metagrad` API for the hot path, backed by
the sm_100a kernels behind include/mgcuda.h.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/metagrad/*.hpp):

  Rng.stream(seed, r)                      rng.hpp:23-25   (device mt19937_64)
  Moment2(decay).step(x)                   moment2.hpp:21-50
  GradientSamplePair(prop, diff, ssn)      meta.hpp:20-24
  MetaEstimator(lr, ...).step(pair, vp, vd) meta.hpp:71-114 (mean/var/alpha_prev injectable)
  Adam(lr, b1, b2, eps).step(grad)         adam.hpp:14-50
  MiniRenderProblem / ExpRateProblem / MultNoiseQuadratic .sample_pair(now, prev, rng)
                                           problems.hpp:74-195
  FusedMetaUpdate                          the one-pass hot path (harness.cpp:144-188)
  ExperimentConfig, run_single, run_experiment   harness.hpp:18-112

Vectors are torch CUDA tensors (float64 = parity mode, float32 = fast mode);
torch is only the device-memory/stream plumbing.  Exceptions: InvalidArgument
(std::invalid_argument), LogicError (std::logic_error), DomainError
(std::domain_error).  There is no CPU fallback.
"""
from __future__ import annotations

from . import _abi  # noqa: F401
from ._lib import DomainError, InvalidArgument, LogicError, MgError, check, load  # noqa: F401
from ._core import (  # noqa: F401
    _p,
    _dtype_code,
    Context,
    mix64,
    Rng,
)
from .estimators import (  # noqa: F401
    Moment2,
    GradientSamplePair,
    MetaEstimator,
    Adam,
    FusedMetaUpdate,
    FusedAdamUpdate,
)
from .problems import (  # noqa: F401
    _Problem,
    MiniRenderProblem,
    ExpRateProblem,
    MultNoiseQuadratic,
    MiniRenderRun,
)
from .scenes import (  # noqa: F401
    QuadTextureProblem,
    QuadTextureRun,
    helix_spheres,
    HelixProblem,
    HelixRun,
    MESH_VIEW_LAYOUT,
    _sphere_triangles,
    mesh_scene_geometry,
    mesh_large_scene_geometry,
    mesh_scene_view,
    smooth_noise_textures,
    MeshScene,
    MeshTextureProblem,
    large_scene_view,
    fixed_finalize,
    MeshLargeProblem,
    MeshTextureRun,
)
from .harness import (  # noqa: F401
    ExperimentConfig,
    STATUS,
    RunRecord,
    SCALED_MIN_PIXELS,
    _scaled_eligible,
    _run_minirender_scaled,
    _run_device,
    run_single,
    SeriesStats,
    AggregateReport,
    _seq_sum,
    _column_stats,
    SERIES_ORDER,
    aggregate,
    aggregate_series_device,
    _run_experiment_device_stats,
    run_experiment,
)

__all__ = ["Context", "Rng", "Moment2", "GradientSamplePair", "MetaEstimator", "Adam",
           "MiniRenderProblem", "ExpRateProblem", "MultNoiseQuadratic", "FusedMetaUpdate",
           "FusedAdamUpdate", "MiniRenderRun", "QuadTextureProblem", "QuadTextureRun",
           "HelixProblem", "HelixRun", "helix_spheres", "MeshScene", "MeshTextureProblem",
           "MeshTextureRun", "mesh_scene_geometry", "mesh_scene_view", "smooth_noise_textures",
           "MeshLargeProblem", "mesh_large_scene_geometry", "large_scene_view",
           "ExperimentConfig", "RunRecord", "AggregateReport", "run_single",
           "run_experiment", "InvalidArgument", "LogicError", "DomainError", "mix64"]
