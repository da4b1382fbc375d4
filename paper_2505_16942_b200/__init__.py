"""B200-native correlation-volume lookup (RAFT / SEA-RAFT), drop-in for corrvol's samplers.

Hot path (BASELINE.json north_star): fmap2 pyramid, per-iteration
(2r+1)^2 bilinear cost lookup around each query's flow estimate, and the
dense / on-demand / partial variant switch — all computed by hand-written
sm_100a kernels in libcorrvol_b200.so (C ABI: include/corrvol_b200.h).
Names and signatures follow corrvol 0.1.0 (corrvol/__init__.py:23-176) for
the hot-path subset.  There is no CPU fallback.
"""

from ._backend import available_backends, default_backend, get_kernels
from .dense import (PYRAMID_MODES, DenseCorrelationVolume, build_dense_volume,
                    build_feature_pyramid, build_volume_pyramid, estimate_dense_bytes,
                    lookup_dense, pool_volume, pooled_dims)
from .analyzer import LevelAccess, record_occupancy
from .flow import cascaded_init, resample_flow
from .ondemand import WorkCount, count_work_on_demand, lookup_on_demand
from .raft import CorrBlock
from .sampler import VARIANTS, BatchCorrSampler, CorrSampler
from .scenario import SyntheticScenario, gen_scenario
from .sparse import (DEFAULT_CACHE_CAP_BYTES, BlockStore, PaddedGrid, ProxyBlock,
                     SparseVolumeState, compute_block_indices, gather_proxy, init_state,
                     init_state_batch,
                     memory_footprint, padded_extent, sample_iteration, sample_iteration_raft,
                     sampled_block_mmm, set_computation_mask)
from .types import (CacheLimitError, CentroidField, CorrvolError, CostMaps,
                    DimensionMismatchError, FeatureMap, FeaturePyramid, GatherMissError,
                    LookupSpec, WorkCounter)

__version__ = "0.1.0"

__all__ = [
    "available_backends", "default_backend", "get_kernels",
    "PYRAMID_MODES", "DenseCorrelationVolume", "build_dense_volume", "build_feature_pyramid",
    "build_volume_pyramid", "estimate_dense_bytes", "lookup_dense", "pool_volume",
    "pooled_dims",
    "WorkCount", "count_work_on_demand", "lookup_on_demand",
    "cascaded_init", "resample_flow", "LevelAccess", "record_occupancy",
    "VARIANTS", "CorrSampler", "BatchCorrSampler", "CorrBlock",
    "SyntheticScenario", "gen_scenario",
    "DEFAULT_CACHE_CAP_BYTES", "BlockStore", "PaddedGrid", "ProxyBlock", "SparseVolumeState",
    "compute_block_indices", "gather_proxy", "init_state", "memory_footprint", "padded_extent",
    "sample_iteration", "sample_iteration_raft", "sampled_block_mmm", "set_computation_mask",
    "CacheLimitError", "CentroidField", "CorrvolError", "CostMaps", "DimensionMismatchError",
    "FeatureMap", "FeaturePyramid", "GatherMissError", "LookupSpec", "WorkCounter",
]
