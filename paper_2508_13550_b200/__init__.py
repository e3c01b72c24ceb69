"""B200-native (sm_100a) cubed-sphere FMM — the hot path of arXiv 2508.13550
(csfs::csfmm_sum, /root/reference/proj/src/summation.cpp:383-421) as hand-written CUDA
behind a C-ABI (include/csfs_b200.h)."""
from .engine import (  # noqa: F401
    BveState,
    BveStepOptions,
    Engine,
    Kernel,
    KernelKind,
    Method,
    ParticleSet,
    PotentialField,
    SalParams,
    SumStats,
    TraversalConfig,
    bve_remesh,
    bve_step,
    csfmm_sum,
    default_engine,
    direct_sum,
    lib,
    summed_potential,
)
