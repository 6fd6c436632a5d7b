"""B200-native RES-PCA (arXiv 1904.07497) solver: the reference's respca::solve
hot path as hand-written sm_100a CUDA behind a C-ABI (include/respca_cu.h).

The Python API mirrors the reference's C++ API (proj/include/respca/*.hpp):
"""
from .respca import (  # noqa: F401
    ConvergenceReport, DecompositionResult, KMeansConfig, KMeansResult, SolverConfig,
    check_convergence, column_l2_norms, column_mean, elementwise_l1, frob_norm, group_scatter,
    kmeans, kmeans_pp_init, kmeans_warm, l21_norm, l_update, lloyd_step, multiplier_update,
    s_update_l1, s_update_l21, solve, synth_generate,
)
