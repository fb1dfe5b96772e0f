"""stgp_b200: B200-native engine for the data-parallel hot path of arXiv 2602.03609.

Vecchia / FITC / VIF negative log-likelihood, gradient and prediction, the
correlation-based neighbour searches and space-time kMeans++ seeding, as
hand-written sm_100a CUDA behind a C ABI (include/stgp_b200.h).  This package
is the Python mirror of the reference's C++ API (proj/include/stgp/*.hpp).
"""
from .api import *  # noqa: F401,F403
from .api import (CovarianceParams, Context, SpaceTimeDataset, NeighborSets, InducingSet, Structure,  # noqa: F401
                  build_vecchia, build_fitc, build_vif, nll, nll_grad, nll_and_grad, evaluate, gls_beta, predict,
                  euclidean_neighbors, correlation_neighbors, residual_neighbors, sts_kmeanspp,
                  joint_kmeanspp_inducing, kmeanspp, order_observations, order_observations_perm,
                  effective_ranges, fit, default_init, read_dataset_csv, write_dataset_csv, write_neighbor_debug_csv, FitConfig, FittedModel, LikelihoodParams, LaplaceState, laplace_marginal, ZcptnPrediction, zcptn_predict, ConfigError, DataError, NumericError, StgpError, LATENT, OBSERVATION)
from ._native import LIB_PATH, exported_symbols  # noqa: F401
from . import synth  # noqa: F401

__version__ = "0.1.0"
