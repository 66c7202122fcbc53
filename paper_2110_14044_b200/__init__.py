"""B200-native iALS++ (arXiv 2110.14044) block solver.

A drop-in for the hot path of the reference package ``blockals`` 0.1.0: the
iALS++ epoch (``ialspp_epoch``) and its pieces, with the same public names.
The numerical work runs in hand-written sm_100a CUDA kernels behind the C ABI
of ``libials_b200.so`` (``include/ials_b200.h``); there is no CPU fallback.
"""

from .data import InteractionDataset, SideView
from .estimator import ImplicitALS
from .evaluation import (MetricReport, evaluate_holdout, fold_in_users, ndcg_at_k, project_user,
                         rank_items, recall_at_k, top_k_from_scores)
from .linalg import SingularMatrixError, check_block, gramian, partial_gramian
from .model import (FactorModel, PredictionCache, SolverConfig, cache_drift, compute_loss,
                    compute_predictions, effective_reg, init_model)
from .solvers import (BlockPartition, DeviceTrainer, EpochReport, block_update,
                      coordinate_update, ials_epoch, ialspp_epoch, icd_epoch, iterate_epochs,
                      partition_dims, train)

__version__ = "0.1.0"

__all__ = [
    "InteractionDataset", "SideView", "ImplicitALS",
    "MetricReport", "evaluate_holdout", "fold_in_users", "ndcg_at_k", "project_user",
    "rank_items", "recall_at_k", "top_k_from_scores",
    "SingularMatrixError", "check_block", "gramian", "partial_gramian",
    "FactorModel", "PredictionCache", "SolverConfig", "cache_drift", "compute_loss",
    "compute_predictions", "effective_reg", "init_model",
    "BlockPartition", "DeviceTrainer", "EpochReport", "block_update", "coordinate_update",
    "ials_epoch", "ialspp_epoch", "icd_epoch", "iterate_epochs", "partition_dims", "train",
]
