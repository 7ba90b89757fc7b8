"""B200-native K-NN descent local join (arXiv 2202.00517).

Drop-in for the hot path of the reference package ``rankdescent``: swap
``import rankdescent as rd`` for ``import paper_2202_00517_b200 as rd`` and
``rd.run(rd.Dataset(points), rd.KlRankingSystem(points), rd.DescentConfig(k=K))``
runs the same algorithm with the per-round local join, co-friend CSR,
initial row sort and FCC statistic in hand-written sm_100a kernels
(libknnd.so, C ABI in include/knnd.h).

The exact K-NN ground truth and recall (evaluation.py:36-137) run on the GPU
too (knnd_exact_knn).  The KL and squared-Euclidean ranking systems
(similarity.py:80-140) are accelerated through the same fused join; other
ranking systems, the metrizability checker and the CLI are out of scope (see
DESIGN.md).  ``paper_2202_00517_b200.bench`` mirrors the reference's experiment
harness (run_experiment / dimension_sweep / emit_report / emit_sweep).
"""

from ._lib import EXPORTS, KnndError, launch_count
from ._lib import load as load_library
from .core import ConfigError, Dataset, ItemId, RankingSystem, ScoredRankingSystem
from .descent import (
    STREAM_DATA,
    STREAM_FCC,
    STREAM_INIT,
    STREAM_RECALL,
    DescentConfig,
    KnnState,
    RoundStats,
    derive_rng,
    fcc_samples,
    friend_clustering_rate,
    init_random_kout,
    propose_new_friend_set,
    random_kout_draws,
    round_budget,
    run,
    run_round,
    run_to_fixed_point,
)
from . import bench, evaluation
from .evaluation import ExactKnnGraph, exact_knn, exact_rows, recall, sampled_recall, uniform_recall_sample
from .similarity import (
    EuclideanRankingSystem,
    KlRankingSystem,
    euclidean_ranking,
    sample_simplex_uniform,
    validate_simplex_points,
)

__version__ = "0.1.0"

__all__ = [
    "ConfigError",
    "Dataset",
    "DescentConfig",
    "EXPORTS",
    "EuclideanRankingSystem",
    "ExactKnnGraph",
    "ItemId",
    "KlRankingSystem",
    "KnndError",
    "KnnState",
    "RankingSystem",
    "RoundStats",
    "STREAM_DATA",
    "STREAM_FCC",
    "STREAM_INIT",
    "STREAM_RECALL",
    "ScoredRankingSystem",
    "derive_rng",
    "euclidean_ranking",
    "bench",
    "evaluation",
    "exact_knn",
    "exact_rows",
    "fcc_samples",
    "friend_clustering_rate",
    "init_random_kout",
    "launch_count",
    "load_library",
    "propose_new_friend_set",
    "random_kout_draws",
    "recall",
    "round_budget",
    "run",
    "run_round",
    "run_to_fixed_point",
    "sample_simplex_uniform",
    "sampled_recall",
    "uniform_recall_sample",
    "validate_simplex_points",
]
