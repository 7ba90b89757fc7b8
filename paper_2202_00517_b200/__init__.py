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
ranking systems, the metrizability checker, the comparator-only engine
(BoundedNeighborSet), point-file IO and the CLI are out of scope (see
DESIGN.md).  The experiment harness (run_experiment / dimension_sweep /
emit_report / emit_sweep, ``paper_2202_00517_b200.bench``) and the small host
helpers (kl_divergence, candidate_set, build_cofriends, verify_total_order)
keep the reference's names and behaviour.
"""

from ._lib import EXPORTS, KnndError, launch_count
from ._lib import load as load_library
from .core import ConfigError, Dataset, ItemId, RankingSystem, ScoredRankingSystem, build_cofriends, verify_total_order
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
    candidate_set,
    run,
    run_round,
    run_to_fixed_point,
)
from . import bench, evaluation
from .bench import (
    ORACLE_GUARD,
    ExperimentReport,
    ExperimentSpec,
    OracleGuardError,
    dimension_sweep,
    emit_report,
    emit_sweep,
    run_experiment,
)
from .evaluation import ExactKnnGraph, exact_knn, exact_rows, recall, sampled_recall, uniform_recall_sample
from .similarity import (
    EuclideanRankingSystem,
    KlRankingSystem,
    euclidean_ranking,
    kl_divergence,
    load_points_csv,
    load_points_f64,
    sample_simplex_uniform,
    save_points_csv,
    save_points_f64,
    validate_simplex_points,
)

__version__ = "0.1.0"

__all__ = [
    "bench",
    "build_cofriends",
    "candidate_set",
    "ConfigError",
    "Dataset",
    "derive_rng",
    "DescentConfig",
    "dimension_sweep",
    "emit_report",
    "emit_sweep",
    "euclidean_ranking",
    "EuclideanRankingSystem",
    "evaluation",
    "exact_knn",
    "exact_rows",
    "ExactKnnGraph",
    "ExperimentReport",
    "ExperimentSpec",
    "EXPORTS",
    "fcc_samples",
    "friend_clustering_rate",
    "init_random_kout",
    "ItemId",
    "kl_divergence",
    "load_points_csv",
    "load_points_f64",
    "save_points_csv",
    "save_points_f64",
    "KlRankingSystem",
    "KnndError",
    "KnnState",
    "launch_count",
    "load_library",
    "ORACLE_GUARD",
    "OracleGuardError",
    "propose_new_friend_set",
    "random_kout_draws",
    "RankingSystem",
    "recall",
    "round_budget",
    "RoundStats",
    "run",
    "run_experiment",
    "run_round",
    "run_to_fixed_point",
    "sample_simplex_uniform",
    "sampled_recall",
    "ScoredRankingSystem",
    "STREAM_DATA",
    "STREAM_FCC",
    "STREAM_INIT",
    "STREAM_RECALL",
    "uniform_recall_sample",
    "validate_simplex_points",
    "verify_total_order",
]
