"""Behavioural tests of the drop-in API on the device engine, restating the
reference's own test_descent.py checks (init / KnnState / run_round / FCC /
run / run_to_fixed_point) on the same small instances, plus the reference's
recorded outcome for each instance (tests/golden/api_cases.json, from
make_api_golden.py): same final table (sha256) and same history."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import paper_2202_00517_b200 as b2
from conftest import load_json

pytestmark = pytest.mark.gpu


def kl_instance(n, d, seed):
    pts = b2.sample_simplex_uniform(d, n, seed)
    return b2.Dataset(pts), b2.KlRankingSystem(pts, validate=False)


def euclid_instance(n, d, seed):
    v = np.random.default_rng(seed).standard_normal((n, d))
    return b2.Dataset(v), b2.EuclideanRankingSystem(v)


def assert_valid_kout(friends, n, k):
    """Out-degree k, ids in range, no self-loops, no repeated targets."""
    assert friends.shape == (n, k)
    assert friends.min() >= 0 and friends.max() < n
    assert not (friends == np.arange(n)[:, None]).any()
    srt = np.sort(friends, axis=1)
    assert not (srt[:, 1:] == srt[:, :-1]).any()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def cases():
    return load_json("api_cases.json")


def hist(h):
    return [[s.round_index, s.fcc, s.comparisons, s.changed_friend_sets] for s in h]


# ---------------------------------------------------------------------------
# init_random_kout (descent.py:177-213)


def test_init_out_degree_and_no_self_loops(cuda):
    ds, rs = kl_instance(5, 3, 0)
    st = b2.init_random_kout(ds, rs, b2.DescentConfig(k=2), b2.derive_rng(0, 2))
    assert_valid_kout(st.friends, 5, 2)


def test_init_forced_case_n_equals_k_plus_one(cuda, cases):
    ds, rs = kl_instance(5, 3, 1)
    st = b2.init_random_kout(ds, rs, b2.DescentConfig(k=4), b2.derive_rng(0, 2))
    for x in range(5):
        assert set(map(int, st.friends[x])) == set(range(5)) - {x}
    assert sha(st.friends) == cases["init_kl_5_3_k4_s1"]["sha"]


@pytest.mark.parametrize("name", ["init_kl_1000_5_k8_s42", "init_kl_300_6_k7_s3", "init_kl_12_3_k6_s4"])
def test_init_matches_reference_and_is_deterministic(cuda, cases, name):
    c = cases[name]
    ds, rs = kl_instance(c["n"], c["d"], c["seed"])
    a = b2.init_random_kout(ds, rs, b2.DescentConfig(k=c["k"]), b2.derive_rng(c["rng_seed"], 2))
    b = b2.init_random_kout(ds, rs, b2.DescentConfig(k=c["k"]), b2.derive_rng(c["rng_seed"], 2))
    assert np.array_equal(a.friends, b.friends)
    assert sha(a.friends) == c["sha"]
    assert_valid_kout(a.friends, c["n"], c["k"])  # 12/6 is the dense (permutation) regime


def test_init_rows_sorted_under_anchor_order(cuda):
    ds, rs = kl_instance(300, 6, 3)
    st = b2.init_random_kout(ds, rs, b2.DescentConfig(k=7), b2.derive_rng(3, 2))
    for x in range(0, 300, 17):
        keys = [(rs.score(x, int(y)), int(y)) for y in st.friends[x]]
        assert keys == sorted(keys)


def test_init_rejects_n_not_greater_than_k(cuda):
    ds, rs = kl_instance(8, 3, 5)
    with pytest.raises(b2.ConfigError):
        b2.init_random_kout(ds, rs, b2.DescentConfig(k=8), b2.derive_rng(0, 2))


# ---------------------------------------------------------------------------
# KnnState and rounds (descent.py:111-148, 282-314)


def test_snapshot_is_read_only(cuda):
    st = b2.KnnState(np.array([[1, 2], [0, 2], [0, 1]]))
    with pytest.raises(ValueError):
        st.friends[0, 0] = 2


def test_out_degree_regular_after_rounds(cuda):
    ds, rs = kl_instance(250, 4, 15)
    cfg = b2.DescentConfig(k=5, seed=15)
    st = b2.init_random_kout(ds, rs, cfg, b2.derive_rng(15, 2))
    for _ in range(4):
        st, _ = b2.run_round(st, rs, cfg)
        assert_valid_kout(st.friends, 250, 5)


def test_monotone_local_improvement(cuda):
    """The K-th best friend of an anchor never gets worse (descent.py:234 keeps
    the current friends in the candidate set)."""
    ds, rs = kl_instance(200, 5, 16)
    cfg = b2.DescentConfig(k=6, seed=16)
    st = b2.init_random_kout(ds, rs, cfg, b2.derive_rng(16, 2))
    for _ in range(3):
        new, _ = b2.run_round(st, rs, cfg)
        for x in range(200):
            old_worst = max((rs.score(x, int(y)), int(y)) for y in st.friends[x])
            new_worst = max((rs.score(x, int(y)), int(y)) for y in new.friends[x])
            assert new_worst <= old_worst
        st = new


def test_comparison_count_bound(cuda):
    ds, rs = kl_instance(500, 5, 17)
    k = 6
    cfg = b2.DescentConfig(k=k, seed=17)
    st = b2.init_random_kout(ds, rs, cfg, b2.derive_rng(17, 2))
    _, stats = b2.run_round(st, rs, cfg)
    assert 0 < stats.comparisons <= 2 * 500 * (k + k * k)


# ---------------------------------------------------------------------------
# friend_clustering_rate (descent.py:317-338)


def test_fcc_fresh_random_kout_is_near_zero(cuda):
    ds, rs = kl_instance(20_000, 10, 18)
    st = b2.init_random_kout(ds, rs, b2.DescentConfig(k=16), b2.derive_rng(18, 2))
    assert b2.friend_clustering_rate(st, 2000, b2.derive_rng(18, 3, 0)) < 0.05


def test_fcc_rejects_bad_arguments(cuda):
    with pytest.raises(b2.ConfigError):
        b2.friend_clustering_rate(b2.KnnState(np.array([[1], [2], [0]])), 10, b2.derive_rng(0, 3, 1))
    with pytest.raises(b2.ConfigError):
        b2.friend_clustering_rate(b2.KnnState(np.array([[1, 2], [0, 2], [0, 1]])), 0, b2.derive_rng(0, 3, 1))


# ---------------------------------------------------------------------------
# run / run_to_fixed_point (descent.py:341-391)


@pytest.mark.parametrize("name", ["run_kl_2000_6_k8_s20", "run_kl_500_5_k6_s23", "run_kl_5_3_k4_s22",
                                  "run_kl_100_4_k4_s19_max1", "run_kl_30_4_k4_s21"])
def test_run_matches_reference(cuda, cases, name):
    c = cases[name]
    ds, rs = kl_instance(c["n"], c["d"], c["seed"])
    friends, h = b2.run(ds, rs, b2.DescentConfig(**c["cfg"]))
    assert hist(h) == c["history"]
    assert sha(friends) == c["sha"]
    assert_valid_kout(friends, c["n"], c["cfg"]["k"])


def test_run_stops_when_rate_stalls(cuda):
    ds, rs = kl_instance(2000, 6, 20)
    _, h = b2.run(ds, rs, b2.DescentConfig(k=8, seed=20))
    rates = [s.fcc for s in h]
    if len(h) < b2.DescentConfig(k=8).resolved_max_rounds(2000):
        assert rates[-1] <= rates[-2]
    for a, b in zip(rates[:-2], rates[1:-1]):
        assert b > a  # strictly increasing before the stopping round


def test_run_max_rounds_one_and_forced_complete_case(cuda):
    ds, rs = kl_instance(100, 4, 19)
    assert len(b2.run(ds, rs, b2.DescentConfig(k=4, seed=19, max_rounds=1))[1]) == 1
    ds, rs = kl_instance(5, 3, 22)
    friends, h = b2.run(ds, rs, b2.DescentConfig(k=4, seed=22))
    for x in range(5):
        assert set(map(int, friends[x])) == set(range(5)) - {x}
    assert len(h) == 2  # rate 1.0 from round 1, stalls at round 2


def test_run_small_instance_recall(cuda):
    ds, rs = kl_instance(30, 4, 21)
    friends, _ = b2.run(ds, rs, b2.DescentConfig(k=4, seed=21))
    assert b2.recall(friends, b2.exact_knn(ds, rs, 4), np.arange(30)) >= 0.9


def test_run_deterministic_replay(cuda):
    ds, rs = kl_instance(500, 5, 23)
    cfg = b2.DescentConfig(k=6, seed=23)
    fa, ha = b2.run(ds, rs, cfg)
    fb, hb = b2.run(ds, rs, cfg)
    assert np.array_equal(fa, fb) and hist(ha) == hist(hb)


def test_run_propagates_config_error(cuda):
    ds, rs = kl_instance(6, 3, 24)
    with pytest.raises(b2.ConfigError):
        b2.run(ds, rs, b2.DescentConfig(k=8, seed=0))


@pytest.mark.parametrize("name", ["fixed_eu_120_3_k4_s25", "fixed_eu_120_3_k4_s26_max2"])
def test_run_to_fixed_point_matches_reference(cuda, cases, name):
    c = cases[name]
    ds, rs = euclid_instance(c["n"], c["d"], c["seed"])
    friends, h = b2.run_to_fixed_point(ds, rs, b2.DescentConfig(**c["cfg"]))
    assert hist(h) == c["history"]
    assert sha(friends) == c["sha"]
    if "max_rounds" in c["cfg"]:
        assert len(h) <= c["cfg"]["max_rounds"]
    else:
        assert h[-1].changed_friend_sets == 0
    assert_valid_kout(friends, c["n"], c["cfg"]["k"])


@pytest.mark.parametrize("n,d,k", [(20_000, 10, 16), (100_000, 20, 20)])
def test_repeated_runs_on_one_ranking_system_agree(cuda, n, d, k):
    """run() twice on the same ranking system (cached device tables, reused
    caching-allocator blocks): identical tables and histories — the check that
    exposed knnd_random_kout's workspace overrun."""
    pts = b2.sample_simplex_uniform(d, n, b2.derive_rng(0, b2.STREAM_DATA, d))
    ds, rs = b2.Dataset(pts), b2.KlRankingSystem(pts, validate=False)
    cfg = b2.DescentConfig(k=k, seed=1, max_rounds=3)
    fa, ha = b2.run(ds, rs, cfg)
    fb, hb = b2.run(ds, rs, cfg)
    fc, hc = b2.run(ds, b2.KlRankingSystem(pts, validate=False), cfg)
    assert np.array_equal(fa, fb) and np.array_equal(fa, fc)
    assert hist(ha) == hist(hb) == hist(hc)


# ---------------------------------------------------------------------------
# candidate_set / propose_new_friend_set (descent.py:216-259)


def test_candidate_set_hand_traces(cuda):
    st = b2.KnnState(np.array([[1, 2], [0, 2], [0, 1]]))
    assert all(b2.candidate_set(x, st).size == 0 for x in range(3))  # saturated triangle
    assert list(b2.candidate_set(0, b2.KnnState(np.array([[1], [2], [0]])))) == [2]  # three-cycle, K = 1


def test_candidate_set_exclusion_and_size_bound(cuda):
    ds, rs = kl_instance(400, 4, 8)
    k = 5
    st = b2.init_random_kout(ds, rs, b2.DescentConfig(k=k), b2.derive_rng(8, 2))
    for x in range(0, 400, 13):
        cand = b2.candidate_set(x, st)
        assert x not in cand and not np.isin(cand, st.friends[x]).any()
        assert len(set(map(int, cand))) == cand.size and np.all(np.diff(cand) > 0)
        cofs = st.cofriends_of(x).size
        assert cand.size <= cofs + k * k + cofs * k


def test_propose_matches_exhaustive_union_sort(cuda):
    """The device join for one anchor equals sorting friends | candidates by (score, id)."""
    ds, rs = euclid_instance(20, 1, 9)
    st = b2.init_random_kout(ds, rs, b2.DescentConfig(k=2), b2.derive_rng(9, 2))
    for x in range(20):
        union = set(map(int, st.friends[x])) | set(map(int, b2.candidate_set(x, st)))
        expected = sorted(union, key=lambda y: (rs.score(x, y), y))[:2]
        assert list(b2.propose_new_friend_set(x, st, rs)) == expected
