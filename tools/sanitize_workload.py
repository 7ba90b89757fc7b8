"""A small run of every libknnd kernel, for compute-sanitizer (memcheck /
racecheck / synccheck; tools/gpu_sanitize.sh, tests/test_sanitize.py) and for
its stand-in on pools where compute-sanitizer is closed: run with
KNND_LIBRARY=checked KNND_GUARD=1 (tests/test_checked.py) it loads the
bounds-checked build and guards every workspace, and fails unless
knnd_check_failures() and the guard zones both report zero.

Covers: kl_prepare, the device PCG64 draws (knnd_random_kout) + row sort,
co-friend CSR, the local join in every size class (warp, 2^12/2^13 128-thread
blocks, 2^14 256-thread, 2^15 512-thread, global-memory hub tables) through a
hub-stress table, K = 64 (two selection registers per lane), the fused peer
stores (a same-device stand-in peer table), FCC, batch_scores, exact K-NN and
the Euclidean path.  Each result is checked against the C oracle so a
sanitizer run is also a parity run.  Prints SANITIZE_OK at the end."""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_00517_b200 as b2  # noqa: E402
from oracle import native, port  # noqa: E402


def hub_table(n, k, hubs, rng):
    t = b2.random_kout_draws(n, k, rng)
    for hub, cnt in hubs:
        rows = rng.choice(np.setdiff1d(np.arange(n), [hub]), size=cnt, replace=False)
        for r in rows:
            if hub not in t[r]:
                t[r, rng.integers(0, k)] = hub
    return t


def check_join(n, d, k, hubs, peers=False):
    rng = np.random.default_rng(n + d + k)
    pts = port.experiment_points(n, d, 3)
    tab = native.Tables(pts)
    table = native.sort_rows(tab, hub_table(n, k, hubs, rng))
    rs = b2.KlRankingSystem(pts, validate=False)
    st = b2.KnnState(table)
    dev = st.device
    out = torch.empty((n, k), dtype=torch.int32, device=dev)
    uc = torch.empty(n, dtype=torch.int32, device=dev)
    tally = torch.zeros(4, dtype=torch.int64, device=dev)
    mirror = torch.full((n, k), -1, dtype=torch.int32, device=dev)
    st._engine.ops.join(rs.device_tables(), st._table, n, k, st._csr, st._max_indeg, out, tally, None, uc,
                        peers=(mirror.data_ptr(),) if peers else ())
    rows, _, o_uc, comps, changed = native.local_join(tab, table)
    assert np.array_equal(uc.cpu().numpy(), o_uc), "join |U| differs"
    assert np.array_equal(out.cpu().numpy(), rows), "join rows differ"
    assert tally.cpu().tolist()[:3] == [comps, changed, 0]
    if peers:
        assert torch.equal(mirror, out), "peer stores differ"
    print(f"join n={n} d={d} K={k} max_indeg={st._max_indeg}: ok", flush=True)


def main():
    torch.cuda.set_device(0)
    # init (device draws + row sort), CSR, two rounds, FCC, batch_scores, exact K-NN
    n, d, k, seed = 4000, 20, 20, 0
    pts = port.experiment_points(n, d, seed)
    rs = b2.KlRankingSystem(pts, validate=False)
    cfg = b2.DescentConfig(k=k, seed=seed)
    st = b2.init_random_kout(b2.Dataset(pts), rs, cfg, b2.derive_rng(seed, 2))
    tab = native.Tables(pts)
    init = native.sort_rows(tab, port.random_kout_draws(n, k, port.substream(seed, port.TAG_INIT)))
    assert np.array_equal(st.friends, init), "init differs"
    for _ in range(2):
        st, _stats = b2.run_round(st, rs, cfg)
    assert rs.batch_scores(5, np.arange(0, n, 7)).shape == (len(range(0, n, 7)),)
    q = np.arange(0, n, 131)
    assert np.array_equal(b2.exact_rows(rs, q, k), native.exact_rows(tab, q, k)), "exact K-NN differs"
    print("init / rounds / fcc / batch_scores / exact: ok", flush=True)
    # every size class, the hub (global-table) class, the peer stores
    check_join(6000, 20, 20, [(7, 1500), (11, 600), (13, 800), (17, 160), (19, 60), (23, 40)], peers=True)
    check_join(3000, 8, 64, [(7, 700), (11, 300)])
    check_join(3000, 7, 12, [(5, 900), (9, 200)])
    check_join(2500, 50, 30, [(3, 800), (8, 250), (21, 90)])  # the 160-byte Q23 rows
    check_join(3000, 7, 2, [(5, 1200), (9, 300)])  # K = 2: the global-memory class with a table below 2^15 slots
    os.environ["KNND_Q23"] = "0"  # the fp32 screen rows (specialised and generic widths)
    try:
        check_join(4000, 20, 20, [(7, 1200), (11, 500), (13, 150), (17, 60)], peers=True)
        check_join(2000, 6, 10, [(5, 500)])
    finally:
        del os.environ["KNND_Q23"]
    # the Euclidean path
    rng = np.random.default_rng(5)
    v = rng.normal(size=(3000, 12))
    ers = b2.EuclideanRankingSystem(v)
    ecfg = b2.DescentConfig(k=10, seed=1)
    est = b2.init_random_kout(b2.Dataset(v), ers, ecfg, b2.derive_rng(1, 2))
    b2.run_round(est, ers, ecfg)
    b2.exact_rows(ers, np.arange(0, 3000, 97), 10)
    torch.cuda.synchronize()
    report_checks()
    print("SANITIZE_OK", flush=True)


def report_checks():
    """Checked build / guarded workspaces: zero failed bounds checks, zero guard bytes touched."""
    import ctypes as C

    from paper_2202_00517_b200 import _lib
    from paper_2202_00517_b200.engine import check_guards

    if os.environ.get("KNND_GUARD") == "1":
        bad = check_guards()
        print(f"guard bytes overwritten: {bad}", flush=True)
        assert bad == 0, f"{bad} workspace guard bytes were overwritten"
    if os.environ.get("KNND_LIBRARY") == "checked":
        cnt, first = C.c_ulonglong(0), C.c_ulonglong(0)
        # positive control first: a kernel whose checks fail on purpose is seen
        lib = _lib.load()
        lib.knnd_internal_check_selftest.argtypes = [C.c_void_p]
        assert lib.knnd_internal_check_selftest(None) == 0
        assert lib.knnd_check_failures(C.byref(cnt), C.byref(first)) == 0, _lib.last_error()
        print(f"self-test: {cnt.value} failures reported, first at {first.value}", flush=True)
        assert cnt.value == 2 and first.value // 100000 == 9, (cnt.value, first.value)
        rc = _lib.load().knnd_check_failures(C.byref(cnt), C.byref(first))
        assert rc == 0, _lib.last_error()
        print(f"device bounds checks failed: {cnt.value} (first at file*100000+line {first.value})", flush=True)
        assert cnt.value == 0, f"{cnt.value} device bounds checks failed, first at {first.value}"


if __name__ == "__main__":
    main()
