"""The Q23 screen's error model, checked on the host: a numpy emulation of
knnd_kl_q23_prepare (prep.cu) and of screen_row_q23 / q23_weights (join_impl.cuh) —
the same quantisation, the same fp32 weights, the same four FMA chains — must
stay within the bound the join's thresholds and certification rely on:

    | v - 2^-23 (ce + sum_j x_j Lmax_j) |  <=  band * v + slack,
    band = (ceil(NQ / 4) + 6) 2^-24,  slack = 2^-23 * (1/2) sum_j x_j h_j (1 + 2^-9)

for every (anchor, candidate) pair, ce the fp64 cross entropy the reference
ranks by (similarity.py:101-106).  The device kernels are checked against the
oracle's tables (tests/test_q23.py); this pins the analysis itself."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import port

F32 = np.float32


def _fma32(a, b, c):
    # fp32 fused multiply-add: the product of two fp32 values is exact in fp64
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(F32)


def _quantise(logs):
    hi, lo = logs.max(axis=0), logs.min(axis=0)
    h = (hi - lo) / 8388607.0
    with np.errstate(divide="ignore", invalid="ignore"):
        q = np.where(h > 0, np.rint((hi - logs) / np.where(h > 0, h, 1.0)), 0.0)
    return np.clip(q, 0, 8388607).astype(np.int64), h, hi


@pytest.mark.parametrize("n,d,seed", [(4000, 20, 0), (3000, 10, 1), (2000, 5, 2), (1500, 16, 3), (1200, 50, 4)])
def test_q23_screen_error_model(n, d, seed):
    pts = port.experiment_points(n, d, seed)
    logs = np.log(pts)
    q, h, hi = _quantise(logs)
    row_bytes = (3 * d + 15) // 16 * 16 if 3 * d <= 64 else 160
    nq = row_bytes // 3
    band = ((nq + 3) // 4 + 6) * 2.0 ** -24
    # denormal floats whose bit pattern is q: q * 2^-149 (exact in fp64)
    Fq = (q.astype(np.float64) * 2.0 ** -149)
    assert np.array_equal(Fq.astype(F32).astype(np.float64), Fq)  # representable: the byte permute builds them
    h32 = h.astype(F32)
    rng = np.random.default_rng(seed)
    anchors = rng.choice(n, 40, replace=False)
    worst = 0.0
    for x in anchors:
        x32 = pts[x].astype(F32)
        w = ((x32 * h32).astype(F32) * F32(2.0 ** 126)).astype(F32)  # q23_weights: (x * h) * 2^126
        s = F32(0)
        for j in range(d):
            s = _fma32(np.abs(w[j]), F32(2.0 ** -75), s)
        slack = float(s) * 2.0 ** -75 * (1 + 2.0 ** -9) + 1e-36
        # screen_row_q23: chain j & 3 accumulates entry j; (a0 + a1) + (a2 + a3)
        a = [np.zeros(n, F32) for _ in range(4)]
        for j in range(d):
            a[j & 3] = _fma32(np.full(n, w[j], F32), Fq[:, j].astype(F32), a[j & 3])
        v = ((a[0] + a[1]).astype(F32) + (a[2] + a[3]).astype(F32)).astype(F32).astype(np.float64)
        ce = -(pts[x][None, :] * logs).sum(axis=1)                      # fp64 cross entropy of every candidate
        exact = 2.0 ** -23 * (ce + (pts[x] * hi).sum())
        err = np.abs(v - exact)
        bound = band * v + slack
        assert (err <= bound).all(), (x, float((err / bound).max()))
        worst = max(worst, float((err / bound).max()))
    assert worst < 1.0


def test_q23_values_order_like_cross_entropy():
    """Screened values differ from the cross entropy by a per-anchor constant and
    scale: candidates further apart than the bound keep their order."""
    n, d = 3000, 20
    pts = port.experiment_points(n, d, 5)
    logs = np.log(pts)
    q, h, hi = _quantise(logs)
    x = 17
    v = 2.0 ** -23 * (q * (pts[x] * h)[None, :]).sum(axis=1)
    ce = -(pts[x][None, :] * logs).sum(axis=1)
    slack = 2.0 ** -23 * 0.5 * (pts[x] * h).sum()
    order = np.argsort(ce)
    gaps = np.diff(v[order])
    assert (gaps > -2 * slack * (1 + 1e-6)).all()
