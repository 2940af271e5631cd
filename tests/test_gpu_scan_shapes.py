"""Pair-scan partition shapes on the B200: grid sizes that are not a multiple of the
2,048-point chunk (and one above 65,536 points: 64-bit packed keys), query counts from a
handful (cell mode, few query slots per warp) through tens of thousands (stream-K), with
QoS-only, budget-only and QoS+budget classes in one batch. Every answer is checked
against the C oracle (itself pinned to the reference) on a stratified sample, and the
whole batch must equal the same plan's prefix-min decide path."""
import numpy as np
import pytest

from paper_2605_21427_b200 import workloads
from paper_2605_21427_b200.wattserve import AnalyticModel, Grid, Plan

pytestmark = pytest.mark.gpu

SHAPES = [
    # (caps, batches, tps) -> n
    (np.linspace(120.0, 390.0, 23), np.arange(1, 98), [1, 2, 4]),        # 6,693 points
    (np.linspace(100.0, 400.0, 61), np.arange(1, 257), [1, 2, 4, 8]),    # 62,464
    (np.linspace(100.0, 400.0, 67), np.arange(1, 257), [1, 2, 4, 8]),    # 68,608 (wide keys)
]


@pytest.mark.parametrize("shape", range(len(SHAPES)))
@pytest.mark.parametrize("nq", [37, 3_000, 40_000])
def test_scan_shapes_vs_oracle(ctx, oracle, shape, nq):
    cfg = workloads.cfg2()
    caps, batches, tps = SHAPES[shape]
    pts = workloads.grid_points(caps, batches, tps)
    plan = Plan(AnalyticModel(ctx, cfg["profile"], cfg["gpu"]), Grid(ctx, pts), cfg["coeffs"])
    th, pn, _ = plan.scores()
    q = workloads.gen_queries(nq, 7 + shape, float(th.max()), "mixed",
                              budget=(float(pn.min()) * 0.9, float(pn.max()) * 1.1))
    # a third of the QoS queries without a budget: classes A, B and C in one batch
    q["has_budget"][::3] = 0
    idx, rs = plan.select(q)
    stats = plan.stats()
    assert stats[:3].sum() > 0
    T, P, _ = oracle.eval(cfg["profile"], cfg["gpu"], pts)
    # every query up to 3,000, a stratified sample of larger batches
    sub = np.unique(np.concatenate([np.arange(0, nq, max(1, nq // 3_000)), [nq - 1]]))
    oi, orr, rc = oracle.select(pts, T, P, cfg["coeffs"], q[sub])
    assert rc == 0
    assert np.array_equal(idx[sub], oi) and np.array_equal(rs[sub], orr)
    plan.set_decide("prefix")
    idx2, rs2 = plan.select(q)
    plan.set_decide("scan")
    assert np.array_equal(idx2, idx) and np.array_equal(rs2, rs)
