"""build_frontier / evaluate_regime (pareto.hpp) on the B200: explicit point sets with
exact ties against the C restatement and the reference build, every profile x regime
of the pareto command against the reference, dense grids (65,536 narrow-key and
589,824 wide-key points) against the restatement."""
import numpy as np
import pytest

from oracle.oracle import oracle_build_frontier, ref_build_frontier, ref_evaluate_regime
from paper_2605_21427_b200 import workloads
from paper_2605_21427_b200.pareto import (FrontierPoint, build_frontier, default_regimes,
                                          evaluate_regime, frontier_indices, peak_efficiency,
                                          regime_by_name, verify_dominance)
from paper_2605_21427_b200.wattserve import AnalyticModel, ConfigError, Grid, Plan
from tests.test_pareto import K_BATCHES, K_CAPS, K_TPS, fp_arrays, random_set

pytestmark = pytest.mark.gpu


def _same_points(pts, idx_a, idx_b, thr, eff):
    assert np.array_equal(pts[idx_a], pts[idx_b])
    assert np.array_equal(thr[idx_a], thr[idx_b]) and np.array_equal(eff[idx_a], eff[idx_b])


def test_reference_cases_gpu(ctx):
    f = build_frontier([FrontierPoint((300.0, 8, 2, 1, 1), 100.0, 0.5)], ctx)
    assert len(f) == 1 and f[0].throughput_tps == 100.0
    f = build_frontier([FrontierPoint((300.0, 8, 2, 1, 1), 100.0, 0.5),
                        FrontierPoint((300.0, 8, 2, 1, 1), 90.0, 0.4)], ctx)
    assert len(f) == 1 and f[0].throughput_tps == 100.0
    f = build_frontier([FrontierPoint((350.0, 8, 2, 1, 1), 100.0, 0.5),
                        FrontierPoint((250.0, 8, 2, 1, 1), 100.0, 0.5)], ctx)
    assert len(f) == 1 and f[0].point[0] == 250.0
    f = build_frontier([FrontierPoint((300.0, 8, 2, 1, 1), t, e)
                        for t, e in [(100.0, 0.5), (200.0, 0.4), (300.0, 0.2)]], ctx)
    dom, wit = verify_dominance(f, f)
    assert dom and not wit
    a = build_frontier([FrontierPoint((300.0, 8, 2, 1, 1), 100.0, 0.5)], ctx)
    b = build_frontier([FrontierPoint((300.0, 8, 2, 1, 1), 120.0, 0.3)], ctx)
    dom, wit = verify_dominance(a, b)
    assert not dom and len(wit) == 1 and wit[0].throughput_tps == 120.0
    with pytest.raises(ConfigError):
        build_frontier([], ctx)
    with pytest.raises(ConfigError, match="valid: sw-only, hw-only, hw-sw, joint"):
        regime_by_name("everything")


@pytest.mark.parametrize("ties", [None, 3, 8])
def test_random_sets_vs_oracle_and_reference(ctx, oracle, reference, ties):
    rng = np.random.default_rng(1000 + (ties or 0))
    for case in range(80):
        n = int(rng.integers(1, 400))
        pts, thr, eff = random_set(rng, n, ties)
        if case % 4 == 0:  # negative / zero efficiencies exercise best_eff = -1.0
            eff = eff - 1.5
        got = frontier_indices(pts, thr, eff, ctx)
        want = oracle_build_frontier(oracle, pts, thr, eff)
        _same_points(pts, got, want, thr, eff)
        rp, rt, re = ref_build_frontier(reference, pts, thr, eff)
        assert np.array_equal(pts[got], rp) and np.array_equal(thr[got], rt), case


def test_regimes_every_profile_vs_reference(ctx, reference, bundle):
    profs, gpu, coeffs = bundle
    for p in profs:
        fr = {}
        for reg in default_regimes():
            f = evaluate_regime(reg, p, gpu, coeffs, K_CAPS, K_BATCHES, K_TPS, ctx)
            rp, rt, re = ref_evaluate_regime(reference, reg.name, p, gpu, coeffs, K_CAPS,
                                             K_BATCHES, K_TPS)
            assert [x.point for x in f] == [tuple(r) for r in rp.tolist()], (p.name, reg.name)
            assert np.array_equal([x.throughput_tps for x in f], rt)
            assert np.array_equal([x.efficiency_tpj for x in f], re)
            fr[reg.name] = f
        # tests/test_analysis.cpp:90-104: the joint frontier covers the single-knob ones
        assert verify_dominance(fr["joint"], fr["hw-only"])[0]
        assert verify_dominance(fr["joint"], fr["sw-only"])[0]
        assert peak_efficiency(fr["joint"]) >= peak_efficiency(fr["hw-sw"])


def test_wide_random_values_vs_oracle(ctx, oracle):
    """A large explicit set (wide keys, > 65,536 points) with a long frontier."""
    rng = np.random.default_rng(77)
    n = 200_000
    pts, thr, eff = random_set(rng, n, None)
    eff = 3000.0 / thr + rng.uniform(-0.5, 0.5, n)  # anti-correlated: frontier of many points
    thr[rng.integers(0, n, 5000)] = thr[rng.integers(0, n, 5000)]  # exact throughput ties
    got = frontier_indices(pts, thr, eff, ctx)
    want = oracle_build_frontier(oracle, pts, thr, eff)
    _same_points(pts, got, want, thr, eff)
    assert len(got) > 50


@pytest.mark.parametrize("which", ["cfg2", "cfg3x"])
def test_dense_grid_frontier_vs_oracle(ctx, oracle, which):
    c = workloads.cfg2() if which == "cfg2" else workloads.cfg3_extended()
    pts = c["points"]
    plan = Plan(AnalyticModel(ctx, c["profile"], c["gpu"]), Grid(ctx, pts), c["coeffs"])
    got = plan.frontier()
    T, P, _ = oracle.eval(c["profile"], c["gpu"], pts)
    th = pts["dp"] * T
    ef = th / (pts["dp"] * (c["coeffs"].alpha * 4 * P + c["coeffs"].beta_watts))
    want = oracle_build_frontier(oracle, pts, th, ef)
    _same_points(pts, got, want, th, ef)
    assert len(got) >= 1
