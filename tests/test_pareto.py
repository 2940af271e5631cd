"""CPU pinning of the build_frontier / evaluate_regime checkers (pareto.hpp): the C
restatement against the reference build on the reference's own test cases
(tests/test_analysis.cpp:26-88), random point sets with exact ties, and every
profile x regime of the pareto command (commands.hpp:205-220)."""
import numpy as np
import pytest

from oracle.oracle import (oracle_build_frontier, ref_build_frontier, ref_evaluate_regime,
                           ref_verify_dominance)
from paper_2605_21427_b200.abi import POINT_DT
from paper_2605_21427_b200.pareto import default_regimes, regime_points

K_CAPS = [150.0, 200.0, 250.0, 300.0, 350.0, 400.0]
K_BATCHES = [1, 4, 8, 16, 32, 64]
K_TPS = [1, 2, 4]


def fp_arrays(items):
    """items: (throughput, efficiency, cap, batch) -> FrontierPoint arrays (fp() of
    tests/test_analysis.cpp:17-19: tp 2, ep 1, dp 1)."""
    pts = np.zeros(len(items), POINT_DT)
    for i, (_, _, cap, batch) in enumerate(items):
        pts[i] = (cap, batch, 2, 1, 1)
    thr = np.array([x[0] for x in items], np.float64)
    eff = np.array([x[1] for x in items], np.float64)
    return pts, thr, eff


def random_set(rng, n, tie_levels=None):
    if tie_levels:
        thr = rng.choice(rng.uniform(10.0, 1000.0, tie_levels), n)
        eff = rng.choice(rng.uniform(0.1, 2.0, tie_levels), n)
    else:
        thr = rng.uniform(10.0, 1000.0, n)
        eff = rng.uniform(0.1, 2.0, n)
    pts = np.zeros(n, POINT_DT)
    pts["cap_watts"] = rng.choice(K_CAPS, n)
    pts["batch"] = rng.choice(K_BATCHES, n)
    pts["tp"], pts["ep"], pts["dp"] = 2, 1, 1
    return pts, thr, eff


def check_same(oracle, reference, pts, thr, eff):
    idx = oracle_build_frontier(oracle, pts, thr, eff)
    rp, rt, re = ref_build_frontier(reference, pts, thr, eff)
    assert np.array_equal(pts[idx], rp)
    assert np.array_equal(thr[idx], rt) and np.array_equal(eff[idx], re)
    return idx


def test_reference_cases(oracle, reference):
    for items, want in [([(100.0, 0.5, 300.0, 8)], [0]),
                        ([(100.0, 0.5, 300.0, 8), (90.0, 0.4, 300.0, 8)], [0]),
                        ([(100.0, 0.5, 350.0, 8), (100.0, 0.5, 250.0, 8)], [1]),
                        ([(100.0, 0.5, 300.0, 8), (200.0, 0.4, 300.0, 8),
                          (300.0, 0.2, 300.0, 8)], [0, 1, 2])]:
        assert check_same(oracle, reference, *fp_arrays(items)).tolist() == want


@pytest.mark.parametrize("ties", [None, 3, 8])
def test_random_sets(oracle, reference, ties):
    rng = np.random.default_rng(99 if ties is None else ties)
    for _ in range(150):
        n = int(rng.integers(1, 120))
        pts, thr, eff = random_set(rng, n, ties)
        idx = check_same(oracle, reference, pts, thr, eff)
        # sorted by throughput with strictly decreasing efficiency (test_analysis.cpp:65-69)
        assert np.all(np.diff(thr[idx]) > 0) and np.all(np.diff(eff[idx]) < 0)


def test_negative_and_zero_efficiency(oracle, reference):
    items = [(100.0, -2.0, 300.0, 8), (90.0, -0.5, 250.0, 4), (80.0, 0.0, 200.0, 1),
             (70.0, -0.0, 150.0, 1), (60.0, 1.0, 150.0, 16)]
    check_same(oracle, reference, *fp_arrays(items))


def test_regimes_every_profile(oracle, reference, bundle):
    profs, gpu, coeffs = bundle
    for p in profs:
        for reg in default_regimes():
            pts = regime_points(reg, p, K_CAPS, K_BATCHES, K_TPS)
            T, P, err = oracle.eval(p, gpu, pts)
            assert not err.any()
            th = pts["dp"] * T
            ef = th / (pts["dp"] * (coeffs.alpha * 4 * P + coeffs.beta_watts))
            idx = oracle_build_frontier(oracle, pts, th, ef)
            rp, rt, re = ref_evaluate_regime(reference, reg.name, p, gpu, coeffs, K_CAPS,
                                             K_BATCHES, K_TPS)
            assert np.array_equal(pts[idx], rp), (p.name, reg.name)
            assert np.array_equal(th[idx], rt) and np.array_equal(ef[idx], re)


def test_verify_dominance_reference_cases(reference):
    dom, cov = ref_verify_dominance(reference, [100.0, 200.0, 300.0], [0.5, 0.4, 0.2],
                                    [100.0, 200.0, 300.0], [0.5, 0.4, 0.2])
    assert dom and cov.all()
    dom, cov = ref_verify_dominance(reference, [100.0], [0.5], [120.0], [0.3])
    assert not dom and cov.tolist() == [False]
