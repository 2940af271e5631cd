"""CPU pinning of the allocate_budget checkers (allocator.hpp:76-186): the C restatement
(or_allocate) against the reference itself (ref_allocate) bit for bit on random clusters,
and the Python restatement used for table/forest sets against both — plus the
reference's own allocator tests (tests/test_controller.cpp:237-283) on the Python one."""
import numpy as np
import pytest

from oracle.oracle import oracle_allocate, ref_allocate
from paper_2605_21427_b200 import workloads
from tests.helpers import alloc_setup, ladder, py_allocate, py_steps

K_ALPHA, K_BETA = 1.05, 345.0  # kCoeffs of tests/test_controller.cpp:12


def _same(a, b):
    for k in ("node_budget", "total", "all_sat", "status"):
        assert np.array_equal(np.asarray(a[k]).view(np.uint8), np.asarray(b[k]).view(np.uint8)), k


@pytest.mark.parametrize("margin,quantum", [(0.0, 25.0), (0.02, 25.0), (0.008, 10.0),
                                            (0.0, 7.3)])
def test_oracle_matches_reference(oracle, reference, margin, quantum):
    s = alloc_setup(oracle)
    prob = workloads.alloc_problems(1500, 31, s["t_max"], s["p_max"], s["gpu"], s["coeffs"])
    args = (s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"], quantum, margin, prob)
    a = oracle_allocate(oracle, *args)
    b = ref_allocate(reference, *args)
    _same(a, b)
    assert (a["status"] == 0).mean() > 0.9 and (a["status"] == 2).any()
    assert 0.1 < a["all_sat"][a["status"] == 0].mean() < 0.95


def test_large_clusters_oracle_matches_reference(oracle, reference):
    s = alloc_setup(oracle)
    prob = workloads.alloc_problems(60, 5, s["t_max"], s["p_max"], s["gpu"], s["coeffs"],
                                    max_nodes=80)
    args = (s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"], 25.0, 0.02, prob)
    _same(oracle_allocate(oracle, *args), ref_allocate(reference, *args))


def test_python_restatement_matches_oracle(oracle):
    s = alloc_setup(oracle)
    k = s["coeffs"]
    unit = k.alpha * 4 * s["gpu"].min_cap_watts + k.beta_watts
    prob = workloads.alloc_problems(120, 9, s["t_max"], s["p_max"], s["gpu"], k)
    want = oracle_allocate(oracle, s["profiles"], s["gpu"], k, s["caps"], s["batches"], 25.0,
                           0.02, prob)
    cache = {}
    for p in range(120):
        lo, hi = prob["off"][p], prob["off"][p + 1]
        steps = []
        for m, d in zip(prob["model"][lo:hi], prob["dp"][lo:hi]):
            if (m, d) not in cache:
                prof = s["profiles"][m]
                pts = workloads.grid_points(s["caps"], s["batches"], [prof.deploy_tp],
                                            [prof.deploy_ep], [d])
                T, P, _ = oracle.eval(prof, s["gpu"], pts)
                cache[m, d] = py_steps(T, P, pts["dp"], k.alpha, k.beta_watts, 0.02)
            steps.append(cache[m, d])
        r = py_allocate(steps, prob["dp"][lo:hi], prob["target"][lo:hi], prob["budget"][p], unit)
        if r is None:
            assert want["status"][p] == 2
            continue
        bud, tot, sat = r
        assert want["status"][p] == 0
        assert np.array_equal(np.array(bud), want["node_budget"][lo:hi])
        assert tot == want["total"][p] and sat == bool(want["all_sat"][p])


def _ladder_steps(n, lo, hi):
    pts, T, P = ladder(n, lo, hi)
    return pts, T, P, py_steps(T, P, pts["dp"], K_ALPHA, K_BETA)


def test_reference_case_one_node_takes_budget_up_to_useful_max():
    """tests/test_controller.cpp:237-254 on the Python restatement."""
    _, _, P, st = _ladder_steps(8, 400.0, 1200.0)
    unit = K_ALPHA * 4 * 100.0 + K_BETA  # GpuSpec{} min_cap_watts = 100 (types.hpp:29)
    max_useful = K_ALPHA * 4 * P[-1] + K_BETA
    bud, tot, _ = py_allocate([st], [1], [3000.0], max_useful + 500.0, unit)
    assert max_useful <= bud[0] <= max_useful + 3 * 25.0
    assert tot <= max_useful + 500.0


def test_reference_case_identical_nodes_split_evenly():
    """tests/test_controller.cpp:256-271."""
    _, _, _, st = _ladder_steps(120, 400.0, 2000.0)
    unit = K_ALPHA * 4 * 100.0 + K_BETA
    bud, _, _ = py_allocate([st, st], [1, 1], [1800.0, 1800.0], 3000.0, unit)
    assert abs(bud[0] - bud[1]) <= 6 * 25.0 and bud[0] + bud[1] <= 3000.0


def test_reference_case_infeasible_floor():
    """tests/test_controller.cpp:273-283."""
    _, _, _, st = _ladder_steps(4, 400.0, 1000.0)
    unit = K_ALPHA * 4 * 100.0 + K_BETA
    assert py_allocate([st] * 3, [1, 1, 1], [0.0] * 3, 100.0, unit) is None
