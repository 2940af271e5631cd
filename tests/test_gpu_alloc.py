"""allocate_budget (allocator.hpp:76-186) on the B200 through libpals_gpu.so: batched
random clusters bit for bit against the C restatement and the reference build; the
reference's own allocator tests (tests/test_controller.cpp:237-283) on table sets;
table and forest scorers against the Python restatement over oracle scores; error
statuses; clusters larger than the per-thread node cache."""
import os

import numpy as np
import pytest

from oracle.oracle import oracle_allocate, oracle_forest_predict, ref_allocate
from paper_2605_21427_b200 import workloads
from paper_2605_21427_b200.abi import Coeffs, GpuSpec
from paper_2605_21427_b200.forest import Bundle, make_forest_model
from paper_2605_21427_b200.wattserve import (Allocator, AnalyticModel, ConfigError, TableModel,
                                             allocate_budget)
from tests.helpers import alloc_setup, ladder, py_allocate, py_steps, table_view

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
K = Coeffs(1.05, 345.0)  # kCoeffs of tests/test_controller.cpp:12
GPU_DEFAULT = GpuSpec(40.0, 100.0, 400.0, 1.0)  # GpuSpec{} (types.hpp:27-31)


def _same(a, b, ok_only_nodes=False):
    for k in ("total", "all_sat", "status"):
        assert np.array_equal(np.asarray(a[k]).view(np.uint8), np.asarray(b[k]).view(np.uint8)), k
    assert np.array_equal(a["node_budget"].view(np.uint64), b["node_budget"].view(np.uint64))


@pytest.fixture(scope="module")
def setup(oracle):
    return alloc_setup(oracle)


@pytest.mark.parametrize("margin,quantum", [(0.0, 25.0), (0.02, 25.0), (0.008, 10.0),
                                            (0.02, 7.3)])
def test_random_clusters_vs_oracle_and_reference(ctx, oracle, reference, setup, margin, quantum):
    s = setup
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    al = Allocator(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                   max_dp=3, selection_margin=margin)
    prob = workloads.alloc_problems(4000, 17, s["t_max"], s["p_max"], s["gpu"], s["coeffs"])
    got = al.allocate(prob["off"], prob["model"], prob["dp"], prob["target"], prob["budget"],
                      quantum)
    args = (s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"], quantum, margin, prob)
    _same(got, oracle_allocate(oracle, *args))
    _same(got, ref_allocate(reference, *args))
    assert (got["status"] == 2).any() and (got["status"] == 0).mean() > 0.9


def test_large_clusters_spill_path(ctx, oracle, setup):
    """Clusters of up to 100 nodes: node state beyond the 32-node local cache."""
    s = setup
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    al = Allocator(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                   max_dp=3, selection_margin=0.02)
    prob = workloads.alloc_problems(300, 3, s["t_max"], s["p_max"], s["gpu"], s["coeffs"],
                                    max_nodes=100)
    assert np.diff(prob["off"]).max() > 32
    got = al.allocate(prob["off"], prob["model"], prob["dp"], prob["target"], prob["budget"])
    _same(got, oracle_allocate(oracle, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                               s["batches"], 25.0, 0.02, prob))


def test_step_tables_match_restatement(ctx, oracle, setup):
    s = setup
    k = s["coeffs"]
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    al = Allocator(ctx, models, s["profiles"], s["gpu"], k, s["caps"], s["batches"], max_dp=3,
                   selection_margin=0.02)
    for m, prof in enumerate(s["profiles"]):
        for d in (1, 2, 3):
            pts = workloads.grid_points(s["caps"], s["batches"], [prof.deploy_tp],
                                        [prof.deploy_ep], [d])
            T, P, _ = oracle.eval(prof, s["gpu"], pts)
            want = np.array(py_steps(T, P, pts["dp"], k.alpha, k.beta_watts, 0.02))
            pw, th = al.steps(m, d)
            assert np.array_equal(pw, want[:, 0]) and np.array_equal(th, want[:, 1])


def _ladder_alloc(ctx, n, lo, hi, names=None, n_sets=1):
    pts, T, P = ladder(n, lo, hi)
    tab = TableModel(ctx, pts, T, P)
    return Allocator.from_sets(ctx, [(tab, pts)] * n_sets, GPU_DEFAULT, K, names=names), P


def test_reference_case_one_node_takes_budget_up_to_useful_max(ctx):
    """tests/test_controller.cpp:237-254."""
    al, P = _ladder_alloc(ctx, 8, 400.0, 1200.0)
    max_useful = K.alpha * 4 * P[-1] + K.beta_watts
    res = allocate_budget(al, [(0, 1, 3000.0)], max_useful + 500.0, 25.0)
    assert max_useful <= res.node_budgets_w[0] <= max_useful + 3 * 25.0
    assert res.total_allocated_w <= max_useful + 500.0


def test_reference_case_identical_nodes_split_evenly(ctx):
    """tests/test_controller.cpp:256-271."""
    al, _ = _ladder_alloc(ctx, 120, 400.0, 2000.0, n_sets=2)
    res = allocate_budget(al, [(0, 1, 1800.0), (1, 1, 1800.0)], 3000.0, 25.0)
    b = res.node_budgets_w
    assert abs(b[0] - b[1]) <= 6 * 25.0 and b[0] + b[1] <= 3000.0


def test_reference_case_infeasible_floor_names_nodes(ctx):
    """tests/test_controller.cpp:273-283: config_error naming the starved nodes."""
    al, _ = _ladder_alloc(ctx, 4, 400.0, 1000.0, names=["starved"])
    with pytest.raises(ConfigError, match="starved"):
        allocate_budget(al, [(0, 1, 0.0)] * 3, 100.0)
    with pytest.raises(ConfigError, match="no nodes"):
        allocate_budget(al, [], 1000.0)


def test_table_sets_vs_restatement(ctx):
    """Random TableScorer sets (duplicates: first match wins) and mixed node dp."""
    rng = np.random.default_rng(41)
    unit = K.alpha * 4 * GPU_DEFAULT.min_cap_watts + K.beta_watts
    for case in range(6):
        sets, py_sets = [], []
        for _ in range(4):
            n = int(rng.integers(1, 200))
            pts, T, P = ladder(n, 100.0, float(rng.uniform(500, 3000)))
            pts["dp"] = rng.integers(1, 4, n)
            dup = rng.integers(0, n, n // 5)
            pts = np.concatenate([pts, pts[dup]])
            T = np.concatenate([T, T[dup] * 1.5])
            P = np.concatenate([P, P[dup] * 0.5])
            tab = TableModel(ctx, pts, T, P)
            cand = pts[rng.permutation(len(pts))[: max(1, len(pts) // 2)]]
            sets.append((tab, cand))
            Ts, Ps, canon = table_view(pts, T, P)
            lut = {tuple(p): i for i, p in reversed(list(enumerate(pts.tolist())))}
            ix = np.array([lut[tuple(p)] for p in cand.tolist()])
            py_sets.append(py_steps(Ts[ix], Ps[ix], cand["dp"], K.alpha, K.beta_watts, 0.01))
        al = Allocator.from_sets(ctx, sets, GPU_DEFAULT, K, selection_margin=0.01)
        for st, py in zip(range(4), py_sets):
            pw, th = al.steps(st)
            assert np.array_equal(pw, np.array([x[0] for x in py])), case
            assert np.array_equal(th, np.array([x[1] for x in py])), case
        nn = rng.integers(1, 7, 50)
        off = np.concatenate([[0], np.cumsum(nn)])
        node_set = rng.integers(0, 4, off[-1]).astype(np.int32)
        node_dp = rng.integers(1, 3, off[-1]).astype(np.int32)
        tgt = rng.uniform(100.0, 4000.0, off[-1])
        budget = rng.uniform(0.8, 4.0, 50) * nn * 1500.0
        got = al.allocate(off, node_set, node_dp, tgt, budget, 25.0)
        for p in range(50):
            lo, hi = off[p], off[p + 1]
            r = py_allocate([py_sets[j] for j in node_set[lo:hi]], node_dp[lo:hi], tgt[lo:hi],
                            budget[p], unit)
            if r is None:
                assert got["status"][p] == 2
                continue
            assert got["status"][p] == 0
            assert np.array_equal(np.array(r[0]), got["node_budget"][lo:hi]), (case, p)
            assert r[1] == got["total"][p] and r[2] == bool(got["all_sat"][p])


def test_forest_sets_vs_restatement(ctx, oracle, bundle):
    """predictor_scorer nodes: forest predictions through the product form."""
    _, gpu, coeffs = bundle
    b = Bundle.load_npz(os.path.join(ROOT, "paper_2605_21427_b200", "data",
                                     "predictor_small.npz"))
    s = workloads.cfg4_setup()
    profs = [p for p in s["profiles"] if bytes(p.name).split(b"\0")[0].decode() in b.model_ids]
    ids = [bytes(p.name).split(b"\0")[0].decode() for p in profs]
    models = [make_forest_model(ctx, b, mid) for mid in ids]
    al = Allocator(ctx, models, profs, gpu, coeffs, s["caps"], s["batches"], max_dp=2,
                   selection_margin=0.02)
    steps = {}
    for m, (prof, mid) in enumerate(zip(profs, ids)):
        for d in (1, 2):
            pts = workloads.grid_points(s["caps"], s["batches"], [prof.deploy_tp],
                                        [prof.deploy_ep], [d])
            T, P, _ = oracle_forest_predict(oracle, b, mid, pts)
            steps[m, d] = py_steps(T, P, pts["dp"], coeffs.alpha, coeffs.beta_watts, 0.02)
            pw, th = al.steps(m, d)
            assert np.array_equal(pw, np.array([x[0] for x in steps[m, d]]))
    rng = np.random.default_rng(5)
    nn = rng.integers(1, 6, 80)
    off = np.concatenate([[0], np.cumsum(nn)])
    nm = rng.integers(0, len(profs), off[-1]).astype(np.int32)
    nd = rng.integers(1, 3, off[-1]).astype(np.int32)
    tgt = rng.uniform(200.0, 2500.0, off[-1])
    budget = rng.uniform(1.0, 3.0, 80) * nn * 1200.0
    got = al.allocate(off, nm, nd, tgt, budget)
    unit = coeffs.alpha * 4 * gpu.min_cap_watts + coeffs.beta_watts
    for p in range(80):
        lo, hi = off[p], off[p + 1]
        r = py_allocate([steps[m, d] for m, d in zip(nm[lo:hi], nd[lo:hi])], nd[lo:hi],
                        tgt[lo:hi], budget[p], unit)
        if r is None:
            assert got["status"][p] == 2
            continue
        assert np.array_equal(np.array(r[0]), got["node_budget"][lo:hi]), p
        assert r[1] == got["total"][p]


def test_error_statuses(ctx, setup):
    s = setup
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    al = Allocator(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                   max_dp=2)
    off = np.array([0, 0, 1, 2, 3, 4])  # empty problem, then bad model, dp 0, dp 3, fine
    got = al.allocate(off, [99, 0, 0, 1], [1, 0, 3, 1], [500.0] * 4, [1e5] * 5)
    assert got["status"].tolist() == [2, 2, 2, 5, 0]
    # an analytic model whose deployment tp is not calibrated rejects every candidate
    bad = [s["profiles"][0]]
    bad_prof = type(bad[0]).from_buffer_copy(bad[0])
    bad_prof.deploy_tp = 3
    al2 = Allocator(ctx, [models[0]], [bad_prof], s["gpu"], s["coeffs"], s["caps"],
                    s["batches"], max_dp=1)
    got = al2.allocate([0, 1, 2], [0, 0], [1, 1], [1.0, 1.0], [1e5, 10.0])
    assert got["status"].tolist() == [2, 2]  # scorer config_error; floors checked first
    with pytest.raises(Exception):
        al.allocate([0, 1], [0], [1], [1.0], [1e5], quantum_w=0.0)
