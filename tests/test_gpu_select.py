"""K1 parity on the B200: grid evaluation and batched select_config through
libpals_gpu.so, bit-exact against the reference's fixtures and the C oracle."""
import numpy as np
import pytest

from paper_2605_21427_b200 import abi, workloads
from paper_2605_21427_b200.wattserve import (AnalyticModel, ConfigError, Grid, OutOfRange, Plan,
                                             TableModel, eval_grid, make_targets, select_config)
from tests.helpers import bits, table_cases, table_view

pytestmark = pytest.mark.gpu


def test_eval_bit_exact_full_grid(ctx, bundle, gold):
    profs, gpu, _ = bundle
    g = gold("eval")
    for i, p in enumerate(profs):
        ok = g["full_err"][i] == 0
        T, P = eval_grid(AnalyticModel(ctx, p, gpu), Grid(ctx, g["full_points"][ok]))
        assert np.array_equal(bits(T), bits(g["full_T"][i][ok]))
        assert np.array_equal(bits(P), bits(g["full_P"][i][ok]))
        ok = g["odd_err"][i] == 0
        T, P = eval_grid(AnalyticModel(ctx, p, gpu), Grid(ctx, g["odd_points"][ok]))
        assert np.array_equal(bits(T), bits(g["odd_T"][i][ok]))
        assert np.array_equal(bits(P), bits(g["odd_P"][i][ok]))


def test_eval_bit_exact_cfg_grids(ctx, gold):
    from oracle.gen_golden import fnv_bits
    g = gold("eval")
    for name, cfg in (("cfg2", workloads.cfg2()), ("cfg3", workloads.cfg3())):
        T, P = eval_grid(AnalyticModel(ctx, cfg["profile"], cfg["gpu"]), Grid(ctx, cfg["points"]))
        assert [fnv_bits(T), fnv_bits(P)] == g[f"{name}_digest"].tolist()


def test_eval_errors_follow_reference(ctx, bundle, gold):
    profs, gpu, _ = bundle
    m = AnalyticModel(ctx, profs[0], gpu)
    bad = workloads.grid_points([150.0, 450.0], [8], [2])
    with pytest.raises(OutOfRange, match="cap outside platform range"):
        eval_grid(m, Grid(ctx, bad))
    bad = workloads.grid_points([150.0], [8], [3])
    with pytest.raises(ConfigError, match="no comm cost calibrated for tp=3"):
        eval_grid(m, Grid(ctx, bad))
    bad = workloads.grid_points([150.0], [0], [2])
    with pytest.raises(ConfigError, match="batch must be >= 1"):
        eval_grid(m, Grid(ctx, bad))


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_select_matches_reference_fixtures(ctx, gold, name):
    cfg = getattr(workloads, name)()
    g = gold("select")
    plan = Plan(AnalyticModel(ctx, cfg["profile"], cfg["gpu"]), Grid(ctx, cfg["points"]),
                cfg["coeffs"])
    idx, rs = plan.select(g[f"{name}_queries"])
    assert np.array_equal(idx, g[f"{name}_idx"])
    assert np.array_equal(rs, g[f"{name}_reason"])
    plan.force_exact(True)
    idx2, rs2 = plan.select(g[f"{name}_queries"])
    assert np.array_equal(idx2, idx) and np.array_equal(rs2, rs)
    assert plan.last_exact_count == len(idx)


def test_select_near_tie_tables(ctx, bundle, gold):
    """Adversarial TableScorer cases (exact ties, 1e-10..4e-9 relative near-ties, chains
    that make better_candidate non-transitive, duplicate points)."""
    _, _, coeffs = bundle
    n_exact = 0
    for pts, T, P, q, want_i, want_r in table_cases(gold):
        _, _, canon = table_view(pts, T, P)
        plan = Plan(TableModel(ctx, pts, T, P), Grid(ctx, pts), coeffs)
        idx, rs = plan.select(q)
        n_exact += plan.last_exact_count
        assert np.array_equal(canon[idx], want_i) and np.array_equal(rs, want_r)
        plan.force_exact(True)
        idx, rs = plan.select(q)
        assert np.array_equal(canon[idx], want_i) and np.array_equal(rs, want_r)
    assert n_exact > 0  # the near-tie fallback was exercised


def test_select_cfg2_all_queries_vs_reference(ctx, reference):
    """Every one of the 1e4 cfg2 bench queries (and 2,000 budget-variant queries) against
    the unmodified select_config + analytic_scorer (oracle/_ref, all host threads)."""
    import os
    cfg = workloads.cfg2()
    model = AnalyticModel(ctx, cfg["profile"], cfg["gpu"])
    plan = Plan(model, Grid(ctx, cfg["points"]), cfg["coeffs"])
    th, pn, ef = plan.scores()
    tref = float(th.max())
    q = workloads.gen_queries(10_000, 2605, tref, "qos")
    idx, rs = plan.select(q)
    threads = os.cpu_count() or 1
    _, ri, rr = reference.bench_select(cfg["profile"], cfg["gpu"], cfg["points"],
                                       cfg["coeffs"], q, threads)
    assert np.array_equal(idx, ri) and np.array_equal(rs, rr)
    # the budget variant
    qb = workloads.gen_queries(2_000, 2606, tref, "qos", budget=(600.0, 2000.0))
    idx, rs = plan.select(qb)
    _, ri, rr = reference.bench_select(cfg["profile"], cfg["gpu"], cfg["points"],
                                       cfg["coeffs"], qb, threads)
    assert np.array_equal(idx, ri) and np.array_equal(rs, rr)


def test_select_cfg3_million_queries(ctx, oracle):
    """Full cfg3 query count on the GPU; a stratified sample against the oracle and an
    exact FP64 feasibility check of every returned point."""
    cfg = workloads.cfg3()
    plan = Plan(AnalyticModel(ctx, cfg["profile"], cfg["gpu"]), Grid(ctx, cfg["points"]),
                cfg["coeffs"])
    th, pn, ef = plan.scores()
    q = workloads.gen_queries(1_000_000, 2605, float(th.max()), "mixed", budget=(600.0, 2000.0))
    idx, rs = plan.select(q)
    assert idx.min() >= 0 and idx.max() < len(cfg["points"])
    T, P, _ = oracle.eval(cfg["profile"], cfg["gpu"], cfg["points"])
    sub = np.arange(0, 1_000_000, 2_000)
    oi, orr, rc = oracle.select(cfg["points"], T, P, cfg["coeffs"], q[sub])
    assert np.array_equal(idx[sub], oi) and np.array_equal(rs[sub], orr)
    # feasibility of every answer, in the reference's FP64 expressions
    target = q["throughput_tps"] * (1.0 + q["target_headroom"])
    budget = q["power_budget_w"] * (1.0 - q["budget_margin"])
    qos = rs == abi.REASON_QOS_FEASIBLE
    assert np.all(~(th[idx[qos]] * q["bias"][qos] < target[qos]))
    assert np.all(pn[idx[qos]] <= budget[qos])
    assert np.all(q["objective"][qos] == abi.OBJ_QOS)
    bud = rs == abi.REASON_BUDGET_MAX_T
    within = pn[idx[bud]] <= budget[bud]
    # budget-constrained picks are within budget unless no point fits (least-power pick)
    assert np.all(within | (pn[idx[bud]] == pn.min()))


def test_select_one_and_errors(ctx, bundle):
    _, _, coeffs = bundle
    from tests.helpers import ladder
    pts, T, P = ladder(8, 1000.0, 2000.0)
    m = TableModel(ctx, pts, T, P)
    # test_controller.cpp:54-60 all feasible: the first (most efficient) point wins
    d = select_config(pts, make_targets(500.0), m, coeffs)
    assert d.reason == abi.REASON_QOS_FEASIBLE and d.point.cap_watts == pts[0]["cap_watts"]
    # :62-67 no candidate reaches the target: max throughput
    pts2, T2, P2 = ladder(8, 100.0, 300.0)
    m2 = TableModel(ctx, pts2, T2, P2)
    d = select_config(pts2, make_targets(1000.0), m2, coeffs)
    assert d.reason == abi.REASON_FALLBACK_MAX_T and d.point.batch == pts2[7]["batch"]
    # :69-79 budget constrains the fallback
    budget = 1.0 * (coeffs.alpha * 4 * P2[3] + coeffs.beta_watts) + 1.0
    d = select_config(pts2, make_targets(1000.0, budget), m2, coeffs)
    assert d.reason == abi.REASON_BUDGET_MAX_T and d.point.batch == pts2[3]["batch"]
    # :81-92 exact ties resolve to the lower cap, then the smaller batch
    tie = np.zeros(2, abi.POINT_DT)
    tie[0] = (300.0, 8, 2, 1, 1)
    tie[1] = (200.0, 8, 2, 1, 1)
    mt = TableModel(ctx, tie, [1000.0, 1000.0], [150.0, 150.0])
    assert select_config(tie, make_targets(100.0), mt, coeffs).point.cap_watts == 200.0
    tie[0] = (200.0, 16, 2, 1, 1)
    mt = TableModel(ctx, tie, [1000.0, 1000.0], [150.0, 150.0])
    assert select_config(tie, make_targets(100.0), mt, coeffs).point.batch == 8
    # :94-98 empty candidate list
    with pytest.raises(ConfigError, match="select_config: empty candidate list"):
        select_config(np.zeros(0, abi.POINT_DT), make_targets(100.0), m, coeffs)
    # unscored candidate (TableScorer throws config_error)
    other = workloads.grid_points([333.0], [3], [2])
    with pytest.raises(ConfigError, match="unscored candidate"):
        select_config(other, make_targets(100.0), m, coeffs)


@pytest.mark.parametrize("nq", [3000, 300_001])
def test_select_pinned_buffers_graph_path(ctx, oracle, nq):
    """pals_select with pinned host buffers runs one graph holding the upload (overlapped
    with the prepare; in chunks pipelined behind their scans for large batches) and
    stores the decisions into the mapped result buffers; replays must read the buffers'
    current contents."""
    import torch

    from paper_2605_21427_b200.abi import QUERY_DT, ptr
    from paper_2605_21427_b200.wattserve import check

    cfg = workloads.cfg2()
    model = AnalyticModel(ctx, cfg["profile"], cfg["gpu"])
    plan = Plan(model, Grid(ctx, cfg["points"]), cfg["coeffs"])
    th, _, _ = plan.scores()
    T, P, _ = oracle.eval(cfg["profile"], cfg["gpu"], cfg["points"])
    step = 7 if nq < 10_000 else 997
    h_q = torch.empty(nq * QUERY_DT.itemsize, dtype=torch.uint8, pin_memory=True)
    h_qn = h_q.numpy().view(QUERY_DT)
    h_idx = torch.empty(nq, dtype=torch.int32, pin_memory=True).numpy()
    h_rs = torch.empty(nq, dtype=torch.uint8, pin_memory=True).numpy()
    for seed in (11, 12, 13):  # same buffers, new contents: the cached graph is replayed
        q = workloads.gen_queries(nq, seed, float(th.max()), "mixed", budget=(700.0, 1900.0))
        h_qn[:] = q
        check(ctx.lib.pals_select(plan.h, ptr(h_qn), nq, ptr(h_idx), ptr(h_rs)))
        idx, rs = plan.select(q)  # pageable path
        assert np.array_equal(h_idx, idx) and np.array_equal(h_rs, rs)
        oi, orr, rc = oracle.select(cfg["points"], T, P, cfg["coeffs"], q[::step])
        assert rc == 0 and np.array_equal(h_idx[::step], oi) and np.array_equal(h_rs[::step], orr)
        assert plan.last_exact_count >= 0


@pytest.mark.parametrize("which", ["cfg2", "cfg3", "cfg3x"])
def test_prefix_decide_equals_scan(ctx, oracle, which):
    """PALS_DECIDE_PREFIX (prefix-min tables; 2-D blocks for QoS+budget queries) decides
    every query exactly as the pair scan does, on the bench grids, and a sample agrees
    with the C oracle."""
    c = {"cfg2": workloads.cfg2, "cfg3": workloads.cfg3,
         "cfg3x": workloads.cfg3_extended}[which]()
    plan = Plan(AnalyticModel(ctx, c["profile"], c["gpu"]), Grid(ctx, c["points"]), c["coeffs"])
    th, _, _ = plan.scores()
    n = {"cfg2": 20_000, "cfg3": 200_000, "cfg3x": 20_000}[which]
    q = workloads.gen_queries(n, 4242, float(th.max()), "mixed", budget=(600.0, 6000.0))
    q["bias"][::3] = np.linspace(0.5, 2.0, len(q["bias"][::3]))
    si, sr = plan.select(q)
    plan.set_decide("prefix")
    pi, pr = plan.select(q)
    assert np.array_equal(si, pi) and np.array_equal(sr, pr)
    assert plan.stats()[1] > 0  # QoS+budget queries took the 2-D path
    T, P, _ = oracle.eval(c["profile"], c["gpu"], c["points"])
    sub = np.arange(0, n, max(1, n // 300))
    oi, orr, _ = oracle.select(c["points"], T, P, c["coeffs"], q[sub])
    assert np.array_equal(pi[sub], oi) and np.array_equal(pr[sub], orr)
