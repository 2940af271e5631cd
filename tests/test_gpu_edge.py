"""Edge cases and the less-travelled code paths on the B200: 64-bit keys (grids
above 65,536 points), the literal-fold path for non-finite / non-positive score
sets, tiny grids, the dense demand-response candidate grid in the replay, and
the reference's error semantics."""
import numpy as np
import pytest

from paper_2605_21427_b200 import abi, workloads
from paper_2605_21427_b200.wattserve import (AnalyticModel, ConfigError, Grid, Plan, TableModel,
                                             replay)
from tests.helpers import table_view

pytestmark = pytest.mark.gpu


def test_select_wide_keys_extended_cfg3(ctx, oracle):
    """589,824 configs (cfg3 x EP x DP): 64-bit packed keys, vs the C oracle."""
    cfg = workloads.cfg3_extended()
    assert len(cfg["points"]) == 589_824
    plan = Plan(AnalyticModel(ctx, cfg["profile"], cfg["gpu"]), Grid(ctx, cfg["points"]),
                cfg["coeffs"])
    th, pn, ef = plan.scores()
    q = workloads.gen_queries(20_000, 99, float(th.max()), "mixed", budget=(600.0, 6000.0))
    idx, rs = plan.select(q)
    T, P, e = oracle.eval(cfg["profile"], cfg["gpu"], cfg["points"])
    assert not e.any()
    sub = np.arange(0, 20_000, 500)
    oi, orr, rc = oracle.select(cfg["points"], T, P, cfg["coeffs"], q[sub])
    assert rc == 0
    assert np.array_equal(idx[sub], oi) and np.array_equal(rs[sub], orr)
    plan.force_exact(True)
    ie, re = plan.select(q[:64])
    assert np.array_equal(ie, idx[:64]) and np.array_equal(re, rs[:64])


def test_select_generic_scores_use_literal_fold(ctx, oracle, bundle):
    """Zero, negative, infinite and NaN scores disable the integer fast path; the
    literal fold must still reproduce the reference (IEEE comparisons included)."""
    _, _, coeffs = bundle
    rng = np.random.default_rng(3)
    for case in range(12):
        n = 40
        pts = workloads.grid_points([150.0, 200.0, 250.0, 300.0, 350.0], [1, 2, 4, 8, 16, 32, 64, 128],
                                    [2])[:n]
        T = rng.uniform(100.0, 3000.0, n)
        P = rng.uniform(60.0, 400.0, n)
        bad = rng.choice(n, 4, replace=False)
        T[bad[0]] = 0.0
        P[bad[1]] = -300.0  # negative p_node
        T[bad[2]] = [np.inf, np.nan, 1e-320][case % 3]
        P[bad[3]] = [np.nan, 1e300, np.inf][case % 3]
        q = np.zeros(30, abi.QUERY_DT)
        q["throughput_tps"] = rng.uniform(50.0, 3000.0, 30)
        q["bias"] = 1.0
        q["has_budget"] = rng.uniform(size=30) < 0.5
        q["power_budget_w"] = rng.uniform(500.0, 2000.0, 30)
        q["objective"] = (rng.uniform(size=30) < 0.3).astype(np.int32)
        plan = Plan(TableModel(ctx, pts, T, P), Grid(ctx, pts), coeffs)
        idx, rs = plan.select(q)
        assert plan.last_exact_count == len(q)  # all routed to the literal fold
        Ts, Ps, canon = table_view(pts, T, P)
        oi, orr, rc = oracle.select(pts, Ts, Ps, coeffs, q)
        assert np.array_equal(canon[idx], oi) and np.array_equal(rs, orr), case


def test_select_tiny_grids(ctx, oracle, bundle):
    profs, gpu, coeffs = bundle
    p = profs[2]
    for caps, batches in (([400.0], [1]), ([100.0, 400.0], [64]), ([250.0], [1, 2, 3])):
        pts = workloads.grid_points(caps, batches, [p.deploy_tp], [p.deploy_ep], [p.deploy_dp])
        plan = Plan(AnalyticModel(ctx, p, gpu), Grid(ctx, pts), coeffs)
        th, _, _ = plan.scores()
        q = workloads.gen_queries(200, 1, float(th.max()), "mixed", budget=(300.0, 2500.0))
        idx, rs = plan.select(q)
        T, P, _ = oracle.eval(p, gpu, pts)
        oi, orr, _ = oracle.select(pts, T, P, coeffs, q)
        assert np.array_equal(idx, oi) and np.array_equal(rs, orr)


def test_plan_errors(ctx, bundle):
    profs, gpu, coeffs = bundle
    m = AnalyticModel(ctx, profs[0], gpu)
    with pytest.raises(ConfigError, match="select_config: empty candidate list"):
        Plan(m, Grid(ctx, np.zeros(0, abi.POINT_DT)), coeffs).select(
            workloads.gen_queries(1, 1, 100.0))
    t = TableModel(ctx, workloads.grid_points([150.0], [1], [2]), [10.0], [100.0])
    with pytest.raises(ConfigError, match="unscored candidate"):
        Plan(t, Grid(ctx, workloads.grid_points([150.0, 200.0], [1], [2])), coeffs).select(
            workloads.gen_queries(1, 1, 100.0))


def test_replay_dense_dr_grid(ctx, oracle):
    """The demand-response scenario's 61 x 24 = 1,464-candidate grid."""
    s = workloads.cfg4_setup()
    caps, batches = workloads.dr_candidates()
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    spec = workloads.replay_spec(160, n_steps=600, seed=515, n_log_traces=8)
    summ, logs = replay(ctx, models, s["profiles"], s["gpu"], s["coeffs"], caps, batches,
                        s["cfg"], spec)
    osumm, ologs = oracle.replay(s["profiles"], s["gpu"], s["coeffs"], caps, batches, s["cfg"],
                                 spec)
    assert np.array_equal(logs, ologs)
    assert np.array_equal(summ, osumm)


@pytest.mark.parametrize("mode", [0, 1])
def test_replay_single_objective(ctx, oracle, mode):
    """All-QoS and all-budget traces (no objective reordering)."""
    s = workloads.cfg4_setup()
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    spec = workloads.replay_spec(300, n_steps=900, seed=21 + mode, objective_mode=mode,
                                 n_log_traces=10)
    summ, logs = replay(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                        s["batches"], s["cfg"], spec)
    osumm, ologs = oracle.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                                 s["cfg"], spec)
    assert np.array_equal(logs, ologs) and np.array_equal(summ, osumm)


def test_select_negative_bias(ctx, reference, bundle):
    """A negative bias makes the QoS-feasible set a suffix of the t_hat order:
    such queries must take the literal fold and still match the reference, including a
    non-positive target (every candidate then passes !(t*bias < target) or none does)."""
    profs, gpu, coeffs = bundle
    p = profs[1]
    pts = workloads.grid_points([150.0 + 10 * i for i in range(24)], list(range(1, 33)),
                                [p.deploy_tp], [p.deploy_ep], [p.deploy_dp])
    plan = Plan(AnalyticModel(ctx, p, gpu), Grid(ctx, pts), coeffs)
    th, _, _ = plan.scores()
    rng = np.random.default_rng(11)
    n = 400
    q = np.zeros(n, abi.QUERY_DT)
    q["throughput_tps"] = rng.uniform(-1.2, 1.0, n) * float(th.max())
    q["bias"] = np.where(rng.uniform(size=n) < 0.7, rng.uniform(-2.0, -0.01, n),
                         rng.uniform(0.5, 2.0, n))
    q["target_headroom"] = 0.05
    q["has_budget"] = rng.uniform(size=n) < 0.5
    q["power_budget_w"] = rng.uniform(600.0, 2500.0, n)
    q["budget_margin"] = 0.02
    q["objective"] = (rng.uniform(size=n) < 0.2).astype(np.int32)
    idx, rs = plan.select(q)
    ri, rr, rc = reference.select_analytic(p, gpu, pts, coeffs, q)
    assert rc == 0, reference.last_error()
    assert np.array_equal(idx, ri) and np.array_equal(rs, rr)
    neg = (q["bias"] < 0) & (q["objective"] == 0)
    assert plan.stats()[4] >= int(neg.sum())  # routed to the literal fold
