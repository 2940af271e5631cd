"""Randomised parity on the B200 against the C oracle (itself pinned to the
reference): many generated score tables with exact ties, tolerance near-ties
and chains of near-ties, random targets/budgets/biases/margins; random
controller configurations for the replay; two contexts driven from two host
threads at once."""
import threading

import numpy as np
import pytest

from paper_2605_21427_b200 import abi, workloads
from paper_2605_21427_b200.abi import default_ctrl_cfg
from paper_2605_21427_b200.wattserve import (AnalyticModel, Context, Grid, Plan, TableModel,
                                             replay)
from tests.helpers import table_view

pytestmark = pytest.mark.gpu


def random_table(rng, n):
    caps = rng.choice([100.0, 150.0, 200.0, 250.0, 300.0, 350.0, 400.0], n)
    pts = np.zeros(n, abi.POINT_DT)
    pts["cap_watts"] = caps
    pts["batch"] = rng.choice([1, 2, 4, 8, 16, 32, 64, 128], n)
    pts["tp"] = rng.choice([1, 2, 4, 8], n)
    pts["ep"] = 1
    pts["dp"] = rng.choice([1, 1, 2, 3], n)
    base_t = rng.uniform(50.0, 5000.0, max(1, n // 4))
    base_p = rng.uniform(50.0, 400.0, max(1, n // 4))
    T = base_t[rng.integers(0, len(base_t), n)]
    P = base_p[rng.integers(0, len(base_p), n)]
    kind = rng.integers(0, 4)
    if kind == 1:
        T = T * (1.0 + rng.choice([0.0, 2e-10, 7e-10, 1.5e-9, 3.9e-9, 4.1e-9, 1e-8], n))
    elif kind == 2:
        P = P * (1.0 + rng.choice([0.0, -5e-10, 9e-10, 2e-9, 5e-9], n))
    elif kind == 3:  # eff chains: consecutive near-ties that make the comparator non-transitive
        k = rng.uniform(0.2, 3.0)
        steps = rng.integers(0, 12, n)
        alpha4 = 1.05 * 4
        pn = P * alpha4 + 345.0
        T = k * pn * (1.0 + 0.95e-9 * steps) / pts["dp"] * pts["dp"]
    return pts, T, P


def random_queries(rng, nq, tmax, pn_min, pn_max):
    q = np.zeros(nq, abi.QUERY_DT)
    q["throughput_tps"] = rng.uniform(0.0, 1.2, nq) * tmax
    q["bias"] = np.where(rng.uniform(size=nq) < 0.4, 1.0, rng.uniform(0.4, 2.5, nq))
    q["target_headroom"] = rng.choice([0.0, 0.05, 0.1], nq)
    q["has_budget"] = rng.uniform(size=nq) < 0.6
    q["power_budget_w"] = rng.uniform(0.8 * pn_min, 1.2 * pn_max, nq)
    q["budget_margin"] = rng.choice([0.0, 0.008, 0.02], nq)
    q["objective"] = (rng.uniform(size=nq) < 0.35).astype(np.int32)
    return q


def test_random_tables_vs_oracle(ctx, oracle, bundle):
    _, _, coeffs = bundle
    rng = np.random.default_rng(20261017)
    total = 0
    for case in range(120):
        n = int(rng.integers(1, 300))
        pts, T, P = random_table(rng, n)
        pn = pts["dp"] * (coeffs.alpha * 4 * P + coeffs.beta_watts)
        q = random_queries(rng, 64, float(np.max(T * pts["dp"])), float(pn.min()), float(pn.max()))
        plan = Plan(TableModel(ctx, pts, T, P), Grid(ctx, pts), coeffs)
        idx, rs = plan.select(q)
        Ts, Ps, canon = table_view(pts, T, P)
        oi, orr, rc = oracle.select(pts, Ts, Ps, coeffs, q)
        assert rc == 0
        # the reference returns a Decision's point: compare points (first equal index)
        assert np.array_equal(canon[idx], canon[oi]), case
        assert np.array_equal(rs, orr), case
        total += len(q)
    assert total == 120 * 64


def test_random_controller_configs_replay_vs_oracle(ctx, oracle):
    """Random gains, sustain counts, clamps, margins and trace shapes."""
    s = workloads.cfg4_setup()
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    rng = np.random.default_rng(7)
    for case in range(6):
        cfg = default_ctrl_cfg(kp=float(rng.uniform(0.0, 1.0)), ki=float(rng.uniform(0.0, 0.3)),
                               kd=float(rng.uniform(0.0, 0.2)),
                               integral_clamp=float(rng.uniform(0.1, 1.0)),
                               sustain_intervals=int(rng.integers(0, 6)),
                               target_headroom=float(rng.choice([0.0, 0.05])),
                               budget_margin=float(rng.choice([0.0, 0.008, 0.02])))
        spec = workloads.replay_spec(120, n_steps=500, seed=100 + case,
                                     objective_mode=int(rng.integers(0, 3)), n_log_traces=6)
        spec.noise_amp = float(rng.uniform(0.0, 0.1))
        spec.seg_min, spec.seg_max = int(rng.integers(1, 40)), int(rng.integers(40, 200))
        spec.budget_mode = int(rng.integers(0, 2))
        spec.budget_lo_frac = float(rng.uniform(0.5, 1.0))
        summ, logs = replay(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                            s["batches"], cfg, spec)
        osumm, ologs = oracle.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                                     s["batches"], cfg, spec)
        assert np.array_equal(logs, ologs), case
        assert np.array_equal(summ, osumm), case


def test_two_contexts_two_threads(oracle, bundle):
    """Calls on different contexts are independent (one host thread per context)."""
    profs, gpu, coeffs = bundle
    c1 = workloads.cfg1()
    T, P, _ = oracle.eval(c1["profile"], gpu, c1["points"])
    q = workloads.gen_queries(4000, 3, float(T.max()), "mixed", budget=(900.0, 1900.0))
    want = oracle.select(c1["points"], T, P, coeffs, q)
    results, errors = {}, []

    def work(k):
        try:
            ctx = Context(0)
            plan = Plan(AnalyticModel(ctx, c1["profile"], gpu), Grid(ctx, c1["points"]), coeffs)
            for _ in range(20):
                idx, rs = plan.select(q)
            results[k] = (idx, rs)
        except Exception as e:  # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors
    for k in range(2):
        assert np.array_equal(results[k][0], want[0]) and np.array_equal(results[k][1], want[1])
