"""K3 parity on the B200: control_step single calls against the reference's
recorded sequences, and the batched replay against the reference-driven fixtures
and the C oracle (full per-step logs + per-trace digests)."""
import numpy as np
import pytest

from paper_2605_21427_b200 import abi, workloads
from paper_2605_21427_b200.abi import CtrlState, Telemetry, default_ctrl_cfg
from paper_2605_21427_b200.wattserve import (AnalyticModel, TableModel, control_step,
                                             make_targets, replay)
from tests.helpers import ladder, run_control_sequences

pytestmark = pytest.mark.gpu


def test_control_sequences_match_reference(ctx, bundle, gold):
    _, _, coeffs = bundle
    cache = {}

    def step(pts, T, P, tel, now, tg, st, cfg):
        key = len(pts)
        if key not in cache:
            cache[key] = TableModel(ctx, pts, T, P)
        return control_step(tel, now, tg, pts, cache[key], coeffs, st, cfg)

    assert run_control_sequences(gold, step) == []


def test_reference_controller_properties(ctx, bundle):
    """test_controller.cpp:140-235 on the GPU path: fixed point, dead-band, target step,
    stale hold, bias convergence."""
    _, _, coeffs = bundle
    cfg = default_ctrl_cfg()
    pts, T, P = ladder(10, 500.0, 1500.0)
    m = TableModel(ctx, pts, T, P)
    st = CtrlState()
    st.bias = 1.0
    st.current = abi.Point(*pts[0].tolist())
    d, st2 = control_step(Telemetry(1.0, T[0]), 1.0, make_targets(T[0]), pts, m, coeffs, st, cfg)
    assert st2.bias == pytest.approx(1.0)
    # stale telemetry holds (:194-205)
    st.current = abi.Point(*pts[3].tolist())
    d, _ = control_step(Telemetry(0.0, 100.0), 10.0, make_targets(2000.0), pts, m, coeffs, st, cfg)
    assert not d.applied and d.reason == abi.REASON_HOLD and d.point.batch == pts[3]["batch"]
    # dead-band: 1000 steps, no reconfiguration (:153-175)
    pts, T, P = ladder(30, 500.0, 1500.0)
    m = TableModel(ctx, pts, T, P)
    st = CtrlState()
    st.bias = 1.0
    st.current = abi.Point(*pts[20].tolist())
    tg = make_targets(T[20])
    st.last_targets = tg
    st.has_last_targets = 1
    rng = np.random.default_rng(7)
    now = 1.0
    for _ in range(300):
        meas = tg.throughput_tps * (1.0 + rng.uniform(-0.049, 0.049))
        d, st = control_step(Telemetry(now, meas), now, tg, pts, m, coeffs, st, cfg)
        assert not d.applied
        now += 0.5
    # target step forces immediate re-selection (:177-192)
    st = CtrlState()
    st.bias = 1.0
    st.current = abi.Point(*pts[29].tolist())
    st.last_targets = make_targets(T[29])
    st.has_last_targets = 1
    d, _ = control_step(Telemetry(1.0, T[29]), 1.0, make_targets(T[5]), pts, m, coeffs, st, cfg)
    assert d.applied and d.point.batch == pts[5]["batch"]
    # bias convergence (:207-235)
    for lam in (0.7, 1.3):
        pts, T, P = ladder(60, 300.0, 2400.0)
        m = TableModel(ctx, pts, T, P)
        st = CtrlState()
        st.bias = 1.0
        st.current = abi.Point(*pts[59].tolist())
        tg = make_targets(1100.0)
        now, meas, settled = 0.5, lam * T[59], -1
        for k in range(40):
            d, st = control_step(Telemetry(now, meas), now, tg, pts, m, coeffs, st, cfg)
            i = int(np.nonzero(pts["batch"] == st.current.batch)[0][0])
            meas = lam * T[i]
            err = abs(tg.throughput_tps - meas) / tg.throughput_tps
            if settled < 0 and err <= 0.05:
                settled = k
            if settled >= 0 and err > 0.05:
                settled = -1
            now += 0.5
        assert 0 <= settled < 20


def test_control_step_analytic_matches_reference(ctx, bundle, reference):
    """Analytic scorer, arbitrary current point (not a candidate) — straight against the
    reference build when it is present."""
    profs, gpu, coeffs = bundle
    c1 = workloads.cfg1()
    m = AnalyticModel(ctx, c1["profile"], gpu)
    cfg = default_ctrl_cfg(target_headroom=0.05, budget_margin=0.02)
    rng = np.random.default_rng(5)
    st = CtrlState()
    st.bias = 1.0
    st.current = abi.Point(275.0, 48, 2, 1, 1)
    rst = CtrlState.from_buffer_copy(st)
    now = 0.5
    for k in range(200):
        tg = make_targets(float(rng.uniform(200, 2500)), None if k % 3 else float(
            rng.uniform(900, 1800)), 0.05, int(k % 7 == 6))
        tel = Telemetry(now, float(rng.uniform(100, 3000)))
        d, st = control_step(tel, now, tg, c1["points"], m, coeffs, st, cfg)
        rd, rst, rc = reference.control_step_analytic(c1["profile"], gpu, c1["points"], tel, now,
                                                      tg, coeffs, rst, cfg)
        assert rc == 0
        assert bytes(d) == bytes(rd) and bytes(st) == bytes(rst), k
        now += 0.5


def test_replay_matches_reference_fixtures(ctx, gold):
    s = workloads.cfg4_setup()
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    g = gold("replay")
    spec = workloads.replay_spec(96, n_steps=720, seed=515, n_log_traces=12)
    summ, logs = replay(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                        s["batches"], s["cfg"], spec)
    assert np.array_equal(logs, g["logs"])
    assert np.array_equal(summ, g["summ"])
    spec = workloads.replay_spec(32, n_steps=720, seed=516, objective_mode=0, n_log_traces=4)
    summ, logs = replay(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                        s["batches"], s["cfg"], spec)
    assert np.array_equal(summ, g["summ_q"]) and np.array_equal(logs, g["logs_q"])


def test_replay_vs_oracle_cfg4_shape(ctx, oracle):
    """cfg4 trace length (3600 steps), 1,000 traces: full logs for 64, digests for all."""
    s = workloads.cfg4_setup()
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    spec = workloads.replay_spec(1000, n_steps=3600, seed=2605, n_log_traces=64)
    summ, logs = replay(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                        s["batches"], s["cfg"], spec)
    osumm, ologs = oracle.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                                 s["cfg"], spec)
    assert np.array_equal(logs, ologs)
    assert np.array_equal(summ, osumm)


def test_replay_shards_compose(ctx):
    """Trace i depends only on (seed, i): a sharded run equals the unsharded run."""
    s = workloads.cfg4_setup()
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    full, _ = replay(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                     s["cfg"], workloads.replay_spec(4096, n_steps=600, seed=9))
    parts = []
    for k in range(4):
        sp = workloads.replay_spec(1024, n_steps=600, seed=9, first=1024 * k)
        parts.append(replay(ctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                            s["batches"], s["cfg"], sp)[0])
    assert np.array_equal(np.concatenate(parts), full)
