"""The warp-per-trace replay layout (BASELINE cfg4's named layout) against the same
oracle / reference fixtures as the thread layout: identical logs and summaries."""
import numpy as np
import pytest

from paper_2605_21427_b200 import workloads
from paper_2605_21427_b200.abi import default_ctrl_cfg
from paper_2605_21427_b200.wattserve import AnalyticModel, Context, replay

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wctx():
    c = Context(0)
    c.set_replay_layout("warp")
    return c


def _models(ctx, s):
    return [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]


def test_warp_layout_matches_reference_fixtures(wctx, gold):
    s = workloads.cfg4_setup()
    models = _models(wctx, s)
    g = gold("replay")
    spec = workloads.replay_spec(96, n_steps=720, seed=515, n_log_traces=12)
    summ, logs = replay(wctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                        s["batches"], s["cfg"], spec)
    assert np.array_equal(logs, g["logs"]) and np.array_equal(summ, g["summ"])
    spec = workloads.replay_spec(32, n_steps=720, seed=516, objective_mode=0, n_log_traces=4)
    summ, logs = replay(wctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                        s["batches"], s["cfg"], spec)
    assert np.array_equal(summ, g["summ_q"]) and np.array_equal(logs, g["logs_q"])


def test_warp_layout_cfg4_shape_equals_thread_layout(wctx, ctx, oracle):
    """3600-step traces: warp layout == thread layout on 4,096 traces, == oracle on 256
    (full logs for 32)."""
    s = workloads.cfg4_setup()
    spec = workloads.replay_spec(4096, n_steps=3600, seed=2605, n_log_traces=32)
    w_summ, w_logs = replay(wctx, _models(wctx, s), s["profiles"], s["gpu"], s["coeffs"],
                            s["caps"], s["batches"], s["cfg"], spec)
    t_summ, t_logs = replay(ctx, _models(ctx, s), s["profiles"], s["gpu"], s["coeffs"],
                            s["caps"], s["batches"], s["cfg"], spec)
    assert np.array_equal(w_summ, t_summ) and np.array_equal(w_logs, t_logs)
    spec = workloads.replay_spec(256, n_steps=3600, seed=2605, n_log_traces=32)
    osumm, ologs = oracle.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"],
                                 s["cfg"], spec)
    assert np.array_equal(w_summ[:256], osumm) and np.array_equal(w_logs, ologs)


def test_warp_layout_dr_grid(wctx, oracle):
    """1,464 candidates: three 32-ary rounds per search, 61-position breaker walks."""
    s = workloads.cfg4_setup()
    caps, batches = workloads.dr_candidates()
    spec = workloads.replay_spec(160, n_steps=600, seed=515, n_log_traces=8)
    summ, logs = replay(wctx, _models(wctx, s), s["profiles"], s["gpu"], s["coeffs"], caps,
                        batches, s["cfg"], spec)
    osumm, ologs = oracle.replay(s["profiles"], s["gpu"], s["coeffs"], caps, batches, s["cfg"],
                                 spec)
    assert np.array_equal(logs, ologs) and np.array_equal(summ, osumm)


def test_warp_layout_random_configs(wctx, oracle):
    """Random gains / sustain / margins / segment lengths; odd step counts (noise rounds
    that end mid-warp)."""
    s = workloads.cfg4_setup()
    models = _models(wctx, s)
    rng = np.random.default_rng(11)
    for case in range(5):
        cfg = default_ctrl_cfg(kp=float(rng.uniform(0.0, 1.0)), ki=float(rng.uniform(0.0, 0.3)),
                               kd=float(rng.uniform(0.0, 0.2)),
                               sustain_intervals=int(rng.integers(0, 6)),
                               target_headroom=float(rng.choice([0.0, 0.05])),
                               budget_margin=float(rng.choice([0.0, 0.02])))
        spec = workloads.replay_spec(97, n_steps=int(rng.integers(1, 700)), seed=300 + case,
                                     objective_mode=int(rng.integers(0, 3)), n_log_traces=5)
        spec.seg_min, spec.seg_max = int(rng.integers(1, 40)), int(rng.integers(40, 200))
        spec.budget_mode = int(rng.integers(0, 2))
        summ, logs = replay(wctx, models, s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                            s["batches"], cfg, spec)
        osumm, ologs = oracle.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                                     s["batches"], cfg, spec)
        assert np.array_equal(logs, ologs), case
        assert np.array_equal(summ, osumm), case
