"""pals_replay_traces on the B200 against the unmodified reference control_step over the
same caller traces (oracle/_ref, replay_trace_one), and against the synthetic path."""
import numpy as np
import pytest

from paper_2605_21427_b200 import workloads
from paper_2605_21427_b200.abi import (PLANT_DT, STATE_DT, TRACE_DT, default_ctrl_cfg)
from paper_2605_21427_b200.wattserve import (AnalyticModel, ConfigError, replay,
                                             replay_traces)
from tests.test_traces import build_dr_traces, ref_plant_constants

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup(ctx, reference):
    s = workloads.cfg4_setup()
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    return s, models, ref_plant_constants(reference, s, s["caps"], s["batches"])


def _args(s, caps=None, batches=None):
    return (s["profiles"], s["gpu"], s["coeffs"], s["caps"] if caps is None else caps,
            s["batches"] if batches is None else batches, s["cfg"])


def test_synthetic_workload_through_traces(ctx, setup):
    """The cfg4 synthetic workload exported as caller traces: same summaries and logs."""
    s, models, (t_max, p_min, p_max) = setup
    spec = workloads.replay_spec(4096, n_steps=3600, seed=2605, n_log_traces=16)
    want, wlogs = replay(ctx, models, *_args(s), spec)
    tr, sig = workloads.synthetic_traces(spec, len(models), t_max, p_min, p_max)
    got = replay_traces(ctx, models, *_args(s), tr, sig, spec.n_steps, n_log_traces=16)
    assert np.array_equal(got["summaries"], want)
    assert np.array_equal(got["logs"], wlogs)


@pytest.mark.parametrize("grid", ["cfg4", "dr"])
def test_dr_trace_vs_reference_with_resume(ctx, reference, setup, grid):
    """The demand-response cluster budget trace (dr_cluster_1h.csv, split over the
    scenario's 3 nodes as assign_budgets does) for one hour of 0.5 s intervals, every
    profile and objective; the GPU replay is split at step 3001 and resumed from its own
    returned states. Logs, details, summaries and final states equal the reference's."""
    s, models, (t_max, _, _) = setup
    caps, batches = (s["caps"], s["batches"]) if grid == "cfg4" else workloads.dr_candidates()
    tr, sig = build_dr_traces(s, t_max, n_per_model=2, n_steps=7200)
    a = _args(s, caps, batches)
    kw = dict(n_log_traces=len(tr), details=True)
    want, _ = reference.replay_traces(*a, tr, sig, 7200, threads=8, **kw)
    full = replay_traces(ctx, models, *a, tr, sig, 7200, **kw)
    for k in ("summaries", "logs", "details", "final_state", "final_plant"):
        assert np.array_equal(full[k], want[k]), k
    p1 = replay_traces(ctx, models, *a, tr, sig, 3001, **kw)
    p2 = replay_traces(ctx, models, *a, tr, sig, 4199, first_step=3001,
                       init=p1["final_state"], init_plant=p1["final_plant"], **kw)
    n = len(tr)
    logs = np.concatenate([p1["logs"].reshape(n, -1), p2["logs"].reshape(n, -1)], 1)
    assert np.array_equal(logs, want["logs"].reshape(n, -1))
    assert np.array_equal(p2["final_state"], want["final_state"])
    assert np.array_equal(p2["final_plant"], want["final_plant"])
    assert (want["logs"]["reason"] == 2).any()  # budget-constrained decisions happened


def test_random_states_vs_reference(ctx, reference, setup):
    """Arbitrary caller states: bias anywhere in [bias_min, bias_max] (negative bias_min
    included), integral / prev_error / sustain values, a current point anywhere on the
    grid, last_targets equal or not to the trace's, plant states off the initial point."""
    s, models, (t_max, _, _) = setup
    rng = np.random.default_rng(17)
    tr, sig = build_dr_traces(s, t_max, n_per_model=24, n_steps=1200, seed=9)
    n = len(tr)
    init = np.zeros(n, STATE_DT)
    init["bias"] = rng.uniform(-0.5, 2.0, n)
    init["integral"] = rng.uniform(-0.5, 0.5, n)
    init["prev_error"] = rng.uniform(-0.3, 0.3, n)
    init["has_prev_error"] = rng.integers(0, 2, n)
    init["sustain_count"] = rng.integers(0, 5, n)
    a_idx = rng.integers(0, len(s["caps"]), n)
    b_idx = rng.integers(0, len(s["batches"]), n)
    for i in range(n):
        p = s["profiles"][int(tr["model"][i])]
        init["current"][i] = (s["caps"][a_idx[i]], s["batches"][b_idx[i]], p.deploy_tp,
                              p.deploy_ep, p.deploy_dp)
    same = rng.uniform(size=n) < 0.6
    lt = init["last_targets"]
    lt["throughput_tps"] = np.where(same, tr["target_tps"], tr["target_tps"] * 1.01)
    lt["epsilon"] = tr["epsilon"]
    lt["objective"] = tr["objective"]
    lt["has_budget"] = rng.integers(0, 2, n)
    lt["power_budget_w"] = 1000.0
    init["last_targets"] = lt
    init["has_last_targets"] = rng.integers(0, 2, n)
    plant = np.zeros(n, PLANT_DT)
    plant["applied_cap_w"] = s["caps"][rng.integers(0, len(s["caps"]), n)]
    plant["inflight_cap_w"] = s["caps"][rng.integers(0, len(s["caps"]), n)]
    plant["batch_cap"] = s["batches"][rng.integers(0, len(s["batches"]), n)]
    cfg = default_ctrl_cfg(target_headroom=0.05, budget_margin=0.02, bias_min=-0.25)
    a = (s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"], cfg)
    kw = dict(init=init, init_plant=plant, first_step=11, n_log_traces=n, details=True)
    want, _ = reference.replay_traces(*a, tr, sig, 1200, threads=8, **kw)
    got = replay_traces(ctx, models, *a, tr, sig, 1200, **kw)
    for k in ("summaries", "logs", "details", "final_state", "final_plant"):
        assert np.array_equal(got[k], want[k]), k
    zero = replay_traces(ctx, models, *a, tr, sig, 0, init=init, init_plant=plant)
    assert np.array_equal(zero["final_state"], init)  # no step: the state passes through
    assert np.array_equal(zero["final_plant"], plant)


def test_invalid_traces_rejected(ctx, setup):
    s, models, (t_max, _, _) = setup
    tr, sig = build_dr_traces(s, t_max, n_per_model=1, n_steps=100)
    bad = tr.copy()
    bad["model"][3] = 99
    with pytest.raises(ConfigError, match="trace 3: model index out of range"):
        replay_traces(ctx, models, *_args(s), bad, sig, 10)
    bad = tr.copy()
    bad["load_off"][2] = len(sig)
    with pytest.raises(ConfigError, match="trace 2: signal outside"):
        replay_traces(ctx, models, *_args(s), bad, sig, 10)
    init = np.zeros(len(tr), STATE_DT)
    init["bias"] = 1.0
    init["current"] = (123.0, 1, 1, 1, 1)
    with pytest.raises(ConfigError, match="not a candidate"):
        replay_traces(ctx, models, *_args(s), tr, sig, 10, init=init)
    assert TRACE_DT.itemsize == 64
