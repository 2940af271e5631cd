"""Caller-trace replay (pals_replay_traces) contract, pinned on the CPU with the
reference harness (oracle/_ref: the unmodified control_step, detail::trace_value and
detail::enforce_cap, sim.hpp:167-205):

* the synthetic fluid-plant workload written out as caller traces
  (workloads.synthetic_traces) replays to the synthetic path's decisions bit for bit;
* a replay split at any step and resumed from the returned ControllerState / plant
  state gives the same per-step decisions and final state as one uninterrupted call.
"""
import numpy as np
import pytest

from paper_2605_21427_b200 import workloads
from paper_2605_21427_b200.abi import SIGNAL_DT, TRACE_DT


def ref_plant_constants(ref, s, caps, batches):
    """(t_max, p_min, p_max) per model from the reference's own throughput/avg_gpu_power."""
    t_max, p_min, p_max = [], [], []
    for p in s["profiles"]:
        pts = workloads.grid_points(caps, batches, [p.deploy_tp], [p.deploy_ep], [p.deploy_dp])
        T, P, _ = ref.eval(p, s["gpu"], pts)
        dp = float(p.deploy_dp)
        pn = dp * (s["coeffs"].alpha * 4.0 * P + s["coeffs"].beta_watts)
        i = int(np.flatnonzero((pts["cap_watts"] == np.max(caps)) &
                               (pts["batch"] == np.max(batches)))[0])
        t_max.append(dp * T[i])
        p_min.append(pn.min())
        p_max.append(pn.max())
    return np.array(t_max), np.array(p_min), np.array(p_max)


def dr_budget(n_nodes=3):
    """Budget: the demand-response cluster trace (proj/data/traces/dr_cluster_1h.csv via
    the package's scenarios.json) split dp-proportionally over the scenario's 3 dp=1 nodes
    exactly as assign_budgets does (cluster_w * dp / total_dp, sim.hpp:332-334); offered
    load: a few piecewise-constant levels per trace."""
    import json
    import os

    from paper_2605_21427_b200 import profiles
    path = os.path.join(os.path.dirname(profiles.__file__), "data", "scenarios.json")
    with open(path) as f:
        trace = json.load(f)["demand_response"]["trace"]
    return np.array([(t, w * 1.0 / n_nodes) for t, w in trace], SIGNAL_DT)


def build_dr_traces(s, t_max, n_per_model=2, n_steps=7200, seed=5):
    budget = dr_budget()
    rng = np.random.default_rng(seed)
    n_models = len(s["profiles"])
    sig = [budget]
    off = len(budget)
    tr = np.zeros(n_models * n_per_model, TRACE_DT)
    for i in range(len(tr)):
        m = i % n_models
        k = int(rng.integers(2, 9))
        ts = np.sort(rng.uniform(0.0, n_steps * 0.5, k))
        ts[0] = rng.choice([0.0, 12.25])  # a first point after t0 = 0 keeps the front value
        ts[k // 2] = ts[k // 2 - 1]  # duplicate timestamp: the later row wins
        lv = rng.uniform(0.3, 1.2, k) * t_max[m]
        load = np.zeros(k, SIGNAL_DT)
        load["t_s"], load["value"] = ts, lv
        sig.append(load)
        tr[i] = (0, off, rng.uniform(0.3, 0.9) * t_max[m], 0.05, 0.04,
                 int(rng.integers(0, 2**63)), len(budget) if i % 3 else 0, k, m, i % 2)
        off += k
    return tr, np.concatenate(sig)


@pytest.fixture(scope="module")
def setup(reference):
    s = workloads.cfg4_setup()
    return s, ref_plant_constants(reference, s, s["caps"], s["batches"])


def test_synthetic_workload_as_caller_traces(reference, setup):
    s, (t_max, p_min, p_max) = setup
    spec = workloads.replay_spec(96, n_steps=900, seed=77, n_log_traces=12)
    want, wlogs = reference.replay(s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                                   s["batches"], s["cfg"], spec)
    tr, sig = workloads.synthetic_traces(spec, len(s["profiles"]), t_max, p_min, p_max)
    got, _ = reference.replay_traces(s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                                     s["batches"], s["cfg"], tr, sig, spec.n_steps,
                                     n_log_traces=12)
    assert np.array_equal(got["summaries"], want)
    assert np.array_equal(got["logs"], wlogs)


def test_resume_from_returned_state(reference, setup):
    s, (t_max, _, _) = setup
    tr, sig = build_dr_traces(s, t_max, n_steps=2400)
    kw = dict(n_log_traces=len(tr), details=True)
    args = (s["profiles"], s["gpu"], s["coeffs"], s["caps"], s["batches"], s["cfg"], tr, sig)
    full, _ = reference.replay_traces(*args, 2400, **kw)
    a, _ = reference.replay_traces(*args, 1001, **kw)
    b, _ = reference.replay_traces(*args, 1399, first_step=1001, init=a["final_state"],
                                   init_plant=a["final_plant"], **kw)
    n = len(tr)
    la = a["logs"].reshape(n, 1001)
    lb = b["logs"].reshape(n, 1399)
    assert np.array_equal(np.concatenate([la, lb], 1), full["logs"].reshape(n, 2400))
    assert np.array_equal(b["final_state"], full["final_state"])
    assert np.array_equal(b["final_plant"], full["final_plant"])
    # the budget signal moved and budgets bound: decisions were made under budget
    assert (full["logs"]["reason"] == 2).any() and full["summaries"]["n_applied"].sum() > 0
