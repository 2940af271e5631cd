"""Synthetic workloads of BASELINE.json's configs.

cfg1  bundled: llama2-7b-like, 6 caps x 6 batches at its deployment tp (36 candidates),
      one target 0.6 x unconstrained throughput, one static 1600 W budget.
cfg2  dense 8B: llama2-7b-like + comm_fixed_by_tp[8] = 2*comm_fixed_by_tp[4];
      caps[i] = 100 + 300 i/63 (64), batches 1..256, tp {1,2,4,8} -> 65,536 configs;
      1e4 QoS targets from splitmix64(2605 ^ q).
cfg3  MoE: mixtral-8x7b-like (+tp8), same 64x256x4 grid at ep=8; 1e6 (target, budget)
      queries, QoS / budget-throughput 50/50, budget U(600, 2000) W, margin 0.02.
cfg4  replay: 1e6 traces x 3600 steps over the 8 profiles, 36 candidates each.
cfg5  replay stress: 1e7 traces as cfg4, sharded over GPUs.

Everything is a pure function of (seed, index), so every arm (GPU, oracle, the
reference build) sees bit-identical inputs.
"""
from __future__ import annotations

import numpy as np

from .abi import (OBJ_BUDGET, OBJ_QOS, POINT_DT, QUERY_DT, SIGNAL_DT, TRACE_DT, ReplaySpec,
                  default_ctrl_cfg)
from .profiles import comm_of, load_bundle, profile_by_name, with_comm

GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """rng.hpp:15-20, vectorised (uint64 arithmetic wraps)."""
    x = np.asarray(x, dtype=np.uint64) + GOLDEN
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def u01(u: np.ndarray) -> np.ndarray:
    return (u >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def cfg2_caps() -> np.ndarray:
    return np.array([100.0 + 300.0 * i / 63.0 for i in range(64)], np.float64)


def grid_points(caps, batches, tps, eps=(1,), dps=(1,)) -> np.ndarray:
    """Canonical sweep nesting cap -> batch -> tp -> ep -> dp (sweep.hpp:134-138)."""
    caps = np.asarray(caps, np.float64)
    b = np.asarray(batches, np.int32)
    t = np.asarray(tps, np.int32)
    e = np.asarray(eps, np.int32)
    d = np.asarray(dps, np.int32)
    C, B, T, E, D = np.meshgrid(caps, b, t, e, d, indexing="ij")
    pts = np.zeros(C.size, POINT_DT)
    pts["cap_watts"] = C.ravel()
    pts["batch"] = B.ravel()
    pts["tp"] = T.ravel()
    pts["ep"] = E.ravel()
    pts["dp"] = D.ravel()
    return pts


def gen_queries(n: int, seed: int, t_ref: float, objective: str = "qos",
                budget: tuple | None = None, headroom: float = 0.05,
                margin: float = 0.02, first: int = 0) -> np.ndarray:
    """Queries q in [first, first+n): target U(0.05,1)*t_ref, bias 1.0 (half) or U(0.5,2)."""
    qi = np.arange(first, first + n, dtype=np.uint64)
    k = splitmix64(np.uint64(seed) ^ qi)
    r = [u01(splitmix64(k + np.uint64((j * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)))
         for j in range(1, 6)]
    q = np.zeros(n, QUERY_DT)
    q["throughput_tps"] = (0.05 + 0.95 * r[0]) * t_ref
    q["bias"] = np.where(r[1] < 0.5, 1.0, 0.5 + 1.5 * r[2])
    q["target_headroom"] = headroom
    if budget is not None:
        q["has_budget"] = 1
        q["power_budget_w"] = budget[0] + (budget[1] - budget[0]) * r[3]
        q["budget_margin"] = margin
    if objective == "qos":
        q["objective"] = OBJ_QOS
    elif objective == "budget":
        q["objective"] = OBJ_BUDGET
    else:  # mixed 50/50
        q["objective"] = np.where(r[4] < 0.5, OBJ_QOS, OBJ_BUDGET)
    return q


def dense_profile(profiles, name: str):
    """Profile + synthetic tp=8 comm cost: 2 x comm_fixed_by_tp[4]."""
    p = profile_by_name(profiles, name)
    return with_comm(p, 8, 2.0 * comm_of(p, 4))


def cfg1():
    profs, gpu, coeffs = load_bundle()
    p = profile_by_name(profs, "llama2-7b-like")
    caps = [150.0, 200.0, 250.0, 300.0, 350.0, 400.0]
    batches = [1, 4, 8, 16, 32, 64]
    pts = grid_points(caps, batches, [p.deploy_tp], [p.deploy_ep], [p.deploy_dp])
    return dict(name="cfg1", profile=p, gpu=gpu, coeffs=coeffs, points=pts, caps=caps,
                batches=batches)


def cfg2(n_queries: int = 10_000, budget: bool = False):
    profs, gpu, coeffs = load_bundle()
    p = dense_profile(profs, "llama2-7b-like")
    pts = grid_points(cfg2_caps(), np.arange(1, 257), [1, 2, 4, 8])
    return dict(name="cfg2", profile=p, gpu=gpu, coeffs=coeffs, points=pts,
                n_queries=n_queries, seed=2605, objective="qos",
                budget=(600.0, 2000.0) if budget else None)


def cfg3(n_queries: int = 1_000_000):
    profs, gpu, coeffs = load_bundle()
    p = dense_profile(profs, "mixtral-8x7b-like")
    pts = grid_points(cfg2_caps(), np.arange(1, 257), [1, 2, 4, 8], [8], [1])
    return dict(name="cfg3", profile=p, gpu=gpu, coeffs=coeffs, points=pts,
                n_queries=n_queries, seed=2605, objective="mixed", budget=(600.0, 2000.0))


def replay_spec(n_traces: int, n_steps: int = 3600, seed: int = 2605, first: int = 0,
                objective_mode: int = 2, n_log_traces: int = 0) -> ReplaySpec:
    """cfg4/cfg5 fluid-plant traces."""
    s = ReplaySpec()
    s.seed = seed
    s.first_trace = first
    s.n_traces = n_traces
    s.n_steps = n_steps
    s.objective_mode = objective_mode
    s.interval_s = 0.5
    s.qos_frac_lo, s.qos_frac_hi = 0.3, 0.9
    s.load_lo, s.load_hi = 0.3, 1.2
    s.noise_amp = 0.04
    s.budget_lo_frac, s.budget_hi_frac = 0.9, 1.1
    s.epsilon = 0.05
    s.seg_min, s.seg_max = 60, 480
    s.budget_mode = 1
    s.n_log_traces = n_log_traces
    return s


def _draw(key, lane: int, ctr) -> np.ndarray:
    """draw(key, lane, ctr) = splitmix64(key ^ lane << 48 ^ ctr)."""
    return splitmix64(key ^ (np.uint64(lane) << np.uint64(48)) ^ np.asarray(ctr, np.uint64))


def synthetic_traces(spec: ReplaySpec, n_models: int, t_max, p_min, p_max):
    """The synthetic replay workload of `spec` written out as caller traces
    for pals_replay_traces: per trace its model, objective, target and noise key, and its
    piecewise-constant budget / offered-load segments as (t_s, value) signal rows starting
    at step S_j (t_s = S_j * interval_s). Replaying these traces gives the synthetic path's
    decisions bit for bit. t_max / p_min / p_max: per model, the plant's unconstrained
    throughput and the min / max p_node over the candidates (what the generator scales by).
    Returns (traces TRACE_DT, signal SIGNAL_DT)."""
    n = int(spec.n_traces)
    t_max, p_min, p_max = (np.asarray(x, np.float64) for x in (t_max, p_min, p_max))
    gi = np.uint64(spec.first_trace) + np.arange(n, dtype=np.uint64)
    key = splitmix64(np.uint64(spec.seed) ^ gi)
    model = (key % np.uint64(n_models)).astype(np.int64)
    if spec.objective_mode == 2:
        obj = (_draw(key, 0, 0) >> np.uint64(63)).astype(np.int32)
    else:
        obj = np.full(n, spec.objective_mode, np.int32)
    qfrac = spec.qos_frac_lo + (spec.qos_frac_hi - spec.qos_frac_lo) * u01(_draw(key, 0, 1))
    span = np.uint64(spec.seg_max - spec.seg_min + 1)

    def segments(lane, lo, hi):
        """Seg::at: segment j starts at S_j = sum of earlier lengths; kept while S_j < n_steps."""
        start = np.zeros(n, np.int64)
        rows_t, rows_v, rows_i = [], [], []
        act = np.arange(n)
        j = 0
        while len(act):
            k = key[act]
            ln = spec.seg_min + (_draw(k, lane, 2 * j) % span).astype(np.int64)
            u = u01(_draw(k, lane, 2 * j + 1))
            lvl = lo[act] + (hi[act] - lo[act]) * u
            rows_i.append(act)
            rows_t.append(start[act].astype(np.float64) * spec.interval_s)
            rows_v.append(lvl)
            start[act] += ln
            act = act[start[act] < spec.n_steps]
            j += 1
        i = np.concatenate(rows_i)
        order = np.argsort(i, kind="stable")  # per trace, in segment order
        cnt = np.bincount(i, minlength=n)
        return np.concatenate(rows_t)[order], np.concatenate(rows_v)[order], cnt

    lt, lv, lc = segments(2, spec.load_lo * t_max[model], spec.load_hi * t_max[model])
    if spec.budget_mode:
        bt, bv, bc = segments(1, spec.budget_lo_frac * p_min[model],
                              spec.budget_hi_frac * p_max[model])
    else:
        bt, bv, bc = np.zeros(0), np.zeros(0), np.zeros(n, np.int64)
    signal = np.zeros(len(bt) + len(lt), SIGNAL_DT)
    signal["t_s"][: len(bt)], signal["value"][: len(bt)] = bt, bv
    signal["t_s"][len(bt):], signal["value"][len(bt):] = lt, lv
    tr = np.zeros(n, TRACE_DT)
    tr["budget_off"] = np.concatenate([[0], np.cumsum(bc)[:-1]]) if n else 0
    tr["n_budget"] = bc
    tr["load_off"] = len(bt) + (np.concatenate([[0], np.cumsum(lc)[:-1]]) if n else 0)
    tr["n_load"] = lc
    tr["target_tps"] = qfrac * t_max[model]
    tr["epsilon"] = spec.epsilon
    tr["noise_amp"] = spec.noise_amp
    tr["noise_key"] = key
    tr["model"] = model
    tr["objective"] = obj
    return tr, signal


def plant_constants(ctx, plant, gpu, coeffs, caps, batches):
    """Per model: (t_max, p_min, p_max) the synthetic generator scales by — the plant's
    unconstrained throughput at (max cap, max batch) (sim.hpp:258-264) and the p_node range
    over the candidates — from the library's own evaluation (pals_eval)."""
    from .wattserve import AnalyticModel, Grid, eval_grid
    t_max, p_min, p_max = [], [], []
    for p in plant:
        pts = grid_points(caps, batches, [p.deploy_tp], [p.deploy_ep], [p.deploy_dp])
        T, P = eval_grid(AnalyticModel(ctx, p, gpu), Grid(ctx, pts))
        dp = float(p.deploy_dp)
        pn = dp * (coeffs.alpha * 4.0 * P + coeffs.beta_watts)
        i = int(np.flatnonzero((pts["cap_watts"] == np.max(caps)) &
                               (pts["batch"] == np.max(batches)))[0])
        t_max.append(dp * T[i])
        p_min.append(float(pn.min()))
        p_max.append(float(pn.max()))
    return np.array(t_max), np.array(p_min), np.array(p_max)


def dr_candidates():
    """The demand-response scenario's dense candidate grid (data/scenarios/
    demand_response.json: caps 100..400 W step 5, 24 batch sizes) = 1,464 points."""
    caps = np.arange(100.0, 400.0 + 1e-9, 5.0)
    batches = np.array([1, 2, 3, 4, 5, 6, 8, 10, 12, 14, 16, 18, 20, 24, 28, 32, 36, 40, 44, 48,
                        52, 56, 60, 64], np.int32)
    return caps, batches


def cfg3_extended():
    """cfg3 with the EP x DP axes: 64 x 256 x TP{1,2,4,8} x EP{1,4,8} x DP{1,2,3} = 589,824."""
    profs, gpu, coeffs = load_bundle()
    p = dense_profile(profs, "mixtral-8x7b-like")
    pts = grid_points(cfg2_caps(), np.arange(1, 257), [1, 2, 4, 8], [1, 4, 8], [1, 2, 3])
    return dict(name="cfg3x", profile=p, gpu=gpu, coeffs=coeffs, points=pts)


def cfg4_setup():
    """8 profiles, 6x6 candidates at each profile's deployment, scenario_io defaults."""
    profs, gpu, coeffs = load_bundle()
    caps = np.array([150.0, 200.0, 250.0, 300.0, 350.0, 400.0])
    batches = np.array([1, 4, 8, 16, 32, 64], np.int32)
    # scenario_io.hpp:60-71: headroom defaults to epsilon, budget_margin to 0.02
    cfg = default_ctrl_cfg(target_headroom=0.05, budget_margin=0.02)
    return dict(profiles=profs, gpu=gpu, coeffs=coeffs, caps=caps, batches=batches, cfg=cfg)


def alloc_problems(n_problems: int, seed: int, t_max, p_max, gpu, coeffs, max_nodes: int = 8,
                   first: int = 0):
    """Independent allocate_budget problems (allocator.hpp:76): each cluster has 1..max_nodes
    nodes drawn from the profiles (model m, dp in {1,2,3}), targets U(0.2,1.0) of the node's
    unconstrained throughput, and a cluster budget between the node floors and 1.15x the
    sum of the nodes' peak draw (3% of problems fall below the floors: the error path).
    t_max[m] / p_max[m]: unconstrained throughput and peak p_node of model m at dp = 1."""
    pi = np.arange(first, first + n_problems, dtype=np.uint64)
    k = splitmix64(np.uint64(seed) ^ pi)
    nn = 1 + (k % np.uint64(max_nodes)).astype(np.int64)
    off = np.zeros(n_problems + 1, np.int64)
    off[1:] = np.cumsum(nn)
    tot = int(off[-1])
    owner = np.repeat(np.arange(n_problems), nn)
    local = np.arange(tot) - off[owner]
    kn = splitmix64(k[owner] ^ (np.uint64(0xA5A5) + local.astype(np.uint64)))
    n_models = len(t_max)
    model = (kn % np.uint64(n_models)).astype(np.int32)
    dp = (1 + (splitmix64(kn + np.uint64(1)) % np.uint64(3))).astype(np.int32)
    u = u01(splitmix64(kn + np.uint64(2)))
    t_max = np.asarray(t_max, np.float64)
    p_max = np.asarray(p_max, np.float64)
    target = (0.2 + 0.8 * u) * t_max[model] * dp
    floor = dp * (coeffs.alpha * 4.0 * gpu.min_cap_watts + coeffs.beta_watts)
    floor_sum = np.add.reduceat(floor, off[:-1])
    peak_sum = np.add.reduceat(p_max[model] * dp, off[:-1])
    ub = u01(splitmix64(k + np.uint64(3)))
    budget = floor_sum + ub * (1.15 * peak_sum - floor_sum)
    below = u01(splitmix64(k + np.uint64(4))) < 0.03
    budget = np.where(below, 0.9 * floor_sum, budget)
    return dict(off=off, model=model, dp=dp, target=target, budget=budget)


def predict_points(n: int, seed: int = 2605) -> np.ndarray:
    """Random operating points for predictor throughput (continuous caps, any batch)."""
    k = splitmix64(np.uint64(seed) ^ np.arange(n, dtype=np.uint64))
    r = [splitmix64(k + np.uint64((j * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF))
         for j in range(1, 6)]
    pts = np.zeros(n, POINT_DT)
    pts["cap_watts"] = 100.0 + 300.0 * u01(r[0])
    pts["batch"] = 1 + (r[1] % np.uint64(256)).astype(np.int32)
    pts["tp"] = np.array([1, 2, 4, 8], np.int32)[(r[2] % np.uint64(4)).astype(np.int64)]
    pts["ep"] = np.array([1, 4, 8], np.int32)[(r[3] % np.uint64(3)).astype(np.int64)]
    pts["dp"] = 1 + (r[4] % np.uint64(3)).astype(np.int32)
    return pts


def max_t_hat(profile, gpu, points) -> float:
    """Reference scale for query targets: max dp*T over the grid, from the GPU eval."""
    from .wattserve import AnalyticModel, Grid, default_context, eval_grid
    ctx = default_context()
    T, _ = eval_grid(AnalyticModel(ctx, profile, gpu), Grid(ctx, points))
    return float(np.max(T * points["dp"]))
