"""Host-side mirror of the reference's decision API, backed by libpals_gpu.so.

Same names and argument meaning as /root/reference/proj/include/wattserve/
controller.hpp, so the parity tests read like the reference's own:

    analytic_scorer(profile, gpu)                    controller.hpp:107-111
    table_scorer(points, t_hat, p_gpu)               tests/test_controller.cpp:17-29
    select_config(cands, targets, scorer, coeffs,
                  bias, target_headroom, budget_margin)    controller.hpp:132-201
    control_step(telemetry, now_s, targets, cands, scorer,
                 coeffs, state, cfg)                  controller.hpp:210-267

plus the batched B200 entry points (Plan.select for many Targets at once,
replay for many traces). Exceptions mirror the reference's: ConfigError for
config_error, OutOfRange for std::out_of_range. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .abi import (OBJ_BUDGET, OBJ_QOS, PLANT_DT, POINT_DT, QUERY_DT, SIGNAL_DT, STATE_DT,
                  STEPDETAIL_DT, STEPLOG_DT, SUMMARY_DT, TRACE_DT, Coeffs, CtrlCfg, CtrlState,
                  Decision, GpuSpec, Point, Profile, ReplaySpec, Targets, Telemetry, TraceBatch,
                  ptr, state_array)
from ._lib import ConfigError, DataError, OutOfRange, PalsError, check  # noqa: F401

__all__ = [
    "Context", "AnalyticModel", "TableModel", "Grid", "Plan", "analytic_scorer",
    "table_scorer", "select_config", "control_step", "replay", "make_targets",
    "default_context", "Allocator", "AllocResult", "allocate_budget", "replay_with_details",
    "decisions_csv", "fnv1a64", "replay_traces", "replay_traces_device", "ConfigError", "DataError", "OutOfRange", "PalsError",
]


class Context:
    """One GPU, one stream (pals_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        check(self.lib.pals_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            self.lib.pals_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, cuda_stream_ptr: int | None):
        check(self.lib.pals_ctx_set_stream(self.h, C.c_void_p(cuda_stream_ptr or 0)))

    @property
    def stream(self) -> int:
        return self.lib.pals_ctx_stream(self.h) or 0

    def sync(self):
        check(self.lib.pals_ctx_sync(self.h))

    def set_replay_layout(self, layout: str):
        """"thread" (one thread per trace, default) or "warp" (one warp per trace)."""
        check(self.lib.pals_ctx_set_replay_layout(self.h, {"thread": 0, "warp": 1}[layout]))

    def set_sim_streaming(self, on: bool = True):
        """Queue-plant runs stream their arrival uploads behind the running simulation (on,
        the default); off draws and uploads everything first (for kernel profilers)."""
        check(self.lib.pals_sim_set_streaming(self.h, 1 if on else 0))

    def set_one_server(self, idle_us: int):
        """Single calls through the resident server kernel, which exits after idle_us without
        a request (0: one kernel launch per call)."""
        check(self.lib.pals_ctx_set_one_server(self.h, int(idle_us)))

    @property
    def launches(self) -> int:
        return int(self.lib.pals_ctx_launch_count(self.h))


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class _Model:
    kind = "?"

    def __init__(self, ctx: Context, handle: C.c_void_p):
        self.ctx = ctx
        self.h = handle

    def __del__(self):
        try:
            if self.h and self.ctx.h:
                self.ctx.lib.pals_model_destroy(self.h)
        except Exception:
            pass


class AnalyticModel(_Model):
    """analytic_scorer(profile, gpu) (controller.hpp:107-111)."""

    kind = "analytic"

    def __init__(self, ctx: Context, profile: Profile, gpu: GpuSpec):
        h = C.c_void_p()
        check(ctx.lib.pals_model_analytic(ctx.h, C.byref(profile), C.byref(gpu), C.byref(h)))
        super().__init__(ctx, h)
        self.profile = profile
        self.gpu = gpu


class TableModel(_Model):
    """TableScorer (tests/test_controller.cpp:17-29): scores by point value, first match."""

    kind = "table"

    def __init__(self, ctx: Context, points: np.ndarray, t_hat, p_gpu):
        pts = np.ascontiguousarray(points, dtype=POINT_DT)
        t = np.ascontiguousarray(t_hat, np.float64)
        p = np.ascontiguousarray(p_gpu, np.float64)
        h = C.c_void_p()
        check(ctx.lib.pals_model_table(ctx.h, ptr(pts), ptr(t), ptr(p), len(pts), C.byref(h)))
        super().__init__(ctx, h)


def analytic_scorer(profile: Profile, gpu: GpuSpec, ctx: Context | None = None) -> AnalyticModel:
    return AnalyticModel(ctx or default_context(), profile, gpu)


def table_scorer(points, t_hat, p_gpu, ctx: Context | None = None) -> TableModel:
    return TableModel(ctx or default_context(), points, t_hat, p_gpu)


class Grid:
    """A candidate list (std::vector<OperatingPoint>) resident on the device."""

    def __init__(self, ctx: Context, points: np.ndarray):
        self.ctx = ctx
        self.points = np.ascontiguousarray(points, dtype=POINT_DT)
        h = C.c_void_p()
        check(ctx.lib.pals_grid_points(ctx.h, ptr(self.points), len(self.points), C.byref(h)))
        self.h = h

    def __len__(self):
        return len(self.points)

    def __del__(self):
        try:
            if self.h and self.ctx.h:
                self.ctx.lib.pals_grid_destroy(self.h)
        except Exception:
            pass


def eval_grid(model: _Model, grid: Grid):
    """CandidateScore for every grid point: (throughput_tps, gpu_power_w)."""
    n = len(grid)
    T = np.empty(n, np.float64)
    P = np.empty(n, np.float64)
    check(model.ctx.lib.pals_eval(model.ctx.h, model.h, grid.h, ptr(T), ptr(P)))
    return T, P


class Plan:
    """Model x candidate grid x SystemPowerCoeffs, prepared for batched select_config."""

    def __init__(self, model: _Model, grid: Grid, coeffs: Coeffs):
        self.ctx = model.ctx
        self.model = model
        self.grid = grid
        self.coeffs = coeffs
        h = C.c_void_p()
        check(self.ctx.lib.pals_plan_create(self.ctx.h, model.h, grid.h, C.byref(coeffs),
                                            C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h and self.ctx.h:
                self.ctx.lib.pals_plan_destroy(self.h)
        except Exception:
            pass

    def prepare(self):
        check(self.ctx.lib.pals_plan_prepare(self.h))

    def select(self, queries: np.ndarray):
        """Host buffers in and out: one select_config per query. Returns (index, reason)."""
        q = np.ascontiguousarray(queries, dtype=QUERY_DT)
        idx = np.empty(len(q), np.int32)
        rs = np.empty(len(q), np.uint8)
        check(self.ctx.lib.pals_select(self.h, ptr(q), len(q), ptr(idx), ptr(rs)))
        return idx, rs

    def select_device(self, d_queries: int, n: int, d_idx: int, d_reason: int):
        """Device pointers (e.g. torch tensors' data_ptr()); async on the context stream."""
        check(self.ctx.lib.pals_plan_select_device(self.h, C.c_void_p(d_queries), n,
                                                   C.c_void_p(d_idx), C.c_void_p(d_reason)))

    def frontier(self) -> np.ndarray:
        """build_frontier over the plan's (t_hat, eff): point indices, throughput ascending."""
        idx = np.empty(max(1, len(self.grid)), np.int32)
        n = C.c_int64(0)
        check(self.ctx.lib.pals_plan_frontier(self.h, ptr(idx), C.byref(n)))
        return idx[: n.value].copy()

    def frontier_device(self, d_idx: int, d_n: int):
        """Async: frontier indices into d_idx (grid-size capacity), count into d_n (int64)."""
        check(self.ctx.lib.pals_plan_frontier_device(self.h, C.c_void_p(d_idx), C.c_void_p(d_n)))

    def run(self, d_queries: int, n: int, d_idx: int, d_reason: int):
        """One full step (evaluate + rank + select) from a cached CUDA graph; async."""
        check(self.ctx.lib.pals_plan_run(self.h, C.c_void_p(d_queries), n, C.c_void_p(d_idx),
                                         C.c_void_p(d_reason)))

    def scores(self):
        n = len(self.grid)
        th, pn, ef = (np.empty(n, np.float64) for _ in range(3))
        check(self.ctx.lib.pals_plan_scores(self.h, ptr(th), ptr(pn), ptr(ef)))
        return th, pn, ef

    @property
    def last_exact_count(self) -> int:
        return int(self.ctx.lib.pals_plan_last_exact_count(self.h))

    def set_decide(self, mode: str):
        """"scan" (default: the pair scan) or "prefix" (prefix-min tables; same results)."""
        check(self.ctx.lib.pals_plan_set_decide(self.h, {"scan": 0, "prefix": 1}[mode]))

    def force_exact(self, on: bool = True):
        check(self.ctx.lib.pals_plan_set_force_exact(self.h, 1 if on else 0))

    def time_scan(self, on: bool = True):
        check(self.ctx.lib.pals_plan_time_scan(self.h, 1 if on else 0))

    def scan_ms(self) -> float:
        return float(self.ctx.lib.pals_plan_scan_ms(self.h))

    def stats(self) -> np.ndarray:
        """Per-class query counts of the last select (see pals_plan_stats)."""
        c = np.zeros(6, np.int64)
        check(self.ctx.lib.pals_plan_stats(self.h, ptr(c)))
        return c


def measure_peaks(ctx: Context):
    """(integer compare+min ops/s, FP64 flop/s) measured on this device."""
    a = C.c_double()
    b = C.c_double()
    check(ctx.lib.pals_measure_peaks(ctx.h, C.byref(a), C.byref(b)))
    return a.value, b.value


def make_targets(throughput_tps: float, power_budget_w: float | None = None,
                 epsilon: float = 0.05, objective: int = OBJ_QOS) -> Targets:
    """Targets (controller.hpp:19-29); power_budget_w None is std::nullopt."""
    t = Targets()
    t.throughput_tps = throughput_tps
    t.has_budget = 0 if power_budget_w is None else 1
    t.power_budget_w = 0.0 if power_budget_w is None else power_budget_w
    t.epsilon = epsilon
    t.objective = objective
    return t


def make_queries(throughput_tps, power_budget_w=None, bias=1.0, target_headroom=0.0,
                 budget_margin=0.0, objective=OBJ_QOS) -> np.ndarray:
    """Vectorised pals_query array; power_budget_w entries that are NaN mean no budget."""
    tps = np.atleast_1d(np.asarray(throughput_tps, np.float64))
    n = len(tps)
    q = np.zeros(n, QUERY_DT)
    q["throughput_tps"] = tps
    if power_budget_w is None:
        q["has_budget"] = 0
    else:
        b = np.broadcast_to(np.asarray(power_budget_w, np.float64), (n,))
        q["has_budget"] = (~np.isnan(b)).astype(np.int32)
        q["power_budget_w"] = np.where(np.isnan(b), 0.0, b)
    q["bias"] = bias
    q["target_headroom"] = target_headroom
    q["budget_margin"] = budget_margin
    q["objective"] = objective
    return q


def _points(candidates) -> np.ndarray:
    if isinstance(candidates, np.ndarray):
        return np.ascontiguousarray(candidates, dtype=POINT_DT)
    pts = np.zeros(len(candidates), POINT_DT)
    for i, c in enumerate(candidates):
        pts[i] = (c.cap_watts, c.batch, c.tp, c.ep, c.dp) if isinstance(c, Point) else tuple(c)
    return pts


def select_config(candidates, targets: Targets, scorer: _Model, coeffs: Coeffs,
                  bias: float = 1.0, target_headroom: float = 0.0,
                  budget_margin: float = 0.0) -> Decision:
    """select_config (controller.hpp:132-201), one call, on the GPU."""
    pts = _points(candidates)
    d = Decision()
    ctx = scorer.ctx
    check(ctx.lib.pals_select_one(ctx.h, scorer.h, ptr(pts), len(pts), C.byref(targets),
                                  C.byref(coeffs), bias, target_headroom, budget_margin,
                                  C.byref(d)))
    return d


def control_step(telemetry: Telemetry, now_s: float, targets: Targets, candidates,
                 scorer: _Model, coeffs: Coeffs, state: CtrlState, cfg: CtrlCfg):
    """control_step (controller.hpp:210-267), one call, on the GPU."""
    pts = _points(candidates)
    d = Decision()
    st = CtrlState()
    ctx = scorer.ctx
    check(ctx.lib.pals_control_step_one(ctx.h, scorer.h, C.byref(telemetry), now_s,
                                        C.byref(targets), ptr(pts), len(pts), C.byref(coeffs),
                                        C.byref(state), C.byref(cfg), C.byref(d), C.byref(st)))
    return d, st


def replay(ctx: Context, models, plant, gpu: GpuSpec, coeffs: Coeffs, caps, batches,
           cfg: CtrlCfg, spec: ReplaySpec, summaries: np.ndarray | None = None):
    """Batched control_step replay over spec.n_traces synthetic traces (host outputs).
    `summaries` may be a caller-owned (e.g. pinned) SUMMARY_DT array of n_traces."""
    n_models = len(models)
    hs = (C.c_void_p * n_models)(*[m.h for m in models])
    profs = (Profile * n_models)(*plant)
    caps = np.ascontiguousarray(caps, np.float64)
    batches = np.ascontiguousarray(batches, np.int32)
    summ = np.zeros(spec.n_traces, SUMMARY_DT) if summaries is None else summaries
    assert summ.dtype == SUMMARY_DT and len(summ) >= spec.n_traces
    nl = min(spec.n_log_traces, spec.n_traces)
    logs = np.zeros(max(1, nl * spec.n_steps), STEPLOG_DT)
    check(ctx.lib.pals_replay(ctx.h, n_models, hs, profs, C.byref(gpu), C.byref(coeffs),
                              ptr(caps), len(caps), ptr(batches), len(batches), C.byref(cfg),
                              C.byref(spec), ptr(summ), ptr(logs) if nl else None))
    return summ, logs[: nl * spec.n_steps]


def replay_with_details(ctx: Context, models, plant, gpu: GpuSpec, coeffs: Coeffs, caps,
                        batches, cfg: CtrlCfg, spec: ReplaySpec):
    """replay() plus the per-step DecisionRecord err_norm / bias (STEPDETAIL_DT) of the
    logged traces: (summaries, logs, details)."""
    n_models = len(models)
    hs = (C.c_void_p * n_models)(*[m.h for m in models])
    profs = (Profile * n_models)(*plant)
    caps = np.ascontiguousarray(caps, np.float64)
    batches = np.ascontiguousarray(batches, np.int32)
    summ = np.zeros(spec.n_traces, SUMMARY_DT)
    nl = min(spec.n_log_traces, spec.n_traces)
    logs = np.zeros(max(1, nl * spec.n_steps), STEPLOG_DT)
    det = np.zeros(max(1, nl * spec.n_steps), STEPDETAIL_DT)
    check(ctx.lib.pals_replay_ex(ctx.h, n_models, hs, profs, C.byref(gpu), C.byref(coeffs),
                                 ptr(caps), len(caps), ptr(batches), len(batches), C.byref(cfg),
                                 C.byref(spec), ptr(summ), ptr(logs) if nl else None,
                                 ptr(det) if nl else None))
    return summ, logs[: nl * spec.n_steps], det[: nl * spec.n_steps]


def decisions_csv(spec: ReplaySpec, plant, caps, batches, summaries, logs, details) -> bytes:
    """The reference's decisions CSV (metrics.hpp:145-157) of a replay's logged traces,
    formatted by libpals_gpu (host code; no device needed)."""
    lib = _lib.load(build_if_missing=False)
    profs = (Profile * len(plant))(*plant)
    caps = np.ascontiguousarray(caps, np.float64)
    batches = np.ascontiguousarray(batches, np.int32)
    summ = np.ascontiguousarray(summaries, SUMMARY_DT)
    logs = np.ascontiguousarray(logs, STEPLOG_DT)
    det = np.ascontiguousarray(details, STEPDETAIL_DT)
    n = C.c_int64(0)
    args = [C.byref(spec), profs, len(plant), ptr(caps), len(caps), ptr(batches), len(batches),
            ptr(summ), ptr(logs), ptr(det)]
    check(lib.pals_decisions_csv(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(max(1, n.value))
    check(lib.pals_decisions_csv(*args, buf, n.value, C.byref(n)))
    return buf.raw[: n.value]


def fnv1a64(data: bytes) -> int:
    """rng.hpp:22-28 — the per-file hash of the reference's run manifests."""
    lib = _lib.load(build_if_missing=False)
    return int(lib.pals_fnv1a64(data, len(data)))


def replay_device(ctx: Context, models, plant, gpu: GpuSpec, coeffs: Coeffs, caps, batches,
                  cfg: CtrlCfg, spec: ReplaySpec, d_summaries: int, d_logs: int = 0):
    """Device-resident outputs; async on the context stream."""
    n_models = len(models)
    hs = (C.c_void_p * n_models)(*[m.h for m in models])
    profs = (Profile * n_models)(*plant)
    caps = np.ascontiguousarray(caps, np.float64)
    batches = np.ascontiguousarray(batches, np.int32)
    check(ctx.lib.pals_replay_device(ctx.h, n_models, hs, profs, C.byref(gpu), C.byref(coeffs),
                                     ptr(caps), len(caps), ptr(batches), len(batches),
                                     C.byref(cfg), C.byref(spec), C.c_void_p(d_summaries),
                                     C.c_void_p(d_logs)))


def _replay_common(models, plant, caps, batches):
    n_models = len(models)
    hs = (C.c_void_p * n_models)(*[m.h for m in models])
    profs = (Profile * n_models)(*plant)
    return (n_models, hs, profs, np.ascontiguousarray(caps, np.float64),
            np.ascontiguousarray(batches, np.int32))


def replay_traces(ctx: Context, models, plant, gpu: GpuSpec, coeffs: Coeffs, caps, batches,
                  cfg: CtrlCfg, traces: np.ndarray, signal: np.ndarray, n_steps: int,
                  interval_s: float = 0.5, first_step: int = 0, init=None, init_plant=None,
                  n_log_traces: int = 0, details: bool = False, summaries=None):
    """control_step replayed over caller traces (pals_replay_traces; host buffers).

    traces: TRACE_DT array (model, objective, target, epsilon, noise, signal slices);
    signal: SIGNAL_DT array of (t_s, value) rows — the reference's budget-trace
    representation, read with detail::trace_value semantics (sim.hpp:167-174).
    init: STATE_DT array / CtrlState list or None (ControllerState{} at max cap and
    batch); init_plant: PLANT_DT array or None. Returns a dict with summaries,
    final_state (STATE_DT), final_plant (PLANT_DT), logs and details."""
    n_models, hs, profs, caps, batches = _replay_common(models, plant, caps, batches)
    tr = np.ascontiguousarray(traces, TRACE_DT)
    sig = np.ascontiguousarray(signal, SIGNAL_DT)
    n = len(tr)
    ini = None if init is None else state_array(init)
    inp = None if init_plant is None else np.ascontiguousarray(init_plant, PLANT_DT)
    summ = np.zeros(n, SUMMARY_DT) if summaries is None else summaries
    fin = np.zeros(n, STATE_DT)
    finp = np.zeros(n, PLANT_DT)
    nl = min(max(n_log_traces, 0), n)
    logs = np.zeros(max(1, nl * n_steps), STEPLOG_DT)
    det = np.zeros(max(1, nl * n_steps), STEPDETAIL_DT) if details else None
    b = TraceBatch(n_traces=n, first_step=first_step, n_steps=n_steps, n_log_traces=nl,
                   interval_s=interval_s, traces=ptr(tr).value if n else None,
                   signal=ptr(sig).value if len(sig) else None, n_signal=len(sig),
                   init=None if ini is None else ptr(ini).value,
                   init_plant=None if inp is None else ptr(inp).value,
                   summaries=ptr(summ).value if n else None, final_state=ptr(fin).value,
                   final_plant=ptr(finp).value, logs=ptr(logs).value if nl else None,
                   details=ptr(det).value if (nl and details) else None)
    check(ctx.lib.pals_replay_traces(ctx.h, n_models, hs, profs, C.byref(gpu), C.byref(coeffs),
                                     ptr(caps), len(caps), ptr(batches), len(batches),
                                     C.byref(cfg), C.byref(b)))
    out = {"summaries": summ[:n], "final_state": fin, "final_plant": finp,
           "logs": logs[: nl * n_steps]}
    if details:
        out["details"] = det[: nl * n_steps]
    return out


def replay_traces_device(ctx: Context, models, plant, gpu: GpuSpec, coeffs: Coeffs, caps,
                         batches, cfg: CtrlCfg, batch: TraceBatch):
    """pals_replay_traces_device: every pointer of `batch` device-resident; async."""
    n_models, hs, profs, caps, batches = _replay_common(models, plant, caps, batches)
    check(ctx.lib.pals_replay_traces_device(ctx.h, n_models, hs, profs, C.byref(gpu),
                                            C.byref(coeffs), ptr(caps), len(caps), ptr(batches),
                                            len(batches), C.byref(cfg), C.byref(batch)))


OBJECTIVES = {"qos": OBJ_QOS, "budget-throughput": OBJ_BUDGET}


class Allocator:
    """Batched allocate_budget (allocator.hpp:76-186) over many independent clusters.

    models[k] scores the candidates of nodes running model k: caps x batches at
    deploy[k]'s deployment tp/ep and the node's dp (sim.hpp:318-331). Step tables for
    every (model, dp <= max_dp) are built once here (pals_alloc_create)."""

    def __init__(self, ctx: Context, models, deploy, gpu: GpuSpec, coeffs: Coeffs, caps,
                 batches, max_dp: int = 8, selection_margin: float = 0.0):
        self.ctx, self.lib = ctx, ctx.lib
        self.models = list(models)  # keep the handles alive
        n = len(self.models)
        hs = (C.c_void_p * n)(*[m.h for m in self.models])
        profs = (Profile * n)(*deploy)
        self.caps = np.ascontiguousarray(caps, np.float64)
        self.batches = np.ascontiguousarray(batches, np.int32)
        self.gpu, self.coeffs, self.max_dp = gpu, coeffs, max_dp
        self.max_cand = max(1, len(self.caps) * len(self.batches))
        self.names = [bytes(p.name).split(b"\0")[0].decode() for p in deploy]
        h = C.c_void_p()
        check(self.lib.pals_alloc_create(ctx.h, n, hs, profs, C.byref(gpu), C.byref(coeffs),
                                         ptr(self.caps), len(self.caps), ptr(self.batches),
                                         len(self.batches), max_dp, selection_margin,
                                         C.byref(h)))
        self.h = h

    @classmethod
    def from_sets(cls, ctx: Context, sets, gpu: GpuSpec, coeffs: Coeffs,
                  selection_margin: float = 0.0, names=None):
        """General AllocRequest form: sets = [(model, candidate points)]; nodes then name a
        set index in node_model (their dp only sets the floor)."""
        self = cls.__new__(cls)
        self.ctx, self.lib = ctx, ctx.lib
        self.models = [m for m, _ in sets]
        pts = [np.ascontiguousarray(p, dtype=POINT_DT) for _, p in sets]
        off = np.zeros(len(sets) + 1, np.int64)
        off[1:] = np.cumsum([len(p) for p in pts])
        allp = np.concatenate(pts) if pts else np.zeros(0, POINT_DT)
        allp = np.ascontiguousarray(allp if len(allp) else np.zeros(1, POINT_DT))
        self.gpu, self.coeffs, self.max_dp = gpu, coeffs, 0
        self.max_cand = max([1] + [len(p) for p in pts])
        self.names = list(names) if names else [str(i) for i in range(len(sets))]
        hs = (C.c_void_p * len(sets))(*[m.h for m in self.models])
        h = C.c_void_p()
        check(self.lib.pals_alloc_create_sets(ctx.h, len(sets), hs, ptr(allp), ptr(off),
                                              C.byref(gpu), C.byref(coeffs), selection_margin,
                                              C.byref(h)))
        self.h = h
        return self

    def close(self):
        if getattr(self, "h", None):
            self.lib.pals_alloc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def steps(self, model: int, dp: int | None = None):
        """detail::throughput_steps (margin-scaled) of one set, (power_w, thr). In the
        (model, dp) form pass both; in the from_sets form pass the set index only."""
        set_ = model if dp is None else model * self.max_dp + dp - 1
        n = C.c_int32(0)
        pw, th = np.empty(self.max_cand), np.empty(self.max_cand)
        check(self.lib.pals_alloc_steps(self.h, set_, ptr(pw), ptr(th), C.byref(n)))
        return pw[: n.value].copy(), th[: n.value].copy()

    def allocate(self, off, node_model, node_dp, node_target, cluster_budget,
                 quantum_w: float = 25.0):
        """Host arrays in/out. Returns dict(node_budget, total, all_sat, status)."""
        off = np.ascontiguousarray(off, np.int64)
        npb = len(off) - 1
        node_model = np.ascontiguousarray(node_model, np.int32)
        node_dp = np.ascontiguousarray(node_dp, np.int32)
        node_target = np.ascontiguousarray(node_target, np.float64)
        cluster_budget = np.ascontiguousarray(cluster_budget, np.float64)
        nn = int(off.max()) if npb > 0 else 0
        if min(len(node_model), len(node_dp), len(node_target)) < nn or len(cluster_budget) < npb:
            raise ConfigError(2, "allocate: node/problem arrays shorter than node_offset implies")
        out = dict(node_budget=np.zeros(nn), total=np.zeros(npb),
                   all_sat=np.zeros(npb, np.uint8), status=np.zeros(npb, np.int32))
        check(self.lib.pals_allocate_budget(
            self.h, quantum_w, npb, ptr(off), ptr(node_model), ptr(node_dp), ptr(node_target),
            ptr(cluster_budget), ptr(out["node_budget"]), ptr(out["total"]), ptr(out["all_sat"]),
            ptr(out["status"])))
        return out

    def run_device(self, quantum_w, n_problems, n_nodes, d_off, d_model, d_dp, d_target,
                   d_budget, d_node_budget, d_total, d_all_sat, d_status):
        """Device pointers (ints); async on the context stream."""
        v = C.c_void_p
        check(self.lib.pals_alloc_run_device(self.h, quantum_w, n_problems, v(d_off), n_nodes,
                                             v(d_model), v(d_dp), v(d_target), v(d_budget),
                                             v(d_node_budget), v(d_total), v(d_all_sat),
                                             v(d_status)))


class AllocResult:
    """AllocResult (allocator.hpp:24-28)."""

    def __init__(self, node_budgets_w, total_allocated_w, all_targets_satisfied):
        self.node_budgets_w = list(node_budgets_w)
        self.total_allocated_w = float(total_allocated_w)
        self.all_targets_satisfied = bool(all_targets_satisfied)


def allocate_budget(allocator: Allocator, nodes, cluster_budget_w: float,
                    quantum_w: float = 25.0) -> AllocResult:
    """allocate_budget(nodes, cluster_budget_w, gpu, coeffs, quantum_w, selection_margin)
    (allocator.hpp:76) for one cluster: nodes = [(model_index, dp, throughput_target_tps)].
    gpu, coeffs, the candidate axes and the margin are the allocator's. Raises ConfigError
    with the reference's message when the budget is below the node floors."""
    nodes = list(nodes)
    if not nodes:
        raise ConfigError(2, "allocate_budget: no nodes")
    m = np.array([n[0] for n in nodes], np.int32)
    d = np.array([n[1] for n in nodes], np.int32)
    t = np.array([n[2] for n in nodes], np.float64)
    out = allocator.allocate([0, len(nodes)], m, d, t, [cluster_budget_w], quantum_w)
    st = int(out["status"][0])
    if st != 0:
        g, k = allocator.gpu, allocator.coeffs
        unit = k.alpha * 4 * g.min_cap_watts + k.beta_watts
        floors = [int(x) * unit for x in d]
        if sum(floors) > cluster_budget_w:  # allocator.hpp:87-95
            parts = ", ".join(f"{allocator.names[i] if 0 <= i < len(allocator.names) else i}"
                              f"={f:g} W" for i, f in zip(m, floors))
            raise ConfigError(st, f"allocate_budget: cluster budget {cluster_budget_w:g} W "
                                  f"below the sum of node floors ({parts})")
        cls = {2: ConfigError, 3: DataError, 5: OutOfRange}.get(st, PalsError)
        raise cls(st, "allocate_budget: a node's scorer rejected its candidates")
    return AllocResult(out["node_budget"], out["total"][0], out["all_sat"][0])
