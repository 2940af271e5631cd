"""Pareto frontier API mirroring /root/reference/proj/include/wattserve/pareto.hpp.

    build_frontier(points)                      pareto.hpp:31-59   (on the GPU)
    evaluate_regime(regime, profile, gpu, ...)  pareto.hpp:114-135 (eval + frontier on the GPU)
    verify_dominance(a, b)                      pareto.hpp:66-83   (host; frontiers are small)
    default_regimes / regime_by_name            pareto.hpp:88-111
    peak_efficiency(frontier)                   pareto.hpp:137-141

The frontier of a dense grid is one prepared plan plus four small kernels
(csrc/frontier.cu). There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import ConfigError, check
from .abi import POINT_DT, Coeffs, GpuSpec, Profile, ptr
from .wattserve import AnalyticModel, Context, Grid, Plan, default_context


@dataclass
class FrontierPoint:
    """FrontierPoint (pareto.hpp:12-16); point = (cap_watts, batch, tp, ep, dp)."""
    point: tuple
    throughput_tps: float
    efficiency_tpj: float


@dataclass
class RegimeSpec:
    """RegimeSpec (pareto.hpp:88-96)."""
    name: str
    sweep_cap: bool = False
    sweep_batch: bool = False
    sweep_tp: bool = False
    fixed_cap_w: float = 300.0
    fixed_batch: int = 64


def default_regimes():
    return [RegimeSpec("sw-only", False, True, True, 300.0, 64),
            RegimeSpec("hw-only", True, False, False, 300.0, 64),
            RegimeSpec("hw-sw", True, True, False, 300.0, 64),
            RegimeSpec("joint", True, True, True, 300.0, 64)]


def regime_by_name(name: str) -> RegimeSpec:
    for r in default_regimes():
        if r.name == name:
            return r
    valid = ", ".join(r.name for r in default_regimes())
    raise ConfigError(2, f"unknown regime '{name}' (valid: {valid})")


def weakly_dominates(p: FrontierPoint, q: FrontierPoint) -> bool:
    return p.throughput_tps >= q.throughput_tps and p.efficiency_tpj >= q.efficiency_tpj


def strictly_dominates(p: FrontierPoint, q: FrontierPoint) -> bool:
    return weakly_dominates(p, q) and (p.throughput_tps > q.throughput_tps or
                                       p.efficiency_tpj > q.efficiency_tpj)


def frontier_indices(points, throughput, efficiency, ctx: Context | None = None) -> np.ndarray:
    """build_frontier on the device over arrays: indices into points, throughput ascending."""
    ctx = ctx or default_context()
    pts = np.ascontiguousarray(points, dtype=POINT_DT)
    thr = np.ascontiguousarray(throughput, np.float64)
    eff = np.ascontiguousarray(efficiency, np.float64)
    if not (len(pts) == len(thr) == len(eff)):
        raise ConfigError(2, "build_frontier: points / throughput / efficiency lengths differ")
    idx = np.empty(max(1, len(pts)), np.int32)
    n = C.c_int64(0)
    check(ctx.lib.pals_frontier_values(ctx.h, ptr(pts), ptr(thr), ptr(eff), len(pts), ptr(idx),
                                       C.byref(n)))
    return idx[: n.value].copy()


def build_frontier(points, ctx: Context | None = None):
    """build_frontier(std::vector<FrontierPoint>) (pareto.hpp:31-59)."""
    points = list(points)
    if not points:
        raise ConfigError(2, "build_frontier: no points")
    pts = np.zeros(len(points), POINT_DT)
    for i, p in enumerate(points):
        pts[i] = tuple(p.point)
    thr = np.array([p.throughput_tps for p in points], np.float64)
    eff = np.array([p.efficiency_tpj for p in points], np.float64)
    return [points[i] for i in frontier_indices(pts, thr, eff, ctx)]


def regime_points(regime: RegimeSpec, profile: Profile, cap_grid, batch_grid, tp_grid):
    """The operating points evaluate_regime scores (pareto.hpp:118-131), in its loop order;
    TP degrees without a calibrated comm cost are skipped."""
    caps = list(cap_grid) if regime.sweep_cap else [regime.fixed_cap_w]
    batches = list(batch_grid) if regime.sweep_batch else [regime.fixed_batch]
    tps = list(tp_grid) if regime.sweep_tp else [profile.deploy_tp]
    keys = set(profile.tp_keys[: profile.n_tp])
    out = [(float(c), int(b), int(t), profile.deploy_ep, 1)
           for c in caps for b in batches for t in tps if t in keys]
    return np.array(out, dtype=POINT_DT)


def evaluate_regime(regime: RegimeSpec, profile: Profile, gpu: GpuSpec, coeffs: Coeffs,
                    cap_grid, batch_grid, tp_grid, ctx: Context | None = None):
    """evaluate_regime (pareto.hpp:114-135): analytic scores + frontier, on the device."""
    ctx = ctx or default_context()
    pts = regime_points(regime, profile, cap_grid, batch_grid, tp_grid)
    if len(pts) == 0:
        raise ConfigError(2, "build_frontier: no points")
    plan = Plan(AnalyticModel(ctx, profile, gpu), Grid(ctx, pts), coeffs)
    idx = plan.frontier()
    th, _, ef = plan.scores()
    return [FrontierPoint(tuple(pts[i].tolist()), float(th[i]), float(ef[i])) for i in idx]


def verify_dominance(a, b):
    """verify_dominance (pareto.hpp:66-83): (dominated, witnesses)."""
    witnesses = [q for q in b if not any(weakly_dominates(p, q) for p in a)]
    return not witnesses, witnesses


def peak_efficiency(frontier) -> float:
    best = 0.0
    for p in frontier:
        best = max(best, p.efficiency_tpj)
    return best
