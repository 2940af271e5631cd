"""Single calls through the resident server kernel (pals_ctx_set_one_server): the same
decisions and states as one kernel launch per call and as the reference, across server
exits (short idle time + host sleeps), relaunches, and candidate-set evictions while a
server is resident."""
import time

import numpy as np
import pytest

from paper_2605_21427_b200 import abi, workloads
from paper_2605_21427_b200.abi import CtrlState, Telemetry, default_ctrl_cfg
from paper_2605_21427_b200.wattserve import (AnalyticModel, Context, control_step, make_targets,
                                             select_config)

pytestmark = pytest.mark.gpu


def _run(ctx, c1, gpu, coeffs, n, sleep_every=0, n_sets=1):
    m = AnalyticModel(ctx, c1["profile"], gpu)
    cfg = default_ctrl_cfg(target_headroom=0.05, budget_margin=0.02)
    rng = np.random.default_rng(11)
    # n_sets distinct candidate sets (prefixes of the grid), visited round-robin
    sets = [c1["points"][: len(c1["points"]) - j] for j in range(n_sets)]
    st = CtrlState()
    st.bias = 1.0
    st.current = abi.Point(275.0, 48, 2, 1, 1)
    out = []
    now = 0.5
    for k in range(n):
        pts = sets[k % n_sets]
        tg = make_targets(float(rng.uniform(200, 2500)), None if k % 3 else float(
            rng.uniform(900, 1800)), 0.05, int(k % 7 == 6))
        tel = Telemetry(now, float(rng.uniform(100, 3000)))
        d, st = control_step(tel, now, tg, pts, m, coeffs, st, cfg)
        s = select_config(pts, tg, m, coeffs, bias=float(rng.uniform(0.6, 1.4)))
        out.append(bytes(d) + bytes(st) + bytes(s))
        if sleep_every and k % sleep_every == sleep_every - 1:
            time.sleep(0.002)
        now += 0.5
    return out


def test_server_matches_launch_per_call(bundle):
    _, gpu, coeffs = bundle
    c1 = workloads.cfg1()
    ctx_l = Context(0)
    ctx_l.set_one_server(0)
    base = _run(ctx_l, c1, gpu, coeffs, 120)
    ctx_s = Context(0)
    assert _run(ctx_s, c1, gpu, coeffs, 120) == base
    # idle exits between calls: the next call relaunches the server
    ctx_s.set_one_server(30)
    assert _run(ctx_s, c1, gpu, coeffs, 120, sleep_every=3) == base
    ctx_s.set_one_server(2000)
    # more sets than the cache holds: evictions while a server is resident
    ctx_l2 = Context(0)
    ctx_l2.set_one_server(0)
    many = _run(ctx_l2, c1, gpu, coeffs, 80, n_sets=20)
    assert _run(ctx_s, c1, gpu, coeffs, 80, n_sets=20) == many


def test_server_against_reference(bundle, reference):
    """The analytic-scorer control_step sequence of test_gpu_control, served."""
    _, gpu, coeffs = bundle
    c1 = workloads.cfg1()
    ctx = Context(0)
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
