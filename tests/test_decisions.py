"""Decision-log wire format: the reference's decisions CSV
(metrics.hpp:145-157, "%.10g" numbers, csvio.hpp:17-21) and its manifest hash
(fnv1a64, rng.hpp:22-28), byte-identical from replay logs.

CPU: the C oracle's replay logs + details through libpals_gpu's formatter (host code)
against fixtures written by the reference's own decisions_csv. GPU: the same from the
CUDA replay, both kernel layouts."""
import numpy as np
import pytest

from oracle.gen_golden import DECISION_SPECS
from paper_2605_21427_b200 import workloads
from paper_2605_21427_b200.wattserve import (AnalyticModel, Context, decisions_csv, fnv1a64,
                                             replay_with_details)


def _setup(name):
    s = workloads.cfg4_setup()
    caps, batches = workloads.dr_candidates() if name == "dr" else (s["caps"], s["batches"])
    return s, caps, batches, workloads.replay_spec(**DECISION_SPECS[name])


@pytest.mark.parametrize("name", sorted(DECISION_SPECS))
def test_oracle_logs_format_to_reference_csv(oracle, gold, name):
    s, caps, batches, spec = _setup(name)
    summ, logs, det = oracle.replay_ex(s["profiles"], s["gpu"], s["coeffs"], caps, batches,
                                       s["cfg"], spec)
    csv = decisions_csv(spec, s["profiles"], caps, batches, summ, logs, det)
    g = gold("decisions")
    assert csv == bytes(g[name])
    assert fnv1a64(csv) == int(g[name + "_fnv"][0])


def test_reference_writer_live(reference, oracle):
    """A fresh spec (not a fixture) through the reference writer vs our formatter."""
    s = workloads.cfg4_setup()
    spec = workloads.replay_spec(10, n_steps=150, seed=4242, n_log_traces=10, first=1000)
    ref_csv, ref_h = reference.replay_decisions_csv(s["profiles"], s["gpu"], s["coeffs"],
                                                    s["caps"], s["batches"], s["cfg"], spec)
    summ, logs, det = oracle.replay_ex(s["profiles"], s["gpu"], s["coeffs"], s["caps"],
                                       s["batches"], s["cfg"], spec)
    ours = decisions_csv(spec, s["profiles"], s["caps"], s["batches"], summ, logs, det)
    # node ids: the reference numbers its SimResult nodes from 0, the formatter from
    # first_trace; everything after the first field is identical
    strip = lambda b: [ln.split(b",", 1)[1] for ln in b.split(b"\n")[1:] if ln]  # noqa: E731
    assert strip(ours) == strip(ref_csv)
    assert ours.split(b"\n", 1)[0] == ref_csv.split(b"\n", 1)[0]
    assert fnv1a64(ref_csv) == ref_h


def test_formatter_errors(oracle):
    from paper_2605_21427_b200._lib import ConfigError
    s, caps, batches, spec = _setup("qos")
    summ, logs, det = oracle.replay_ex(s["profiles"], s["gpu"], s["coeffs"], caps, batches,
                                       s["cfg"], spec)
    bad = logs.copy()
    bad["idx"][3] = 10_000
    with pytest.raises(ConfigError):
        decisions_csv(spec, s["profiles"], caps, batches, summ, bad, det)
    empty = workloads.replay_spec(0, n_steps=10)
    assert decisions_csv(empty, s["profiles"], caps, batches, summ[:0], logs[:0], det[:0]) == (
        b"node,model,t_s,cap_w,batch,tp,ep,dp,applied,reason,err_norm,bias\n")


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["thread", "warp"])
@pytest.mark.parametrize("name", sorted(DECISION_SPECS))
def test_gpu_replay_decisions_csv(gold, name, layout):
    ctx = Context(0)
    ctx.set_replay_layout(layout)
    s, caps, batches, spec = _setup(name)
    models = [AnalyticModel(ctx, p, s["gpu"]) for p in s["profiles"]]
    summ, logs, det = replay_with_details(ctx, models, s["profiles"], s["gpu"], s["coeffs"],
                                          caps, batches, s["cfg"], spec)
    csv = decisions_csv(spec, s["profiles"], caps, batches, summ, logs, det)
    g = gold("decisions")
    assert csv == bytes(g[name])
    assert fnv1a64(csv) == int(g[name + "_fnv"][0])
