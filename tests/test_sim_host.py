"""Host side of the queue-plant simulator (no GPU): the scenario parser against the
reference's scenario_from_json (scenario_io.hpp:35-93) on the bundled files, the
shipped scenario data against the reference's data directory, and the CSV
writers' formats."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from paper_2605_21427_b200.abi import SIM_DEC_DT, SIM_TEL_DT
from paper_2605_21427_b200.sim import (bundled_scenarios, decisions_csv, n_intervals,
                                       scenario_from_dict, telemetry_csv)

REF_SCEN = "/root/reference/proj/data/scenarios"


def _digest(sc: dict) -> str:
    g = lambda v: "%.17g" % v  # noqa: E731
    o = [f"name={sc['name']}", f"duration_s={g(sc['duration_s'])}",
         f"interval_s={g(sc['interval_s'])}", f"seed={sc['seed']}",
         f"mean_tokens={g(sc['mean_tokens'])}", f"log_sigma={g(sc['log_sigma'])}",
         "cluster_budget_w=" + ("none" if sc["cluster_budget_w"] is None
                                else g(sc["cluster_budget_w"])),
         "trace=" + "".join(f"{g(t)}:{g(w)};" for t, w in sc["trace"]),
         f"policy={sc['policy']}", f"objective={sc['objective']}"]
    from paper_2605_21427_b200.abi import default_ctrl_cfg
    c = default_ctrl_cfg(**sc["controller"])
    o += [f"kp={g(c.kp)}", f"ki={g(c.ki)}", f"kd={g(c.kd)}",
          f"sustain_intervals={c.sustain_intervals}", f"integral_clamp={g(c.integral_clamp)}",
          f"target_headroom={g(c.target_headroom)}", f"budget_margin={g(c.budget_margin)}",
          f"epsilon={g(sc['epsilon'])}", "caps=" + "".join(g(v) + ";" for v in sc["caps"]),
          "batches=" + "".join(f"{v};" for v in sc["batches"]),
          f"initial={g(sc['initial_cap_w'])}:{sc['initial_batch']}"]
    for n in sc["nodes"]:
        o.append(f"node={n['model']}:{g(n['qos_fraction'])}:{n['tp']}:{n['ep']}:{n['dp']}:"
                 f"{g(n['arrival_rate_per_s'])}:{n['initial_backlog']}")
    return "\n".join(o) + "\n"


@pytest.mark.skipif(not os.path.isdir(REF_SCEN), reason="reference data absent")
@pytest.mark.parametrize("name", ["single_node", "multinode_qos", "demand_response"])
def test_parser_matches_reference_loader(reference, name):
    L = reference.lib
    L.ref_scenario_digest.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.c_void_p]
    path = os.path.join(REF_SCEN, name + ".json").encode()
    n = C.c_int64(0)
    assert L.ref_scenario_digest(path, None, 0, C.byref(n)) == 0
    buf = C.create_string_buffer(n.value)
    L.ref_scenario_digest(path, buf, n.value, C.byref(n))
    ours = bundled_scenarios()[name]
    assert _digest(ours) == buf.raw.decode()


def test_parser_defaults():
    """scenario_io.hpp defaults: headroom = epsilon, margin 0.02 (no controller block);
    initial = max cap / max batch; interval 0.5; output length 200 / 0.4."""
    sc = scenario_from_dict({"name": "x", "duration_s": 10, "seed": 3,
                             "nodes": [{"model": "olmoe-like", "arrival_rate_per_s": 1}]})
    assert sc["controller"] == {"target_headroom": 0.05, "budget_margin": 0.02}
    assert (sc["initial_cap_w"], sc["initial_batch"]) == (400.0, 64)
    assert sc["interval_s"] == 0.5 and (sc["mean_tokens"], sc["log_sigma"]) == (200.0, 0.4)
    assert n_intervals(sc) == 20
    with pytest.raises(ValueError):
        scenario_from_dict(dict(name="x", duration_s=1, seed=1, policy="greedy", nodes=[]))


def test_csv_formats():
    sc = bundled_scenarios()["single_node"]
    n = n_intervals(sc)
    tel = np.zeros((1, n), SIM_TEL_DT)
    dec = np.zeros((1, n), SIM_DEC_DT)
    tel["t_s"] = np.arange(1, n + 1) * 0.5
    tel["sys_power_w"] = 1234.5678901234
    dec["cap_w"], dec["batch"], dec["reason"], dec["bias"] = 400.0, 64, 3, 1.0
    t = telemetry_csv(sc, tel).decode().splitlines()
    d = decisions_csv(sc, tel, dec).decode().splitlines()
    assert t[0].startswith("node,model,t_s,gpu_power_w") and len(t) == n + 1
    assert t[1] == "0,olmoe-like,0.5,0,1234.56789,0,0,0,0,0,0,0"
    assert d[1] == "0,olmoe-like,0.5,400,64,2,8,1,0,hold-hysteresis,0,1"


def test_shipped_scenarios_match_reference_files():
    if not os.path.isdir(REF_SCEN):
        pytest.skip("reference data absent")
    for name, sc in bundled_scenarios().items():
        with open(os.path.join(REF_SCEN, name + ".json")) as f:
            j = json.load(f)
        assert sc["name"] == j["name"] and sc["seed"] == j["seed"]
        assert len(sc["nodes"]) == len(j["nodes"])
