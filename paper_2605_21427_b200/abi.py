"""ctypes / numpy mirrors of the POD structs in include/pals_gpu.h.

Every struct mirrors one reference type (paths under
/root/reference/proj/include/wattserve/): pals_profile <- ModelProfile
(types.hpp:66-107), pals_point <- OperatingPoint (types.hpp:110-116),
pals_query <- select_config's Targets + bias/headroom/margin
(controller.hpp:132-135), pals_ctrl_cfg <- ControllerConfig
(controller.hpp:37-53), pals_ctrl_state <- ControllerState
(controller.hpp:55-63), pals_decision <- Decision (controller.hpp:85-89).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

PALS_OK = 0
PALS_ECONFIG = 2
PALS_EDATA = 3
PALS_ERUNTIME = 4
PALS_ERANGE = 5

OBJ_QOS = 0
OBJ_BUDGET = 1

REASON_QOS_FEASIBLE = 0
REASON_FALLBACK_MAX_T = 1
REASON_BUDGET_MAX_T = 2
REASON_HOLD = 3
REASON_ORACLE = 4
REASON_NAMES = {
    0: "qos-feasible-max-efficiency",
    1: "fallback-max-throughput",
    2: "budget-constrained-max-throughput",
    3: "hold-hysteresis",
    4: "oracle-exhaustive",
}  # controller.hpp:73-83

MAX_TP_KEYS = 8


class GpuSpec(C.Structure):
    _fields_ = [("idle_watts", C.c_double), ("min_cap_watts", C.c_double),
                ("max_cap_watts", C.c_double), ("max_frequency", C.c_double)]


class Coeffs(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta_watts", C.c_double)]


class Profile(C.Structure):
    _fields_ = [
        ("name", C.c_char * 64),
        ("compute_fixed", C.c_double),
        ("compute_per_seq", C.c_double),
        ("comm_per_seq", C.c_double),
        ("internode_factor", C.c_double),
        ("knee_watts", C.c_double),
        ("compute_power_base", C.c_double),
        ("compute_power_per_seq", C.c_double),
        ("comm_power", C.c_double),
        ("overlap", C.c_double),
        ("comm_fixed", C.c_double * MAX_TP_KEYS),
        ("total_params_b", C.c_double),
        ("active_params_b", C.c_double),
        ("tp_keys", C.c_int32 * MAX_TP_KEYS),
        ("n_tp", C.c_int32),
        ("num_experts", C.c_int32),
        ("top_k", C.c_int32),
        ("deploy_tp", C.c_int32),
        ("deploy_ep", C.c_int32),
        ("deploy_dp", C.c_int32),
    ]


class Point(C.Structure):
    _fields_ = [("cap_watts", C.c_double), ("batch", C.c_int32), ("tp", C.c_int32),
                ("ep", C.c_int32), ("dp", C.c_int32)]


class Query(C.Structure):
    _fields_ = [("throughput_tps", C.c_double), ("power_budget_w", C.c_double),
                ("bias", C.c_double), ("target_headroom", C.c_double),
                ("budget_margin", C.c_double), ("objective", C.c_int32),
                ("has_budget", C.c_int32)]


class Targets(C.Structure):
    _fields_ = [("throughput_tps", C.c_double), ("power_budget_w", C.c_double),
                ("epsilon", C.c_double), ("has_budget", C.c_int32), ("objective", C.c_int32)]


class CtrlCfg(C.Structure):
    _fields_ = [("kp", C.c_double), ("ki", C.c_double), ("kd", C.c_double),
                ("integral_clamp", C.c_double), ("bias_min", C.c_double),
                ("bias_max", C.c_double), ("interval_s", C.c_double),
                ("target_headroom", C.c_double), ("budget_margin", C.c_double),
                ("sustain_intervals", C.c_int32), ("_pad", C.c_int32)]


class CtrlState(C.Structure):
    _fields_ = [("bias", C.c_double), ("integral", C.c_double), ("prev_error", C.c_double),
                ("current", Point), ("last_targets", Targets),
                ("has_prev_error", C.c_int32), ("sustain_count", C.c_int32),
                ("has_last_targets", C.c_int32), ("_pad", C.c_int32)]


class Decision(C.Structure):
    _fields_ = [("point", Point), ("applied", C.c_int32), ("reason", C.c_int32)]


class Telemetry(C.Structure):
    _fields_ = [("t_s", C.c_double), ("throughput_tps", C.c_double)]


class ReplaySpec(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("first_trace", C.c_int64), ("n_traces", C.c_int64),
        ("n_steps", C.c_int32), ("objective_mode", C.c_int32),
        ("interval_s", C.c_double), ("qos_frac_lo", C.c_double), ("qos_frac_hi", C.c_double),
        ("load_lo", C.c_double), ("load_hi", C.c_double), ("noise_amp", C.c_double),
        ("budget_lo_frac", C.c_double), ("budget_hi_frac", C.c_double),
        ("epsilon", C.c_double),
        ("seg_min", C.c_int32), ("seg_max", C.c_int32), ("budget_mode", C.c_int32),
        ("n_log_traces", C.c_int32),
    ]


POINT_DT = np.dtype([("cap_watts", "<f8"), ("batch", "<i4"), ("tp", "<i4"), ("ep", "<i4"),
                     ("dp", "<i4")], align=True)
QUERY_DT = np.dtype([("throughput_tps", "<f8"), ("power_budget_w", "<f8"), ("bias", "<f8"),
                     ("target_headroom", "<f8"), ("budget_margin", "<f8"),
                     ("objective", "<i4"), ("has_budget", "<i4")], align=True)
SUMMARY_DT = np.dtype([("digest", "<u8"), ("final_bias", "<f8"), ("energy_j", "<f8"),
                       ("tokens", "<f8"), ("n_applied", "<i4"), ("final_idx", "<i4"),
                       ("model", "<i4"), ("objective", "<i4")], align=True)
STEPLOG_DT = np.dtype([("idx", "<i4"), ("applied", "u1"), ("reason", "u1"),
                       ("cap_tenths", "<u2")], align=True)

assert C.sizeof(Point) == POINT_DT.itemsize == 24
assert C.sizeof(Query) == QUERY_DT.itemsize == 48
STEPDETAIL_DT = np.dtype([("err_norm", "<f8"), ("bias", "<f8")], align=True)

# ---- caller-trace replay (pals_replay_traces) ----
# pals_signal_point = the reference's budget-trace row std::pair<double,double>{t_s, value}
SIGNAL_DT = np.dtype([("t_s", "<f8"), ("value", "<f8")], align=True)
# pals_trace
TRACE_DT = np.dtype([("budget_off", "<i8"), ("load_off", "<i8"), ("target_tps", "<f8"),
                     ("epsilon", "<f8"), ("noise_amp", "<f8"), ("noise_key", "<u8"),
                     ("n_budget", "<i4"), ("n_load", "<i4"), ("model", "<i4"),
                     ("objective", "<i4")], align=True)
# pals_plant_state = NodeRuntime applied_cap / inflight_cap / batch_cap (sim.hpp:155-157)
PLANT_DT = np.dtype([("applied_cap_w", "<f8"), ("inflight_cap_w", "<f8"),
                     ("batch_cap", "<i4"), ("_pad", "<i4")], align=True)
_TARGETS_DT = np.dtype([("throughput_tps", "<f8"), ("power_budget_w", "<f8"),
                        ("epsilon", "<f8"), ("has_budget", "<i4"), ("objective", "<i4")],
                       align=True)
# pals_ctrl_state = ControllerState (controller.hpp:55-63), as an array element
STATE_DT = np.dtype([("bias", "<f8"), ("integral", "<f8"), ("prev_error", "<f8"),
                     ("current", POINT_DT), ("last_targets", _TARGETS_DT),
                     ("has_prev_error", "<i4"), ("sustain_count", "<i4"),
                     ("has_last_targets", "<i4"), ("_pad", "<i4")], align=True)


class TraceBatch(C.Structure):  # pals_trace_batch
    _fields_ = [("n_traces", C.c_int64), ("first_step", C.c_int64), ("n_steps", C.c_int32),
                ("n_log_traces", C.c_int32), ("interval_s", C.c_double),
                ("traces", C.c_void_p), ("signal", C.c_void_p), ("n_signal", C.c_int64),
                ("init", C.c_void_p), ("init_plant", C.c_void_p), ("summaries", C.c_void_p),
                ("final_state", C.c_void_p), ("final_plant", C.c_void_p), ("logs", C.c_void_p),
                ("details", C.c_void_p)]


assert SIGNAL_DT.itemsize == 16 and TRACE_DT.itemsize == 64 and PLANT_DT.itemsize == 24
assert STATE_DT.itemsize == C.sizeof(CtrlState) == 96 and C.sizeof(TraceBatch) == 112


def state_array(states) -> np.ndarray:
    """STATE_DT array from CtrlState structs (or pass a STATE_DT array through)."""
    if isinstance(states, np.ndarray):
        return np.ascontiguousarray(states, STATE_DT)
    out = np.zeros(len(states), STATE_DT)
    C.memmove(out.ctypes.data, (CtrlState * len(states))(*states), out.nbytes)
    return out


def state_struct(row) -> CtrlState:
    """CtrlState from one STATE_DT element."""
    s = CtrlState()
    C.memmove(C.addressof(s), np.ascontiguousarray(row).ctypes.data, C.sizeof(s))
    return s


# ---- queue-plant scenarios (sim.hpp:47-145; pals_run_scenarios) ----
POLICY_FIXED, POLICY_ADAPTIVE_BATCH, POLICY_ADAPTIVE_CAP, POLICY_JOINT, POLICY_ORACLE = range(5)
POLICIES = {"fixed": 0, "adaptive-batch": 1, "adaptive-cap": 2, "joint": 3, "oracle": 4}
SIM_MAX_NODES = 32


class SimNode(C.Structure):  # ScenarioNode (sim.hpp:52-60)
    _fields_ = [("model", C.c_int32), ("tp", C.c_int32), ("ep", C.c_int32), ("dp", C.c_int32),
                ("qos_fraction", C.c_double), ("arrival_rate_per_s", C.c_double),
                ("initial_backlog", C.c_int32), ("_pad", C.c_int32)]


class Scenario(C.Structure):  # Scenario (sim.hpp:62-94)
    _fields_ = [("duration_s", C.c_double), ("interval_s", C.c_double), ("seed", C.c_uint64),
                ("mean_tokens", C.c_double), ("log_sigma", C.c_double),
                ("has_cluster_budget", C.c_int32), ("n_trace", C.c_int32),
                ("cluster_budget_w", C.c_double), ("trace_t", C.c_void_p),
                ("trace_w", C.c_void_p), ("policy", C.c_int32), ("objective", C.c_int32),
                ("controller", CtrlCfg), ("epsilon", C.c_double), ("cand_caps", C.c_void_p),
                ("cand_batches", C.c_void_p), ("n_caps", C.c_int32), ("n_batches", C.c_int32),
                ("initial_cap_w", C.c_double), ("initial_batch", C.c_int32),
                ("n_nodes", C.c_int32), ("nodes", C.c_void_p)]


SIM_NODE_RESULT_DT = np.dtype([
    ("tokens_per_joule", "<f8"), ("qos_violation_rate", "<f8"), ("power_tracking_mae_w", "<f8"),
    ("total_tokens", "<f8"), ("total_energy_j", "<f8"), ("mean_throughput_tps", "<f8"),
    ("throughput_target_tps", "<f8"), ("final_bias", "<f8"), ("arrival_stream_hash", "<u8"),
    ("n_requests", "<i8"), ("n_completed", "<i8"), ("n_applied", "<i4"), ("final_idx", "<i4")],
    align=True)
SIM_RESULT_DT = np.dtype([
    ("tokens_per_joule", "<f8"), ("qos_violation_rate", "<f8"), ("power_tracking_mae_w", "<f8"),
    ("total_tokens", "<f8"), ("total_energy_j", "<f8"), ("mean_throughput_tps", "<f8"),
    ("cluster_tracking_mae_w", "<f8"), ("sim_total_energy_j", "<f8"), ("n_intervals", "<i4"),
    ("n_budget_changes", "<i4")], align=True)
SIM_TEL_DT = np.dtype([
    ("t_s", "<f8"), ("gpu_power_w", "<f8"), ("sys_power_w", "<f8"), ("throughput_tps", "<f8"),
    ("utilization", "<f8"), ("node_budget_w", "<f8"), ("applied_cap_w", "<f8"),
    ("queue_depth", "<i4"), ("active_batch", "<i4"), ("applied_batch_cap", "<i4"),
    ("_pad", "<i4")], align=True)
SIM_DEC_DT = np.dtype([
    ("err_norm", "<f8"), ("bias", "<f8"), ("cap_w", "<f8"), ("batch", "<i4"), ("applied", "u1"),
    ("reason", "u1"), ("_pad", "<u2")], align=True)
SIM_REQ_DT = np.dtype([("id", "<i8"), ("arrival_s", "<f8"), ("output_tokens", "<i4"),
                       ("_pad", "<i4"), ("generated", "<f8"), ("completed_s", "<f8")], align=True)
assert SIM_REQ_DT.itemsize == 40
assert C.sizeof(SimNode) == 40 and C.sizeof(Scenario) == 216
assert SIM_NODE_RESULT_DT.itemsize == 96 and SIM_RESULT_DT.itemsize == 72
assert SIM_TEL_DT.itemsize == 72 and SIM_DEC_DT.itemsize == 32

assert SUMMARY_DT.itemsize == 48 and STEPLOG_DT.itemsize == 8 and STEPDETAIL_DT.itemsize == 16
assert C.sizeof(Profile) == 272


def ptr(a: np.ndarray | None) -> C.c_void_p:
    """Raw data pointer of a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return C.c_void_p(0)
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return C.c_void_p(a.ctypes.data)


def default_ctrl_cfg(**kw) -> CtrlCfg:
    """ControllerConfig defaults (controller.hpp:37-53)."""
    c = CtrlCfg(kp=0.5, ki=0.1, kd=0.05, integral_clamp=0.5, bias_min=0.5, bias_max=2.0,
                interval_s=0.5, target_headroom=0.0, budget_margin=0.0, sustain_intervals=3)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def default_ctrl_state(current: Point | None = None) -> CtrlState:
    """ControllerState defaults (controller.hpp:55-63); OperatingPoint default is 400 W, batch 1."""
    s = CtrlState()
    s.bias = 1.0
    s.current = current if current is not None else Point(400.0, 1, 1, 1, 1)
    return s


def make_points(caps, batches, tps=(1,), eps=(1,), dps=(1,)) -> np.ndarray:
    """Grid in canonical sweep nesting cap -> batch -> tp -> ep -> dp (sweep.hpp:134-138)."""
    n = len(caps) * len(batches) * len(tps) * len(eps) * len(dps)
    pts = np.zeros(n, dtype=POINT_DT)
    i = 0
    for c in caps:
        for b in batches:
            for t in tps:
                for e in eps:
                    for d in dps:
                        pts[i] = (c, b, t, e, d)
                        i += 1
    return pts
