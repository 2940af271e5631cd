"""TEST INFRASTRUCTURE ONLY — ctypes front-end to the two CPU checkers.

* ``Oracle``: the plain-C restatement (oracle/liboracle.so, pals_oracle.c).
* ``Reference``: the unmodified reference headers behind oracle/ref_harness.cpp
  (oracle/_ref/libwsref.so). Built here from /root/reference by oracle/Makefile;
  shipped prebuilt to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module. The product (paper_2605_21427_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2605_21427_b200.abi import (PLANT_DT, POINT_DT, QUERY_DT, SIGNAL_DT, STATE_DT,
                                       STEPDETAIL_DT, STEPLOG_DT, SUMMARY_DT, TRACE_DT, Coeffs,
                                       CtrlCfg, CtrlState, Decision, GpuSpec, Profile,
                                       ReplaySpec, Targets, Telemetry, TraceBatch, ptr,
                                       state_array)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwsref.so")

_VP = C.c_void_p
_P = C.POINTER


def build(quiet: bool = True) -> None:
    """Compile both checkers (the reference one only where /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


class Oracle:
    """Plain-C restatement of the reference hot path (pals_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        L = self.lib = _load(path)
        L.or_splitmix64.restype = C.c_uint64
        L.or_splitmix64.argtypes = [C.c_uint64]
        L.or_effective_frequency.restype = C.c_double
        L.or_effective_frequency.argtypes = [C.c_double, _VP, _VP, _P(C.c_int)]
        L.or_eval.argtypes = [_VP, _VP, _VP, C.c_int64, _VP, _VP, _VP]
        L.or_select_scored.argtypes = [_VP, C.c_int64, _VP, _VP, _VP, _VP, _VP, _VP]
        L.or_control_step_scored.argtypes = [_VP, C.c_int64, _VP, _VP, C.c_double, C.c_int,
                                             _VP, C.c_double, _VP, _VP, _VP, _VP, _VP, _VP]
        L.or_replay.argtypes = [C.c_int, _VP, _VP, _VP, _VP, C.c_int, _VP, C.c_int, _VP, _VP,
                                _VP, _VP]

    def splitmix64(self, x: int) -> int:
        return self.lib.or_splitmix64(x)

    def effective_frequency(self, cap, prof: Profile, gpu: GpuSpec):
        e = C.c_int(0)
        f = self.lib.or_effective_frequency(cap, C.byref(prof), C.byref(gpu), C.byref(e))
        return f, e.value

    def eval(self, prof: Profile, gpu: GpuSpec, pts: np.ndarray):
        n = len(pts)
        T = np.empty(n, np.float64)
        P = np.empty(n, np.float64)
        err = np.empty(n, np.int32)
        self.lib.or_eval(C.byref(prof), C.byref(gpu), ptr(pts), n, ptr(T), ptr(P), ptr(err))
        return T, P, err

    def select(self, pts: np.ndarray, T: np.ndarray, P: np.ndarray, coeffs: Coeffs,
               queries: np.ndarray):
        """select_config per query over pre-scored candidates; returns (idx, reason, rc)."""
        pts = np.ascontiguousarray(pts, dtype=POINT_DT)
        T = np.ascontiguousarray(T, np.float64)
        P = np.ascontiguousarray(P, np.float64)
        nq = len(queries)
        idx = np.empty(nq, np.int32)
        rs = np.empty(nq, np.uint8)
        rc = 0
        for j in range(nq):
            q = np.ascontiguousarray(queries[j:j + 1], dtype=QUERY_DT)
            rc = self.lib.or_select_scored(ptr(pts), len(pts), ptr(T), ptr(P), C.byref(coeffs),
                                           ptr(q), ptr(idx[j:]), ptr(rs[j:]))
            if rc:
                return idx, rs, rc
        return idx, rs, rc

    def control_step(self, pts, T, P, cur_T, cur_ok, tel: Telemetry, now, tg: Targets,
                     coeffs: Coeffs, st: CtrlState, cfg: CtrlCfg):
        d = Decision()
        st2 = CtrlState()
        rc = self.lib.or_control_step_scored(ptr(pts), len(pts), ptr(T), ptr(P), cur_T,
                                             int(cur_ok), C.byref(tel), now, C.byref(tg),
                                             C.byref(coeffs), C.byref(st), C.byref(cfg),
                                             C.byref(d), C.byref(st2))
        return d, st2, rc

    def replay(self, plant, gpu, coeffs, caps, batches, cfg: CtrlCfg, spec: ReplaySpec):
        profs = (Profile * len(plant))(*plant)
        caps = np.ascontiguousarray(caps, np.float64)
        batches = np.ascontiguousarray(batches, np.int32)
        summ = np.zeros(spec.n_traces, SUMMARY_DT)
        logs = np.zeros(max(1, spec.n_log_traces * spec.n_steps), STEPLOG_DT)
        rc = self.lib.or_replay(len(plant), profs, C.byref(gpu), C.byref(coeffs), ptr(caps),
                                len(caps), ptr(batches), len(batches), C.byref(cfg),
                                C.byref(spec), ptr(summ), ptr(logs))
        if rc:
            raise RuntimeError(f"or_replay rc={rc}")
        return summ, logs[: spec.n_log_traces * spec.n_steps]

    def replay_ex(self, plant, gpu, coeffs, caps, batches, cfg: CtrlCfg, spec: ReplaySpec):
        """replay() plus the per-step (err_norm, bias) of the logged traces."""
        L = self.lib
        L.or_replay_ex.argtypes = [C.c_int, _VP, _VP, _VP, _VP, C.c_int, _VP, C.c_int, _VP,
                                   _VP, _VP, _VP, _VP]
        profs = (Profile * len(plant))(*plant)
        caps = np.ascontiguousarray(caps, np.float64)
        batches = np.ascontiguousarray(batches, np.int32)
        summ = np.zeros(spec.n_traces, SUMMARY_DT)
        nl = spec.n_log_traces * spec.n_steps
        logs = np.zeros(max(1, nl), STEPLOG_DT)
        det = np.zeros(max(1, nl), STEPDETAIL_DT)
        rc = L.or_replay_ex(len(plant), profs, C.byref(gpu), C.byref(coeffs), ptr(caps),
                            len(caps), ptr(batches), len(batches), C.byref(cfg), C.byref(spec),
                            ptr(summ), ptr(logs), ptr(det))
        if rc:
            raise RuntimeError(f"or_replay_ex rc={rc}")
        return summ, logs[:nl], det[:nl]

    def replay_scored(self, plant, gpu, coeffs, caps, batches, cfg: CtrlCfg, spec: ReplaySpec,
                      scorer_T: np.ndarray, scorer_P: np.ndarray):
        """Replay with a non-analytic scorer given as [n_models, n_candidates] tables."""
        L = self.lib
        L.or_replay_scored.argtypes = [C.c_int, _VP, _VP, _VP, _VP, C.c_int, _VP, C.c_int, _VP,
                                       _VP, _VP, _VP, _VP, _VP]
        profs = (Profile * len(plant))(*plant)
        caps = np.ascontiguousarray(caps, np.float64)
        batches = np.ascontiguousarray(batches, np.int32)
        sT = np.ascontiguousarray(scorer_T, np.float64)
        sP = np.ascontiguousarray(scorer_P, np.float64)
        summ = np.zeros(spec.n_traces, SUMMARY_DT)
        logs = np.zeros(max(1, spec.n_log_traces * spec.n_steps), STEPLOG_DT)
        rc = L.or_replay_scored(len(plant), profs, C.byref(gpu), C.byref(coeffs), ptr(caps),
                                len(caps), ptr(batches), len(batches), C.byref(cfg),
                                C.byref(spec), ptr(sT), ptr(sP), ptr(summ), ptr(logs))
        if rc:
            raise RuntimeError(f"or_replay_scored rc={rc}")
        return summ, logs[: spec.n_log_traces * spec.n_steps]


class Reference:
    """The unmodified reference (oracle/_ref/libwsref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_splitmix64.restype = C.c_uint64
        L.ref_splitmix64.argtypes = [C.c_uint64]
        L.ref_eval.argtypes = [_VP, _VP, _VP, C.c_int64, _VP, _VP, _VP]
        L.ref_effective_frequency.restype = C.c_double
        L.ref_effective_frequency.argtypes = [C.c_double, _VP, _VP, _P(C.c_int)]
        L.ref_validate.argtypes = [_VP, _VP]
        L.ref_select_analytic.argtypes = [_VP, _VP, _VP, C.c_int64, _VP, _VP, C.c_int64, _VP,
                                          _VP]
        L.ref_select_table.argtypes = [_VP, C.c_int64, _VP, _VP, _VP, _VP, C.c_int64, _VP, _VP]
        L.ref_control_step_table.argtypes = [_VP, C.c_int64, _VP, _VP, _VP, C.c_double, _VP,
                                             _VP, _VP, _VP, _VP, _VP]
        L.ref_control_step_analytic.argtypes = [_VP, _VP, _VP, C.c_int64, _VP, C.c_double, _VP,
                                                _VP, _VP, _VP, _VP, _VP]
        L.ref_replay.argtypes = [C.c_int, _VP, _VP, _VP, _VP, C.c_int, _VP, C.c_int, _VP, _VP,
                                 _VP, _VP]
        L.ref_bench_select.restype = C.c_double
        L.ref_bench_select.argtypes = [_VP, _VP, _VP, C.c_int64, _VP, _VP, C.c_int64, C.c_int,
                                       _VP, _VP]
        L.ref_bench_replay.restype = C.c_double
        L.ref_bench_replay.argtypes = [C.c_int, _VP, _VP, _VP, _VP, C.c_int, _VP, C.c_int, _VP,
                                       _VP, C.c_int, _VP]
        L.ref_replay_traces.argtypes = [C.c_int, _VP, _VP, _VP, _VP, C.c_int, _VP, C.c_int,
                                        _VP, _VP, C.c_int, _P(C.c_double)]
        L.ref_load_profile.argtypes = [C.c_char_p, _VP]
        L.ref_load_platform.argtypes = [C.c_char_p, _VP, _VP]

    def last_error(self) -> str:
        return self.lib.ref_last_error().decode()

    def eval(self, prof: Profile, gpu: GpuSpec, pts: np.ndarray):
        n = len(pts)
        T = np.empty(n, np.float64)
        P = np.empty(n, np.float64)
        err = np.empty(n, np.int32)
        self.lib.ref_eval(C.byref(prof), C.byref(gpu), ptr(pts), n, ptr(T), ptr(P), ptr(err))
        return T, P, err

    def effective_frequency(self, cap, prof: Profile, gpu: GpuSpec):
        e = C.c_int(0)
        f = self.lib.ref_effective_frequency(cap, C.byref(prof), C.byref(gpu), C.byref(e))
        return f, e.value

    def select_analytic(self, prof, gpu, pts, coeffs, queries):
        nq = len(queries)
        idx = np.empty(nq, np.int32)
        rs = np.empty(nq, np.uint8)
        q = np.ascontiguousarray(queries, dtype=QUERY_DT)
        rc = self.lib.ref_select_analytic(C.byref(prof), C.byref(gpu), ptr(pts), len(pts),
                                          C.byref(coeffs), ptr(q), nq, ptr(idx), ptr(rs))
        return idx, rs, rc

    def select_table(self, pts, T, P, coeffs, queries):
        nq = len(queries)
        idx = np.empty(nq, np.int32)
        rs = np.empty(nq, np.uint8)
        q = np.ascontiguousarray(queries, dtype=QUERY_DT)
        T = np.ascontiguousarray(T, np.float64)
        P = np.ascontiguousarray(P, np.float64)
        rc = self.lib.ref_select_table(ptr(pts), len(pts), ptr(T), ptr(P), C.byref(coeffs),
                                       ptr(q), nq, ptr(idx), ptr(rs))
        return idx, rs, rc

    def control_step_table(self, pts, T, P, tel, now, tg, coeffs, st, cfg):
        d = Decision()
        st2 = CtrlState()
        rc = self.lib.ref_control_step_table(ptr(pts), len(pts), ptr(T), ptr(P), C.byref(tel),
                                             now, C.byref(tg), C.byref(coeffs), C.byref(st),
                                             C.byref(cfg), C.byref(d), C.byref(st2))
        return d, st2, rc

    def control_step_analytic(self, prof, gpu, pts, tel, now, tg, coeffs, st, cfg):
        d = Decision()
        st2 = CtrlState()
        rc = self.lib.ref_control_step_analytic(C.byref(prof), C.byref(gpu), ptr(pts), len(pts),
                                                C.byref(tel), now, C.byref(tg), C.byref(coeffs),
                                                C.byref(st), C.byref(cfg), C.byref(d),
                                                C.byref(st2))
        return d, st2, rc

    def replay(self, plant, gpu, coeffs, caps, batches, cfg, spec):
        profs = (Profile * len(plant))(*plant)
        caps = np.ascontiguousarray(caps, np.float64)
        batches = np.ascontiguousarray(batches, np.int32)
        summ = np.zeros(spec.n_traces, SUMMARY_DT)
        logs = np.zeros(max(1, spec.n_log_traces * spec.n_steps), STEPLOG_DT)
        rc = self.lib.ref_replay(len(plant), profs, C.byref(gpu), C.byref(coeffs), ptr(caps),
                                 len(caps), ptr(batches), len(batches), C.byref(cfg),
                                 C.byref(spec), ptr(summ), ptr(logs))
        if rc:
            raise RuntimeError(f"ref_replay rc={rc}: {self.last_error()}")
        return summ, logs[: spec.n_log_traces * spec.n_steps]

    def replay_decisions_csv(self, plant, gpu, coeffs, caps, batches, cfg, spec):
        """The reference's decisions_csv (metrics.hpp:145-157) of the logged traces of a
        fluid-plant replay driven through the unmodified control_step: (bytes, fnv1a64)."""
        L = self.lib
        L.ref_replay_decisions_csv.argtypes = [C.c_int, _VP, _VP, _VP, _VP, C.c_int, _VP,
                                               C.c_int, _VP, _VP, _VP, C.c_int64, _VP, _VP]
        profs = (Profile * len(plant))(*plant)
        caps = np.ascontiguousarray(caps, np.float64)
        batches = np.ascontiguousarray(batches, np.int32)
        n = C.c_int64(0)
        h = C.c_uint64(0)
        args = [len(plant), profs, C.byref(gpu), C.byref(coeffs), ptr(caps), len(caps),
                ptr(batches), len(batches), C.byref(cfg), C.byref(spec)]
        rc = L.ref_replay_decisions_csv(*args, None, 0, C.byref(n), C.byref(h))
        if rc:
            raise RuntimeError(f"ref_replay_decisions_csv rc={rc}: {self.last_error()}")
        buf = C.create_string_buffer(max(1, n.value))
        L.ref_replay_decisions_csv(*args, buf, n.value, C.byref(n), C.byref(h))
        return buf.raw[: n.value], int(h.value)

    def run_scenario(self, scenario: dict, profiles, gpu, coeffs, bundle_path=None,
                     logs: bool = True, want_csv: bool = False):
        """The unmodified run_scenario + summarize for one scenario dict
        (paper_2605_21427_b200.sim format): (node_results, result, tel, dec[, csv])."""
        from paper_2605_21427_b200.abi import (SIM_DEC_DT, SIM_NODE_RESULT_DT, SIM_RESULT_DT,
                                               SIM_TEL_DT)
        from paper_2605_21427_b200.sim import _CScenario, _model_index, n_intervals
        L = self.lib
        L.ref_run_scenario.argtypes = [_VP, C.c_int, _VP, C.c_char_p, _VP, _VP, _VP, _VP,
                                       C.c_int64, _VP, _VP, _VP, C.c_int64, _VP]
        cs = _CScenario(scenario, _model_index(profiles))
        profs = (Profile * len(profiles))(*profiles)
        nn = len(scenario["nodes"])
        stride = n_intervals(scenario)
        nres = np.zeros(nn, SIM_NODE_RESULT_DT)
        res = np.zeros(1, SIM_RESULT_DT)
        tel = np.zeros((nn, stride), SIM_TEL_DT) if logs else None
        dec = np.zeros((nn, stride), SIM_DEC_DT) if logs else None
        n = C.c_int64(0)
        bp = bundle_path.encode() if bundle_path else None
        args = [C.byref(cs.c), len(profiles), profs, bp, C.byref(gpu), C.byref(coeffs), ptr(nres),
                ptr(res), stride, ptr(tel), ptr(dec)]
        rc = L.ref_run_scenario(*args, None, 0, C.byref(n) if want_csv else None)
        if rc:
            raise RuntimeError(f"ref_run_scenario rc={rc}: {self.last_error()}")
        out = (nres, res[0], tel, dec)
        if want_csv:
            buf = C.create_string_buffer(max(1, n.value))
            L.ref_run_scenario(*args, buf, n.value, C.byref(n))
            tcsv, dcsv, rcsv = buf.raw[: n.value].split(b"\0")
            out = out + ((tcsv, dcsv, rcsv),)
        return out

    def bench_scenarios(self, scenarios, profiles, gpu, coeffs, bundle_path, threads,
                        want_results=False):
        """Wall seconds of run_scenario + summarize over the scenario dicts, threads-way;
        with want_results also (node_results, results) in scenario order."""
        from paper_2605_21427_b200.abi import SIM_NODE_RESULT_DT, SIM_RESULT_DT, Scenario
        from paper_2605_21427_b200.sim import _CScenario, _model_index
        L = self.lib
        L.ref_bench_scenarios.restype = C.c_double
        L.ref_bench_scenarios.argtypes = [C.c_int, _VP, C.c_int, _VP, C.c_char_p, _VP, _VP,
                                          C.c_int, _VP, _VP]
        idx = _model_index(profiles)
        cs = [_CScenario(s, idx) for s in scenarios]
        arr = (Scenario * len(cs))(*[c.c for c in cs])
        profs = (Profile * len(profiles))(*profiles)
        nres = np.zeros(sum(len(s["nodes"]) for s in scenarios), SIM_NODE_RESULT_DT)
        res = np.zeros(len(scenarios), SIM_RESULT_DT)
        secs = L.ref_bench_scenarios(len(cs), arr, len(profiles), profs,
                                     bundle_path.encode() if bundle_path else None,
                                     C.byref(gpu), C.byref(coeffs), threads,
                                     ptr(nres) if want_results else None,
                                     ptr(res) if want_results else None)
        if secs < 0:
            raise RuntimeError("ref_bench_scenarios: a scenario failed")
        return (secs, nres, res) if want_results else secs

    def bench_select(self, prof, gpu, pts, coeffs, queries, threads, want_results=True):
        nq = len(queries)
        idx = np.empty(nq, np.int32) if want_results else None
        rs = np.empty(nq, np.uint8) if want_results else None
        q = np.ascontiguousarray(queries, dtype=QUERY_DT)
        secs = self.lib.ref_bench_select(C.byref(prof), C.byref(gpu), ptr(pts), len(pts),
                                         C.byref(coeffs), ptr(q), nq, threads, ptr(idx), ptr(rs))
        return secs, idx, rs

    def replay_traces(self, plant, gpu, coeffs, caps, batches, cfg, traces, signal, n_steps,
                      interval_s=0.5, first_step=0, init=None, init_plant=None,
                      n_log_traces=0, details=False, threads=1):
        """The unmodified control_step over caller traces (the pals_replay_traces
        contract; see replay_trace_one in ref_harness.cpp). Returns (dict, seconds)."""
        profs = (Profile * len(plant))(*plant)
        caps = np.ascontiguousarray(caps, np.float64)
        batches = np.ascontiguousarray(batches, np.int32)
        tr = np.ascontiguousarray(traces, TRACE_DT)
        sig = np.ascontiguousarray(signal, SIGNAL_DT)
        n = len(tr)
        ini = None if init is None else state_array(init)
        inp = None if init_plant is None else np.ascontiguousarray(init_plant, PLANT_DT)
        summ = np.zeros(max(n, 1), SUMMARY_DT)
        fin = np.zeros(max(n, 1), STATE_DT)
        finp = np.zeros(max(n, 1), PLANT_DT)
        nl = min(max(n_log_traces, 0), n)
        logs = np.zeros(max(1, nl * n_steps), STEPLOG_DT)
        det = np.zeros(max(1, nl * n_steps), STEPDETAIL_DT)
        b = TraceBatch(n_traces=n, first_step=first_step, n_steps=n_steps, n_log_traces=nl,
                       interval_s=interval_s, traces=ptr(tr).value if n else None,
                       signal=ptr(sig).value if len(sig) else None, n_signal=len(sig),
                       init=None if ini is None else ptr(ini).value,
                       init_plant=None if inp is None else ptr(inp).value,
                       summaries=ptr(summ).value, final_state=ptr(fin).value,
                       final_plant=ptr(finp).value, logs=ptr(logs).value if nl else None,
                       details=ptr(det).value if (nl and details) else None)
        secs = C.c_double(0.0)
        rc = self.lib.ref_replay_traces(len(plant), profs, C.byref(gpu), C.byref(coeffs),
                                        ptr(caps), len(caps), ptr(batches), len(batches),
                                        C.byref(cfg), C.byref(b), threads, C.byref(secs))
        if rc:
            raise RuntimeError(f"ref_replay_traces rc={rc}: {self.last_error()}")
        out = {"summaries": summ[:n], "final_state": fin[:n], "final_plant": finp[:n],
               "logs": logs[: nl * n_steps]}
        if details:
            out["details"] = det[: nl * n_steps]
        return out, secs.value

    def bench_replay(self, plant, gpu, coeffs, caps, batches, cfg, spec, threads):
        profs = (Profile * len(plant))(*plant)
        caps = np.ascontiguousarray(caps, np.float64)
        batches = np.ascontiguousarray(batches, np.int32)
        summ = np.zeros(spec.n_traces, SUMMARY_DT)
        secs = self.lib.ref_bench_replay(len(plant), profs, C.byref(gpu), C.byref(coeffs),
                                         ptr(caps), len(caps), ptr(batches), len(batches),
                                         C.byref(cfg), C.byref(spec), threads, ptr(summ))
        return secs, summ

    def load_profile(self, path: str) -> Profile:
        p = Profile()
        rc = self.lib.ref_load_profile(path.encode(), C.byref(p))
        if rc:
            raise RuntimeError(self.last_error())
        return p

    def load_platform(self, path: str):
        g = GpuSpec()
        k = Coeffs()
        rc = self.lib.ref_load_platform(path.encode(), C.byref(g), C.byref(k))
        if rc:
            raise RuntimeError(self.last_error())
        return g, k


_ALLOC_ARGS = [C.c_int, _VP, _VP, _VP, _VP, C.c_int, _VP, C.c_int, C.c_double, C.c_double,
               C.c_int64] + [_VP] * 9


def _alloc_call(fn, plant, gpu, coeffs, caps, batches, quantum, margin, prob, extra=()):
    """Shared marshalling for or_allocate / ref_allocate / ref_bench_allocate: ``prob`` is the
    dict of workloads.alloc_problems (off, model, dp, target, budget)."""
    profs = (Profile * len(plant))(*plant)
    caps = np.ascontiguousarray(caps, np.float64)
    batches = np.ascontiguousarray(batches, np.int32)
    off = np.ascontiguousarray(prob["off"], np.int64)
    model = np.ascontiguousarray(prob["model"], np.int32)
    dp = np.ascontiguousarray(prob["dp"], np.int32)
    tgt = np.ascontiguousarray(prob["target"], np.float64)
    bud = np.ascontiguousarray(prob["budget"], np.float64)
    npb = len(off) - 1
    nb_out = np.zeros(len(model), np.float64)
    total = np.zeros(npb, np.float64)
    sat = np.zeros(npb, np.uint8)
    status = np.zeros(npb, np.int32)
    r = fn(len(plant), profs, C.byref(gpu), C.byref(coeffs), ptr(caps), len(caps), ptr(batches),
           len(batches), quantum, margin, npb, ptr(off), ptr(model), ptr(dp), ptr(tgt), ptr(bud),
           ptr(nb_out), ptr(total), ptr(sat), ptr(status), *extra)
    return r, dict(node_budget=nb_out, total=total, all_sat=sat, status=status)


def oracle_allocate(orc: Oracle, plant, gpu, coeffs, caps, batches, quantum, margin, prob):
    """allocate_budget per problem, restated in C (pals_oracle.c or_allocate)."""
    orc.lib.or_allocate.argtypes = _ALLOC_ARGS
    _, out = _alloc_call(orc.lib.or_allocate, plant, gpu, coeffs, caps, batches, quantum,
                         margin, prob)
    return out


def ref_allocate(ref: Reference, plant, gpu, coeffs, caps, batches, quantum, margin, prob):
    """The reference's allocate_budget (allocator.hpp:76) per problem."""
    ref.lib.ref_allocate.argtypes = _ALLOC_ARGS
    _, out = _alloc_call(ref.lib.ref_allocate, plant, gpu, coeffs, caps, batches, quantum,
                         margin, prob)
    return out


def ref_bench_allocate(ref: Reference, plant, gpu, coeffs, caps, batches, quantum, margin, prob,
                       threads: int):
    L = ref.lib
    L.ref_bench_allocate.restype = C.c_double
    L.ref_bench_allocate.argtypes = _ALLOC_ARGS + [C.c_int]
    secs, out = _alloc_call(L.ref_bench_allocate, plant, gpu, coeffs, caps, batches, quantum,
                            margin, prob, extra=(threads,))
    return secs, out


def _forest_args(fs):
    return [fs.n_trees, ptr(fs.tree_offset), ptr(fs.feature), ptr(fs.threshold), ptr(fs.left),
            ptr(fs.right), ptr(fs.value)]


def oracle_forest_predict(orc: Oracle, bundle, model_id: str, pts: np.ndarray):
    """PredictorBundle::predict restated in C (pals_oracle.c or_forest_predict)."""
    L = orc.lib
    L.or_forest_predict.argtypes = [C.c_int, C.c_int, _VP] + [C.c_int] + [_VP] * 6 + \
        [C.c_int] + [_VP] * 6 + [_VP, C.c_int64, _VP, _VP, _VP]
    pts = np.ascontiguousarray(pts, dtype=POINT_DT)
    n = len(pts)
    T, P, E = (np.empty(n) for _ in range(3))
    rc = L.or_forest_predict(len(bundle.model_ids), bundle.model_index(model_id),
                             C.byref(bundle.coeffs), *_forest_args(bundle.throughput),
                             *_forest_args(bundle.power), ptr(pts), n, ptr(T), ptr(P), ptr(E))
    assert rc == 0
    return T, P, E


def ref_train_bundle(ref: Reference, profiles, gpu, coeffs, path: str, n_trees=100,
                     max_depth=14, min_leaf=2, seed=2605) -> None:
    """Train a PredictorBundle with the reference's own pipeline (run_sweep + train_bundle)."""
    L = ref.lib
    L.ref_train_bundle.argtypes = [_VP, C.c_int, _VP, _VP, C.c_int, C.c_int, C.c_int,
                                   C.c_uint64, C.c_char_p]
    arr = (Profile * len(profiles))(*profiles)
    rc = L.ref_train_bundle(arr, len(profiles), C.byref(gpu), C.byref(coeffs), n_trees,
                            max_depth, min_leaf, seed, path.encode())
    if rc:
        raise RuntimeError(ref.last_error())


def ref_bundle_predict(ref: Reference, path: str, model_id: str, pts: np.ndarray):
    L = ref.lib
    L.ref_bundle_predict.argtypes = [C.c_char_p, C.c_char_p, _VP, C.c_int64, _VP, _VP, _VP]
    pts = np.ascontiguousarray(pts, dtype=POINT_DT)
    n = len(pts)
    T, P, E = (np.empty(n) for _ in range(3))
    rc = L.ref_bundle_predict(path.encode(), model_id.encode(), ptr(pts), n, ptr(T), ptr(P),
                              ptr(E))
    if rc:
        raise RuntimeError(ref.last_error())
    return T, P, E


def ref_select_forest(ref: Reference, path: str, model_id: str, pts, coeffs, queries):
    L = ref.lib
    L.ref_select_forest.argtypes = [C.c_char_p, C.c_char_p, _VP, C.c_int64, _VP, _VP, C.c_int64,
                                    _VP, _VP]
    q = np.ascontiguousarray(queries, dtype=QUERY_DT)
    idx = np.empty(len(q), np.int32)
    rs = np.empty(len(q), np.uint8)
    rc = L.ref_select_forest(path.encode(), model_id.encode(), ptr(pts), len(pts),
                             C.byref(coeffs), ptr(q), len(q), ptr(idx), ptr(rs))
    if rc:
        raise RuntimeError(ref.last_error())
    return idx, rs


def ref_bench_predict(ref: Reference, path: str, model_id: str, pts, threads: int) -> float:
    L = ref.lib
    L.ref_bench_predict.restype = C.c_double
    L.ref_bench_predict.argtypes = [C.c_char_p, C.c_char_p, _VP, C.c_int64, C.c_int]
    pts = np.ascontiguousarray(pts, dtype=POINT_DT)
    return L.ref_bench_predict(path.encode(), model_id.encode(), ptr(pts), len(pts), threads)


# ---- Pareto frontier (pareto.hpp) -------------------------------------------------
def oracle_build_frontier(orc: Oracle, pts, thr, eff) -> np.ndarray:
    """build_frontier restated in C: frontier indices into pts, throughput ascending."""
    L = orc.lib
    L.or_build_frontier.argtypes = [_VP, _VP, _VP, C.c_int64, _VP, _VP]
    pts = np.ascontiguousarray(pts, dtype=POINT_DT)
    thr = np.ascontiguousarray(thr, np.float64)
    eff = np.ascontiguousarray(eff, np.float64)
    out = np.empty(max(1, len(pts)), np.int64)
    n = C.c_int64(0)
    rc = L.or_build_frontier(ptr(pts), ptr(thr), ptr(eff), len(pts), ptr(out), C.byref(n))
    if rc:
        raise RuntimeError(f"or_build_frontier rc={rc}")
    return out[: n.value].copy()


def _frontier_out(n):
    return (np.zeros(max(1, n), POINT_DT), np.empty(max(1, n)), np.empty(max(1, n)))


def ref_build_frontier(ref: Reference, pts, thr, eff):
    """The reference's build_frontier: (points, throughput, efficiency) of the frontier."""
    L = ref.lib
    L.ref_build_frontier.argtypes = [_VP, _VP, _VP, C.c_int64, _VP, _VP, _VP, _VP]
    pts = np.ascontiguousarray(pts, dtype=POINT_DT)
    thr = np.ascontiguousarray(thr, np.float64)
    eff = np.ascontiguousarray(eff, np.float64)
    op, ot, oe = _frontier_out(len(pts))
    n = C.c_int64(0)
    rc = L.ref_build_frontier(ptr(pts), ptr(thr), ptr(eff), len(pts), ptr(op), ptr(ot), ptr(oe),
                              C.byref(n))
    if rc:
        raise RuntimeError(f"ref_build_frontier rc={rc}: {ref.last_error()}")
    k = n.value
    return op[:k].copy(), ot[:k].copy(), oe[:k].copy()


def ref_evaluate_regime(ref: Reference, regime: str, prof, gpu, coeffs, caps, batches, tps):
    L = ref.lib
    L.ref_evaluate_regime.argtypes = [C.c_char_p, _VP, _VP, _VP, _VP, C.c_int, _VP, C.c_int, _VP,
                                      C.c_int, _VP, _VP, _VP, _VP]
    caps = np.ascontiguousarray(caps, np.float64)
    batches = np.ascontiguousarray(batches, np.int32)
    tps = np.ascontiguousarray(tps, np.int32)
    op, ot, oe = _frontier_out(len(caps) * len(batches) * len(tps) + 1)
    n = C.c_int64(0)
    rc = L.ref_evaluate_regime(regime.encode(), C.byref(prof), C.byref(gpu), C.byref(coeffs),
                               ptr(caps), len(caps), ptr(batches), len(batches), ptr(tps),
                               len(tps), ptr(op), ptr(ot), ptr(oe), C.byref(n))
    if rc:
        raise RuntimeError(f"ref_evaluate_regime rc={rc}: {ref.last_error()}")
    k = n.value
    return op[:k].copy(), ot[:k].copy(), oe[:k].copy()


def ref_verify_dominance(ref: Reference, a_thr, a_eff, b_thr, b_eff):
    L = ref.lib
    L.ref_verify_dominance.argtypes = [_VP, _VP, C.c_int64, _VP, _VP, C.c_int64, _VP, _VP]
    a_thr, a_eff, b_thr, b_eff = (np.ascontiguousarray(x, np.float64)
                                  for x in (a_thr, a_eff, b_thr, b_eff))
    cov = np.zeros(max(1, len(b_thr)), np.uint8)
    dom = C.c_int(0)
    L.ref_verify_dominance(ptr(a_thr), ptr(a_eff), len(a_thr), ptr(b_thr), ptr(b_eff),
                           len(b_thr), ptr(cov), C.byref(dom))
    return bool(dom.value), cov[: len(b_thr)].astype(bool)


def ref_bench_frontier(ref: Reference, prof, gpu, coeffs, pts, reps: int = 1):
    L = ref.lib
    L.ref_bench_frontier.restype = C.c_double
    L.ref_bench_frontier.argtypes = [_VP, _VP, _VP, _VP, C.c_int64, C.c_int, _VP]
    pts = np.ascontiguousarray(pts, dtype=POINT_DT)
    n = C.c_int64(0)
    t = L.ref_bench_frontier(C.byref(prof), C.byref(gpu), C.byref(coeffs), ptr(pts), len(pts),
                             reps, C.byref(n))
    return t, n.value
