"""Multi-GPU driver (pals_multi_*): one worker thread and one context per device,
contiguous shards of queries / traces, results straight to host or gathered into
device 0 over NVLink (cudaMemcpyPeerAsync). Mirrors the single-context calls of
wattserve.py with the same arguments and results; see include/pals_gpu.h."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .abi import (PLANT_DT, POINT_DT, QUERY_DT, SIGNAL_DT, STATE_DT, STEPDETAIL_DT, STEPLOG_DT,
                  SUMMARY_DT, TRACE_DT, Coeffs, CtrlCfg, GpuSpec, Profile, ReplaySpec,
                  TraceBatch, ptr, state_array)
from ._lib import check


class Multi:
    """pals_multi over `devices` (a device may repeat: several contexts on one GPU)."""

    def __init__(self, devices):
        self.lib = _lib.load()
        devs = (C.c_int32 * len(devices))(*devices)
        h = C.c_void_p()
        check(self.lib.pals_multi_create(devs, len(devices), C.byref(h)))
        self.h = h
        self.devices = list(devices)

    def close(self):
        if self.h:
            self.lib.pals_multi_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self):
        return int(self.lib.pals_multi_size(self.h))

    def set_gather(self, to_device0: bool):
        check(self.lib.pals_multi_set_gather(self.h, 1 if to_device0 else 0))

    def launches(self) -> int:
        return sum(int(self.lib.pals_ctx_launch_count(self.lib.pals_multi_ctx(self.h, r)))
                   for r in range(len(self)))

    def last_ms(self) -> np.ndarray:
        ms = np.zeros(len(self))
        check(self.lib.pals_multi_last_ms(self.h, ptr(ms)))
        return ms

    def model_analytic(self, profile: Profile, gpu: GpuSpec) -> int:
        i = C.c_int32()
        check(self.lib.pals_multi_model_analytic(self.h, C.byref(profile), C.byref(gpu),
                                                 C.byref(i)))
        return i.value

    def model_table(self, points, t_hat, p_gpu) -> int:
        pts = np.ascontiguousarray(points, POINT_DT)
        t = np.ascontiguousarray(t_hat, np.float64)
        p = np.ascontiguousarray(p_gpu, np.float64)
        i = C.c_int32()
        check(self.lib.pals_multi_model_table(self.h, ptr(pts), ptr(t), ptr(p), len(pts),
                                              C.byref(i)))
        return i.value

    def select(self, model: int, points, coeffs: Coeffs, queries, index=None, reason=None):
        pts = np.ascontiguousarray(points, POINT_DT)
        q = np.ascontiguousarray(queries, QUERY_DT)
        idx = np.empty(len(q), np.int32) if index is None else index
        rs = np.empty(len(q), np.uint8) if reason is None else reason
        check(self.lib.pals_multi_select(self.h, model, ptr(pts), len(pts), C.byref(coeffs),
                                         ptr(q), len(q), ptr(idx), ptr(rs)))
        return idx, rs

    def replay(self, models, plant, gpu: GpuSpec, coeffs: Coeffs, caps, batches, cfg: CtrlCfg,
               spec: ReplaySpec, details: bool = False, summaries=None):
        ids = (C.c_int32 * len(models))(*models)
        profs = (Profile * len(plant))(*plant)
        caps = np.ascontiguousarray(caps, np.float64)
        batches = np.ascontiguousarray(batches, np.int32)
        summ = np.zeros(spec.n_traces, SUMMARY_DT) if summaries is None else summaries
        nl = min(spec.n_log_traces, spec.n_traces)
        logs = np.zeros(max(1, nl * spec.n_steps), STEPLOG_DT)
        det = np.zeros(max(1, nl * spec.n_steps), STEPDETAIL_DT)
        check(self.lib.pals_multi_replay(self.h, len(models), ids, profs, C.byref(gpu),
                                         C.byref(coeffs), ptr(caps), len(caps), ptr(batches),
                                         len(batches), C.byref(cfg), C.byref(spec), ptr(summ),
                                         ptr(logs) if nl else None,
                                         ptr(det) if (nl and details) else None))
        out = (summ, logs[: nl * spec.n_steps])
        return out + (det[: nl * spec.n_steps],) if details else out

    def replay_traces(self, models, plant, gpu: GpuSpec, coeffs: Coeffs, caps, batches,
                      cfg: CtrlCfg, traces, signal, n_steps: int, interval_s: float = 0.5,
                      first_step: int = 0, init=None, init_plant=None, n_log_traces: int = 0,
                      details: bool = False):
        ids = (C.c_int32 * len(models))(*models)
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
        check(self.lib.pals_multi_replay_traces(self.h, len(models), ids, profs, C.byref(gpu),
                                                C.byref(coeffs), ptr(caps), len(caps),
                                                ptr(batches), len(batches), C.byref(cfg),
                                                C.byref(b)))
        out = {"summaries": summ[:n], "final_state": fin[:n], "final_plant": finp[:n],
               "logs": logs[: nl * n_steps]}
        if details:
            out["details"] = det[: nl * n_steps]
        return out
