"""The C-ABI boundary, checked without a GPU: the library loads, exports every
symbol include/pals_gpu.h declares, its struct layouts match the Python mirrors,
and with no device it fails loudly instead of falling back to the CPU."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2605_21427_b200 import _lib, abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pals_gpu.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pals_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (pals_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(names) <= bound, set(names) - bound
    for n in names:
        assert getattr(lib, n) is not None


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_struct_layouts_match_c():
    prog = r"""
#include <stdio.h>
#include <stddef.h>
#include "pals_gpu.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n",
  sizeof(pals_gpu_spec), sizeof(pals_coeffs), sizeof(pals_profile), sizeof(pals_point),
  sizeof(pals_query), sizeof(pals_targets), sizeof(pals_ctrl_cfg), sizeof(pals_ctrl_state),
  sizeof(pals_decision), sizeof(pals_telemetry), sizeof(pals_replay_spec),
  sizeof(pals_trace_summary), sizeof(pals_step_log));
 printf("%zu %zu %zu %zu\n", offsetof(pals_profile, tp_keys), offsetof(pals_ctrl_state, current),
  offsetof(pals_ctrl_state, last_targets), offsetof(pals_replay_spec, seg_min));
 return 0;}
"""
    d = os.environ.get("TMPDIR", "/tmp")
    src = os.path.join(d, "pals_layout.c")
    exe = os.path.join(d, "pals_layout")
    with open(src, "w") as f:
        f.write(prog)
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
    sizes, offs = [list(map(int, ln.split())) for ln in
                   subprocess.run([exe], capture_output=True, text=True).stdout.splitlines()]
    want = [C.sizeof(t) for t in (abi.GpuSpec, abi.Coeffs, abi.Profile, abi.Point, abi.Query,
                                  abi.Targets, abi.CtrlCfg, abi.CtrlState, abi.Decision,
                                  abi.Telemetry, abi.ReplaySpec)]
    want += [abi.SUMMARY_DT.itemsize, abi.STEPLOG_DT.itemsize]
    assert sizes == want
    assert offs == [abi.Profile.tp_keys.offset, abi.CtrlState.current.offset,
                    abi.CtrlState.last_targets.offset, abi.ReplaySpec.seg_min.offset]
    assert abi.POINT_DT.itemsize == C.sizeof(abi.Point)
    assert abi.QUERY_DT.itemsize == C.sizeof(abi.Query)


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device failure mode")
def test_no_device_fails_loudly():
    from paper_2605_21427_b200.wattserve import Context, PalsError
    with pytest.raises(PalsError, match="no CUDA device"):
        Context(0)


def test_error_codes_map_to_reference_exceptions():
    from paper_2605_21427_b200 import wattserve as ws
    assert issubclass(ws.ConfigError, ws.PalsError)
    assert _lib._ERR[abi.PALS_ECONFIG] is ws.ConfigError
    assert _lib._ERR[abi.PALS_ERANGE] is ws.OutOfRange
    assert _lib._ERR[abi.PALS_EDATA] is ws.DataError


def test_workload_generators_are_deterministic():
    from paper_2605_21427_b200 import workloads
    a = workloads.gen_queries(1000, 2605, 5000.0, "mixed", budget=(600.0, 2000.0))
    b = workloads.gen_queries(1000, 2605, 5000.0, "mixed", budget=(600.0, 2000.0))
    assert a.tobytes() == b.tobytes()
    c = workloads.gen_queries(500, 2605, 5000.0, "mixed", budget=(600.0, 2000.0), first=500)
    assert c.tobytes() == a[500:].tobytes()  # shards compose
    assert 0.3 < np.mean(a["objective"]) < 0.7
    assert np.all((a["throughput_tps"] >= 0.05 * 5000.0) & (a["throughput_tps"] <= 5000.0))
    pts = workloads.cfg2()["points"]
    assert len(pts) == 65536
    # canonical sweep nesting cap -> batch -> tp (sweep.hpp:134-138)
    assert pts[0]["tp"] == 1 and pts[1]["tp"] == 2 and pts[4]["batch"] == 2
    assert pts[1024]["cap_watts"] == 100.0 + 300.0 * 1 / 63.0


def test_splitmix_matches_reference(oracle):
    from paper_2605_21427_b200 import workloads
    xs = np.array([0, 1, 2605, 2 ** 63 + 5, 2 ** 64 - 1], dtype=np.uint64)
    got = workloads.splitmix64(xs)
    for x, g in zip(xs.tolist(), got.tolist()):
        assert oracle.splitmix64(x) == g
