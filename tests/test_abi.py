"""The C-ABI boundary on CPU (no GPU needed): libmppi_b200.so loads, exports every symbol
include/mppi.h declares, the ctypes mirror matches the C struct layout, and argument
validation fails cleanly before touching a device."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mppi.h")


@pytest.fixture(scope="module")
def capi():
    from paper_1509_01149_b200 import build
    build.build()
    from paper_1509_01149_b200 import _capi
    _capi.lib()
    return _capi


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mppi_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(capi):
    funcs = header_functions()
    assert len(funcs) >= 15
    L = capi.lib()
    for f in funcs:
        assert hasattr(L, f), f
    assert sorted(capi.EXPORTS) == funcs
    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (mppi_\w+)", out))
    assert set(funcs) <= exported
    assert capi.lib().mppi_abi_version() == 1


def test_probe_library_exports_its_header():
    """libmppi_probe.so (FP32 peak probe, BM32 sweep probe) exports what include/mppi_probe.h declares."""
    from paper_1509_01149_b200 import probe_build
    lib = probe_build.build()
    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "mppi_probe.h")).read(), flags=re.S)
    funcs = sorted(set(re.findall(r"\b(mppi_[a-z0-9_]+)\s*\(", src)))
    assert funcs == ["mppi_probe_bm32", "mppi_probe_fp32"]
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    assert set(funcs) <= set(re.findall(r" T (mppi_\w+)", out))


def test_library_is_sm100a(capi):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _c_layout():
    """sizeof/offsetof of the public structs as the C compiler sees them."""
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "mppi.h"
#define P(T) printf(#T " %zu\n", sizeof(T));
#define O(T, f) printf(#T "." #f " %zu\n", offsetof(T, f));
int main(void) {
  P(mppi_dynamics_t) P(mppi_cost_t) P(mppi_info_t) P(mppi_stats_t) P(mppi_dist_t)
  P(mppi_quadrotor_cost_t) P(mppi_linear_dynamics_t) P(mppi_racecar_dynamics_t)
  O(mppi_dynamics_t, p) O(mppi_cost_t, p) O(mppi_quadrotor_cost_t, n_obstacles)
  O(mppi_quadrotor_cost_t, obstacles_xy) O(mppi_info_t, workspace_bytes) O(mppi_stats_t, eta)
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "l.c")
        exe = os.path.join(d, "l")
        open(src, "w").write(prog)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, src])
        out = subprocess.run([exe], capture_output=True, text=True).stdout
    return dict(line.rsplit(" ", 1) for line in out.strip().splitlines())


def test_ctypes_layout_matches_header(capi):
    c = {k: int(v) for k, v in _c_layout().items()}
    A = capi
    assert c["mppi_dynamics_t"] == C.sizeof(A.dynamics_t)
    assert c["mppi_cost_t"] == C.sizeof(A.cost_t)
    assert c["mppi_info_t"] == C.sizeof(A.info_t)
    assert c["mppi_stats_t"] == C.sizeof(A.stats_t)
    assert c["mppi_dist_t"] == C.sizeof(A.dist_t)
    assert c["mppi_quadrotor_cost_t"] == C.sizeof(A.quadrotor_cost_t)
    assert c["mppi_linear_dynamics_t"] == C.sizeof(A.linear_dynamics_t)
    assert c["mppi_racecar_dynamics_t"] == C.sizeof(A.racecar_dynamics_t)
    assert c["mppi_dynamics_t.p"] == A.dynamics_t.p.offset
    assert c["mppi_cost_t.p"] == A.cost_t.p.offset
    assert c["mppi_quadrotor_cost_t.n_obstacles"] == A.quadrotor_cost_t.n_obstacles.offset
    assert c["mppi_quadrotor_cost_t.obstacles_xy"] == A.quadrotor_cost_t.obstacles_xy.offset
    assert c["mppi_info_t.workspace_bytes"] == A.info_t.workspace_bytes.offset
    assert c["mppi_stats_t.eta"] == A.stats_t.eta.offset


def _create(capi, plant="cartpole", K=256, T=10, dt=0.02, lam=5e-3, nu=1.0, m=None, Sigma=None,
            R=None, dist=None, struct_size_delta=0):
    from paper_1509_01149_b200.plants import PlantSpec
    spec = PlantSpec(plant)
    spec.dyn.struct_size += struct_size_delta
    m = spec.m if m is None else m
    S = np.eye(m) * 0.005 if Sigma is None else np.asarray(Sigma, np.float64)
    Rm = np.eye(m) if R is None else np.asarray(R, np.float64)
    S = np.ascontiguousarray(S)
    Rm = np.ascontiguousarray(Rm)
    ctx = C.c_void_p()
    st = capi.lib().mppi_create(C.byref(spec.dyn), C.byref(spec.cost), K, T, dt, lam, nu, m,
                                S.ctypes.data_as(C.POINTER(C.c_double)),
                                Rm.ctypes.data_as(C.POINTER(C.c_double)),
                                C.byref(dist) if dist is not None else None, None, C.byref(ctx))
    return st, ctx


@pytest.mark.parametrize("kw,status", [
    (dict(K=0), 1), (dict(K=254), 1), (dict(T=0), 1), (dict(T=5000), 1), (dict(dt=0.0), 1),
    (dict(dt=float("nan")), 1), (dict(lam=0.0), 1), (dict(lam=-1.0), 1), (dict(nu=0.5), 1),
    (dict(nu=float("inf")), 1), (dict(m=2), 1), (dict(struct_size_delta=4), 1),
    (dict(Sigma=[[-1.0]]), 2), (dict(R=[[0.0]]), 2),
    (dict(plant="racecar", Sigma=[[1.0, 2.0], [2.0, 1.0]]), 2),
    (dict(plant="racecar", Sigma=[[1.0, 0.5], [0.4, 1.0]]), 2),
])
def test_validation_errors(capi, kw, status):
    st, ctx = _create(capi, **kw)
    assert st == status
    assert not ctx.value
    assert len(capi.lib().mppi_last_error()) > 0


def test_quadrotor_negative_position_weight_rejected(capi):
    """The rollout folds sqrt(w) into the position differences, so w_xy, w_z < 0 are refused
    (include/mppi.h, mppi_quadrotor_cost_t) -- before any device is touched."""
    from paper_1509_01149_b200.plants import PlantSpec
    for field in ("w_xy", "w_z"):
        spec = PlantSpec("quadrotor")
        setattr(spec.cost.p.quadrotor, field, -1.0)
        S = np.ascontiguousarray(np.eye(4) * 0.005)
        Rm = np.ascontiguousarray(np.eye(4))
        ctx = C.c_void_p()
        st = capi.lib().mppi_create(C.byref(spec.dyn), C.byref(spec.cost), 256, 10, 0.02, 5e-3, 1.0, 4,
                                    S.ctypes.data_as(C.POINTER(C.c_double)),
                                    Rm.ctypes.data_as(C.POINTER(C.c_double)), None, None, C.byref(ctx))
        assert st == 1 and not ctx.value
        assert b"w_xy and w_z" in capi.lib().mppi_last_error()


def test_dist_validation(capi):
    st, _ = _create(capi, K=256, dist=capi.dist_t(2, 2))
    assert st == 1
    st, _ = _create(capi, K=1000, dist=capi.dist_t(0, 8))     # 125 per rank: not a multiple of 4
    assert st == 1
    st, _ = _create(capi, K=256, dist=capi.dist_t(0, 3))      # not divisible
    assert st == 1


def test_null_arguments(capi):
    L = capi.lib()
    assert L.mppi_optimize(None, None, None, 0, 0, None) == 1
    assert L.mppi_info(None, None) == 1
    L.mppi_destroy(None)
    assert L.mppi_last_launch_count(None) == 0
    assert L.mppi_gather_record_len(None) == -1
    assert L.mppi_accumulate_record(None, None) == 1
    assert L.mppi_apply_gathered(None, None, None, 1) == 1
    assert capi.lib().mppi_status_string(2) == b"MPPI_ERR_NOT_SPD"


def test_create_without_gpu_fails_loudly(capi):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    st, ctx = _create(capi)
    assert st == 4 and not ctx.value       # MPPI_ERR_CUDA, no CPU fallback
