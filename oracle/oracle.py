"""fp64 CPU oracle for one MPPI step — Python face of oracle/liboracle.so.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.  It shares no
code with paper_1509_01149_b200/ (the CUDA path) and never imports it.

Paper: Williams, Aldrich & Theodorou, "Model Predictive Path Integral Control
using Covariance Variable Importance Sampling", arXiv:1509.01149.
Every numeric default below is either printed in the paper (cited by PAPER.md
line) or is a reading recorded in SURVEY.md §8.3 / Appendix A and DESIGN.md.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

from . import build as _build

PLANT_CARTPOLE, PLANT_RACECAR, PLANT_QUADROTOR, PLANT_LINEAR = 1, 2, 3, 4
PLANT_IDS = {"cartpole": 1, "racecar": 2, "quadrotor": 3, "linear": 4}
STATE_DIM = {"cartpole": 4, "racecar": 6, "quadrotor": 16}
CONTROL_DIM = {"cartpole": 1, "racecar": 2, "quadrotor": 4}


def paper_params(plant: str) -> np.ndarray:
    """Plant + cost parameter vector of the oracle (fp64), layout per plant.

    cartpole  [g, l, kv, w_p, w_theta, w_thetadot, w_pdot]
        kv = 10 and the cost weights 1, 500, 1, 1: PAPER.md:395.  g = 9.81, l = 1:
        SPEC.md:344 / SURVEY A10.
    racecar   [mass, Iz, lf, lr, B, C, mu, Cm, Cr, Cd, vmin, g, steer_max, thr_min, thr_max,
               track_a, track_b, w_track, w_speed, v_ref]
        cost 100 d^2 + (vx - 7)^2 with axes 13, 6: PAPER.md:398.  Vehicle: SURVEY Appendix A
        (the paper's [HindThesis] model is unavailable).
    quadrotor [mass, arm, Ixx, Iyy, Izz, gamma, km, g, umin, umax, cphi_min,
               gx, gy, gz, w_xy, w_z, w_yaw, w_vel, w_obs, obs_len, w_crash, ground_z, radius]
        cost weights 2.5, 150, 50, 1, 350, 12, 1000: PAPER.md:431.  Vehicle, goal, radius:
        SURVEY Appendix A / A12 / A13 (GRASP model [michael2010grasp] only cited).
    """
    if plant == "cartpole":
        return np.array([9.81, 1.0, 10.0, 1.0, 500.0, 1.0, 1.0])
    if plant == "racecar":
        return np.array([21.88, 1.6, 0.34, 0.23, 4.0, 1.5, 0.9, 100.0, 1.0, 0.8, 2.0, 9.81,
                         0.6, -1.0, 1.0, 13.0, 6.0, 100.0, 1.0, 7.0])
    if plant == "quadrotor":
        return np.array([0.5, 0.175, 2.32e-3, 2.32e-3, 4.0e-3, 0.0245, 20.0, 9.81, 0.0, 4.0,
                         0.05, 50.0, 0.0, 2.0, 2.5, 150.0, 50.0, 1.0, 350.0, 12.0, 1000.0,
                         0.0, 0.5])
    raise ValueError(plant)


class _Problem(C.Structure):
    _fields_ = [("plant", C.c_int32), ("n", C.c_int32), ("m", C.c_int32), ("T", C.c_int32),
                ("dt", C.c_double), ("lam", C.c_double), ("nu", C.c_double),
                ("Sigma", C.POINTER(C.c_double)), ("R", C.POINTER(C.c_double)),
                ("params", C.POINTER(C.c_double)), ("n_params", C.c_int32),
                ("n_obstacles", C.c_int32), ("obstacles", C.POINTER(C.c_double)),
                ("penalty", C.c_double), ("At", C.POINTER(C.c_double))]


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = _build.build()
        L = C.CDLL(path)
        dp = C.POINTER(C.c_double)
        fp = C.POINTER(C.c_float)
        up = C.POINTER(C.c_uint32)
        ip = C.POINTER(C.c_int32)
        lp = C.POINTER(C.c_int64)
        pp = C.POINTER(_Problem)
        L.oracle_philox4x32_10.argtypes = [up, up, up]
        L.oracle_bm_radius.argtypes = [C.c_uint32]
        L.oracle_bm_radius.restype = C.c_float
        L.oracle_bm_angle.argtypes = [C.c_uint32, fp, fp]
        L.oracle_bm_normals.argtypes = [up, fp]
        L.oracle_bm_radius_words.argtypes = [up, C.c_int64, fp]
        L.oracle_bm_angle_words.argtypes = [up, C.c_int64, fp, fp]
        L.oracle_bm_accuracy.argtypes = [dp] * 5
        L.oracle_noise.argtypes = [C.c_uint64, C.c_uint64, C.c_int32, C.c_int64, C.c_int64,
                                   C.c_int32, fp]
        L.oracle_deriv.argtypes = [pp, dp, dp, dp]
        L.oracle_state_cost.argtypes = [pp, dp, C.c_int32]
        L.oracle_state_cost.restype = C.c_double
        L.oracle_obstacle_distance.argtypes = [pp, dp]
        L.oracle_obstacle_distance.restype = C.c_double
        L.oracle_plant_step.argtypes = [pp, dp, dp, ip]
        L.oracle_plant_step.restype = C.c_double
        L.oracle_rollout_costs.argtypes = [pp, dp, dp, fp, C.c_int64, C.c_int32, C.c_int32,
                                           dp, ip]
        L.oracle_update.argtypes = [pp, dp, fp, C.c_int64, dp, lp, dp, dp, dp]
        L.oracle_optimize.argtypes = [pp, dp, dp, fp, C.c_int64, C.c_int32, dp, lp, dp]
        L.oracle_shift.argtypes = [dp, C.c_int32, C.c_int32, dp]
        L.oracle_rollout_stepcosts.argtypes = [pp, dp, dp, fp, C.c_int64, C.c_int32, dp, C.c_int32]
        L.oracle_update_ctg.argtypes = [pp, dp, fp, C.c_int64, dp, dp, dp]
        L.oracle_crash_margin.argtypes = [pp, dp, dp, fp, C.c_int64, C.c_int32, dp]
        L.oracle_euler_margin.argtypes = [pp, dp, dp, fp, C.c_int64, C.c_int32, dp]
        L.oracle_trajectory.argtypes = [pp, dp, dp, fp, C.c_int64, C.c_int64, dp]
        _LIB = L
    return _LIB


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


class Problem:
    """One MPPI problem (Alg. 1 "Given" block) for the oracle."""

    def __init__(self, plant, T, dt, lam, nu, Sigma, R, params=None, obstacles=None,
                 n=None, m=None, penalty=1e30, At=None):
        self.plant = plant
        self.plant_id = PLANT_IDS[plant]
        if plant == "linear":
            assert n is not None and m is not None and params is not None
            self.n, self.m = int(n), int(m)
        else:
            self.n, self.m = STATE_DIM[plant], CONTROL_DIM[plant]
        self.T = int(T)
        self.dt, self.lam, self.nu = float(dt), float(lam), float(nu)
        self.Sigma = np.ascontiguousarray(np.asarray(Sigma, np.float64).reshape(self.m, self.m))
        self.R = np.ascontiguousarray(np.asarray(R, np.float64).reshape(self.m, self.m))
        self.params = np.ascontiguousarray(
            paper_params(plant) if params is None else np.asarray(params, np.float64))
        obs = np.zeros((0, 2)) if obstacles is None else np.asarray(obstacles, np.float64)
        self.obstacles = np.ascontiguousarray(obs.reshape(-1, 2))
        self.penalty = float(penalty)
        # NEXT-3: per-step sampling transforms A_t [T][m][m] (None: A_t = sqrt(nu) I)
        self.At = None if At is None else np.ascontiguousarray(
            np.asarray(At, np.float64).reshape(self.T, self.m, self.m))
        self._s = _Problem(self.plant_id, self.n, self.m, self.T, self.dt, self.lam, self.nu,
                           _dp(self.Sigma), _dp(self.R), _dp(self.params), len(self.params),
                           len(self.obstacles),
                           _dp(self.obstacles) if len(self.obstacles) else None, self.penalty,
                           _dp(self.At) if self.At is not None else None)

    def ptr(self):
        return C.byref(self._s)


# --------------------------------------------------------------------------- noise
def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(np.asarray(ctr, np.uint32))
    k = np.ascontiguousarray(np.asarray(key, np.uint32))
    out = np.zeros(4, np.uint32)
    up = C.POINTER(C.c_uint32)
    lib().oracle_philox4x32_10(c.ctypes.data_as(up), k.ctypes.data_as(up), out.ctypes.data_as(up))
    return out


def bm_normals(w):
    w = np.ascontiguousarray(np.asarray(w, np.uint32))
    z = np.zeros(4, np.float32)
    lib().oracle_bm_normals(w.ctypes.data_as(C.POINTER(C.c_uint32)), _fp(z))
    return z


def bm_radius_words(w):
    """r(w) of Appendix B "Radius" for every word of the uint32 array w."""
    w = np.ascontiguousarray(np.asarray(w, np.uint32))
    r = np.empty(w.shape, np.float32)
    lib().oracle_bm_radius_words(w.ctypes.data_as(C.POINTER(C.c_uint32)), w.size, _fp(r))
    return r


def bm_angle_words(w):
    """(sin theta(w), cos theta(w)) of Appendix B "Angle" for every word of the uint32 array w."""
    w = np.ascontiguousarray(np.asarray(w, np.uint32))
    s = np.empty(w.shape, np.float32)
    c = np.empty(w.shape, np.float32)
    lib().oracle_bm_angle_words(w.ctypes.data_as(C.POINTER(C.c_uint32)), w.size, _fp(s), _fp(c))
    return s, c


def bm_accuracy():
    v = [C.c_double() for _ in range(5)]
    lib().oracle_bm_accuracy(*[C.byref(x) for x in v])
    return dict(zip(["ln_ulp", "r_ulp", "sin_err", "cos_err", "max_abs_z"], [x.value for x in v]))


def noise(seed, step, T, K, m, k0=0):
    """eps [T][K][m] fp32 for global samples k0..k0+K-1."""
    out = np.zeros((T, K, m), np.float32)
    rc = lib().oracle_noise(seed, step, T, k0, K, m, _fp(out))
    assert rc == 0
    return out


# --------------------------------------------------------------------------- plants
def deriv(pb: Problem, x, v):
    x = np.ascontiguousarray(np.asarray(x, np.float64))
    v = np.ascontiguousarray(np.asarray(v, np.float64))
    xd = np.zeros(pb.n)
    assert lib().oracle_deriv(pb.ptr(), _dp(x), _dp(v), _dp(xd)) == 0
    return xd


def state_cost(pb: Problem, x, crashed=0):
    x = np.ascontiguousarray(np.asarray(x, np.float64))
    return lib().oracle_state_cost(pb.ptr(), _dp(x), int(crashed))


def obstacle_distance(pb: Problem, x):
    x = np.ascontiguousarray(np.asarray(x, np.float64))
    return lib().oracle_obstacle_distance(pb.ptr(), _dp(x))


def plant_step(pb: Problem, x, v, crashed=0):
    """x <- x + F(x, v) dt; returns (x', q(x'), crashed')."""
    x = np.array(x, np.float64)
    v = np.ascontiguousarray(np.asarray(v, np.float64))
    c = C.c_int32(int(crashed))
    q = lib().oracle_plant_step(pb.ptr(), _dp(x), _dp(v), C.byref(c))
    return x, q, c.value


# --------------------------------------------------------------------------- MPPI step
MODES = {"fp64": 0, "twin_f32": 1, "twin_f32_via_f64": 2}


def rollout_costs(pb: Problem, x0, U, eps, mode="fp64", nthreads=0, return_crashed=False):
    x0 = np.ascontiguousarray(np.asarray(x0, np.float64))
    U = np.ascontiguousarray(np.asarray(U, np.float64).reshape(pb.T, pb.m))
    eps = np.ascontiguousarray(np.asarray(eps, np.float32))
    assert eps.shape[0] == pb.T and eps.shape[2] == pb.m
    K = eps.shape[1]
    costs = np.zeros(K)
    crashed = np.zeros(K, np.int32)
    rc = lib().oracle_rollout_costs(pb.ptr(), _dp(x0), _dp(U), _fp(eps), K, MODES[mode],
                                    nthreads, _dp(costs),
                                    crashed.ctypes.data_as(C.POINTER(C.c_int32)))
    if rc:
        raise ValueError("oracle_rollout_costs rc=%d" % rc)
    return (costs, crashed) if return_crashed else costs


def update(pb: Problem, costs, eps, U):
    """PAPER.md:318-321 given costs: returns (U', k*, S_min, eta, weights)."""
    costs = np.ascontiguousarray(np.asarray(costs, np.float64))
    eps = np.ascontiguousarray(np.asarray(eps, np.float32))
    U2 = np.array(U, np.float64).reshape(pb.T, pb.m).copy()
    K = len(costs)
    kstar = C.c_int64()
    smin = C.c_double()
    eta = C.c_double()
    w = np.zeros(K)
    rc = lib().oracle_update(pb.ptr(), _dp(costs), _fp(eps), K, _dp(U2), C.byref(kstar),
                             C.byref(smin), C.byref(eta), _dp(w))
    if rc:
        raise ValueError("oracle_update rc=%d" % rc)
    return U2, kstar.value, smin.value, eta.value, w


def optimize(pb: Problem, x0, U, eps, nthreads=0):
    """One full MPPI step (fp64): returns dict(U, costs, kstar, smin, eta, weights)."""
    costs = rollout_costs(pb, x0, U, eps, nthreads=nthreads)
    U2, kstar, smin, eta, w = update(pb, costs, eps, U)
    return dict(U=U2, costs=costs, kstar=kstar, smin=smin, eta=eta, weights=w)


def rollout_stepcosts(pb: Problem, x0, U, eps, nthreads=0, mode="fp64"):
    """q~_{t,k} of every step, shape [K][T] (fp64; or an fp32 conditioning twin, see MODES)."""
    x0 = np.ascontiguousarray(np.asarray(x0, np.float64))
    U = np.ascontiguousarray(np.asarray(U, np.float64).reshape(pb.T, pb.m))
    eps = np.ascontiguousarray(np.asarray(eps, np.float32))
    K = eps.shape[1]
    out = np.zeros((K, pb.T))
    assert lib().oracle_rollout_stepcosts(pb.ptr(), _dp(x0), _dp(U), _fp(eps), K, nthreads, _dp(out),
                                          MODES[mode]) == 0
    return out


def cost_to_go(stepcosts):
    """S~_{t,k} = sum_{j >= t} q~_{j,k}, shape [T][K] from [K][T] step costs."""
    return np.cumsum(np.asarray(stepcosts)[:, ::-1], axis=1)[:, ::-1].T


def well_conditioned_ctg(pb: Problem, x0, U, eps, rel=1e-5, nthreads=0):
    """SURVEY A19 applied to the cost-to-go: sample k is well-conditioned iff at every t the fp32
    twins' S~_{t,k} (the three of `well_conditioned`) are within rel * max(|S~_{0,k}|, 1) of fp64
    and its crash and Euler-guard margins pass (A19', A19'').  Returns (mask[K], ctg fp64 [T][K])."""
    ref = cost_to_go(rollout_stepcosts(pb, x0, U, eps, nthreads))
    scale = np.maximum(np.abs(ref[0]), 1.0)
    ok = np.ones(ref.shape[1], bool)
    for mode, e in (("twin_f32", eps), ("twin_f32_via_f64", eps), ("twin_f32", perturb_ulp(eps))):
        tw = cost_to_go(rollout_stepcosts(pb, x0, U, e, nthreads, mode))
        ok &= np.all(np.abs(tw - ref) <= rel * scale, axis=0)
    ok &= crash_margin(pb, x0, U, eps, nthreads) >= CRASH_MARGIN
    ok &= euler_margin(pb, x0, U, eps, nthreads) >= EULER_MARGIN
    return ok, ref


def update_ctg(pb: Problem, stepcosts, eps, U):
    """PAPER.md:320/:367 with per-timestep cost-to-go weights: returns (U', smin[T], eta[T])."""
    sc = np.ascontiguousarray(np.asarray(stepcosts, np.float64))
    eps = np.ascontiguousarray(np.asarray(eps, np.float32))
    U2 = np.array(U, np.float64).reshape(pb.T, pb.m).copy()
    K = sc.shape[0]
    smin = np.zeros(pb.T)
    eta = np.zeros(pb.T)
    assert lib().oracle_update_ctg(pb.ptr(), _dp(sc), _fp(eps), K, _dp(U2), _dp(smin), _dp(eta)) == 0
    return U2, smin, eta


def shift(U, u_init):
    U2 = np.array(U, np.float64).copy()
    T, m = U2.shape
    ui = np.ascontiguousarray(np.asarray(u_init, np.float64).reshape(m))
    lib().oracle_shift(_dp(U2), T, m, _dp(ui))
    return U2


def trajectory(pb: Problem, x0, U, eps, k):
    x0 = np.ascontiguousarray(np.asarray(x0, np.float64))
    U = np.ascontiguousarray(np.asarray(U, np.float64).reshape(pb.T, pb.m))
    eps = np.ascontiguousarray(np.asarray(eps, np.float32))
    xs = np.zeros((pb.T + 1, pb.n))
    assert lib().oracle_trajectory(pb.ptr(), _dp(x0), _dp(U), _fp(eps), eps.shape[1], k,
                                   _dp(xs)) == 0
    return xs


def crash_margin(pb: Problem, x0, U, eps, nthreads=0):
    """Per-sample distance of the fp64 crash decisions from their thresholds (quadrotor; +inf
    otherwise), over the steps up to the first crash (reading A19')."""
    x0 = np.ascontiguousarray(np.asarray(x0, np.float64))
    U = np.ascontiguousarray(np.asarray(U, np.float64).reshape(pb.T, pb.m))
    eps = np.ascontiguousarray(np.asarray(eps, np.float32))
    out = np.zeros(eps.shape[1])
    assert lib().oracle_crash_margin(pb.ptr(), _dp(x0), _dp(U), _fp(eps), eps.shape[1], nthreads, _dp(out)) == 0
    return out


def euler_margin(pb: Problem, x0, U, eps, nthreads=0):
    """Per-sample min |cos phi| of the fp64 rollout over the steps up to the first crash
    (quadrotor; +inf otherwise): the distance of the ZXY Euler-rate guard from its sign decision
    (reading A19'')."""
    x0 = np.ascontiguousarray(np.asarray(x0, np.float64))
    U = np.ascontiguousarray(np.asarray(U, np.float64).reshape(pb.T, pb.m))
    eps = np.ascontiguousarray(np.asarray(eps, np.float32))
    out = np.zeros(eps.shape[1])
    assert lib().oracle_euler_margin(pb.ptr(), _dp(x0), _dp(U), _fp(eps), eps.shape[1], nthreads, _dp(out)) == 0
    return out


CRASH_MARGIN = 1e-4     # m; reading A19' (>= 10x the fp32 position error at 50 m)
EULER_MARGIN = 1e-4     # |cos phi|; reading A19'' (the guard's sign decision)


def perturb_ulp(eps):
    """eps with every element moved by exactly one ulp, up or down by a fixed hash of its own bits
    (deterministic, independent of how the columns are chunked): the input of the third
    conditioning twin (reading A19, round 2) -- a rollout whose cost moves by more than
    the twin tolerance under last-bit changes of its inputs is not rolled out stably in fp32."""
    e = np.ascontiguousarray(np.asarray(eps, np.float32))
    b = e.view(np.uint32).astype(np.uint64)
    up = ((b * np.uint64(0x9E3779B1)) >> np.uint64(31)) & np.uint64(1)
    return np.nextafter(e, np.where(up == 1, np.float32(np.inf), np.float32(-np.inf))).astype(np.float32)


def well_conditioned(pb: Problem, x0, U, eps, ref_costs=None, rel=1e-5, nthreads=0,
                     crash_tol=CRASH_MARGIN, euler_tol=EULER_MARGIN, perturbed=True):
    """sample k is well-conditioned iff the fp32 twins are within rel * max(|S_k|, 1)
    of the fp64 cost -- twin 1 (libm fp32), twin 2 (fma updates, fp64 transcendentals) and
    (round 2) twin 1 on the one-ulp-perturbed noise `perturb_ulp(eps)` -- and no decision of its
    fp64 rollout lies within the fp32 resolution of its threshold: crash (reading A19', crash_tol
    m) and the sign of the Euler-rate guard (reading A19'', |cos phi| >= euler_tol).
    Returns (mask, ref_costs)."""
    if ref_costs is None:
        ref_costs = rollout_costs(pb, x0, U, eps, "fp64", nthreads)
    scale = np.maximum(np.abs(ref_costs), 1.0)
    mask = np.ones(len(ref_costs), bool)
    twins = [("twin_f32", eps), ("twin_f32_via_f64", eps)]
    if perturbed:
        twins.append(("twin_f32", perturb_ulp(eps)))
    for mode, e in twins:
        mask &= np.abs(rollout_costs(pb, x0, U, e, mode, nthreads) - ref_costs) <= rel * scale
    if crash_tol:
        mask &= crash_margin(pb, x0, U, eps, nthreads) >= crash_tol
    if euler_tol:
        mask &= euler_margin(pb, x0, U, eps, nthreads) >= euler_tol
    return mask, ref_costs


def closed_loop(pb: Problem, x0, U0, steps, seed, u_init=None, K=None, nthreads=0):
    """Alg. 1 receding horizon with the oracle: optimise, send u_0,
    plant step (noise-free), shift.  Returns (states [steps+1][n], costs per step)."""
    U = np.array(U0, np.float64).reshape(pb.T, pb.m).copy()
    ui = np.zeros(pb.m) if u_init is None else np.asarray(u_init, np.float64)
    x = np.array(x0, np.float64)
    xs, qs = [x.copy()], []
    crashed = 0
    for step in range(steps):
        eps = noise(seed, step, pb.T, K, pb.m)
        r = optimize(pb, x, U, eps, nthreads=nthreads)
        U = r["U"]
        x, q, crashed = plant_step(pb, x, U[0], crashed)
        xs.append(x.copy())
        qs.append(q)
        U = shift(U, ui)
    return np.array(xs), np.array(qs)
