"""Python face of libmppi_b200.so: one MPPI optimisation step on a B200.

Thin binding over include/mppi.h with the same names (mppi_create -> MPPI(...),
mppi_optimize -> MPPI.optimize, ...).  PyTorch provides device memory and the stream;
every step of the path runs in the library's CUDA kernels.  There is no CPU fallback.
"""
import ctypes as C

import numpy as np
import torch

from . import _capi as A
from .plants import PlantSpec


def _fptr(t):
    return C.c_void_p(t.data_ptr())


def _check_dev(t, shape, dtype, name, device=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("%s must be a CUDA tensor" % name)
    if device is not None and t.device != device:
        # a pointer into another GPU's memory would reach the library as a foreign address
        raise ValueError("%s is on %s but this MPPI context lives on %s" % (name, t.device, device))
    if t.dtype != dtype or not t.is_contiguous() or tuple(t.shape) != tuple(shape):
        raise ValueError("%s must be a contiguous %s tensor of shape %s (got %s %s)"
                         % (name, dtype, tuple(shape), t.dtype, tuple(t.shape)))


def _host_f32(a, n, name):
    a = np.ascontiguousarray(np.asarray(a, np.float32).reshape(-1))
    if a.size != n:
        raise ValueError("%s must have %d entries" % (name, n))
    return a


class MPPI:
    """mppi_create(dynamics, cost, K, T, dt, lambda, nu, Sigma, R) — PAPER.md:346-352."""

    def __init__(self, plant, K, T, dt, lam, nu, Sigma, R, dynamics=None, cost=None,
                 obstacles=None, penalty=1e30, linear=None, rank=0, world=1, device=None):
        self.lib = A.lib()
        if device is not None:
            torch.cuda.set_device(device)
        self.spec = PlantSpec(plant, dynamics, cost, obstacles, penalty, linear)
        self.n, self.m = self.spec.n, self.spec.m
        self.K, self.T = int(K), int(T)
        self.Sigma = np.ascontiguousarray(np.asarray(Sigma, np.float64).reshape(self.m, self.m))
        self.R = np.ascontiguousarray(np.asarray(R, np.float64).reshape(self.m, self.m))
        self._stream = torch.cuda.current_stream().cuda_stream
        d = A.dist_t(rank, world)
        ctx = C.c_void_p()
        A.check(self.lib.mppi_create(
            C.byref(self.spec.dyn), C.byref(self.spec.cost), self.K, self.T, dt, lam, nu, self.m,
            self.Sigma.ctypes.data_as(C.POINTER(C.c_double)),
            self.R.ctypes.data_as(C.POINTER(C.c_double)), C.byref(d),
            C.c_void_p(self._stream), C.byref(ctx)))
        self.ctx = ctx
        inf = self.info()
        self.K_loc, self.k_offset = inf.K_loc, inf.k_offset
        self.device = torch.device("cuda", torch.cuda.current_device())

    def _check_dev(self, t, shape, dtype, name):
        _check_dev(t, shape, dtype, name, self.device)

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "ctx", None):
            self.lib.mppi_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self):
        out = A.info_t()
        A.check(self.lib.mppi_info(self.ctx, C.byref(out)))
        return out

    def _sync_stream(self):
        s = torch.cuda.current_stream().cuda_stream
        if s != self._stream:
            A.check(self.lib.mppi_set_stream(self.ctx, C.c_void_p(s)))
            self._stream = s

    def _x0(self, x0):
        return _host_f32(x0.detach().cpu().numpy() if isinstance(x0, torch.Tensor) else x0,
                         self.n, "x0")

    # ------------------------------------------------------------------ the step
    def optimize(self, x0, U, seed=0, step=0, noise=None):
        """mppi_optimize: U (CUDA float32 [T][m]) updated in place."""
        self._check_dev(U, (self.T, self.m), torch.float32, "U")
        if noise is not None:
            self._check_dev(noise, (self.T, self.K_loc, self.m), torch.float32, "noise")
        self._sync_stream()
        x = self._x0(x0)
        A.check(self.lib.mppi_optimize(self.ctx, x.ctypes.data_as(C.POINTER(C.c_float)), _fptr(U),
                                       seed, step, _fptr(noise) if noise is not None else None))
        return U

    def use_graph(self, enable=True):
        """mppi_use_graph: replay mppi_optimize as one CUDA graph (default on)."""
        A.check(self.lib.mppi_use_graph(self.ctx, 1 if enable else 0))

    def set_option(self, option, value):
        """mppi_set_option (A.MPPI_OPTION_*): execution options that never change results."""
        A.check(self.lib.mppi_set_option(self.ctx, option, int(value)))

    def optimize_host(self, x0, U, seed=0, step=0):
        """mppi_optimize_host: U is a host float32 array [T][m], updated in place (synchronous)."""
        if not (isinstance(U, np.ndarray) and U.dtype == np.float32 and U.flags.c_contiguous
                and U.shape == (self.T, self.m)):
            raise ValueError("U must be a C-contiguous float32 numpy array of shape (T, m)")
        self._sync_stream()
        x = self._x0(x0)
        A.check(self.lib.mppi_optimize_host(self.ctx, x.ctypes.data_as(C.POINTER(C.c_float)),
                                            U.ctypes.data_as(C.POINTER(C.c_float)), seed, step))
        return U

    def rollout_costs(self, x0, U, seed=0, step=0, noise=None, costs=None, min_key=None):
        self._check_dev(U, (self.T, self.m), torch.float32, "U")
        if noise is not None:
            self._check_dev(noise, (self.T, self.K_loc, self.m), torch.float32, "noise")
        if costs is None:
            costs = torch.empty(self.K_loc, dtype=torch.float32, device=U.device)
        self._check_dev(costs, (self.K_loc,), torch.float32, "costs")
        if min_key is None:
            min_key = torch.empty(1, dtype=torch.int64, device=U.device)
        self._check_dev(min_key, (1,), torch.int64, "min_key")
        self._sync_stream()
        x = self._x0(x0)
        A.check(self.lib.mppi_rollout_costs(
            self.ctx, x.ctypes.data_as(C.POINTER(C.c_float)), _fptr(U), seed, step,
            _fptr(noise) if noise is not None else None, _fptr(costs), _fptr(min_key)))
        return costs, min_key

    def accumulate(self, global_min_key=None, buf=None):
        if buf is None:
            buf = torch.empty(1 + self.T * self.m, dtype=torch.float32, device=self.device)
        self._check_dev(buf, (1 + self.T * self.m,), torch.float32, "buf")
        if global_min_key is not None:
            self._check_dev(global_min_key, (1,), torch.int64, "global_min_key")
        self._sync_stream()
        A.check(self.lib.mppi_accumulate(
            self.ctx, _fptr(global_min_key) if global_min_key is not None else None, _fptr(buf)))
        return buf

    def gather_record_len(self):
        return int(self.lib.mppi_gather_record_len(self.ctx))

    def accumulate_record(self, out=None):
        """mppi_accumulate_record: this rank's [key, eta, A] record against its own minimum (CUDA fp32)."""
        n = self.gather_record_len()
        if out is None:
            out = torch.empty(n, dtype=torch.float32, device=self.device)
        self._check_dev(out, (n,), torch.float32, "record")
        self._sync_stream()
        A.check(self.lib.mppi_accumulate_record(self.ctx, _fptr(out)))
        return out

    def apply_gathered(self, U, records):
        """mppi_apply_gathered: records [n][len] (CUDA fp32, e.g. an all-gather in rank order)."""
        self._check_dev(U, (self.T, self.m), torch.float32, "U")
        n = records.shape[0] if records.dim() == 2 else 1
        self._check_dev(records, (n, self.gather_record_len()) if records.dim() == 2 else (self.gather_record_len(),),
                        torch.float32, "records")
        self._sync_stream()
        A.check(self.lib.mppi_apply_gathered(self.ctx, _fptr(U), _fptr(records), n))
        return U

    def apply(self, U, buf):
        self._check_dev(U, (self.T, self.m), torch.float32, "U")
        self._check_dev(buf, (1 + self.T * self.m,), torch.float32, "buf")
        self._sync_stream()
        A.check(self.lib.mppi_apply(self.ctx, _fptr(U), _fptr(buf)))
        return U

    # ------------------------------------------------------------------ helpers
    def shift(self, U, u_init=None):
        self._check_dev(U, (self.T, self.m), torch.float32, "U")
        ui = _host_f32(np.zeros(self.m) if u_init is None else u_init, self.m, "u_init")
        self._sync_stream()
        A.check(self.lib.mppi_shift(self.ctx, _fptr(U), ui.ctypes.data_as(C.POINTER(C.c_float))))
        return U

    def noise(self, seed=0, step=0, out=None):
        if out is None:
            out = torch.empty((self.T, self.K_loc, self.m), dtype=torch.float32, device=self.device)
        self._check_dev(out, (self.T, self.K_loc, self.m), torch.float32, "out")
        self._sync_stream()
        A.check(self.lib.mppi_noise(self.ctx, seed, step, _fptr(out)))
        return out

    def attach_nccl(self, group=None):
        """mppi_nccl_attach: rank 0 draws an NCCL unique id, torch.distributed broadcasts it (when
        initialised), every rank attaches; afterwards optimize() runs the whole sharded step."""
        buf = (C.c_uint8 * A.MPPI_NCCL_ID_BYTES)()
        import torch.distributed as dist
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
        rank = dist.get_rank(group) if multi else 0
        if rank == 0:
            A.check(self.lib.mppi_nccl_unique_id(buf))
        if multi:
            t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
            buf = (C.c_uint8 * A.MPPI_NCCL_ID_BYTES)(*t.cpu().tolist())
        A.check(self.lib.mppi_nccl_attach(self.ctx, buf))

    def set_sampling_transform(self, At=None):
        """mppi_set_sampling_transform: per-step A_t [T][m][m] (fp64, Theorem 1) or None for sqrt(nu) I."""
        if At is None:
            A.check(self.lib.mppi_set_sampling_transform(self.ctx, None))
            return
        self._At = np.ascontiguousarray(np.asarray(At, np.float64).reshape(self.T, self.m, self.m))
        A.check(self.lib.mppi_set_sampling_transform(self.ctx, self._At.ctypes.data_as(C.POINTER(C.c_double))))

    def set_weighting(self, cost_to_go):
        """mppi_set_weighting: per-timestep cost-to-go weights or trajectory."""
        A.check(self.lib.mppi_set_weighting(
            self.ctx, A.MPPI_WEIGHTS_COST_TO_GO if cost_to_go else A.MPPI_WEIGHTS_TRAJECTORY))

    def cost_to_go(self, out=None):
        """mppi_cost_to_go: S~_{t,k} of the last cost-to-go step, CUDA [T][K_loc]."""
        if out is None:
            out = torch.empty((self.T, self.K_loc), dtype=torch.float32, device=self.device)
        self._check_dev(out, (self.T, self.K_loc), torch.float32, "out")
        self._sync_stream()
        A.check(self.lib.mppi_cost_to_go(self.ctx, _fptr(out)))
        return out

    def closed_loop(self, x, U, n_steps, seed=0, step0=0, u_init=None, reset_crash=True, log=True):
        """mppi_closed_loop: n_steps of Alg. 1 on the device (x: CUDA [n], U: CUDA [T][m], in/out).
        Returns (x_log [n_steps+1][n], u_log [n_steps][m], q_log [n_steps]) CUDA tensors or None."""
        self._check_dev(x, (self.n,), torch.float32, "x")
        self._check_dev(U, (self.T, self.m), torch.float32, "U")
        ui = _host_f32(np.zeros(self.m) if u_init is None else u_init, self.m, "u_init")
        xl = ul = ql = None
        if log:
            xl = torch.empty((n_steps + 1, self.n), dtype=torch.float32, device=x.device)
            ul = torch.empty((n_steps, self.m), dtype=torch.float32, device=x.device)
            ql = torch.empty((n_steps,), dtype=torch.float32, device=x.device)
        self._sync_stream()
        A.check(self.lib.mppi_closed_loop(
            self.ctx, _fptr(x), _fptr(U), seed, step0, int(n_steps), ui.ctypes.data_as(C.POINTER(C.c_float)),
            1 if reset_crash else 0, _fptr(xl) if log else None, _fptr(ul) if log else None,
            _fptr(ql) if log else None))
        return (xl, ul, ql) if log else None

    def feynman_kac(self, x0, seed=0, step=0):
        """mppi_feynman_kac: returns (log_psi, se_log_psi, s_min)."""
        x = self._x0(x0)
        out = np.zeros(3, np.float64)
        self._sync_stream()
        A.check(self.lib.mppi_feynman_kac(self.ctx, x.ctypes.data_as(C.POINTER(C.c_float)), seed, step,
                                          out.ctypes.data_as(C.POINTER(C.c_double))))
        return float(out[0]), float(out[1]), float(out[2])

    def plant_step(self, x, u, crashed=0):
        """mppi_plant_step: host fp32 Euler step; returns (x', q(x'), crashed')."""
        xs = _host_f32(x, self.n, "x").copy()
        us = _host_f32(u, self.m, "u")
        c = C.c_int32(int(crashed))
        q = C.c_float()
        A.check(self.lib.mppi_plant_step(self.ctx, xs.ctypes.data_as(C.POINTER(C.c_float)),
                                         us.ctypes.data_as(C.POINTER(C.c_float)), C.byref(c),
                                         C.byref(q)))
        return xs, q.value, c.value

    def stats(self):
        out = A.stats_t()
        A.check(self.lib.mppi_get_stats(self.ctx, C.byref(out)))
        return dict(k_star=out.k_star, s_min=out.s_min, eta=out.eta)

    def replay_count(self):
        """mppi_replay_count: rollouts re-run after their step loop since creation (telemetry of
        the slow path; results are identical either way)."""
        out = C.c_int64()
        A.check(self.lib.mppi_replay_count(self.ctx, C.byref(out)))
        return out.value

    def profile_enable(self, enable=True):
        A.check(self.lib.mppi_profile_enable(self.ctx, 1 if enable else 0))

    def profile_read(self):
        """{kernel: (total_ms, launches)} since the last read (synchronous)."""
        out = A.kernel_times_t()
        A.check(self.lib.mppi_profile_read(self.ctx, C.byref(out)))
        return {n: (out.total_ms[i], out.launches[i]) for i, n in enumerate(A.KERNEL_NAMES)}

    def last_launch_count(self):
        return self.lib.mppi_last_launch_count(self.ctx)

    def last_kernels(self):
        """Device-function names of the last call's kernel launches, in launch order."""
        n = 4096
        buf = C.create_string_buffer(n)
        need = self.lib.mppi_last_kernels(self.ctx, buf, n)
        if need >= n:
            buf = C.create_string_buffer(need + 1)
            self.lib.mppi_last_kernels(self.ctx, buf, need + 1)
        s = buf.value.decode()
        return s.split(",") if s else []


def from_workload(w, K=None, world=1, rank=0, **kw):
    """MPPI context for an mppi_inputs.Workload (configs C1-C5)."""
    obstacles = w.obstacles if w.plant == "quadrotor" else None
    return MPPI(w.plant, K or w.K, w.T, w.dt, w.lam, w.nu, w.Sigma, w.R, obstacles=obstacles,
                rank=rank, world=world, **kw)
