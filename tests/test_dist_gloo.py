"""Multi-rank host logic on CPU (gloo, world size 2): paper_1509_01149_b200.dist.ShardedMPPI
drives the split-phase step (rollout_costs -> allreduce MIN key -> accumulate -> allreduce SUM
[eta, A] -> apply) over a K-sharded problem.  The per-rank compute here is an oracle-backed
shard stepper (tests may call the oracle); the result must equal the single-process oracle
step: the sharding algebra of SURVEY §8.5 / PAPER.md:320 (sums over k split across ranks)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from mppi_inputs import get


def _key(cost, k):
    b = int(np.array(cost, np.float32).view(np.int32))
    b = b if b >= 0 else b ^ 0x7FFFFFFF
    return (b << 32) | int(k)


def _unkey(key):
    b = key >> 32
    b = b if b >= 0 else b ^ 0x7FFFFFFF
    return float(np.array(b, np.int32).view(np.float32)), key & 0xFFFFFFFF


class OracleShard:
    """rollout_costs / accumulate / apply over global samples [k0, k0 + K_loc) in fp64."""

    def __init__(self, O, pb, K, rank, world):
        from paper_1509_01149_b200.dist import shard_range
        self.O, self.pb = O, pb
        self.k0, self.K_loc = shard_range(K, rank, world)
        self.L = np.linalg.cholesky(pb.Sigma) * math.sqrt(pb.nu)

    def rollout_costs(self, x0, U, seed, step, noise=None):
        self.eps = self.O.noise(seed, step, self.pb.T, self.K_loc, self.pb.m, k0=self.k0)
        # costs rounded to fp32 exactly as the CUDA path stores them
        self.costs = self.O.rollout_costs(self.pb, x0, U.numpy(), self.eps).astype(np.float32)
        k = int(np.argmin(self.costs))
        return torch.tensor(self.costs), torch.tensor([_key(self.costs[k], self.k0 + k)], dtype=torch.int64)

    def accumulate(self, key):
        smin, _ = _unkey(int(key.item()))
        w = np.exp(-(self.costs.astype(np.float64) - smin) / self.pb.lam)
        A = np.einsum("k,tkj->tj", w, self.eps.astype(np.float64))
        return torch.tensor(np.concatenate([[w.sum()], A.ravel()]), dtype=torch.float64)

    def apply(self, U, buf):
        b = buf.numpy()
        A = b[1:].reshape(self.pb.T, self.pb.m)
        U += torch.tensor((A @ self.L.T) / b[0], dtype=U.dtype)
        return U

    # the one-collective form (MPPI_OPTION_GATHER_COMBINE): [S_min,r, k*_r, eta_r, A_r] against
    # this shard's own minimum; the combine rescales by exp(-(S_min,r - S_min)/lambda)
    def accumulate_record(self):
        k = int(np.argmin(self.costs))
        smin = float(self.costs[k])
        w = np.exp(-(self.costs.astype(np.float64) - smin) / self.pb.lam)
        A = np.einsum("k,tkj->tj", w, self.eps.astype(np.float64))
        return torch.tensor(np.concatenate([[smin, self.k0 + k, w.sum()], A.ravel()]), dtype=torch.float64)

    def apply_gathered(self, U, recs):
        r = recs.numpy()
        smin = r[:, 0].min()
        c = np.exp(-(r[:, 0] - smin) / self.pb.lam)
        eta = np.sum(c * r[:, 2])
        A = (c[:, None] * r[:, 3:]).sum(axis=0).reshape(self.pb.T, self.pb.m)
        U += torch.tensor((A @ self.L.T) / eta, dtype=U.dtype)
        return U


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, K, q, combine="allreduce"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_1509_01149_b200.dist import ShardedMPPI
    w = get(cfg)
    pb = O.Problem(w.plant, T=w.T, dt=w.dt, lam=w.lam, nu=w.nu, Sigma=w.Sigma, R=w.R,
                   obstacles=w.obstacles if w.plant == "quadrotor" else None)
    sh = ShardedMPPI(OracleShard(O, pb, K, rank, world), combine=combine)
    assert sh.world == world
    U = torch.tensor(w.U0.astype(np.float64))
    for step in range(2):
        sh.optimize(w.x0, U, w.seed, step)
    q.put((rank, U.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,K,combine", [("C1", 256, "allreduce"), ("C3", 512, "allreduce"),
                                           ("C1", 256, "gather"), ("C3", 512, "gather")])
def test_sharded_step_world2_matches_single(oracle, cfg, K, combine):
    """Both combines (MIN + SUM all-reduce; one all-gather of per-rank records rescaled to the
    global minimum) give the single-process step (PAPER.md:320 is invariant to the shift)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, K, q, combine)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single process: the same shard stepper over all K (world 1)
    w = get(cfg)
    pb = oracle.Problem(w.plant, T=w.T, dt=w.dt, lam=w.lam, nu=w.nu, Sigma=w.Sigma, R=w.R)
    one = OracleShard(oracle, pb, K, 0, 1)
    U = torch.tensor(w.U0.astype(np.float64))
    for step in range(2):
        c, key = one.rollout_costs(w.x0, U, w.seed, step)
        one.apply(U, one.accumulate(key))
    assert np.array_equal(res[0], res[1])                  # replicas stay identical
    assert np.max(np.abs(res[0] - U.numpy())) < 1e-12


def test_shard_range():
    from paper_1509_01149_b200.dist import shard_range
    assert shard_range(4096, 3, 4) == (3072, 1024)
    with pytest.raises(ValueError):
        shard_range(1000, 0, 3)
    with pytest.raises(ValueError):
        shard_range(1000, 0, 8)     # 125 per rank is not a multiple of 4
