"""NEXT-2 on the GPU: Algorithm 1's receding-horizon loop on the device (mppi_closed_loop,
PAPER.md:356-378) against the fp64 oracle step by step (optimisation, device plant step, shift)
and over the first 10 steps, against the host-driven loop through the same API, plus the Fig. 1
trend (average running cost falls with the exploration variance nu)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from mppi_inputs import get  # noqa: E402
from mppi_inputs.configs import cartpole  # noqa: E402
from paper_1509_01149_b200 import from_workload  # noqa: E402


def host_loop(m, w, steps, seed):
    U = torch.tensor(w.U0, device="cuda")
    x, c, xs, us = w.x0.copy(), 0, [w.x0.copy()], []
    for i in range(steps):
        m.optimize(x, U, seed, i)
        u0 = U[0].cpu().numpy()
        x, q, c = m.plant_step(x, u0, c)
        m.shift(U, np.zeros(w.m, np.float32))
        xs.append(x.copy())
        us.append(u0)
    return np.array(xs), np.array(us)


@pytest.mark.parametrize("cfg", ["C2", "C4"])
def test_device_loop_tracks_host_loop(cfg):
    w = get(cfg)
    if cfg == "C4":
        w.K = 8192
    m = from_workload(w)
    steps = 12
    xs_h, us_h = host_loop(m, w, steps, w.seed)
    x = torch.tensor(w.x0, device="cuda")
    U = torch.tensor(w.U0, device="cuda")
    xl, ul, ql = m.closed_loop(x, U, steps, seed=w.seed, step0=0, u_init=np.zeros(w.m))
    xl, ul = xl.cpu().numpy(), ul.cpu().numpy()
    assert np.array_equal(xl[0], w.x0)
    # the optimisations are identical; only the plant's sin/cos differ (libdevice vs host libm),
    # so the loops agree closely over a short horizon
    assert np.allclose(ul, us_h, rtol=1e-3, atol=1e-4)
    assert np.allclose(xl, xs_h, rtol=1e-3, atol=1e-4)
    assert np.array_equal(x.cpu().numpy(), xl[-1])


def test_device_loop_swings_up_c2():
    w = get("C2")
    m = from_workload(w)
    x = torch.tensor(w.x0, device="cuda")
    U = torch.tensor(w.U0, device="cuda")
    xl, ul, ql = m.closed_loop(x, U, w.steps, seed=w.seed)
    up = 1 + np.cos(xl.cpu().numpy()[1:, 2])
    assert up.min() < 0.05 and int(np.argmax(up < 0.05)) < 100
    assert ql.cpu().numpy()[-50:].mean() < 50.0


def test_fig1_trend_cost_falls_with_nu():
    """PAPER.md:396 / Fig. 1: larger exploration variance swings the pole up faster; natural
    variance (nu = 1) stays near the hanging cost for the first seconds."""
    mean_cost = {}
    for nu in (1.0, 10.0, 100.0, 1000.0):
        costs = []
        for seed in (1, 2):
            w = cartpole(1024, 50, nu, steps=500)
            m = from_workload(w)
            x = torch.tensor(w.x0, device="cuda")
            U = torch.tensor(w.U0, device="cuda")
            _, _, ql = m.closed_loop(x, U, 500, seed=seed)
            costs.append(float(ql.mean().item()))
        mean_cost[nu] = np.mean(costs)
    v = [mean_cost[nu] for nu in (1.0, 10.0, 100.0, 1000.0)]
    assert v == sorted(v, reverse=True), mean_cost
    assert v[0] > 2 * v[-1]


@pytest.mark.parametrize("cfg,K", [("C2", 4096), ("C4", 65536)])
def test_sharded_closed_loop_single_rank_equals_graph_loop(cfg, K):
    """mppi_closed_loop through the library's communicator (single-rank: one GPU per call here)
    steps the same states and controls as the single-GPU graph loop -- bit for bit at C2; at C4
    size the sharded step runs the fused noise and reduction (the graph loop draws the noise in
    a separate pass and reduces with K3), so the controls agree to rounding."""
    w = get(cfg)
    a = from_workload(w, K=K)
    b = from_workload(w, K=K)
    b.attach_nccl()
    steps = 8
    outs = []
    for m in (a, b):
        x = torch.tensor(w.x0, device="cuda")
        U = torch.tensor(w.U0, device="cuda")
        xl, ul, ql = m.closed_loop(x, U, steps, seed=w.seed, step0=3, u_init=np.zeros(w.m))
        outs.append((xl.cpu().numpy(), ul.cpu().numpy()))
    if K < 65536:
        assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    else:
        assert np.allclose(outs[0][1], outs[1][1], rtol=1e-4, atol=1e-5)
        assert np.allclose(outs[0][0], outs[1][0], rtol=1e-4, atol=1e-5)
    a.close()
    b.close()


# ----------------------------------------------------------------------------- against the oracle
def _problem(oracle, w):
    return oracle.Problem(w.plant, T=w.T, dt=w.dt, lam=w.lam, nu=w.nu, Sigma=w.Sigma, R=w.R,
                          obstacles=w.obstacles if w.plant == "quadrotor" else None)


@pytest.mark.parametrize("cfg,K", [("C2", 4096), ("C3", 4096), ("C4", 8192)])
def test_device_loop_step_by_step_against_oracle(oracle, cfg, K):
    """Each of the first 10 receding-horizon steps of mppi_closed_loop against
    the fp64 oracle, from the device's own state and controls (so fp32/fp64 chaos cannot build
    up):  the optimisation (decoupled U within 1e-5 on the GPU's costs and noise; coupled within
    1e-5 whenever the A20 bound allows), the device plant step x_{i+1} = x_i + F(x_i, u_0) dt
    (the advance kernel, :377) and q(x_{i+1}) element-wise, and the shift (:372-375) bitwise.
    The 10-step graph loop then reproduces the step-by-step states and controls bit for bit."""
    w = get(cfg)
    w.K = K
    g = from_workload(w)
    pb = _problem(oracle, w)
    ui = np.zeros(w.m, np.float32)
    x = torch.tensor(w.x0, device="cuda")
    U = torch.tensor(w.U0, device="cuda")
    steps, crashed, coupled, worst = 10, 0, 0, 0.0
    xs, us = [w.x0.copy()], []
    for i in range(steps):
        x_i = x.cpu().numpy().copy()
        U_before = U.cpu().numpy().copy()
        xl, ul, ql = g.closed_loop(x, U, 1, seed=w.seed, step0=i, u_init=ui, reset_crash=(i == 0))
        xl, ul, ql = xl.cpu().numpy(), ul.cpu().numpy(), float(ql.cpu().numpy()[0])
        U_now = U.cpu().numpy()
        assert np.array_equal(xl[0], x_i)
        U_after = np.concatenate([ul, U_now[:-1]], axis=0).astype(np.float64)
        # optimisation of step i
        costs, _ = g.rollout_costs(x_i, torch.tensor(U_before, device="cuda"), w.seed, i)
        c = costs.cpu().numpy().astype(np.float64)
        eps = g.noise(w.seed, i).cpu().numpy()
        Ud = oracle.update(pb, c, eps, U_before)[0]
        assert np.max(np.abs(U_after - Ud)) <= 1e-5, (i, np.max(np.abs(U_after - Ud)))
        full = oracle.optimize(pb, x_i, U_before, eps)
        wbar = full["weights"] / full["weights"].sum()
        du = math.sqrt(w.nu) * np.einsum("ij,tkj->tki", np.linalg.cholesky(w.Sigma), eps.astype(np.float64))
        dev = np.abs(du - np.einsum("k,tki->ti", wbar, du)[:, None, :]).max(axis=(0, 2))
        if np.sum(wbar * np.abs(c - full["costs"]) * dev) / w.lam <= 5e-6:
            assert np.max(np.abs(U_after - full["U"])) <= 1e-5
            coupled += 1
        # device plant step and its cost
        x_ref, q_ref, crashed = oracle.plant_step(pb, x_i.astype(np.float64), ul[0].astype(np.float64), crashed)
        scale = np.maximum(np.abs(x_ref), 1.0)
        assert np.all(np.abs(xl[1] - x_ref) <= 1e-5 * scale), (i, np.abs(xl[1] - x_ref) / scale)
        assert abs(ql - q_ref) <= 1e-5 * max(abs(q_ref), 1.0)
        # shift
        assert np.array_equal(U_now, oracle.shift(U_after.astype(np.float32), ui).astype(np.float32))
        worst = max(worst, float(np.max(np.abs(xl[1] - x_ref) / scale)))
        xs.append(xl[1].copy())
        us.append(ul[0].copy())
    assert coupled >= steps // 2, "coupled U check ran on %d of %d steps" % (coupled, steps)
    print("PARITY closed loop %s K=%d: 10 steps vs oracle, coupled U on %d steps, max plant-step rel err %.3g"
          % (cfg, K, coupled, worst))
    # the 10-step graph loop equals the step-by-step loop
    x = torch.tensor(w.x0, device="cuda")
    U = torch.tensor(w.U0, device="cuda")
    xl, ul, _ = g.closed_loop(x, U, steps, seed=w.seed, step0=0, u_init=ui)
    assert np.array_equal(xl.cpu().numpy(), np.array(xs)) and np.array_equal(ul.cpu().numpy(), np.array(us))
    g.close()


@pytest.mark.parametrize("cfg,K", [("C2", 4096), ("C4", 8192)])
def test_device_loop_tracks_oracle_closed_loop(oracle, cfg, K):
    """The first 10 steps of the device loop against oracle.closed_loop (fp64 all the way): in the
    argmin regime both pick the same samples, so states agree to fp32 rounding."""
    w = get(cfg)
    w.K = K
    g = from_workload(w)
    steps = 10
    x = torch.tensor(w.x0, device="cuda")
    U = torch.tensor(w.U0, device="cuda")
    xl, ul, ql = g.closed_loop(x, U, steps, seed=w.seed, step0=0, u_init=np.zeros(w.m))
    xs, qs = oracle.closed_loop(_problem(oracle, w), w.x0, w.U0, steps, w.seed, K=K)
    xl = xl.cpu().numpy().astype(np.float64)
    assert np.allclose(xl, xs, rtol=1e-4, atol=1e-5), np.max(np.abs(xl - xs))
    assert np.allclose(ql.cpu().numpy(), qs, rtol=1e-4, atol=1e-4)
    g.close()


def test_closed_loop_graph_reuse_equals_fresh_context():
    """A second mppi_closed_loop call of the same length reuses the instantiated loop graph with
    updated node arguments (seed, step, pointers): bitwise the results of a fresh context."""
    w = get("C2")
    w.K = 1024
    a = from_workload(w)
    b = from_workload(w)
    n = 6
    x, U = torch.tensor(w.x0, device="cuda"), torch.tensor(w.U0, device="cuda")
    a.closed_loop(x, U, n, seed=3, step0=0, u_init=np.zeros(w.m))          # builds the graph
    outs = []
    for m in (a, b):                                                       # a reuses, b builds
        x, U = torch.tensor(w.x0, device="cuda"), torch.tensor(w.U0, device="cuda")
        xl, ul, ql = m.closed_loop(x, U, n, seed=5, step0=40, u_init=np.zeros(w.m))
        outs.append((xl.cpu().numpy(), ul.cpu().numpy(), ql.cpu().numpy(), U.cpu().numpy()))
    for u, v in zip(outs[0], outs[1]):
        assert np.array_equal(u, v)
    a.close()
    b.close()
