"""Row (a2) for a GENERAL sampling covariance and control cost, against the fp64 oracle.

delta u = sqrt(nu) L eps with L = chol(Sigma_u) (PAPER.md:185-187 B_E = A B_c, :308 A = sqrt(nu) I,
:312), and the importance-sampling terms 1/2 (1 - 1/nu) du' R du + U' R du + 1/2 U' R U with a full
R.  The configs use diagonal Sigma_u and R; here both carry off-diagonals of
about 20 % (correlation), which routes the GPU through its general kernels: the one-sample
`!DIAG` rollout at K = 4096, and at K = 65536 + 4 the packed quadrotor kernel's general variant
with in-kernel noise and the fused reduction (a ragged last CTA).  Bars as everywhere
(SURVEY A19/A20): per-sample costs within 1e-4 relative on the samples the oracle calls
well-conditioned, the decoupled U within 1e-5, the coupled U within 1e-5 when the first-order
bound allows (asserted to have run at the config's lambda)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import MPPI  # noqa: E402

COST_RTOL = 1e-4
U_ATOL = 1e-5


def correlated(m, scale, rho, sign_pattern=True):
    """scale * C with C_ii = 1, C_ij = rho * s_ij (s_ij = +-1 alternating), SPD for rho < 1/(m-1)."""
    C = np.eye(m)
    for i in range(m):
        for j in range(m):
            if i != j:
                C[i, j] = rho * ((-1.0) ** (i + j) if sign_pattern else 1.0)
    assert np.all(np.linalg.eigvalsh(C) > 0)
    return scale * C


def workload(cfg):
    """Correlated Sigma_u (natural variance 0.005, correlations +-0.2) and a full SPD R scaled
    by 100, so that the importance-sampling terms -- and R's off-diagonals in them -- move the
    costs by far more than the 1e-4 tolerance (checked in run())."""
    w = get(cfg)
    w.Sigma = correlated(w.m, 0.005, 0.2)
    w.R = 100.0 * (correlated(w.m, 1.0, 0.2, sign_pattern=False) + np.diag(np.linspace(0.0, 0.3, w.m)))
    return w


def run(oracle, w, K, lam, seed=3, step=0):
    g = MPPI(w.plant, K, w.T, w.dt, lam, w.nu, w.Sigma, w.R,
             obstacles=w.obstacles if w.plant == "quadrotor" else None)
    U = torch.tensor(w.U0, device="cuda")
    costs, key = g.rollout_costs(w.x0, U, seed, step)
    costs = costs.cpu().numpy().astype(np.float64)
    eps = g.noise(seed, step).cpu().numpy()
    g.optimize(w.x0, U, seed, step)
    kernels = g.last_kernels()
    U_gpu = U.cpu().numpy().astype(np.float64)
    st = g.stats()
    g.close()
    ref_eps = oracle.noise(seed, step, w.T, K, w.m)
    assert np.array_equal(eps.view(np.uint32), ref_eps.view(np.uint32))
    pb = oracle.Problem(w.plant, T=w.T, dt=w.dt, lam=lam, nu=w.nu, Sigma=w.Sigma, R=w.R,
                        obstacles=w.obstacles if w.plant == "quadrotor" else None)
    ok, ref = oracle.well_conditioned(pb, w.x0, w.U0, ref_eps)
    # the parity below is evidence about R's off-diagonals only if dropping them moves the costs
    # by much more than the tolerance
    pb_diag = oracle.Problem(w.plant, T=w.T, dt=w.dt, lam=lam, nu=w.nu, Sigma=w.Sigma, R=np.diag(np.diag(w.R)),
                             obstacles=w.obstacles if w.plant == "quadrotor" else None)
    ref_diag = oracle.rollout_costs(pb_diag, w.x0, w.U0, ref_eps[:, :4096])
    assert np.median(np.abs(ref[:4096] - ref_diag) / np.maximum(np.abs(ref[:4096]), 1.0)) > 10 * COST_RTOL
    err = np.abs(costs - ref) / np.maximum(np.abs(ref), 1.0)
    bad = np.nonzero(ok & (err > COST_RTOL))[0]
    assert bad.size == 0, "well-conditioned samples over 1e-4: %s (max %.3g)" % (bad[:10], err[ok].max())
    assert ok.mean() >= 0.95, "excluded fraction %.4f" % (1 - ok.mean())
    # (i) decoupled: the oracle's reduction of the GPU's costs and noise
    Ud, kstar, smin, eta, wts = oracle.update(pb, costs, eps, w.U0)
    assert np.max(np.abs(U_gpu - Ud)) <= U_ATOL
    assert st["k_star"] == kstar
    # (ii) coupled: the whole fp64 step, when the first-order bound (A20) permits
    full = oracle.optimize(pb, w.x0, w.U0, ref_eps)
    wbar = full["weights"] / full["weights"].sum()
    du = math.sqrt(w.nu) * np.einsum("ij,tkj->tki", np.linalg.cholesky(w.Sigma), eps.astype(np.float64))
    dev = np.abs(du - np.einsum("k,tki->ti", wbar, du)[:, None, :]).max(axis=(0, 2))
    bound = np.sum(wbar * np.abs(costs - full["costs"]) * dev) / lam
    coupled = bound <= 5e-6
    if coupled:
        assert np.max(np.abs(U_gpu - full["U"])) <= U_ATOL
    print("PARITY general Sigma/R %s K=%d lambda=%g: max rel err %.3g (excluded %.4f), decoupled |dU| %.3g, "
          "coupled %s" % (w.name, K, lam, err[ok].max(), 1 - ok.mean(), np.max(np.abs(U_gpu - Ud)),
                          "%.3g" % np.max(np.abs(U_gpu - full["U"])) if coupled else "not asserted"))
    return dict(kernels=kernels, excluded=1 - ok.mean(), coupled=coupled, err=err[ok].max())


@pytest.mark.parametrize("cfg", ["C3", "C4"])
@pytest.mark.parametrize("K", [4096, 65536 + 4])
def test_correlated_sigma_and_full_R_match_oracle(oracle, cfg, K):
    w = workload(cfg)
    r = run(oracle, w, K, w.lam)
    if cfg == "C4" and K > 65536:
        # the packed general variant with in-kernel noise and the fused reduction ran
        assert any("rollout_kernel_x2" in n for n in r["kernels"]), r["kernels"]
        assert any("epi_combine" in n for n in r["kernels"]), r["kernels"]
    assert r["coupled"], "coupled U check did not run (argmin regime expected at lambda = 5e-3)"


@pytest.mark.parametrize("cfg,K", [("C3", 4096), ("C4", 65536 + 4)])
def test_correlated_sigma_nondegenerate_lambda(oracle, cfg, K):
    """lambda = std_k of the oracle costs: many samples carry weight (decoupled U bar)."""
    w = workload(cfg)
    pb = oracle.Problem(w.plant, T=w.T, dt=w.dt, lam=w.lam, nu=w.nu, Sigma=w.Sigma, R=w.R,
                        obstacles=w.obstacles if w.plant == "quadrotor" else None)
    ref_costs = oracle.rollout_costs(pb, w.x0, w.U0, oracle.noise(3, 0, w.T, 4096, w.m))
    run(oracle, w, K, float(np.std(ref_costs)))
