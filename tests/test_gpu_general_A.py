"""NEXT-3 on the GPU: per-step variance transforms A_t (mppi_set_sampling_transform, Theorem 1)
against the oracle on the same noise; A_t = sqrt(nu) I reproduces the special case."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import MPPI, MppiError  # noqa: E402


def _rand_A(rng, T, m):
    return np.array([rng.normal(size=(m, m)) * 0.4 + 1.5 * np.eye(m) for _ in range(T)])


@pytest.mark.parametrize("cfg,K", [("C1", 256), ("C3", 2048), ("C4", 2048)])
def test_general_A_matches_oracle(oracle, cfg, K):
    w = get(cfg)
    rng = np.random.default_rng(3)
    At = _rand_A(rng, w.T, w.m)
    lam = 50.0
    m = MPPI(w.plant, K, w.T, w.dt, lam, w.nu, w.Sigma, w.R,
             obstacles=w.obstacles if w.plant == "quadrotor" else None)
    m.set_sampling_transform(At)
    U = torch.tensor(w.U0, device="cuda")
    costs, _ = m.rollout_costs(w.x0, U, 6, 0)
    m.optimize(w.x0, U, 6, 0)
    eps = m.noise(6, 0).cpu().numpy()
    pb = oracle.Problem(w.plant, T=w.T, dt=w.dt, lam=lam, nu=w.nu, Sigma=w.Sigma, R=w.R, At=At,
                        obstacles=w.obstacles if w.plant == "quadrotor" else None)
    ok, ref = oracle.well_conditioned(pb, w.x0, w.U0, eps)
    c = costs.cpu().numpy().astype(np.float64)
    err = np.abs(c - ref) / np.maximum(np.abs(ref), 1.0)
    assert np.max(err[ok]) <= 1e-4 and ok.mean() >= 0.9
    Ud = oracle.update(pb, c, eps, w.U0)[0]                     # decoupled update check
    assert np.max(np.abs(U.cpu().numpy() - Ud)) <= 1e-5


def test_sqrt_nu_identity_equals_default():
    w = get("C3")
    K = 2048
    a = MPPI(w.plant, K, w.T, w.dt, 5.0, w.nu, w.Sigma, w.R)
    b = MPPI(w.plant, K, w.T, w.dt, 5.0, w.nu, w.Sigma, w.R)
    b.set_sampling_transform(np.tile(math.sqrt(w.nu) * np.eye(2), (w.T, 1, 1)))
    ca, _ = a.rollout_costs(w.x0, torch.tensor(w.U0, device="cuda"), 1, 0)
    cb, _ = b.rollout_costs(w.x0, torch.tensor(w.U0, device="cuda"), 1, 0)
    assert torch.allclose(ca, cb, rtol=2e-6, atol=0)
    b.set_sampling_transform(None)                              # back to the diagonal fast path
    cc, _ = b.rollout_costs(w.x0, torch.tensor(w.U0, device="cuda"), 1, 0)
    assert torch.equal(ca, cc)


def test_singular_A_rejected():
    w = get("C3")
    m = MPPI(w.plant, 256, w.T, w.dt, 5.0, w.nu, w.Sigma, w.R)
    At = np.tile(np.eye(2), (w.T, 1, 1))
    At[3] = [[1.0, 2.0], [2.0, 4.0]]
    with pytest.raises(MppiError):
        m.set_sampling_transform(At)
