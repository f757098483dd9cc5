"""NEXT-1 on the GPU: per-timestep cost-to-go weights (Alg. 1 :367) against the
oracle (decoupled: the oracle update applied to the GPU's own cost-to-go and noise; and the
cost-to-go itself against the oracle's per-step costs), and u_0 against the trajectory weighting."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import MPPI, from_workload  # noqa: E402


@pytest.mark.parametrize("cfg,K,lam", [("C1", 256, None), ("C3", 4096, None), ("C4", 4096, None),
                                        ("C1", 256, 50.0), ("C4", 1 << 16, 500.0)])
def test_cost_to_go_update_matches_oracle(oracle, cfg, K, lam):
    w = get(cfg)
    lam = lam or w.lam
    m = MPPI(w.plant, K, w.T, w.dt, lam, w.nu, w.Sigma, w.R,
             obstacles=w.obstacles if w.plant == "quadrotor" else None)
    m.set_weighting(True)
    U = torch.tensor(w.U0, device="cuda")
    m.optimize(w.x0, U, 3, 1)
    ctg = m.cost_to_go().cpu().numpy().astype(np.float64)        # [T][K]
    eps = m.noise(3, 1).cpu().numpy()
    pb = oracle.Problem(w.plant, T=w.T, dt=w.dt, lam=lam, nu=w.nu, Sigma=w.Sigma, R=w.R,
                        obstacles=w.obstacles if w.plant == "quadrotor" else None)
    # (a) the cost-to-go against the oracle's fp64 per-step costs (suffix sums) on the same noise
    ok, ref = oracle.well_conditioned_ctg(pb, w.x0, w.U0, oracle.noise(3, 1, w.T, K, w.m))
    rel = np.abs(ctg - ref) / np.maximum(np.abs(ref[0:1, :]), 1.0)  # scale: the sample's total cost
    assert np.max(rel[:, ok]) <= 1e-4
    assert ok.mean() >= 0.95
    # (b) decoupled update: the oracle's cost-to-go reduction on the GPU's S~_{t,k} and noise.  The
    # oracle takes per-step costs, so feed back differences of the GPU suffix sums.
    gpu_steps = np.diff(np.vstack([ctg, np.zeros((1, K))]), axis=0) * -1.0
    Ud, smin, eta = oracle.update_ctg(pb, gpu_steps.T, eps, w.U0)
    assert np.max(np.abs(U.cpu().numpy() - Ud)) <= 1e-5


def test_u0_matches_trajectory_weighting():
    w = get("C4")
    K = 8192
    a = MPPI(w.plant, K, w.T, w.dt, 500.0, w.nu, w.Sigma, w.R, obstacles=w.obstacles)
    b = MPPI(w.plant, K, w.T, w.dt, 500.0, w.nu, w.Sigma, w.R, obstacles=w.obstacles)
    b.set_weighting(True)
    Ua, Ub = torch.tensor(w.U0, device="cuda"), torch.tensor(w.U0, device="cuda")
    ca, _ = a.rollout_costs(w.x0, torch.tensor(w.U0, device="cuda"), 2, 0)
    a.optimize(w.x0, Ua, 2, 0)
    b.optimize(w.x0, Ub, 2, 0)
    # S~_{0,k} is the same sum of q~ in another fp32 order: |dS| <= a few ulp of S, so by the
    # first-order bound of SURVEY A20 |du_0| <= max|dS| / lambda * max|du - mean du|
    S = ca.cpu().numpy().astype(np.float64)
    dS = 4 * np.spacing(np.abs(S).astype(np.float32)).max()
    du = math.sqrt(w.nu) * math.sqrt(w.Sigma[0, 0]) * np.abs(b.noise(2, 0)[0].cpu().numpy()).max() * 2
    assert torch.max(torch.abs(Ua[0] - Ub[0])).item() <= dS / 500.0 * du
    assert not torch.allclose(Ua[5:], Ub[5:])
    # switching back restores the trajectory weighting exactly
    b.set_weighting(False)
    Uc = torch.tensor(w.U0, device="cuda")
    b.optimize(w.x0, Uc, 2, 0)
    assert torch.equal(Uc, Ua)


@pytest.mark.parametrize("K,sampling,lam", [(65536 + 4, "diag", None), (1 << 17, "diag", 500.0),
                                             (65536 + 4, "A_t", 500.0)])
def test_fused_cost_to_go_pass_is_bitwise(K, sampling, lam):
    """The packed rollout's fused cost-to-go pass (suffix sums of each thread's own q~ rows, per-t
    CTA minima) gives bit for bit the separate ctg_kernel's S~_{t,k}; its fused reduction (weights
    against the per-(CTA, t) minima, rescaled by epi_combine_ctg_kernel) gives the separate
    reduction's update to rounding: ragged last CTA, diagonal Sigma and per-step transforms A_t,
    one-hot (config lambda) and dense (lambda = 500) weights."""
    from paper_1509_01149_b200 import _capi as A
    w = get("C4")
    if lam is not None:
        w.lam = lam
    ms = [from_workload(w, K=K) for _ in range(2)]
    ms[1].set_option(A.MPPI_OPTION_FUSED_REDUCTION, 0)
    if sampling == "A_t":
        rng = np.random.default_rng(5)
        At = np.array([rng.normal(size=(w.m, w.m)) * 0.2 + 1.2 * np.eye(w.m) for _ in range(w.T)])
    for m in ms:
        m.set_weighting(True)
        if sampling == "A_t":
            m.set_sampling_transform(At)
    Us = [torch.tensor(w.U0, device="cuda") for _ in ms]
    for i in range(2):
        for m, U in zip(ms, Us):
            m.optimize(w.x0, U, 9, i)
        ka, kb = ms[0].last_kernels(), ms[1].last_kernels()
        # mangled names: "10ctg_kernel" is the separate suffix-sum kernel
        assert not any("10ctg_kernel" in n for n in ka) and any("ctg_min_kernel" in n for n in ka), ka
        assert any("epi_combine_ctg" in n for n in ka) and not any("wsum_ctg" in n for n in ka), ka
        assert any("10ctg_kernel" in n for n in kb) and any("wsum_ctg" in n for n in kb), kb
        assert torch.equal(ms[0].cost_to_go(), ms[1].cost_to_go())
        torch.testing.assert_close(Us[0], Us[1], rtol=1e-5, atol=1e-6)
        Us[1].copy_(Us[0])
    for m in ms:
        m.close()
