"""The default C5 kernel (packed two-sample quadrotor rollout drawing its own noise, obstacle
candidate grid, fused reduction) against the fp64 oracle at FULL horizon, sample by sample, plus
the edge cases of the step.

  * every sample of K = 65536, T = 200 (C4 = C5's smallest K), costs within 1e-4 relative on
    the well-conditioned samples (A19), the excluded fraction reported and bounded;
  * 4096 random columns of C5 itself (K = 2^22, T = 200): noise bit-exact, costs as above;
  * exact ties (duplicated supplied-noise columns, including the two lanes of one packed
    thread and another CTA): tied costs bitwise equal, k* the smallest tied index, each tied
    sample weight 1;
  * all samples penalised (every rollout overflows): costs all 1e30, uniform weights, eta = K
    exactly, U += mean du;
  * NaN/Inf injected into supplied noise on the packed path: those samples get the penalty,
    every other sample keeps its bits."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import from_workload  # noqa: E402

COST_RTOL = 1e-4
U_ATOL = 1e-5
PENALTY = np.float32(1e30)


def problem(oracle, w, lam=None):
    return oracle.Problem(w.plant, T=w.T, dt=w.dt, lam=lam or w.lam, nu=w.nu, Sigma=w.Sigma, R=w.R,
                          obstacles=w.obstacles if w.plant == "quadrotor" else None)


def cuda_u(w):
    return torch.tensor(w.U0, device="cuda")


def key_k(key):
    return int(key.item()) & 0xFFFFFFFF


def test_every_sample_at_k65536_full_horizon(oracle):
    w = get("C4")                       # K = 65536, T = 200: the C5 kernels' smallest K
    K = w.K
    g = from_workload(w)
    costs, key = g.rollout_costs(w.x0, cuda_u(w), w.seed, 0)
    kern = g.last_kernels()
    assert any("rollout_kernel_x2" in n for n in kern) and not any("noise_kernel" in n for n in kern), kern
    c = costs.cpu().numpy().astype(np.float64)
    eps = oracle.noise(w.seed, 0, w.T, K, w.m)
    ok, ref = oracle.well_conditioned(problem(oracle, w), w.x0, w.U0, eps)
    err = np.abs(c - ref) / np.maximum(np.abs(ref), 1.0)
    excluded = 1.0 - ok.mean()
    print("PARITY C5 kernel K=65536 T=200 every sample: excluded %.5f, max rel err on kept %.3g, overall %.3g"
          % (excluded, err[ok].max(), err.max()))
    bad = np.nonzero(ok & (err > COST_RTOL))[0]
    assert bad.size == 0, "well-conditioned samples over 1e-4: %s" % bad[:10]
    assert excluded <= 0.01
    kk = key_k(key)
    assert kk == int(np.argmin(c))
    order = np.sort(ref)
    if order[1] - order[0] > 2 * np.max(np.abs(c - ref)[ok]) and ok[np.argmin(ref)]:
        assert kk == int(np.argmin(ref))


def test_4096_random_columns_of_c5(oracle):
    w = get("C5")
    K = w.K
    g = from_workload(w)
    costs, key = g.rollout_costs(w.x0, cuda_u(w), w.seed, 0)
    kern = g.last_kernels()
    assert any("rollout_kernel_x2" in n for n in kern), kern
    rng = np.random.default_rng(2024)
    ks = np.sort(np.concatenate([rng.choice(K, 4094, replace=False), [0, K - 1]]))
    ks = np.unique(ks)
    assert ks.size >= 4096 - 2
    eps_dev = g.noise(w.seed, 0)
    got = eps_dev[:, torch.as_tensor(ks, device="cuda"), :].cpu().numpy()
    del eps_dev
    ref_eps = np.concatenate([oracle.noise(w.seed, 0, w.T, 1, 4, k0=int(k)) for k in ks], axis=1)
    assert np.array_equal(got.view(np.uint32), ref_eps.view(np.uint32))
    ok, ref = oracle.well_conditioned(problem(oracle, w), w.x0, w.U0, ref_eps)
    c = costs.cpu().numpy()[ks].astype(np.float64)
    err = np.abs(c - ref) / np.maximum(np.abs(ref), 1.0)
    print("PARITY C5 K=2^22 4096 columns: noise bitwise, excluded %.5f, max rel err on kept %.3g"
          % (1 - ok.mean(), err[ok].max()))
    assert np.all(err[ok] <= COST_RTOL)
    assert ok.mean() >= 0.99


@pytest.mark.parametrize("K", [65536 + 4, 4096])
def test_exact_ties_take_smallest_index_and_weight_one(oracle, K):
    """A16: duplicated noise columns give bitwise-equal costs; k* is the smallest tied index and
    every tied sample gets w = exp(0) = 1 (eta counts them), U is the oracle's update."""
    w = get("C4")
    g = from_workload(w, K=K)
    eps = g.noise(w.seed, 0)
    c0, key0 = g.rollout_costs(w.x0, cuda_u(w), 0, 0, noise=eps)
    k0 = key_k(key0)
    ties = sorted({k0, k0 ^ 1, (k0 + K // 2 + 256) % K, 2 if k0 != 2 else 3})
    eps2 = eps.clone()
    for j in ties:
        eps2[:, j, :] = eps[:, k0, :]
    c2, key2 = g.rollout_costs(w.x0, cuda_u(w), 0, 0, noise=eps2)
    c2n = c2.cpu().numpy()
    assert len({c2n[j].tobytes() for j in ties}) == 1
    assert key_k(key2) == ties[0]
    assert c2n[ties[0]] == c2n.min()
    U = cuda_u(w)
    g.optimize(w.x0, U, 0, 0, noise=eps2)
    st = g.stats()
    assert st["k_star"] == ties[0]
    Ud, kstar, smin, eta, wts = oracle.update(problem(oracle, w), c2n.astype(np.float64),
                                              eps2.cpu().numpy(), w.U0)
    assert kstar == ties[0]
    assert all(wts[j] == 1.0 for j in ties)
    assert eta >= len(ties) and st["eta"] == pytest.approx(eta, rel=1e-6)
    assert np.max(np.abs(U.cpu().numpy() - Ud)) <= U_ATOL


@pytest.mark.parametrize("cfg,K", [("C4", 65536 + 4), ("C4", 4096), ("C1", 256)])
def test_all_samples_penalised_gives_uniform_weights(oracle, cfg, K):
    """A15: every rollout overflows (initial speed 3e38 m/s) -> every cost is the penalty, all
    weights exp(0) = 1, eta = K exactly and U' = U + mean_k du_k."""
    w = get(cfg)
    x0 = w.x0.copy()
    x0[1 if cfg == "C1" else 3] = 3e38
    g = from_workload(w, K=K)
    costs, key = g.rollout_costs(x0, cuda_u(w), 5, 0)
    c = costs.cpu().numpy()
    assert np.all(c == PENALTY)
    assert key_k(key) == 0
    U = cuda_u(w)
    g.optimize(x0, U, 5, 0)
    st = g.stats()
    assert st["eta"] == float(K) and st["k_star"] == 0
    eps = g.noise(5, 0).cpu().numpy().astype(np.float64)
    L = np.linalg.cholesky(w.Sigma)
    want = w.U0 + math.sqrt(w.nu) * eps.mean(axis=1) @ L.T
    assert np.max(np.abs(U.cpu().numpy() - want)) <= U_ATOL


def test_nan_injection_on_packed_path():
    """A15 on the C5 kernels (K >= 65536, supplied noise): NaN / Inf in a sample's noise gives that
    sample the penalty; the other lane of the same packed thread and every other sample keep
    their bits, and k* is unchanged."""
    w = get("C4")
    K = 65536 + 4
    g = from_workload(w, K=K)
    eps = g.noise(7, 0)
    c0, key0 = g.rollout_costs(w.x0, cuda_u(w), 0, 0, noise=eps)
    k0 = key_k(key0)
    hit = [j for j in (0, 1, 257, 40000, K - 1, K - 4) if j != k0 and j != (k0 ^ 1)]
    eps2 = eps.clone()
    for i, j in enumerate(hit):
        eps2[(37 * i) % w.T, j, i % 4] = float("nan") if i % 2 == 0 else float("inf")
    c2, key2 = g.rollout_costs(w.x0, cuda_u(w), 0, 0, noise=eps2)
    a, b = c0.cpu().numpy(), c2.cpu().numpy()
    assert np.all(b[hit] == PENALTY)
    keep = np.setdiff1d(np.arange(K), hit)
    assert np.array_equal(a[keep].view(np.uint32), b[keep].view(np.uint32))
    assert key_k(key2) == k0


@pytest.mark.parametrize("K", [65536, 262144 + 4])
def test_fused_reduction_step_agrees_with_the_rollout_pass(oracle, K):
    """The optimise step's rollout (fused reduction epilogue) and mppi_rollout_costs' rollout of the
    same noise give a bitwise-equal minimum cost and k*, and the update equals the separate
    reduction's to rounding (K = 2^16 and a ragged 2^18 + 4)."""
    from paper_1509_01149_b200 import _capi as A
    w = get("C4")
    m = from_workload(w, K=K)
    U = cuda_u(w)
    m.optimize(w.x0, U, 3, 1)
    assert any("rollout_kernel_x2" in n for n in m.last_kernels()) and any("epi_combine" in n for n in m.last_kernels())
    st = m.stats()
    c, key = m.rollout_costs(w.x0, cuda_u(w), 3, 1)
    cn = c.cpu().numpy()
    assert st["k_star"] == key_k(key) == int(np.argmin(cn))
    assert np.float32(st["s_min"]).view(np.uint32) == cn.min().view(np.uint32)
    sep = from_workload(w, K=K)
    sep.set_option(A.MPPI_OPTION_FUSED_REDUCTION, 0)
    U2 = cuda_u(w)
    sep.optimize(w.x0, U2, 3, 1)
    assert np.max(np.abs(U.cpu().numpy() - U2.cpu().numpy())) <= 1e-6
