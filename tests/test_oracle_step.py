"""Pins for the oracle's reduction/update and the whole step: P4 (simplex, shift invariance),
P5 (lambda -> 0), P6 (lambda -> inf), P7 (nu = 1), P10 (linear-quadratic closed form),
P11 (tiny brute force), P12 (closed-loop behaviour), plus penalty and shift semantics.
PAPER.md:318-322, :356-378, :396."""
import math

import numpy as np
import pytest
from mppi_inputs import get

from lq_fixture import lq_setup as _lq_setup


def cartpole_problem(oracle, T=8, nu=4.0, lam=0.5, **kw):
    return oracle.Problem("cartpole", T=T, dt=0.02, lam=lam, nu=nu, Sigma=[[0.005]], R=[[1.0]], **kw)


def _setup(oracle, K=64, T=8, nu=4.0, lam=0.5, seed=3):
    pb = cartpole_problem(oracle, T=T, nu=nu, lam=lam)
    rng = np.random.default_rng(seed)
    U = rng.normal(size=(T, 1)) * 0.3
    x0 = np.array([0.0, 0.0, 0.2, 0.0])
    eps = oracle.noise(seed, 0, T, K, 1)
    return pb, U, x0, eps


def test_weights_simplex_and_shift_invariance(oracle):
    """weights non-negative and sum to 1 +- 1e-12; S~ + c leaves U' unchanged."""
    pb, U, x0, eps = _setup(oracle)
    costs = oracle.rollout_costs(pb, x0, U, eps)
    U1, kstar, smin, eta, w = oracle.update(pb, costs, eps, U)
    assert np.all(w >= 0) and abs(w.sum() / eta - 1.0) < 1e-12
    assert w[kstar] == 1.0 and costs[kstar] == smin == costs.min()
    U2 = oracle.update(pb, costs + 12345.678, eps, U)[0]
    assert np.max(np.abs(U1 - U2)) < 1e-12


def test_lambda_to_zero_selects_argmin(oracle):
    """P5 / SPEC.md:291: lambda = 1e-8 * spread with a unique minimum gives U' = U + du_{k*}."""
    pb, U, x0, eps = _setup(oracle)
    costs = oracle.rollout_costs(pb, x0, U, eps)
    spread = costs.max() - costs.min()
    pb0 = cartpole_problem(oracle, lam=1e-8 * spread)
    U1, kstar, _, eta, _ = oracle.update(pb0, costs, eps, U)
    assert kstar == int(np.argmin(costs)) and eta == 1.0
    du = math.sqrt(4.0) * np.linalg.cholesky(np.array([[0.005]])) @ eps[:, kstar, :].T.astype(float)
    assert np.max(np.abs(U1 - (U + du.T))) < 1e-15


def test_lambda_to_infinity_gives_noise_mean(oracle):
    """P6: lambda = 1e30 -> every w = 1, eta = K, U' = U + mean_k du."""
    pb, U, x0, eps = _setup(oracle, K=48)
    costs = oracle.rollout_costs(pb, x0, U, eps)
    pbi = cartpole_problem(oracle, lam=1e30)
    U1, _, _, eta, w = oracle.update(pbi, costs, eps, U)
    assert np.all(w == 1.0) and eta == 48.0
    du = 2.0 * math.sqrt(0.005) * eps.astype(float).mean(axis=1)
    assert np.max(np.abs(U1 - (U + du))) < 1e-15


def test_argmin_ties_take_smallest_index(oracle):
    """k* = smallest k among exact ties; every tied minimum gets weight 1."""
    pb = cartpole_problem(oracle, T=2)
    eps = oracle.noise(1, 0, 2, 6, 1)
    costs = np.array([5.0, 3.0, 4.0, 3.0, 9.0, 3.0])
    _, kstar, smin, eta, w = oracle.update(pb, costs, eps, np.zeros((2, 1)))
    assert kstar == 1 and smin == 3.0
    assert w[1] == w[3] == w[5] == 1.0


def test_nu_one_is_the_mean_shift_cost(oracle):
    """P7 / SPEC.md:195, :198, :555: nu = 1 makes the (1 - 1/nu)/2 term exactly zero, so
    S~ - S = sum_t (u'R du + 1/2 u'R u) on the same trajectory; with u = 0 and nu = 1, S~ = S
    exactly; for nu > 1 and u = 0 the difference is (1 - 1/nu)/2 sum du'R du."""
    T, K = 6, 32
    eps = oracle.noise(5, 0, T, K, 1)
    x0 = np.array([0.0, 0.0, 0.4, 0.0])
    U = np.random.default_rng(1).normal(size=(T, 1)) * 0.4
    for nu in (1.0, 9.0):
        pb = cartpole_problem(oracle, T=T, nu=nu)
        pb0 = oracle.Problem("cartpole", T=T, dt=0.02, lam=0.5, nu=nu, Sigma=[[0.005]], R=[[0.0]])
        du = math.sqrt(nu) * math.sqrt(0.005) * eps[:, :, 0].astype(float)       # [T][K]
        # u = 0
        St = oracle.rollout_costs(pb, x0, np.zeros((T, 1)), eps)
        S = oracle.rollout_costs(pb0, x0, np.zeros((T, 1)), eps)
        if nu == 1.0:
            assert np.array_equal(St, S)
        else:
            assert np.allclose(St - S, 0.5 * (1 - 1 / nu) * (du ** 2).sum(0), rtol=1e-10, atol=1e-12)
        # u != 0
        St = oracle.rollout_costs(pb, x0, U, eps)
        S = oracle.rollout_costs(pb0, x0, U, eps)
        want = 0.5 * (1 - 1 / nu) * (du ** 2).sum(0) + (U * du).sum(0) + 0.5 * (U ** 2).sum()
        assert np.allclose(St - S, want, rtol=1e-10, atol=1e-12)


def test_tiny_brute_force_update(oracle):
    """P11: K <= 8, T <= 3 with supplied eps, the update expanded by hand:
    K=2, lambda=1, S~ = (0, ln 3) -> weights (0.75, 0.25); du = (+1, -1) -> u' = 0.5."""
    pb = oracle.Problem("cartpole", T=1, dt=0.02, lam=1.0, nu=1.0, Sigma=[[1.0]], R=[[1.0]])
    eps = np.array([[[1.0], [-1.0]]], np.float32)
    U1, kstar, _, eta, w = oracle.update(pb, np.array([0.0, math.log(3.0)]), eps, np.zeros((1, 1)))
    assert w / eta == pytest.approx([0.75, 0.25], abs=1e-15)
    assert U1[0, 0] == pytest.approx(0.5, abs=1e-15) and kstar == 0
    # K = 3, T = 2, m = 2 with a full Cholesky factor: du = sqrt(nu) L eps by hand
    Sig = np.array([[2.0, 0.6], [0.6, 1.0]])
    L = np.array([[math.sqrt(2.0), 0.0], [0.6 / math.sqrt(2.0), math.sqrt(1.0 - 0.18)]])
    pb = oracle.Problem("racecar", T=2, dt=0.02, lam=2.0, nu=9.0, Sigma=Sig, R=np.eye(2))
    eps = np.array([[[1, 2], [0, -1], [3, 0]], [[-1, 1], [2, 2], [0, 0.5]]], np.float32)
    costs = np.array([4.0, 1.0, 2.5])
    U0 = np.array([[0.1, 0.2], [0.3, 0.4]])
    U1 = oracle.update(pb, costs, eps, U0)[0]
    w = [math.exp(-(c - 1.0) / 2.0) for c in costs]
    for t in range(2):
        num = sum(w[k] * 3.0 * (L @ eps[t, k].astype(float)) for k in range(3))
        assert np.allclose(U1[t], U0[t] + num / sum(w), rtol=0, atol=1e-15)


def test_penalty_for_non_finite_rollouts(oracle):
    """a rollout with a non-finite cost is charged the penalty (default 1e30);
    if every sample is penalised the weights are uniform."""
    T, K = 3, 8
    pb = cartpole_problem(oracle, T=T)
    eps = oracle.noise(1, 0, T, K, 1)
    eps[1, 2, 0] = np.nan
    eps[0, 5, 0] = np.inf
    costs = oracle.rollout_costs(pb, np.zeros(4), np.zeros((T, 1)), eps)
    assert costs[2] == 1e30 and costs[5] == 1e30
    assert np.all(np.isfinite(costs)) and np.all(costs[[0, 1, 3, 4, 6, 7]] < 1e30)
    allbad = np.full_like(eps, np.nan)
    costs = oracle.rollout_costs(pb, np.zeros(4), np.zeros((T, 1)), allbad)
    _, _, _, eta, w = oracle.update(pb, costs, eps, np.zeros((T, 1)))
    assert np.all(w == 1.0) and eta == K


def test_shift(oracle):
    """Alg. 1 / SPEC.md:275: U=(a,b,c) -> (b,c,u_init)."""
    U = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]])
    assert np.array_equal(oracle.shift(U, [7.0, 8.0]), [[3, 4], [5, 6], [7, 8]])


def test_thread_count_independence(oracle):
    """results are identical for 1 and many worker threads."""
    w = get("C1")
    pb = cartpole_problem(oracle, T=w.T, nu=300.0, lam=5e-3)
    eps = oracle.noise(w.seed, 0, w.T, w.K, 1)
    a = oracle.optimize(pb, w.x0, w.U0, eps, nthreads=1)
    b = oracle.optimize(pb, w.x0, w.U0, eps, nthreads=8)
    assert np.array_equal(a["costs"], b["costs"]) and np.array_equal(a["U"], b["U"])


def test_linear_quadratic_closed_form(oracle):
    """P10: linear plant + quadratic cost make S~ quadratic in du, so the exp(-S~/lambda)-tilted
    sampling Gaussian is Gaussian with mean mu* = -P^{-1} g / lambda, P = (nu Sigma_u)^{-1} (x) I_T
    + H/lambda.  The Monte-Carlo update of the oracle converges to U + mu* at 1/sqrt(ESS)
    (PAPER.md:315 is this expectation; :320 its K-sample estimate)."""
    pb, x0, U, mu, Pinv = _lq_setup(oracle)
    for K in (1 << 12, 1 << 16):
        eps = oracle.noise(11, 0, pb.T, K, 1)
        r = oracle.optimize(pb, x0, U, eps)
        w = r["weights"] / r["weights"].sum()
        ess = 1.0 / np.sum(w ** 2)
        err = (r["U"] - U)[:, 0] - mu
        z = err / np.sqrt(np.diag(Pinv) / ess)
        assert np.max(np.abs(z)) < 5.0, (K, z)
    # a wrong sign on the u'R du term or a dropped factor 1/2 moves mu* by >> the MC error
    assert np.max(np.abs(err)) < 0.1 * np.max(np.abs(mu))


@pytest.mark.slow
def test_closed_loop_cartpole_behaviour(oracle):
    """P12: "The MPPI controller is able to swing-up the pole faster with
    increasing exploration variance"; with only the natural variance (nu = 1) the average cost
    stays near the hanging cost 2000 (SPEC.md:558 5a: >= 1500) over the first 2 s.  Under our
    cart-pole reading nu = 1 does swing up eventually (after ~3.3 s), which the
    paper's "never" does not: recorded in DESIGN.md, and the trend is what is pinned here."""
    T, K = 50, 512
    first_up = []
    for nu in (1.0, 10.0, 100.0, 1000.0):
        pb = oracle.Problem("cartpole", T=T, dt=0.02, lam=5e-3, nu=nu, Sigma=[[0.005]], R=[[1.0]])
        xs, qs = oracle.closed_loop(pb, np.zeros(4), np.zeros((T, 1)), 250, seed=1, K=K)
        up = 1 + np.cos(xs[:, 2]) < 0.05
        assert up.any()
        first_up.append(int(np.argmax(up)))
        if nu == 1.0:
            assert qs[:100].mean() >= 1500.0
        if nu == 1000.0:
            assert qs[:100].mean() < 500.0 and qs[-50:].mean() < 10.0
    assert first_up == sorted(first_up, reverse=True) and first_up[0] > 2 * first_up[-1]
