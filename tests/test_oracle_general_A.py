"""NEXT-3 pins: generalized importance sampling with per-step variance transforms
A_t (Theorem 1; running-cost form :271-284).  The oracle samples
du_t = A_t L eps and charges 1/2 du'(R - A_t^{-T} R A_t^{-1}) du + u'R du + 1/2 u'R u."""
import math

import numpy as np
import pytest
from scipy.stats import multivariate_normal


def _rand_spd(rng, n):
    A = rng.normal(size=(n, n))
    return A @ A.T + n * np.eye(n)


def _rand_A(rng, T, m):
    return np.array([rng.normal(size=(m, m)) * 0.4 + 1.5 * np.eye(m) for _ in range(T)])


def test_sqrt_nu_identity_reproduces_special_case(oracle):
    """A_t = sqrt(nu) I is exactly the special case of PAPER.md:303-331."""
    rng = np.random.default_rng(0)
    T, K, nu = 6, 64, 7.0
    Sig = _rand_spd(rng, 2) * 0.01
    R = _rand_spd(rng, 2)
    base = oracle.Problem("racecar", T=T, dt=0.02, lam=0.5, nu=nu, Sigma=Sig, R=R)
    gen = oracle.Problem("racecar", T=T, dt=0.02, lam=0.5, nu=nu, Sigma=Sig, R=R,
                         At=np.tile(math.sqrt(nu) * np.eye(2), (T, 1, 1)))
    x0 = [13.0, 0.0, math.pi / 2, 7.0, 0.0, 0.0]
    U = np.tile([0.0, 0.5], (T, 1)) + rng.normal(size=(T, 2)) * 0.1
    eps = oracle.noise(4, 0, T, K, 2)
    a = oracle.rollout_costs(base, x0, U, eps)
    b = oracle.rollout_costs(gen, x0, U, eps)
    assert np.allclose(a, b, rtol=1e-12, atol=0)
    assert np.allclose(oracle.update(base, a, eps, U)[0], oracle.update(gen, b, eps, U)[0], rtol=1e-12)


@pytest.mark.parametrize("plant", ["linear", "quadrotor"])
def test_general_A_weights_equal_density_ratio(oracle, plant):
    """The importance-sampling identity with a changed mean AND a general per-step covariance
    A_t Sigma_u A_t^T (the point of Theorem 1): with R = lambda Sigma_u^{-1}
    (Eq. 7), exp(-S~/lambda) equals exp(-S/lambda) p(tau)/q(tau) up to a sample-independent
    constant, p: v_t ~ N(0, Sigma_u), q: v_t ~ N(U_t, A_t Sigma_u A_t^T)."""
    rng = np.random.default_rng(1)
    T, K, lam = 5, 48, 0.9
    if plant == "linear":
        n, m = 3, 2
        params = np.concatenate([(rng.normal(size=(n, n)) * 0.3).ravel(), rng.normal(size=(n, m)).ravel(),
                                 np.diag([1.0, 2.0, 0.5]).ravel()])
        kw, x0 = dict(params=params, n=n, m=m), rng.normal(size=n)
        U = rng.normal(size=(T, m)) * 0.2
    else:
        m, kw = 4, {}
        x0 = np.zeros(16); x0[2] = 2.0; x0[12:] = 0.5 * 9.81 / 4
        U = np.full((T, m), 0.5 * 9.81 / 4) + rng.normal(size=(T, m)) * 0.05
    Sig = _rand_spd(rng, m) * 0.01
    R = lam * np.linalg.inv(Sig)
    At = _rand_A(rng, T, m)
    pb = oracle.Problem(plant, T=T, dt=0.02, lam=lam, nu=1.0, Sigma=Sig, R=R, At=At, **kw)
    pb0 = oracle.Problem(plant, T=T, dt=0.02, lam=lam, nu=1.0, Sigma=Sig, R=np.zeros((m, m)), At=At, **kw)
    eps = rng.normal(size=(T, K, m)).astype(np.float32)
    St = oracle.rollout_costs(pb, x0, U, eps)
    S = oracle.rollout_costs(pb0, x0, U, eps)
    L = np.linalg.cholesky(Sig)
    logpq = np.zeros(K)
    for k in range(K):
        for t in range(T):
            v = U[t] + At[t] @ L @ eps[t, k].astype(np.float64)
            logpq[k] += multivariate_normal.logpdf(v, mean=np.zeros(m), cov=Sig)
            logpq[k] -= multivariate_normal.logpdf(v, mean=U[t], cov=At[t] @ Sig @ At[t].T)
    diff = St / lam - (S / lam - logpq)
    assert np.ptp(diff) < 1e-9 * max(np.max(np.abs(St / lam)), 1.0)


def test_general_A_lambda_infinity_update(oracle):
    """lambda -> inf: U' = U + mean_k A_t L eps_{t,k} (the update uses the same per-step factor)."""
    rng = np.random.default_rng(2)
    T, K = 4, 40
    Sig = _rand_spd(rng, 2) * 0.01
    At = _rand_A(rng, T, 2)
    pb = oracle.Problem("racecar", T=T, dt=0.02, lam=1e30, nu=1.0, Sigma=Sig, R=np.eye(2), At=At)
    eps = oracle.noise(9, 0, T, K, 2)
    U0 = np.zeros((T, 2))
    costs = oracle.rollout_costs(pb, [13.0, 0, math.pi / 2, 7.0, 0, 0], U0, eps)
    U1 = oracle.update(pb, costs, eps, U0)[0]
    L = np.linalg.cholesky(Sig)
    want = np.array([At[t] @ L @ eps[t].astype(np.float64).mean(axis=0) for t in range(T)])
    assert np.allclose(U1, want, rtol=1e-12, atol=1e-15)


def test_singular_A_is_rejected(oracle):
    At = np.tile(np.eye(2), (3, 1, 1))
    At[1] = [[1.0, 2.0], [2.0, 4.0]]
    pb = oracle.Problem("racecar", T=3, dt=0.02, lam=1.0, nu=1.0, Sigma=np.eye(2), R=np.eye(2), At=At)
    with pytest.raises(ValueError):
        oracle.rollout_costs(pb, np.zeros(6), np.zeros((3, 2)), oracle.noise(1, 0, 3, 8, 2))
