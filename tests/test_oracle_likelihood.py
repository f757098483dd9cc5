"""Pins P8 (importance-sampling identity on the oracle's augmented costs) and P9 (Theorem 1
against a brute-force product of Gaussian densities).  PAPER.md:135-138, :177-301, :323-331."""
import numpy as np
import pytest
from scipy.stats import multivariate_normal

from oracle import likelihood as LR


def _rand_spd(rng, n):
    A = rng.normal(size=(n, n))
    return A @ A.T + n * np.eye(n)


def test_theorem1_matches_brute_force():
    """SPEC.md:554 acceptance 1: >= 1000 random instances (n_c <= 3, N <= 5), rel. err <= 1e-8."""
    rng = np.random.default_rng(1)
    worst = 0.0
    for _ in range(1000):
        n = int(rng.integers(1, 4))
        N = int(rng.integers(1, 6))
        dt = float(rng.uniform(0.01, 0.5))
        zs = [rng.normal(size=n) for _ in range(N)]
        mus = [rng.normal(size=n) for _ in range(N)]
        Ss = [_rand_spd(rng, n) for _ in range(N)]
        As = []
        for _ in range(N):
            A = rng.normal(size=(n, n)) + 2 * np.eye(n)
            As.append(A)
        a = LR.theorem1_log_ratio(zs, mus, Ss, As, dt)
        b = LR.brute_force_log_ratio(zs, mus, Ss, As, dt)
        worst = max(worst, abs(a - b) / max(1.0, abs(b)))
    assert worst < 1e-8


def test_theorem1_printed_gamma_is_garbled():
    """Reading A5: with a non-symmetric A, the printed Lambda = A^T Sigma A
    does NOT reproduce the density ratio, while Lambda = A Sigma A^T does."""
    rng = np.random.default_rng(2)
    n = 2
    S = _rand_spd(rng, n)
    A = np.array([[1.5, 0.7], [0.0, 2.0]])
    z, mu = rng.normal(size=n), rng.normal(size=n)
    good = LR.theorem1_log_ratio([z], [mu], [S], [A], 0.1)
    brute = LR.brute_force_log_ratio([z], [mu], [S], [A], 0.1)
    assert good == pytest.approx(brute, rel=1e-10)
    Ginv_printed = np.linalg.inv(S) - np.linalg.inv(A.T @ S @ A)
    printed = np.log(abs(np.linalg.det(A))) - 0.05 * LR.Q_term(z, mu, S, Ginv_printed)
    assert abs(printed - brute) > 1e-3


def test_girsanov_degeneration():
    """SPEC.md:555 / PAPER.md:267-269: A = I gives Gamma^{-1} = 0 exactly, leaving the
    Girsanov terms 2 mu^T Sigma^{-1}(z - mu) + mu^T Sigma^{-1} mu."""
    rng = np.random.default_rng(3)
    S = _rand_spd(rng, 3)
    assert np.all(LR.gamma_inverse(S, np.eye(3)) == 0.0)
    z, mu = rng.normal(size=3), rng.normal(size=3)
    Si = np.linalg.inv(S)
    assert LR.Q_term(z, mu, S, np.zeros((3, 3))) == pytest.approx(2 * mu @ Si @ (z - mu) + mu @ Si @ mu)
    # SPEC.md:154-155 worked values: scalar z=1, mu=.5, Sigma=1: A=1 -> 0.75; A=sqrt(2) -> 0.875
    one = np.eye(1)
    assert LR.Q_term(np.array([1.0]), np.array([0.5]), one, LR.gamma_inverse(one, one)) == pytest.approx(0.75)
    A = np.sqrt(2) * one
    assert LR.Q_term(np.array([1.0]), np.array([0.5]), one, LR.gamma_inverse(one, A)) == pytest.approx(0.875)
    # Sigma=4, A=sqrt 2 -> 1/8; Sigma = I, A = 2 I -> 0.75 I
    assert LR.gamma_inverse(4 * one, A)[0, 0] == pytest.approx(1 / 8)
    assert np.allclose(LR.gamma_inverse(np.eye(2), 2 * np.eye(2)), 0.75 * np.eye(2))


def test_special_case_reduction():
    """with A = sqrt(nu) I, z - mu = G du, mu = G u, Sigma = G G^T / rho and
    Eq. 7 (B_c B_c^T = lambda G R^{-1} G^T with B = G/sqrt(rho)) forcing R = lambda rho dt I in
    reading A2, dt/2 Q equals q~'s IS terms / lambda
    (SPEC.md:556 acceptance 3 on random instances, to 1e-10)."""
    rng = np.random.default_rng(4)
    for _ in range(1000):
        m = int(rng.integers(1, 3))
        G = rng.normal(size=(m, m)) + 3 * np.eye(m)
        rho, dt, lam, nu = rng.uniform(10, 1e4), rng.uniform(0.005, 0.1), rng.uniform(0.01, 5), rng.uniform(1, 200)
        u, du = rng.normal(size=m), rng.normal(size=m)
        S = G @ G.T / rho
        A = np.sqrt(nu) * np.eye(m)
        mu = G @ u
        z = mu + G @ du
        dtQ2 = 0.5 * dt * LR.Q_term(z, mu, S, LR.gamma_inverse(S, A))
        R = lam * rho * dt * np.eye(m)
        assert dtQ2 == pytest.approx(LR.special_case_is_terms(u, du, R, nu) / lam, rel=1e-10, abs=1e-12)
    # SPEC.md:182 worked value: q=1, u=2, du=1, R=1, nu=2 -> 5.25
    assert 1.0 + LR.special_case_is_terms(np.array([2.0]), np.array([1.0]), np.eye(1), 2.0) == 5.25


@pytest.mark.parametrize("plant", ["cartpole", "linear", "quadrotor"])
def test_augmented_weights_equal_density_ratio(oracle, plant):
    """P8 on the oracle's C rollout: when R = lambda Sigma_u^{-1} (Eq. 7, in
    reading A2) the weights exp(-S~/lambda) equal exp(-S/lambda) p(tau)/q(tau) up to a constant,
    where S is the pure state cost on the same trajectory (oracle run with R = 0) and p, q are
    the explicit densities of v_t = U_t + du_t under N(0, Sigma_u) and N(U_t, nu Sigma_u)
    (§III-B "any terms which do not depend on the state ... cancel")."""
    rng = np.random.default_rng(5)
    T, K, lam, nu = 6, 64, 0.7, 5.0
    if plant == "linear":
        n, m = 3, 2
        A = rng.normal(size=(n, n)) * 0.3
        B = rng.normal(size=(n, m))
        Qm = np.diag([1.0, 2.0, 0.5])
        params = np.concatenate([A.ravel(), B.ravel(), Qm.ravel()])
        x0 = rng.normal(size=n)
        kw = dict(params=params, n=n, m=m)
    elif plant == "cartpole":
        m, kw, x0 = 1, {}, np.array([0.1, 0.0, 0.3, 0.0])
    else:
        m, kw = 4, {}
        x0 = np.zeros(16); x0[2] = 2.0; x0[12:] = 0.5 * 9.81 / 4
    Sig = _rand_spd(rng, m) * 0.01
    R = lam * np.linalg.inv(Sig)
    pb = oracle.Problem(plant, T=T, dt=0.02, lam=lam, nu=nu, Sigma=Sig, R=R, **kw)
    pb0 = oracle.Problem(plant, T=T, dt=0.02, lam=lam, nu=nu, Sigma=Sig, R=np.zeros((m, m)), **kw)
    U = rng.normal(size=(T, m)) * 0.2 + (0.5 * 9.81 / 4 if plant == "quadrotor" else 0)
    eps = rng.normal(size=(T, K, m)).astype(np.float32)
    St = oracle.rollout_costs(pb, x0, U, eps)
    S = oracle.rollout_costs(pb0, x0, U, eps)
    L = np.linalg.cholesky(Sig)
    logp = np.zeros(K)
    logq = np.zeros(K)
    for k in range(K):
        for t in range(T):
            du = np.sqrt(nu) * L @ eps[t, k].astype(np.float64)
            v = U[t] + du
            logp[k] += multivariate_normal.logpdf(v, mean=np.zeros(m), cov=Sig)
            logq[k] += multivariate_normal.logpdf(v, mean=U[t], cov=nu * Sig)
    diff = St / lam - (S / lam - logp + logq)
    scale = np.max(np.abs(St / lam))
    assert np.ptp(diff) < 1e-10 * max(scale, 1.0)
