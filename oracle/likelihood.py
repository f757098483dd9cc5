"""Theorem 1 of arXiv:1509.01149 and its brute-force check, fp64 numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings:
  A5  Gamma^{-1} = Sigma^{-1} - Lambda^{-1} with Lambda = A Sigma A^T (the proof, PAPER.md:226,
      :252); the theorem statement's "(Sigma^{-1} - A^T Sigma A)^{-1}" is garbled.
  A6  Sigma_i = B_c B_c^T (no dt) inside the quadratic forms, so that a one-step transition has
      density N(z; mu, Sigma/dt) and the exponent is -dt/2 (z-mu)^T Sigma^{-1} (z-mu).
"""
import numpy as np


def gamma_inverse(Sigma, A):
    """Gamma^{-1} = Sigma^{-1} - (A Sigma A^T)^{-1}."""
    Lam = A @ Sigma @ A.T
    return np.linalg.inv(Sigma) - np.linalg.inv(Lam)


def Q_term(z, mu, Sigma, Ginv):
    """Q = (z-mu)^T Gamma^{-1} (z-mu) + 2 mu^T Sigma^{-1} (z-mu) + mu^T Sigma^{-1} mu."""
    Si = np.linalg.inv(Sigma)
    d = z - mu
    return d @ Ginv @ d + 2.0 * mu @ Si @ d + mu @ Si @ mu


def theorem1_log_ratio(zs, mus, Sigmas, As, dt):
    """log p/q = sum_i log|det A_i| - dt/2 sum_i Q_i."""
    out = 0.0
    for z, mu, S, A in zip(zs, mus, Sigmas, As):
        out += np.log(abs(np.linalg.det(A))) - 0.5 * dt * Q_term(z, mu, S, gamma_inverse(S, A))
    return out


def gaussian_logpdf(x, mean, cov):
    """Explicit multivariate normal log-density."""
    d = x - mean
    k = len(x)
    sign, logdet = np.linalg.slogdet(cov)
    assert sign > 0
    return -0.5 * (k * np.log(2 * np.pi) + logdet + d @ np.linalg.solve(cov, d))


def brute_force_log_ratio(zs, mus, Sigmas, As, dt):
    """Product of one-step densities: under p, z_i ~ N(0, Sigma_i/dt);
    under q, z_i ~ N(mu_i, A_i Sigma_i A_i^T / dt)."""
    out = 0.0
    for z, mu, S, A in zip(zs, mus, Sigmas, As):
        out += gaussian_logpdf(z, np.zeros_like(z), S / dt)
        out -= gaussian_logpdf(z, mu, A @ S @ A.T / dt)
    return out


def special_case_is_terms(u, du, R, nu):
    """the likelihood-ratio part of q~ in the special case A = sqrt(nu) I:
    (1 - 1/nu)/2 du^T R du + u^T R du + 1/2 u^T R u."""
    return 0.5 * (1.0 - 1.0 / nu) * du @ R @ du + u @ R @ du + 0.5 * u @ R @ u
