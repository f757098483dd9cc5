"""Feynman-Kac path-integral estimate and its exact scalar-LQ value.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Psi(x0) = E_P[ exp(-S(tau)/lambda) ],  S = sum_{t=0}^{T-1} q(x_{t+1})   (A2, A3)
under the uncontrolled discrete dynamics x_{t+1} = x_t + (f(x_t) + G du_t) dt, du_t ~ N(0, Sigma_u)
(the natural noise: U = 0, nu = 1, so the importance-sampling terms of q~ vanish).
"""
import math

import numpy as np

from . import oracle as O


def mc_estimate(pb, x0, eps):
    """Monte-Carlo log Psi-hat and its standard error from the oracle's fp64 rollouts.
    pb must have nu = 1; the controls are U = 0.  Returns (log_psi, se_log_psi, S)."""
    assert pb.nu == 1.0
    S = O.rollout_costs(pb, x0, np.zeros((pb.T, pb.m)), eps)
    smin = S.min()
    w = np.exp(-(S - smin) / pb.lam)
    K = len(S)
    mean = w.mean()
    se = w.std(ddof=1) / math.sqrt(K) / mean           # delta method: se(log m) = se(m) / m
    return -smin / pb.lam + math.log(mean), se, S


def scalar_lq_log_psi(a, b, dt, sigma_u, Q, lam, T, x0):
    """Exact log Psi_0(x0) for x_{t+1} = phi x_t + b dt du_t, du_t ~ N(0, sigma_u), q = Q x^2.

    Backward recursion ("discrete Riccati recursion"): with Psi_{t+1}(x) =
    c exp(-p x^2 / lambda) and x' ~ N(phi x, w), w = (b dt)^2 sigma_u,
      E[exp(-alpha x'^2)] = (1 + 2 alpha w)^(-1/2) exp(-alpha (phi x)^2 / (1 + 2 alpha w)),
    alpha = (Q + p) / lambda, so p <- lambda alpha phi^2 / (1 + 2 alpha w) and
    log c <- log c - log(1 + 2 alpha w) / 2, starting from p = 0, log c = 0 at t = T.
    Returns log Psi_0(x0) = log c - p x0^2 / lambda."""
    phi = 1.0 + a * dt
    w = (b * dt) ** 2 * sigma_u
    p, logc = 0.0, 0.0
    for _ in range(T):
        alpha = (Q + p) / lam
        den = 1.0 + 2.0 * alpha * w
        p = lam * alpha * phi * phi / den
        logc -= 0.5 * math.log(den)
    return logc - p * x0 * x0 / lam
