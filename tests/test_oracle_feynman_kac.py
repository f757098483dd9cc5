"""NEXT-4 pins: the Feynman-Kac estimate Psi = E_P[exp(-S/lambda)]
of the oracle against an exact Gaussian backward recursion."""
import math

import numpy as np
import pytest

from oracle import feynman_kac as FK


def scalar_problem(oracle, T=10, Q=1.0, a=-0.5, b=1.0, dt=0.1, sig=0.4, lam=0.7):
    params = np.array([a, b, Q])            # A (1x1), B (1x1), Q (1x1)
    return oracle.Problem("linear", T=T, dt=dt, lam=lam, nu=1.0, Sigma=[[sig]], R=[[1.0]],
                          params=params, n=1, m=1)


def test_zero_cost_gives_psi_one(oracle):
    """q = 0 -> Psi = 1 exactly, zero variance."""
    pb = scalar_problem(oracle, Q=0.0)
    eps = oracle.noise(3, 0, pb.T, 1024, 1)
    log_psi, se, S = FK.mc_estimate(pb, np.array([0.8]), eps)
    assert log_psi == 0.0 and se == 0.0 and np.all(S == 0.0)
    assert FK.scalar_lq_log_psi(-0.5, 1.0, 0.1, 0.4, 0.0, 0.7, 10, 0.8) == 0.0


def test_recursion_one_step_closed_form():
    """T = 1 by hand: x' ~ N(phi x0, w), E exp(-Q x'^2/lam) = (1 + 2Qw/lam)^(-1/2) exp(-Q phi^2 x0^2 /
    (lam (1 + 2Qw/lam)))."""
    a, b, dt, sig, Q, lam, x0 = -0.5, 1.0, 0.1, 0.4, 2.0, 0.7, 0.8
    phi, w = 1 + a * dt, (b * dt) ** 2 * sig
    den = 1 + 2 * Q * w / lam
    want = -0.5 * math.log(den) - Q * phi ** 2 * x0 ** 2 / (lam * den)
    assert FK.scalar_lq_log_psi(a, b, dt, sig, Q, lam, 1, x0) == pytest.approx(want, rel=1e-14)


def test_recursion_matches_numerical_integration():
    """T = 2 against direct numerical integration over (x1, x2) on a fine grid."""
    a, b, dt, sig, Q, lam, x0 = -0.5, 1.0, 0.5, 0.3, 1.0, 0.9, 0.6
    phi, w = 1 + a * dt, (b * dt) ** 2 * sig
    g = np.linspace(-4, 4, 2001)
    dx = g[1] - g[0]
    pdf = lambda x, m: np.exp(-(x - m) ** 2 / (2 * w)) / math.sqrt(2 * math.pi * w)
    inner = np.array([np.sum(pdf(g, phi * x1) * np.exp(-Q * g ** 2 / lam)) * dx for x1 in g])
    psi = np.sum(pdf(g, phi * x0) * np.exp(-Q * g ** 2 / lam) * inner) * dx
    assert FK.scalar_lq_log_psi(a, b, dt, sig, Q, lam, 2, x0) == pytest.approx(math.log(psi), rel=1e-6)


def test_monte_carlo_matches_recursion(oracle):
    """SPEC.md:557 acceptance 4: |log Psi-hat - log Psi| <= 3 standard errors at K = 1e5 (scalar LQ)."""
    pb = scalar_problem(oracle)
    K = 100000
    eps = oracle.noise(11, 0, pb.T, K, 1)
    x0 = 0.8
    log_psi, se, _ = FK.mc_estimate(pb, np.array([x0]), eps)
    exact = FK.scalar_lq_log_psi(-0.5, 1.0, 0.1, 0.4, 1.0, 0.7, pb.T, x0)
    assert abs(log_psi - exact) <= 3 * se, (log_psi, exact, se)
    assert se < 0.01
