"""Linear-quadratic fixture for pin P10 (shared by the oracle test and the GPU parity test).

Linear plant x_{t+1} = x_t + (A x_t + B v_t) dt with q = x'Qx makes S~ quadratic in the stacked
du (PAPER.md:329-331 adds only quadratic/linear du terms), so the exp(-S~/lambda)-tilted sampling
Gaussian N(0, nu Sigma_u (x) I_T) is Gaussian with precision P = (nu Sigma_u)^{-1} (x) I + H/lambda
and mean mu* = -P^{-1} g / lambda: the expectation PAPER.md:315 estimates with K samples (:320).
"""
import numpy as np


def lq_setup(oracle, T=4, lam=1.0, nu=2.0):
    A = np.array([[0.0, 1.0], [-1.0, -0.3]])
    B = np.array([[0.0], [1.0]])
    Q = np.array([[2.0, 0.0], [0.0, 0.5]])
    dt, Sig, R = 0.1, np.array([[0.3]]), np.array([[0.8]])
    pb = oracle.Problem("linear", T=T, dt=dt, lam=lam, nu=nu, Sigma=Sig, R=R,
                        params=np.concatenate([A.ravel(), B.ravel(), Q.ravel()]), n=2, m=1)
    x0 = np.array([1.0, -0.5])
    U = np.array([[0.2], [-0.1], [0.3], [0.0]])[:T]
    # x_{t+1} = Phi x_t + Bd v_t; stack x_{1..T} = xbar + G d with d = du stacked
    Phi = np.eye(2) + dt * A
    Bd = dt * B
    xbar = []
    x = x0.copy()
    for t in range(T):
        x = Phi @ x + Bd @ U[t]
        xbar.append(x.copy())
    G = np.zeros((2 * T, T))
    for t in range(T):
        for s in range(t + 1):
            G[2 * t:2 * t + 2, s] = (np.linalg.matrix_power(Phi, t - s) @ Bd)[:, 0]
    Qh = np.kron(np.eye(T), Q)
    c1 = 0.5 * (1 - 1 / nu)
    H = 2 * (G.T @ Qh @ G + c1 * R[0, 0] * np.eye(T))
    g = 2 * G.T @ Qh @ np.concatenate(xbar) + R[0, 0] * U[:, 0]
    P0 = np.eye(T) / (nu * Sig[0, 0])
    P = P0 + H / lam
    mu = -np.linalg.solve(P, g / lam)
    return pb, x0, U, mu, np.linalg.inv(P)


