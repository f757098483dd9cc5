"""NEXT-1 pins: per-timestep cost-to-go weights, PAPER.md:320-322 / Alg. 1 :367
("S(tau_{i,k}) is the cost-to-go of the k-th rollout from time t_i onward")."""
import math

import numpy as np
import pytest


def _pb(oracle, T=8, lam=0.5, nu=4.0):
    return oracle.Problem("cartpole", T=T, dt=0.02, lam=lam, nu=nu, Sigma=[[0.005]], R=[[1.0]])


def test_stepcosts_sum_to_trajectory_cost(oracle):
    """SPEC.md:228, :293 telescoping: S~(tau_{0,k}) = sum_t q~_{t,k} = the trajectory cost."""
    pb = _pb(oracle)
    rng = np.random.default_rng(0)
    U = rng.normal(size=(pb.T, 1)) * 0.3
    eps = oracle.noise(3, 0, pb.T, 64, 1)
    sc = oracle.rollout_stepcosts(pb, [0, 0, 0.3, 0], U, eps)
    S = oracle.rollout_costs(pb, [0, 0, 0.3, 0], U, eps)
    assert np.allclose(sc.sum(axis=1), S, rtol=1e-13)


def test_u0_equals_trajectory_weighting(oracle):
    """S~(tau_{0,k}) is the trajectory cost, so u_0 is the same under both readings."""
    pb = _pb(oracle)
    U = np.zeros((pb.T, 1))
    eps = oracle.noise(5, 0, pb.T, 128, 1)
    sc = oracle.rollout_stepcosts(pb, [0, 0, 0.2, 0], U, eps)
    Uc, smin, eta = oracle.update_ctg(pb, sc, eps, U)
    Ut = oracle.update(pb, sc.sum(axis=1), eps, U)[0]
    assert abs(Uc[0, 0] - Ut[0, 0]) < 1e-13
    assert not np.allclose(Uc[1:], Ut[1:])      # later steps weight by their own cost-to-go


def test_last_step_weights_by_last_cost_only(oracle):
    """Brute force: u_{T-1} is weighted by q~_{T-1,k} alone; u_t by the suffix sums."""
    pb = _pb(oracle, T=3, lam=2.0)
    eps = np.array([[[1.0], [-1.0], [0.5]], [[0.2], [0.0], [-0.4]], [[-1.0], [2.0], [1.0]]], np.float32)
    sc = np.array([[1.0, 2.0, 3.0], [0.5, 0.5, 5.0], [2.0, 0.1, 0.2]])      # [K][T]
    U1, smin, eta = oracle.update_ctg(pb, sc, eps, np.zeros((3, 1)))
    s = math.sqrt(4.0) * math.sqrt(0.005)
    for t in range(3):
        ctg = sc[:, t:].sum(axis=1)
        w = np.exp(-(ctg - ctg.min()) / 2.0)
        want = (w * s * eps[t, :, 0]).sum() / w.sum()
        assert U1[t, 0] == pytest.approx(want, abs=1e-15)
        assert smin[t] == pytest.approx(ctg.min(), rel=1e-15) and eta[t] == pytest.approx(w.sum(), rel=1e-14)


def test_ctg_simplex_and_lambda_limits(oracle):
    pb = _pb(oracle, lam=1e-14)
    U = np.zeros((pb.T, 1))
    eps = oracle.noise(7, 0, pb.T, 32, 1)
    sc = oracle.rollout_stepcosts(pb, [0, 0, 0.3, 0], U, eps)
    U1, smin, eta = oracle.update_ctg(pb, sc, eps, U)
    ctg = np.cumsum(sc[:, ::-1], axis=1)[:, ::-1]
    s = 2.0 * math.sqrt(0.005)
    checked = 0
    for t in range(pb.T):       # lambda -> 0: each u_t takes the noise of its own argmin
        order = np.sort(ctg[:, t])
        if order[1] - order[0] < 1e-11:      # (near-)tie: several weights survive
            continue
        k = int(np.argmin(ctg[:, t]))
        assert abs(U1[t, 0] - s * float(eps[t, k, 0])) < 1e-15 and eta[t] == 1.0
        checked += 1
    assert checked >= pb.T - 1
