"""NEXT-4 on the GPU: mppi_feynman_kac against the oracle on the same noise and
against the exact scalar-LQ value (oracle/feynman_kac.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import feynman_kac as FK  # noqa: E402
from paper_1509_01149_b200 import MPPI, MppiError  # noqa: E402
from mppi_inputs import get  # noqa: E402


def test_feynman_kac_scalar_lq(oracle):
    T, dt, sig, lam, x0 = 10, 0.1, 0.4, 0.7, 0.8
    lin = dict(A=[[-0.5]], B=[[1.0]], Q=[[1.0]])
    K = 1 << 17
    m = MPPI("linear", K, T, dt, lam, 1.0, [[sig]], [[1.0]], linear=lin)
    log_psi, se, smin = m.feynman_kac([x0], seed=11, step=0)
    pb = oracle.Problem("linear", T=T, dt=dt, lam=lam, nu=1.0, Sigma=[[sig]], R=[[1.0]],
                        params=np.array([-0.5, 1.0, 1.0]), n=1, m=1)
    ref, ref_se, _ = FK.mc_estimate(pb, np.array([x0]), oracle.noise(11, 0, T, K, 1))
    assert abs(log_psi - ref) < 1e-4 and abs(se - ref_se) < 1e-3 * ref_se + 1e-9
    exact = FK.scalar_lq_log_psi(-0.5, 1.0, dt, sig, 1.0, lam, T, x0)
    assert abs(log_psi - exact) <= 3 * se


def test_feynman_kac_cartpole_matches_oracle(oracle):
    w = get("C1")
    K = 4096
    m = MPPI("cartpole", K, w.T, w.dt, 50.0, 1.0, w.Sigma, w.R)
    log_psi, se, smin = m.feynman_kac(w.x0, seed=2, step=1)
    pb = oracle.Problem("cartpole", T=w.T, dt=w.dt, lam=50.0, nu=1.0, Sigma=w.Sigma, R=w.R)
    ref, ref_se, S = FK.mc_estimate(pb, w.x0, oracle.noise(2, 1, w.T, K, 1))
    assert abs(smin - S.min()) <= 1e-4 * abs(S.min())
    assert abs(log_psi - ref) <= 1e-4 * abs(ref)


def test_feynman_kac_requires_nu_one():
    w = get("C1")
    m = MPPI("cartpole", 256, w.T, w.dt, 1.0, 2.0, w.Sigma, w.R)
    with pytest.raises(MppiError):
        m.feynman_kac(w.x0)


def test_feynman_kac_through_nccl_equals_direct():
    """Sharded path of mppi_feynman_kac on a single-rank communicator (one GPU per call here):
    NCCL MIN of the key and SUM of the fp64 partials give the direct estimate bit for bit; a
    world-2 context without a communicator is refused."""
    from mppi_inputs import get as get_w
    from paper_1509_01149_b200 import from_workload
    w = get_w("C4")
    w.nu = 1.0
    a = from_workload(w, K=1 << 16)
    b = from_workload(w, K=1 << 16)
    b.attach_nccl()
    ra = a.feynman_kac(w.x0, seed=4, step=2)
    rb = b.feynman_kac(w.x0, seed=4, step=2)
    assert ra == rb and np.isfinite(ra[0])
    a.close()
    b.close()
    c = from_workload(w, K=1024, rank=0, world=2)
    with pytest.raises(MppiError):
        c.feynman_kac(w.x0)
    c.close()
