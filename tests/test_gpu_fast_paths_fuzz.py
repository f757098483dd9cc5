"""Seeded random combinations of plant, K (ragged), T, Sigma (diagonal or correlated), per-step
A_t, cost-to-go weighting, forest and start state: every execution option that claims identical
results (CUDA graph, packed samples, in-kernel noise, obstacle grid, bulk-copy reduction, PDL,
sparse reduction) switched on versus all switched off must give the same costs, k* and U bit for
bit over several receding-horizon steps."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from mppi_inputs import get  # noqa: E402
from mppi_inputs.forest import generate_forest  # noqa: E402
from paper_1509_01149_b200 import MPPI, _capi as A  # noqa: E402

FAST = {"CUDA_GRAPH": 1, "PACKED_SAMPLES": 1, "FUSED_NOISE": 1, "OBSTACLE_GRID": 1, "BULK_REDUCTION": 1,
        "PDL": 1, "SPARSE_REDUCTION": 1}


def _combo(i):
    rng = np.random.default_rng(100 + i)
    cfg = ["C1", "C3", "C4", "C4", "C4"][i % 5]
    w = get(cfg)
    T = int(rng.integers(5, 60))
    K = int(rng.choice([256, 4100, 65536, 65536 + 4 * int(rng.integers(1, 500)), 131072]))
    m = w.m
    Sig = np.array(w.Sigma, np.float64)
    if rng.random() < 0.4 and m > 1:
        B = rng.normal(size=(m, m)) * 0.02
        Sig = Sig + B @ B.T
    lam = float(rng.choice([w.lam, 0.5, 50.0]))
    obstacles = None
    x0 = w.x0.copy()
    if w.plant == "quadrotor":
        f = generate_forest(spacing=float(rng.choice([3.0, 4.0, 5.0])), seed=int(rng.integers(0, 99)))
        obstacles = np.array(f["centers"], np.float32)[:120]
        x0[0], x0[1] = rng.uniform(-5, 40), rng.uniform(-8, 8)
        x0[3] = rng.uniform(-3, 6)
    At = None
    if rng.random() < 0.25:
        At = np.array([rng.normal(size=(m, m)) * 0.2 + 2.0 * np.eye(m) for _ in range(T)])
    ctg = rng.random() < 0.3
    U0 = np.resize(w.U0, (T, m)).astype(np.float32)
    return w, T, K, Sig, lam, obstacles, x0, At, ctg, U0


@pytest.mark.parametrize("i", range(30))
def test_all_fast_paths_bitwise(i):
    w, T, K, Sig, lam, obstacles, x0, At, ctg, U0 = _combo(i)
    ctxs = []
    for fast in (True, False):
        m = MPPI(w.plant, K, T, w.dt, lam, w.nu, Sig, w.R, obstacles=obstacles)
        for k, v in FAST.items():
            m.set_option(getattr(A, "MPPI_OPTION_" + k), v if fast else 0)
        m.set_option(A.MPPI_OPTION_FUSED_REDUCTION, 0)   # changes rounding: tested on its own
        if At is not None:
            m.set_sampling_transform(At)
        if ctg:
            m.set_weighting(True)
        ctxs.append(m)
    Us = [torch.tensor(U0, device="cuda") for _ in ctxs]
    for step in range(3):
        for m, U in zip(ctxs, Us):
            m.optimize(x0, U, 11, step)
        torch.cuda.synchronize()
        assert torch.equal(Us[0], Us[1]), (i, step, float((Us[0] - Us[1]).abs().max()))
        assert ctxs[0].stats() == ctxs[1].stats()
    c0, k0 = ctxs[0].rollout_costs(x0, Us[0], 12, 0)
    c1, k1 = ctxs[1].rollout_costs(x0, Us[1], 12, 0)
    assert torch.equal(c0, c1) and int(k0.item()) == int(k1.item())
    for m in ctxs:
        m.close()
