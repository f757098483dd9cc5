"""MPPI_OPTION_NOISE_AHEAD (opt-in): below the in-kernel-noise threshold the step graph also
draws the noise of (seed, step + 1) beside the rollouts, and the next call with that (seed,
step) skips its noise kernel.  Noise is a pure function of (seed, step, k),
so every result must be bitwise the plain path's -- through hits, misses (other steps or seeds),
and calls that rewrite the context's noise buffer in between (split phase, direct launches,
supplied noise, the on-device closed loop)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import _capi as A, from_workload  # noqa: E402


def bits(t):
    return t.detach().cpu().numpy().view(np.uint32).copy()


def run(m, w, U, script):
    out = []
    for op, a in script:
        if op == "opt":
            seed, step = a
            m.optimize(w.x0, U, seed, step)
            st = m.stats()
            out.append(("opt", bits(U), st["k_star"], np.float32(st["eta"]).view(np.uint32)))
        elif op == "costs":
            c, key = m.rollout_costs(w.x0, U, a[0], a[1])
            out.append(("costs", bits(c), int(key.item())))
        elif op == "direct":
            m.use_graph(False)
            m.optimize(w.x0, U, a[0], a[1])
            m.use_graph(True)
            out.append(("direct", bits(U)))
        elif op == "supplied":
            eps = m.noise(a[0] + 7, a[1])
            m.optimize(w.x0, U, a[0], a[1], noise=eps)
            out.append(("supplied", bits(U)))
    return out


SCRIPT = [("opt", (1, 0)), ("opt", (1, 1)), ("opt", (1, 2)), ("opt", (1, 3)),   # hits
          ("opt", (1, 7)), ("opt", (2, 8)), ("opt", (2, 9)),                     # misses, then a hit
          ("costs", (2, 10)), ("opt", (2, 10)), ("opt", (2, 11)),                # split phase between
          ("direct", (2, 12)), ("opt", (2, 13)), ("opt", (2, 14)),               # direct launches
          ("supplied", (2, 15)), ("opt", (2, 16)), ("opt", (2, 17))]             # supplied noise


@pytest.mark.parametrize("cfg,K", [("C1", 256), ("C3", 4096), ("C4", 4096), ("C2", 4096)])
def test_noise_ahead_is_bitwise_the_plain_path(cfg, K):
    w = get(cfg)
    a = from_workload(w, K=K)
    a.set_option(A.MPPI_OPTION_NOISE_AHEAD, 1)
    b = from_workload(w, K=K)
    b.set_option(A.MPPI_OPTION_NOISE_AHEAD, 0)
    Ua = torch.tensor(w.U0, device="cuda")
    Ub = Ua.clone()
    ra = run(a, w, Ua, SCRIPT)
    rb = run(b, w, Ub, SCRIPT)
    assert len(ra) == len(rb)
    for x, y in zip(ra, rb):
        assert x[0] == y[0]
        for u, v in zip(x[1:], y[1:]):
            assert np.array_equal(np.asarray(u), np.asarray(v)), x[0]
    # a hit's graph launches no noise kernel on the chain: the same launch count as the plain
    # path (the side branch's noise kernel replaces it)
    assert a.last_launch_count() == b.last_launch_count()


def test_noise_ahead_across_the_device_closed_loop():
    """mppi_closed_loop rewrites the noise buffer: an optimize after it must not use the noise
    drawn ahead before it."""
    w = get("C2")
    a = from_workload(w, K=1024)
    a.set_option(A.MPPI_OPTION_NOISE_AHEAD, 1)
    b = from_workload(w, K=1024)
    b.set_option(A.MPPI_OPTION_NOISE_AHEAD, 0)
    res = []
    for m in (a, b):
        U = torch.tensor(w.U0, device="cuda")
        x = torch.tensor(w.x0, device="cuda")
        m.optimize(w.x0, U, 3, 0)                 # draws (3, 1) ahead
        m.closed_loop(x, U, 5, seed=3, step0=1)   # uses steps 1..5 through its own graph
        m.optimize(w.x0, U, 3, 1)                 # must redraw (3, 1)
        m.optimize(w.x0, U, 3, 2)
        res.append(bits(U))
    assert np.array_equal(res[0], res[1])
