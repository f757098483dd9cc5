"""Does the rollout slow down as U converges (more pairs replayed after the loop)?  Times the
step with the initial U and with U after N optimisation steps from the same x0, with the obstacle
grid on and off (off: the exact full 50-cylinder search, so no grid-miss replays).
    CFG=C4 [K=...] python scripts/replay_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import _capi as A, from_workload  # noqa: E402

w = get(os.environ.get("CFG", "C4"))
if os.environ.get("K"):
    w.K = int(os.environ["K"])


def timed(m, U0, n=20, seed0=1000):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    Ut = U0.clone()
    m.optimize(w.x0, Ut, w.seed, seed0)
    torch.cuda.synchronize()
    e0.record()
    for i in range(n):
        Ut.copy_(U0)
        m.optimize(w.x0, Ut, w.seed, seed0 + 1 + i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


m = from_workload(w)
mg = from_workload(w)
mg.set_option(A.MPPI_OPTION_OBSTACLE_GRID, 0)
U0 = torch.tensor(w.U0, device="cuda")
U = U0.clone()
print("%s K=%d: fresh U: %.1f us (grid) %.1f us (full search)" % (w.name, w.K, timed(m, U0), timed(mg, U0)))
done = 0
for n in (10, 40, 150, 300):
    while done < n:
        m.optimize(w.x0, U, w.seed, done)
        done += 1
    torch.cuda.synchronize()
    Uc = U.clone()
    print("after %3d steps: %.1f us (grid) %.1f us (full search); U mean %s" %
          (n, timed(m, Uc), timed(mg, Uc), np.round(Uc.mean(0).cpu().numpy(), 3)))
