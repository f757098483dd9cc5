"""Feynman-Kac estimate (NEXT-4) wall time on the quadrotor forest (nu = 1, U = 0) and the
scalar cart-pole, K = 2^20 / 2^22; synchronous calls (the estimate is returned to the host)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import MPPI  # noqa: E402

for cfg, K in (("C4", 1 << 20), ("C4", 1 << 22), ("C2", 1 << 20)):
    w = get(cfg)
    m = MPPI(w.plant, K, w.T, w.dt, w.lam, 1.0, w.Sigma, w.R,
             obstacles=w.obstacles if w.plant == "quadrotor" else None)
    for i in range(2):
        m.feynman_kac(w.x0, 1, i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(5):
        r = m.feynman_kac(w.x0, 1, 2 + i)
    dt = (time.perf_counter() - t0) / 5
    print("%s K=%d T=%d: %.3f ms per estimate (%.3g K*T/s), log_psi %.3f +- %.3f" % (cfg, K, w.T, dt * 1e3, K * w.T / dt, r[0], r[1]), flush=True)
    m.close()
