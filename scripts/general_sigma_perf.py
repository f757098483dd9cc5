"""C5 step time with a diagonal vs a correlated Sigma (the general one-sample path) vs per-step
transforms A_t (NEXT-3), all with the in-kernel noise and the obstacle grid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import MPPI  # noqa: E402

w = get("C5")
K = int(os.environ.get("K", w.K))
rng = np.random.default_rng(5)
B = rng.normal(size=(4, 4)) * 0.02
for name in ("diagonal", "correlated", "A_t"):
    Sig = np.array(w.Sigma, np.float64) + (B @ B.T if name == "correlated" else 0.0)
    m = MPPI(w.plant, K, w.T, w.dt, w.lam, w.nu, Sig, w.R, obstacles=w.obstacles)
    if name == "A_t":
        m.set_sampling_transform(np.array([rng.normal(size=(4, 4)) * 0.3 + 3.0 * np.eye(4) for _ in range(w.T)]))
    U = torch.tensor(w.U0, device="cuda")
    for i in range(3):
        m.optimize(w.x0, U, 1, i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(5):
        m.optimize(w.x0, U, 1, 3 + i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print("%-10s K=%d ms/step %.3f K*T/s %.3g" % (name, K, ms, K * w.T / ms * 1e3), flush=True)
    m.close()
