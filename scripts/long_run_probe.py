"""Long optimisation run from the same x0: step time and replayed rollouts per block of steps
(does anything data-dependent creep in as U converges?).  CFG=C5 K=1048576 N=1000 python ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import from_workload  # noqa: E402

w = get(os.environ.get("CFG", "C5"))
if os.environ.get("K"):
    w.K = int(os.environ["K"])
N = int(os.environ.get("N", "1000"))
B = 100
m = from_workload(w)
U = torch.tensor(w.U0, device="cuda")
for i in range(5):
    m.optimize(w.x0, U, w.seed, i)
torch.cuda.synchronize()
for b in range(N // B):
    r0 = m.replay_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(B):
        m.optimize(w.x0, U, w.seed, 5 + b * B + i)
    e1.record()
    torch.cuda.synchronize()
    st = m.stats()
    print("%s K=%d steps %4d-%4d: %.3f ms/step, replayed %d, S_min %.6g, eta %.4g, U finite %s, U mean %s"
          % (w.name, w.K, b * B, (b + 1) * B, e0.elapsed_time(e1) / B, m.replay_count() - r0, st["s_min"],
             st["eta"], bool(torch.isfinite(U).all()), np.round(U.mean(0).cpu().numpy(), 3)), flush=True)
