"""How much of the small-K rollout time is the in-kernel noise: the packed rollout drawing its
noise vs reading a pre-generated tensor (cp.async ring), across K."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from mppi_inputs import get
from paper_1509_01149_b200 import from_workload
w = get("C4")
for K in (1 << 16, 1 << 17, 1 << 18, 1 << 20):
    m = from_workload(w, K=K)
    U = torch.tensor(w.U0, device="cuda")
    eps = m.noise(1, 0)
    res = {}
    for mode in ("gen", "read", "gen", "read"):
        for i in range(2):
            m.rollout_costs(w.x0, U, 1, 0, noise=eps if mode == "read" else None)
        m.profile_enable(True)
        for i in range(10):
            m.rollout_costs(w.x0, U, 1, 0, noise=eps if mode == "read" else None)
        t = m.profile_read()
        m.profile_enable(False)
        res[mode] = t["rollout"][0] / t["rollout"][1]
    print("K=%7d rollout: draws noise %.4f ms, reads noise %.4f ms (ratio %.3f)" % (K, res["gen"], res["read"], res["read"] / res["gen"]), flush=True)
    m.close()
