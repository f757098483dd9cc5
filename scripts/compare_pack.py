"""Rollout time of the one-sample and two-sample (packed) quadrotor kernels across K."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import _capi as A, from_workload  # noqa: E402

w = get("C4")
for K in (1 << 14, 1 << 15, 1 << 16, 1 << 17, 1 << 18, 1 << 19, 1 << 20, 1 << 22):
    row = []
    for packed in (0, 1):
        m = from_workload(w, K=K)
        m.set_option(A.MPPI_OPTION_PACKED_SAMPLES, packed)
        U = torch.tensor(w.U0, device="cuda")
        for i in range(3):
            m.rollout_costs(w.x0, U, 1, i)
        m.profile_enable(True)
        for i in range(10):
            m.rollout_costs(w.x0, U, 1, i)
        t = m.profile_read()["rollout"]
        row.append(t[0] / t[1])
        m.close()
    print("K=%8d  one-sample %.4f ms  packed %.4f ms  ratio %.3f" % (K, row[0], row[1], row[1] / row[0]), flush=True)
