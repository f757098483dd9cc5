"""Minimal driver for ncu / compute-sanitizer: N MPPI steps of one config through the C ABI."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import from_workload  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C5")
p.add_argument("--K", type=int, default=0)
p.add_argument("--steps", type=int, default=2)
a = p.parse_args()
w = get(a.config)
m = from_workload(w, K=a.K or w.K)
from paper_1509_01149_b200 import _capi as A  # noqa: E402
if os.environ.get("CTG"):
    m.set_weighting(True)
for kv in filter(None, os.environ.get("MPPI_OPTS", "").split(",")):   # e.g. OBSTACLE_GRID=0
    k, v = kv.split("=")
    m.set_option(getattr(A, "MPPI_OPTION_" + k), int(v))
U = torch.tensor(w.U0, device="cuda")
for i in range(a.steps):
    m.optimize(w.x0, U, w.seed, i)
torch.cuda.synchronize()
assert torch.isfinite(U).all()
print("ok", a.config, a.K or w.K, m.stats())
