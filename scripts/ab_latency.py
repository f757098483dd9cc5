"""A/B of control-update latency (graph replay, device p50/p99 and host p50) per option setting.
usage: CFG=C1 ab_latency.py SMALL_STEP=1 SMALL_STEP=0"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import _capi as A, from_workload  # noqa: E402

w = get(os.environ.get("CFG", "C1"))
for spec in sys.argv[1:]:
    m = from_workload(w)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        m.set_option(getattr(A, "MPPI_OPTION_" + k), int(v))
    U = torch.tensor(w.U0, device="cuda")
    for i in range(20):
        m.optimize(w.x0, U, w.seed, i)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
    host = []
    for i in range(200):
        t0 = time.perf_counter()
        evs[i][0].record()
        m.optimize(w.x0, U, w.seed, 20 + i)
        evs[i][1].record()
        u0 = U[0].cpu()
        host.append((time.perf_counter() - t0) * 1e6)
    torch.cuda.synchronize()
    dev = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)
    host.sort()
    print(os.environ.get("CFG", "C1"), spec, "device p50 %.1f p99 %.1f us, host p50 %.1f us, launches %d"
          % (dev[100], dev[197], host[100], m.last_launch_count()), flush=True)
    m.close()
