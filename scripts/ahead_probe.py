"""NOISE_AHEAD on/off: per-call host time of mppi_optimize (enqueue only), back-to-back device
time per call, and synchronous per-call device time.  CFG=C3 python scripts/ahead_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import _capi as A, from_workload  # noqa: E402

w = get(os.environ.get("CFG", "C3"))
N = 200


def q(xs, p):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(round(p * (len(xs) - 1))))]


for rep in range(2):
    for ahead in (1, 0):
        m = from_workload(w)
        m.set_option(A.MPPI_OPTION_NOISE_AHEAD, ahead)
        U = torch.tensor(w.U0, device="cuda")
        for i in range(20):
            m.optimize(w.x0, U, w.seed, i)
        torch.cuda.synchronize()
        host = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(N):
            t = time.perf_counter()
            m.optimize(w.x0, U, w.seed, 20 + i)
            host.append((time.perf_counter() - t) * 1e6)
        e1.record()
        torch.cuda.synchronize()
        b2b = e0.elapsed_time(e1) * 1e3 / N
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
        hs = []
        for i in range(N):
            evs[i][0].record()
            t = time.perf_counter()
            m.optimize(w.x0, U, w.seed, 20 + N + i)
            hs.append((time.perf_counter() - t) * 1e6)
            evs[i][1].record()
            torch.cuda.synchronize()
        d = [a.elapsed_time(b) * 1e3 for a, b in evs]
        print("%s rep %d ahead=%d: enqueue p50 %.1f us (b2b loop) %.1f us (sync loop); back-to-back %.1f us/call; "
              "sync device p50 %.1f p99 %.1f" % (w.name, rep, ahead, q(host, .5), q(hs, .5), b2b, q(d, .5), q(d, .99)),
              flush=True)
        m.close()
