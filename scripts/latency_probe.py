"""Control-update latency vs back-to-back throughput at one config: where does a synchronous
call's extra device time come from?  CFG=C4 python scripts/latency_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import from_workload  # noqa: E402

w = get(os.environ.get("CFG", "C4"))
m = from_workload(w)
U = torch.tensor(w.U0, device="cuda")
for i in range(20):
    m.optimize(w.x0, U, w.seed, i)
torch.cuda.synchronize()
N = 200


def q(xs, p):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(round(p * (len(xs) - 1))))]


# 1. back to back
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(N):
    m.optimize(w.x0, U, w.seed, i)
e1.record()
torch.cuda.synchronize()
print("back-to-back: %.1f us per call" % (e0.elapsed_time(e1) * 1e3 / N))
# 2. per-call events, back to back
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
for i in range(N):
    evs[i][0].record()
    m.optimize(w.x0, U, w.seed, i)
    evs[i][1].record()
torch.cuda.synchronize()
d = [a.elapsed_time(b) * 1e3 for a, b in evs]
print("per-call events, no sync: p50 %.1f p99 %.1f us" % (q(d, .5), q(d, .99)))
# 3. per-call events + synchronize after each
for gap_us in (0, 50, 500, 5000):
    for i in range(N):
        evs[i][0].record()
        m.optimize(w.x0, U, w.seed, i)
        evs[i][1].record()
        torch.cuda.synchronize()
        if gap_us:
            t = time.perf_counter()
            while (time.perf_counter() - t) * 1e6 < gap_us:
                pass
    d = [a.elapsed_time(b) * 1e3 for a, b in evs]
    print("per-call sync, host gap %d us: p50 %.1f p99 %.1f us" % (gap_us, q(d, .5), q(d, .99)))
# 4. the same with per-kernel events (direct launches)
m.profile_enable(True)
for i in range(N):
    m.optimize(w.x0, U, w.seed, i)
    torch.cuda.synchronize()
kt = m.profile_read()
m.profile_enable(False)
print("per-call sync, per-kernel:", {k: round(v[0] / v[1] * 1e3, 1) for k, v in kt.items() if v[1]})
m.profile_enable(True)
for i in range(N):
    m.optimize(w.x0, U, w.seed, i)
torch.cuda.synchronize()
kt = m.profile_read()
m.profile_enable(False)
print("back-to-back, per-kernel:", {k: round(v[0] / v[1] * 1e3, 1) for k, v in kt.items() if v[1]})
