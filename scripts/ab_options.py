"""A/B timing of execution options at C5: per-kernel CUDA-event times for each setting.
usage: ab_options.py OPTION=V[,OPTION=V...] ...   e.g. ab_options.py OBSTACLE_GRID=0 OBSTACLE_GRID=1"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import _capi as A, from_workload  # noqa: E402

w = get(os.environ.get("CFG", "C5"))
if os.environ.get("K"):
    w.K = int(os.environ["K"])
for spec in sys.argv[1:]:
    m = from_workload(w)
    if os.environ.get("CTG"):
        m.set_weighting(True)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        m.set_option(int(k) if k.isdigit() else getattr(A, "MPPI_OPTION_" + k), int(v))
    U = torch.tensor(w.U0, device="cuda")
    for i in range(3):
        m.optimize(w.x0, U, w.seed, i)
    torch.cuda.synchronize()
    m.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(10):
        m.optimize(w.x0, U, w.seed, 3 + i)
    e1.record()
    torch.cuda.synchronize()
    kt = m.profile_read()
    print(spec, "step %.3f ms" % (e0.elapsed_time(e1) / 10),
          {k: round(v[0] / v[1], 3) for k, v in kt.items() if v[1]}, flush=True)
    m.close()
