"""How sparse are the MPPI weights? Counts samples with exp(-(S - S_min)/lambda) > 0 in fp32
(and the share of 256-sample column blocks that hold one) over a few receding-horizon steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import from_workload  # noqa: E402

for cfg in sys.argv[1:] or ["C5"]:
    w = get(cfg)
    m = from_workload(w)
    U = torch.tensor(w.U0, device="cuda")
    for step in range(4):
        costs, key = m.rollout_costs(w.x0, U, w.seed, step)
        smin = costs.min()
        wts = torch.exp(-((costs - smin) / w.lam).float())
        nz = (wts > 0)
        blk = nz.view(-1, 256).any(dim=1) if costs.numel() % 256 == 0 else nz
        print(cfg, "step", step, "K", costs.numel(), "nonzero w", int(nz.sum()), "blocks", int(blk.sum()), "/", blk.numel(),
              "eta %.3f" % float(wts.sum()), flush=True)
        m.optimize(w.x0, U, w.seed, step)
    m.close()
