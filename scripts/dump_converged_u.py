"""Save U after N optimisation steps from the same x0 (C4) for offline analysis."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import from_workload  # noqa: E402

w = get(os.environ.get("CFG", "C4"))
m = from_workload(w)
U = torch.tensor(w.U0, device="cuda")
for n in range(int(os.environ.get("N", "150"))):
    m.optimize(w.x0, U, w.seed, n)
np.save("gpurun_out/U_%s_%s.npy" % (w.name, os.environ.get("N", "150")), U.cpu().numpy())
print("saved")
