"""Per-step cost profile of chosen C5 samples: GPU (packed kernel, cost-to-go mode, differenced)
against the fp64 oracle and both fp32 twins; prints |q_gpu - q64| and |q_twin - q64| per step with
the fp64 |cos phi| (distance from the ZXY Euler singularity).
    python tests/tools/c5_profile_samples.py 1168267 575396"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from mppi_inputs import get  # noqa: E402
from paper_1509_01149_b200 import from_workload  # noqa: E402

CH = 65536


def main():
    import oracle.oracle as oracle
    w = get("C5")
    T, m = w.T, w.m
    pb = oracle.Problem(w.plant, T=T, dt=w.dt, lam=w.lam, nu=w.nu, Sigma=w.Sigma, R=w.R,
                        obstacles=w.obstacles)
    gc = from_workload(w, K=CH)
    gc.set_weighting(True)
    U = torch.tensor(w.U0, device="cuda")
    for k in map(int, sys.argv[1:]):
        k0 = (k // CH) * CH
        eps = oracle.noise(w.seed, 0, T, CH, m, k0=k0)
        j = k - k0
        gc.optimize(w.x0, U.clone(), 0, 0, noise=torch.from_numpy(eps).cuda())
        s = gc.cost_to_go().cpu().numpy()[:, j].astype(np.float64)
        qg = s - np.append(s[1:], 0.0)
        e1 = np.ascontiguousarray(eps[:, j:j + 1, :])
        q64 = oracle.rollout_stepcosts(pb, w.x0, w.U0, e1)[0]
        qa = oracle.rollout_stepcosts(pb, w.x0, w.U0, e1, mode="twin_f32")[0]
        qb = oracle.rollout_stepcosts(pb, w.x0, w.U0, e1, mode="twin_f32_via_f64")[0]
        xs = oracle.trajectory(pb, w.x0, w.U0, e1, 0)
        print("k=%d S gpu %.9g fp64 %.9g twinA %.9g twinB %.9g" % (k, s[0], q64.sum(), qa.sum(), qb.sum()))
        for t in range(T):
            print("  t=%3d |cos phi| %.5f  dq gpu %+.4e  twinA %+.4e  twinB %+.4e  (q64 %.3f)"
                  % (t, abs(np.cos(xs[t + 1][6])), qg[t] - q64[t], qa[t] - q64[t], qb[t] - q64[t], q64[t]))
    return 0


if __name__ == "__main__":
    sys.exit(main())
