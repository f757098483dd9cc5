"""Diagnose the C5 samples whose GPU cost misses the oracle by more than 1e-4 although both fp32
conditioning twins agree with fp64 (scripts/c5_every_sample.py): for each listed chunk of 65536
samples, rerun the chunk on the GPU with the oracle's noise (packed kernel, supplied noise: bitwise
the C5 kernel's costs), find the offending samples, and compare the per-step costs q~_t of the GPU
(cost-to-go mode, differenced) with the fp64 oracle and both twins to locate the first divergent
step; print the fp64 state around it.

    python tests/tools/c5_outliers.py 8 17 48 51 53 59
"""
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
    np.set_printoptions(precision=6, suppress=True, linewidth=220)
    w = get("C5")
    T, m = w.T, w.m
    full = from_workload(w)
    U = torch.tensor(w.U0, device="cuda")
    c_full, _ = full.rollout_costs(w.x0, U, w.seed, 0)
    c_full = c_full.cpu().numpy()
    full.close()
    pb = oracle.Problem(w.plant, T=T, dt=w.dt, lam=w.lam, nu=w.nu, Sigma=w.Sigma, R=w.R,
                        obstacles=w.obstacles)
    g = from_workload(w, K=CH)
    gc = from_workload(w, K=CH)
    gc.set_weighting(True)
    for ci in map(int, sys.argv[1:]):
        k0 = ci * CH
        eps = oracle.noise(w.seed, 0, T, CH, m, k0=k0)
        ed = torch.from_numpy(eps).cuda()
        c, _ = g.rollout_costs(w.x0, U, 0, 0, noise=ed)
        c = c.cpu().numpy()
        same = np.array_equal(c.view(np.uint32), c_full[k0:k0 + CH].view(np.uint32))
        ok, ref = oracle.well_conditioned(pb, w.x0, w.U0, eps)
        err = np.abs(c - ref) / np.maximum(np.abs(ref), 1.0)
        bad = np.nonzero(ok & (err > 1e-4))[0]
        print("chunk %d: supplied-noise costs bitwise the C5 run's: %s; bad %s" % (ci, same, (bad + k0).tolist()))
        Ud = U.clone()
        gc.optimize(w.x0, Ud, 0, 0, noise=ed)
        ctg = gc.cost_to_go().cpu().numpy()          # [T][K]
        for j in bad:
            e1 = np.ascontiguousarray(eps[:, j:j + 1, :])
            q64 = oracle.rollout_stepcosts(pb, w.x0, w.U0, e1)[0]
            qa = oracle.rollout_stepcosts(pb, w.x0, w.U0, e1, mode="twin_f32")[0]
            qb = oracle.rollout_stepcosts(pb, w.x0, w.U0, e1, mode="twin_f32_via_f64")[0]
            s = ctg[:, j].astype(np.float64)
            qg = s - np.append(s[1:], 0.0)
            d = np.abs(qg - q64)
            first = int(np.argmax(d > 1e-3 * np.maximum(np.abs(q64), 1.0))) if np.any(d > 1e-3 * np.maximum(np.abs(q64), 1.0)) else -1
            xs = oracle.trajectory(pb, w.x0, w.U0, e1, 0)
            print("  k=%d: S gpu %.9g ctg0 %.9g fp64 %.9g twins %.9g %.9g rel err %.3g; crash margin %.3g; first "
                  "divergent step %d" % (k0 + j, c[j], s[0], ref[j], qa.sum(), qb.sum(), err[j],
                                         oracle.crash_margin(pb, w.x0, w.U0, e1)[0], first))
            lo = max(first - 3, 0) if first >= 0 else int(np.argmax(d))
            for t in range(lo, min(lo + 7, T)):
                print("    t=%3d q gpu %.6f fp64 %.6f twinA %.6f twinB %.6f | x_{t+1} fp64 %s"
                      % (t, qg[t], q64[t], qa[t], qb[t], xs[t + 1]))
    return 0


if __name__ == "__main__":
    sys.exit(main())
