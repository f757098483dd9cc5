"""Cylinder forest for the quadrotor task ("randomly generated three
forests ... 3 / 4 / 5 meters apart"; SURVEY.md Appendix A "Forest").

Jittered grid: one cylinder per cell of side `spacing` over x in [x0, x1],
y in [y0, y1]; centre jitter uniform in +-40 % of the cell; cylinders whose
surface is closer than `clearance` to the start or goal are dropped.  Seeded and
deterministic.  The 4 m forest used by configs C4/C5 is committed as
forest_4m.json (regenerate with `python -m mppi_inputs.forest`).
"""
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
FOREST_4M = os.path.join(HERE, "forest_4m.json")


def generate_forest(spacing=4.0, x_range=(5.0, 45.0), y_range=(-10.0, 10.0), radius=0.5,
                    jitter=0.4, clearance=1.5, start=(0.0, 0.0), goal=(50.0, 0.0), seed=4):
    rng = np.random.default_rng(seed)
    nx = int(round((x_range[1] - x_range[0]) / spacing))
    ny = int(round((y_range[1] - y_range[0]) / spacing))
    out = []
    for i in range(nx):
        for j in range(ny):
            cx = x_range[0] + (i + 0.5) * spacing + rng.uniform(-jitter, jitter) * spacing
            cy = y_range[0] + (j + 0.5) * spacing + rng.uniform(-jitter, jitter) * spacing
            ok = True
            for px, py in (start, goal):
                if np.hypot(cx - px, cy - py) - radius < clearance:
                    ok = False
            if ok:
                out.append((float(np.float32(cx)), float(np.float32(cy))))
    return {"spacing": spacing, "radius": radius, "seed": seed, "centers": out}


def forest_4m():
    """The committed 4 m forest: dict(spacing, radius, seed, centers=[(x, y), ...])."""
    with open(FOREST_4M) as f:
        d = json.load(f)
    d["centers"] = [tuple(c) for c in d["centers"]]
    return d


if __name__ == "__main__":
    d = generate_forest()
    with open(FOREST_4M, "w") as f:
        json.dump(d, f, indent=1)
    print(len(d["centers"]), "cylinders ->", FOREST_4M)
