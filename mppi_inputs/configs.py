"""BASELINE.json configs C1-C5 made concrete (SURVEY.md §8.4 "Concrete synthetic inputs").

Shared inputs only: sizes, initial state x0, initial control sequence U0, the
sampling covariance Sigma_u, control cost R, temperature lambda, variance scale
nu and the Philox seed.  Values and their sources:
  * dt = 0.02 (50 Hz); cart-pole horizon 1 s -> T = 50
  * 1/sqrt(rho) = 0.01, R = 1 -> natural du covariance
    Sigma_u = 1/(rho dt) = 0.005 per channel
  * lambda = R/(rho dt) = 5e-3 (noise/cost coupling)
  * nu: 1 (C1), 1000 (C2, PAPER.md:396 range 1..1500), 150 (C3, PAPER.md:402 range
    50..300), 10 (C4/C5)
"""
from dataclasses import dataclass, field
import math

import numpy as np

from .forest import forest_4m


@dataclass
class Workload:
    name: str
    plant: str
    K: int
    T: int
    dt: float
    nu: float
    lam: float
    Sigma: np.ndarray
    R: np.ndarray
    x0: np.ndarray
    U0: np.ndarray
    seed: int = 1
    step: int = 0
    steps: int = 1                 # receding-horizon steps (C2)
    obstacles: np.ndarray = field(default_factory=lambda: np.zeros((0, 2), np.float32))
    description: str = ""

    @property
    def m(self):
        return self.U0.shape[1]

    @property
    def n(self):
        return self.x0.shape[0]


def _f32(a):
    return np.asarray(a, np.float32)


def cartpole(K, T, nu, steps=1, name="cartpole"):
    return Workload(name=name, plant="cartpole", K=K, T=T, dt=0.02, nu=nu, lam=5e-3,
                    Sigma=np.eye(1) * 0.005, R=np.eye(1),
                    x0=_f32([0, 0, 0, 0]),           # hanging at rest (theta = 0)
                    U0=np.zeros((T, 1), np.float32), steps=steps,
                    description="cart-pole swing-up from hanging rest")


def racecar(K=16384, T=150, nu=150.0):
    return Workload(name="racecar", plant="racecar", K=K, T=T, dt=0.02, nu=nu, lam=5e-3,
                    Sigma=np.eye(2) * 0.005, R=np.eye(2),
                    # on the ellipse at (13, 0), heading +y (counter-clockwise), 7 m/s
                    x0=_f32([13.0, 0.0, math.pi / 2, 7.0, 0.0, 0.0]),
                    U0=np.tile(_f32([0.0, 0.5]), (T, 1)),
                    description="race car on the 13 x 6 m elliptical track")


HOVER = 0.5 * 9.81 / 4.0   # mg/4 with m = 0.5 kg


def quadrotor(K=65536, T=200, nu=10.0, name="quadrotor"):
    f = forest_4m()
    x0 = np.zeros(16, np.float32)
    x0[2] = 2.0
    x0[12:16] = HOVER
    return Workload(name=name, plant="quadrotor", K=K, T=T, dt=0.02, nu=nu, lam=5e-3,
                    Sigma=np.eye(4) * 0.005, R=np.eye(4), x0=x0,
                    U0=np.full((T, 4), HOVER, np.float32),
                    obstacles=_f32(f["centers"]).reshape(-1, 2),
                    description="quadrotor through the 4 m cylinder forest to (50, 0, 2)")


CONFIGS = {
    "C1": lambda: cartpole(256, 50, 1.0, name="C1-cartpole-step"),
    "C2": lambda: cartpole(4096, 100, 1000.0, steps=200, name="C2-cartpole-closed-loop"),
    "C3": lambda: racecar(),
    "C4": lambda: quadrotor(),
    "C5": lambda: quadrotor(K=1 << 22, name="C5-quadrotor-sweep"),
}


def get(name, **overrides):
    w = CONFIGS[name]()
    for k, v in overrides.items():
        setattr(w, k, v)
    if "T" in overrides and w.U0.shape[0] != w.T:
        w.U0 = np.resize(w.U0, (w.T, w.U0.shape[1])).astype(np.float32)
    return w
