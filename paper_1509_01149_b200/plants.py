"""Plant / cost parameter defaults of the three paper tasks and their C-ABI structs.

Product-side defaults, written from the paper (PAPER.md line cited per field) and the
readings of SURVEY.md §8.3 / Appendix A where the paper is silent.  The oracle keeps its
own independent copy (oracle/oracle.py::paper_params); parity tests catch any drift.
"""
import ctypes as C
import math

import numpy as np

from . import _capi as A

PLANTS = {"cartpole": A.MPPI_PLANT_CARTPOLE, "racecar": A.MPPI_PLANT_RACECAR,
          "quadrotor": A.MPPI_PLANT_QUADROTOR, "linear": A.MPPI_PLANT_LINEAR}
STATE_DIM = {"cartpole": 4, "racecar": 6, "quadrotor": 16}
CONTROL_DIM = {"cartpole": 1, "racecar": 2, "quadrotor": 4}

DEFAULT_DYNAMICS = {
    # PAPER.md:395 "p'' = 10(u - p')"; pole g, l: SURVEY A10
    "cartpole": dict(g=9.81, pole_length=1.0, vel_gain=10.0),
    # SURVEY Appendix A (the paper's tire model [HindThesis] is unavailable)
    "racecar": dict(mass=21.88, Iz=1.6, lf=0.34, lr=0.23, tire_B=4.0, tire_C=1.5, mu=0.9,
                    Cm=100.0, Cr=1.0, Cd=0.8, v_min=2.0, g=9.81, steer_max=0.6,
                    throttle_min=-1.0, throttle_max=1.0),
    # SURVEY Appendix A / A12 (GRASP quadrotor [michael2010grasp])
    "quadrotor": dict(mass=0.5, arm=0.175, Ixx=2.32e-3, Iyy=2.32e-3, Izz=4.0e-3,
                      yaw_coeff=0.0245, motor_gain=20.0, g=9.81, thrust_min=0.0,
                      thrust_max=4.0, cos_phi_min=0.05),
}

DEFAULT_COST = {
    # q = p^2 + 500(1 + cos th)^2 + th'^2 + p'^2
    "cartpole": dict(w_p=1.0, w_theta=500.0, w_thetadot=1.0, w_pdot=1.0),
    # q = 100 d^2 + (vx - 7)^2, d = |(x/13)^2 + (y/6)^2 - 1|
    "racecar": dict(track_a=13.0, track_b=6.0, w_track=100.0, w_speed=1.0, v_ref=7.0),
    # 2.5 dx^2 + 2.5 dy^2 + 150 dz^2 + 50 psi^2 + |v|^2 + 350 exp(-d/12) + 1000 C;
    # goal and radius: SURVEY A13 / Appendix A
    "quadrotor": dict(goal=(50.0, 0.0, 2.0), w_xy=2.5, w_z=150.0, w_yaw=50.0, w_vel=1.0,
                      w_obs=350.0, obs_length=12.0, w_crash=1000.0, ground_z=0.0,
                      obstacle_radius=0.5),
}


class PlantSpec:
    """Builds (and keeps alive) the mppi_dynamics_t / mppi_cost_t structs of one plant."""

    def __init__(self, plant, dynamics=None, cost=None, obstacles=None, penalty=1e30,
                 linear=None):
        self.name = plant
        self.plant = PLANTS[plant]
        self.dyn = A.dynamics_t()
        self.dyn.struct_size = C.sizeof(A.dynamics_t)
        self.dyn.plant = self.plant
        self.cost = A.cost_t()
        self.cost.struct_size = C.sizeof(A.cost_t)
        self.cost.penalty = penalty
        self._obs = None
        if plant == "linear":
            # linear = dict(A=[n][n], B=[n][m], Q=[n][n])
            Am = np.asarray(linear["A"], np.float32)
            Bm = np.asarray(linear["B"], np.float32)
            Qm = np.asarray(linear["Q"], np.float32)
            n, m = Bm.shape
            self.n, self.m = n, m
            d = self.dyn.p.linear
            d.n = n
            for i, v in enumerate(Am.ravel()):
                d.A[i] = float(v)
            for i, v in enumerate(Bm.ravel()):
                d.B[i] = float(v)
            for i, v in enumerate(Qm.ravel()):
                self.cost.p.linear.Q[i] = float(v)
            return
        self.n, self.m = STATE_DIM[plant], CONTROL_DIM[plant]
        dd = dict(DEFAULT_DYNAMICS[plant])
        dd.update(dynamics or {})
        dstruct = getattr(self.dyn.p, plant)
        for k, v in dd.items():
            setattr(dstruct, k, float(v))
        cc = dict(DEFAULT_COST[plant])
        cc.update(cost or {})
        cstruct = getattr(self.cost.p, plant)
        for k, v in cc.items():
            if k == "goal":
                for i in range(3):
                    cstruct.goal[i] = float(v[i])
            else:
                setattr(cstruct, k, float(v))
        if plant == "quadrotor":
            obs = np.zeros((0, 2), np.float32) if obstacles is None else \
                np.ascontiguousarray(np.asarray(obstacles, np.float32).reshape(-1, 2))
            self._obs = obs
            cstruct.n_obstacles = len(obs)
            cstruct.obstacles_xy = obs.ctypes.data_as(C.POINTER(C.c_float)) if len(obs) else None
