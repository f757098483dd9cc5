"""Pins P3 for the oracle's plants and state costs: the worked values SPEC.md prints
(hand-checked in SURVEY §4), plus closed forms and invariants that a dropped term,
wrong sign or transposed index would break."""
import math

import numpy as np
import pytest


def P(oracle, plant, **kw):
    m = oracle.CONTROL_DIM[plant]
    args = dict(T=5, dt=0.02, lam=5e-3, nu=1.0, Sigma=np.eye(m) * 0.005, R=np.eye(m))
    args.update(kw)
    return oracle.Problem(plant, **args)


# ----------------------------------------------------------------------------- cart-pole
def test_cartpole_costs_spec_examples(oracle):
    pb = P(oracle, "cartpole")
    assert oracle.state_cost(pb, [0, 0, math.pi, 0]) == pytest.approx(0.0, abs=1e-20)
    assert oracle.state_cost(pb, [0, 0, 0, 0]) == 2000.0
    assert oracle.state_cost(pb, [1, 2, math.pi, 3]) == pytest.approx(14.0, abs=1e-12)


def test_cartpole_dynamics_spec_examples(oracle):
    pb = P(oracle, "cartpole")
    assert np.all(oracle.deriv(pb, [0, 0, 0, 0], [0]) == 0)
    xd = oracle.deriv(pb, [0, 0, math.pi, 0], [0])
    assert abs(xd[3]) < 1e-14
    xd = oracle.deriv(pb, [0, 0, math.pi / 2, 0], [0])
    assert xd[3] == pytest.approx(-9.81, abs=1e-12)
    # PAPER.md:395 p'' = 10 (u - p'): Euler step from rest with u = 1, dt = 0.02 -> p' = 0.2
    x, q, _ = oracle.plant_step(pb, [0, 0, 0, 0], [1.0])
    assert x[1] == pytest.approx(0.2, abs=1e-15)
    assert x[0] == 0.0
    # pole couples to cart acceleration with -cos(theta)/l: hanging pole swings back when the cart accelerates
    xd = oracle.deriv(pb, [0, 0, 0, 0], [1.0])
    assert xd[1] == 10.0 and xd[3] == pytest.approx(-10.0)


def test_cartpole_rollout_from_rest(oracle):
    """U = 0, du = 0 from hanging rest -> q = 2000 every step, S~ = 2000 T."""
    T = 7
    pb = P(oracle, "cartpole", T=T, nu=3.0)
    eps = np.zeros((T, 3, 1), np.float32)
    costs = oracle.rollout_costs(pb, [0, 0, 0, 0], np.zeros((T, 1)), eps)
    assert np.all(costs == 2000.0 * T)


# ----------------------------------------------------------------------------- race car
def test_racecar_costs_spec_examples(oracle):
    pb = P(oracle, "racecar")
    assert oracle.state_cost(pb, [13, 0, 0, 7, 0, 0]) == 0.0
    assert oracle.state_cost(pb, [0, 0, 0, 7, 0, 0]) == 100.0
    assert oracle.state_cost(pb, [13, 0, 0, 0, 0, 0]) == 49.0
    # d is symmetric in x and y and lies on the ellipse at (0, 6)
    a = oracle.state_cost(pb, [3.0, -2.0, 0, 7, 0, 0])
    assert a == oracle.state_cost(pb, [-3.0, -2.0, 0, 7, 0, 0]) == oracle.state_cost(pb, [3.0, 2.0, 0, 7, 0, 0])
    assert oracle.state_cost(pb, [0, 6, 0, 7, 0, 0]) == 0.0


def test_racecar_straight_line(oracle):
    """coasting straight with zero steer -> no lateral/yaw acceleration; only
    drag decelerates: vx' = (-Cr vx - Cd vx|vx|)/m."""
    pb = P(oracle, "racecar")
    xd = oracle.deriv(pb, [0, 0, 0.3, 5.0, 0, 0], [0, 0])
    assert xd[4] == 0.0 and xd[5] == 0.0
    assert xd[3] == pytest.approx((-1.0 * 5 - 0.8 * 25) / 21.88, rel=1e-14)
    assert xd[0] == pytest.approx(5 * math.cos(0.3)) and xd[1] == pytest.approx(5 * math.sin(0.3))


def test_racecar_terminal_speed(oracle):
    """full throttle from rest accelerates monotonically to the drag balance
    Cm = Cr v + Cd v^2 -> v* = (-Cr + sqrt(Cr^2 + 4 Cd Cm)) / (2 Cd)."""
    pb = P(oracle, "racecar")
    x = np.zeros(6)
    prev = -1
    for _ in range(3000):
        x, _, _ = oracle.plant_step(pb, x, [0.0, 1.0])
        assert x[3] >= prev
        prev = x[3]
    vstar = (-1.0 + math.sqrt(1.0 + 4 * 0.8 * 100.0)) / (2 * 0.8)
    assert x[3] == pytest.approx(vstar, rel=1e-6)


def test_racecar_kinematic_limit(oracle):
    """small steering at low speed -> yaw rate ~ vx tan(delta)/(lf+lr) within 10 %."""
    pb = P(oracle, "racecar")
    v, delta = 2.0, 0.05
    tau = (1.0 * v + 0.8 * v * v) / 100.0
    x = np.array([0, 0, 0, v, 0, 0], float)
    for _ in range(1000):
        x, _, _ = oracle.plant_step(pb, x, [delta, tau])
    kin = x[3] * math.tan(delta) / (0.34 + 0.23)
    assert abs(x[5] / kin - 1) < 0.10


def test_racecar_saturation(oracle):
    """steering saturates at +-0.6 rad and throttle at [-1, 1] inside F."""
    pb = P(oracle, "racecar")
    x = [1.0, 2.0, 0.1, 6.0, 0.3, 0.2]
    assert np.array_equal(oracle.deriv(pb, x, [5.0, 3.0]), oracle.deriv(pb, x, [0.6, 1.0]))
    assert np.array_equal(oracle.deriv(pb, x, [-5.0, -3.0]), oracle.deriv(pb, x, [-0.6, -1.0]))


# ----------------------------------------------------------------------------- quadrotor
HOVER = 0.5 * 9.81 / 4


def quad_state(pos=(0, 0, 2), vel=(0, 0, 0), ang=(0, 0, 0), rates=(0, 0, 0), F=(HOVER,) * 4):
    return np.array(list(pos) + list(vel) + list(ang) + list(rates) + list(F), float)


def test_quad_hover_equilibrium(oracle):
    pb = P(oracle, "quadrotor")
    xd = oracle.deriv(pb, quad_state(), [HOVER] * 4)
    assert np.max(np.abs(xd)) < 1e-15


def test_quad_free_fall_and_rotor_lag(oracle):
    pb = P(oracle, "quadrotor")
    xd = oracle.deriv(pb, quad_state(F=(0, 0, 0, 0)), [0, 0, 0, 0])
    assert xd[5] == -9.81 and xd[3] == 0 and xd[4] == 0
    # F_i' = km (sat(u_i) - F_i) with saturation to [0, 4]
    xd = oracle.deriv(pb, quad_state(F=(1, 1, 1, 1)), [10.0, -3.0, 2.0, 1.0])
    assert np.allclose(xd[12:], [20 * 3, 20 * -1, 20 * 1, 0])


def test_quad_torques(oracle):
    """I w' = [L(F2-F4), L(F3-F1), gamma(F1-F2+F3-F4)] - w x I w."""
    pb = P(oracle, "quadrotor")
    h = HOVER
    xd = oracle.deriv(pb, quad_state(F=(h, h + 0.1, h, h)), [h] * 4)
    assert xd[9] == pytest.approx(0.175 * 0.1 / 2.32e-3)
    assert xd[10] == 0 and xd[11] == pytest.approx(-0.0245 * 0.1 / 4.0e-3)
    xd = oracle.deriv(pb, quad_state(F=(h, h, h + 0.1, h)), [h] * 4)
    assert xd[10] == pytest.approx(0.175 * 0.1 / 2.32e-3)
    # gyroscopic coupling: with p, r != 0 and Ixx == Iyy only q' picks up r p (Ixx - Izz)/Iyy
    xd = oracle.deriv(pb, quad_state(rates=(1.0, 0.0, 2.0)), [h] * 4)
    assert xd[9] == 0 and xd[11] == 0
    assert xd[10] == pytest.approx(-2.0 * 1.0 * (2.32e-3 - 4.0e-3) / 2.32e-3)


def _rot_zxy(phi, th, psi):
    cz, sz, cx, sx, cy, sy = (math.cos(psi), math.sin(psi), math.cos(phi), math.sin(phi),
                              math.cos(th), math.sin(th))
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]])
    Rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    return Rz @ Rx @ Ry


def test_quad_attitude_kinematics_against_rotation_matrices(oracle):
    """Independent check of the ZXY Euler-rate and thrust-direction equations: the angle
    rates the oracle returns must satisfy dR/dt = R [w]_x for R = Rz(psi) Rx(phi) Ry(theta),
    and v' = (sum F/m) R e3 - g e3 (finite differences of explicit rotation matrices)."""
    pb = P(oracle, "quadrotor")
    rng = np.random.default_rng(0)
    for _ in range(20):
        ang = rng.uniform(-0.6, 0.6, 3)
        w = rng.uniform(-2, 2, 3)
        F = rng.uniform(0.5, 2.0, 4)
        x = quad_state(ang=ang, rates=w, F=F)
        xd = oracle.deriv(pb, x, F)
        rates = xd[6:9]
        h = 1e-6
        R = _rot_zxy(*ang)
        dR = (_rot_zxy(*(ang + h * rates)) - _rot_zxy(*(ang - h * rates))) / (2 * h)
        W = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
        assert np.allclose(dR, R @ W, atol=1e-7)
        acc = F.sum() / 0.5 * R[:, 2] - np.array([0, 0, 9.81])
        assert np.allclose(xd[3:6], acc, rtol=1e-12, atol=1e-12)


def test_quad_costs_spec_examples(oracle):
    goal = quad_state(pos=(50, 0, 2))
    pb = P(oracle, "quadrotor")                      # no obstacles: d = +inf
    assert oracle.state_cost(pb, goal, 0) == 0.0
    assert oracle.state_cost(pb, goal, 1) == 1000.0
    pb = P(oracle, "quadrotor", obstacles=[[50.0, 12.5]])   # surface distance exactly 12
    assert oracle.obstacle_distance(pb, goal) == 12.0
    assert oracle.state_cost(pb, goal, 0) == pytest.approx(350 * math.exp(-1))           # 128.76
    assert oracle.state_cost(pb, goal, 0) == pytest.approx(128.76, abs=5e-3)
    # each weighted term of PAPER.md:431 separately
    pb = P(oracle, "quadrotor")
    assert oracle.state_cost(pb, quad_state(pos=(51, 0, 2)), 0) == 2.5
    assert oracle.state_cost(pb, quad_state(pos=(50, -1, 2)), 0) == 2.5
    assert oracle.state_cost(pb, quad_state(pos=(50, 0, 3)), 0) == 150.0
    assert oracle.state_cost(pb, quad_state(pos=(50, 0, 2), ang=(0.3, 0.2, 1.0)), 0) == 50.0
    assert oracle.state_cost(pb, quad_state(pos=(50, 0, 2), vel=(1, 2, 2)), 0) == 9.0


def test_quad_obstacle_distance(oracle):
    pb = P(oracle, "quadrotor", obstacles=[[3.0, 4.0], [10.0, 0.0], [-1.0, -1.0]])
    assert oracle.obstacle_distance(pb, quad_state(pos=(0, 0, 2))) == pytest.approx(math.sqrt(2) - 0.5)
    assert oracle.obstacle_distance(pb, quad_state(pos=(3.2, 4.0, 2))) == 0.0   # inside -> 0
    pb = P(oracle, "quadrotor", obstacles=[[3.0, 4.0]])
    assert oracle.obstacle_distance(pb, quad_state(pos=(0, 0, 2))) == 4.5


def test_quad_crash_freeze(oracle):
    """after C = 1 the rollout stops simulating and the vehicle remains where it
    is; the frozen state keeps being charged, including 1000 C, every step."""
    T = 40
    pb = P(oracle, "quadrotor", T=T)
    x0 = quad_state(pos=(0, 0, 0.05), F=(0, 0, 0, 0))
    U = np.zeros((T, 4))
    eps = np.zeros((T, 1, 4), np.float32)
    xs = oracle.trajectory(pb, x0, U, eps, 0)
    crash_t = int(np.argmax(xs[:, 2] <= 0.0))
    assert crash_t > 0
    assert np.all(xs[crash_t:] == xs[crash_t])
    costs, crashed = oracle.rollout_costs(pb, x0, U, eps, return_crashed=True)
    assert crashed[0] == 1
    frozen_q = oracle.state_cost(pb, xs[crash_t], 1)
    assert frozen_q >= 1000.0
    tail = (T - crash_t + 1) * frozen_q
    head = sum(oracle.state_cost(pb, xs[t], 0) for t in range(1, crash_t))
    assert costs[0] == pytest.approx(head + tail, rel=1e-12)
    # crashing into a cylinder also freezes
    pb = P(oracle, "quadrotor", T=T, obstacles=[[0.6, 0.0]])
    x0 = quad_state(vel=(2.0, 0, 0))
    xs = oracle.trajectory(pb, x0, np.full((T, 4), HOVER), eps, 0)
    c = int(np.argmax(xs[:, 0] >= 0.1))
    assert c > 0 and np.all(xs[c:] == xs[c])


def test_quad_crash_margin_closed_form(oracle):
    """Reading A19' filter: free fall from z0 with zero thrust (explicit Euler: z_t = z0 -
    g dt^2 t(t-1)/2) beside a cylinder at horizontal surface distance s: the margin is the
    smaller of s and the closest approach of z_t to the ground up to the first crash."""
    T, dt, g = 60, 0.02, 9.81
    z0, s = 1.0, 0.37
    pb = P(oracle, "quadrotor", T=T, obstacles=[[0.5 + s, 0.0]])
    x0 = quad_state(pos=(0, 0, z0), F=(0, 0, 0, 0))
    U = np.zeros((T, 4))
    eps = np.zeros((T, 1, 4), np.float32)
    t = np.arange(1, T + 1)
    z = z0 - g * dt * dt * t * (t - 1) / 2
    first = int(np.argmax(z <= 0.0))
    want = min(s, float(np.min(np.abs(z[:first + 1]))))
    assert oracle.crash_margin(pb, x0, U, eps)[0] == pytest.approx(want, rel=1e-9)
    # the ground margin alone (cylinder far away), and +inf for another plant
    pb = P(oracle, "quadrotor", T=T, obstacles=[[40.0, 0.0]])
    assert oracle.crash_margin(pb, x0, U, eps)[0] == pytest.approx(float(np.min(np.abs(z[:first + 1]))), rel=1e-9)
    pc = P(oracle, "cartpole", T=5)
    assert np.isinf(oracle.crash_margin(pc, [0, 0, 0, 0], np.zeros((5, 1)), np.zeros((5, 1, 1), np.float32))[0])


# ----------------------------------------------------------------------------- linear
def test_linear_plant(oracle):
    A = np.array([[0.0, 1.0], [-2.0, -0.5]])
    B = np.array([[0.0], [1.0]])
    Q = np.array([[3.0, 0.5], [0.5, 1.0]])
    pb = oracle.Problem("linear", T=3, dt=0.1, lam=1.0, nu=1.0, Sigma=[[1.0]], R=[[1.0]],
                        params=np.concatenate([A.ravel(), B.ravel(), Q.ravel()]), n=2, m=1)
    x = np.array([0.3, -0.7])
    assert np.allclose(oracle.deriv(pb, x, [2.0]), A @ x + B @ [2.0])
    x1, q, _ = oracle.plant_step(pb, x, [2.0])
    assert np.allclose(x1, x + 0.1 * (A @ x + B @ [2.0]))
    assert q == pytest.approx(x1 @ Q @ x1)


def test_quad_euler_margin_closed_form(oracle):
    """Reading A19'' filter: a constant roll rate p with equal thrusts and theta = r = 0 keeps every
    other rate zero, so explicit Euler gives phi_t = t p dt exactly up to rounding and the margin is
    min_{t=1..T} |cos(t p dt)| (no crash: z0 high, thrust at hover).  Choosing p dt = (pi/2)/k
    puts step k on the singularity (margin ~ 0)."""
    T, dt = 40, 0.02
    pb = P(oracle, "quadrotor", T=T, obstacles=[[40.0, 0.0]])
    U = np.full((T, 4), HOVER)
    eps = np.zeros((T, 1, 4), np.float32)
    for prate in (3.1, 5.0, -7.3):
        x0 = quad_state(pos=(0, 0, 50.0), rates=(prate, 0, 0))
        t = np.arange(1, T + 1)
        want = float(np.min(np.abs(np.cos(t * prate * dt))))
        assert oracle.euler_margin(pb, x0, U, eps)[0] == pytest.approx(want, rel=1e-9, abs=1e-14)
    x0 = quad_state(pos=(0, 0, 50.0), rates=(math.pi / 2 / (7 * dt), 0, 0))
    assert oracle.euler_margin(pb, x0, U, eps)[0] < 1e-12
    pc = P(oracle, "cartpole", T=5)
    assert np.isinf(oracle.euler_margin(pc, [0, 0, 0, 0], np.zeros((5, 1)), np.zeros((5, 1, 1), np.float32))[0])


def test_perturb_ulp_moves_every_element_by_one_ulp(oracle):
    """The third conditioning twin's input: every element exactly one ulp away (up or down), a
    fixed function of the element's own bits (so chunking the columns does not change it), both
    directions used."""
    e = oracle.noise(3, 0, 7, 301, 4)
    p = oracle.perturb_ulp(e)
    assert p.dtype == np.float32 and p.shape == e.shape
    up = np.nextafter(e, np.float32(np.inf))
    dn = np.nextafter(e, np.float32(-np.inf))
    assert np.all((p == up) | (p == dn)) and np.all(p != e)
    frac_up = np.mean(p == up)
    assert 0.4 < frac_up < 0.6
    assert np.array_equal(oracle.perturb_ulp(e[:, 100:200]), p[:, 100:200])


def test_twin2_uses_fused_updates_and_twins_stay_close(oracle):
    """twin 2 runs the Euler and cost updates with fmaf, so its rounding sequence
    differs from twin 1's (not bitwise equal on a tumbling quadrotor batch) while both stay
    within the fp32 resolution of fp64 on well-behaved samples; the fp64 reference is unchanged by
    the twins' code (its pins elsewhere stay exact)."""
    T = 60
    pb = P(oracle, "quadrotor", T=T, nu=50.0, obstacles=[[3.0, 0.5], [-2.0, 4.0]])
    x0 = quad_state()
    U = np.full((T, 4), HOVER)
    eps = oracle.noise(11, 0, T, 512, 4)
    ref = oracle.rollout_costs(pb, x0, U, eps)
    a = oracle.rollout_costs(pb, x0, U, eps, "twin_f32")
    b = oracle.rollout_costs(pb, x0, U, eps, "twin_f32_via_f64")
    assert not np.array_equal(a, b)
    ok = oracle.well_conditioned(pb, x0, U, eps, ref_costs=ref)[0]
    assert ok.mean() > 0.9
    rel = np.abs(np.stack([a, b]) - ref) / np.maximum(np.abs(ref), 1.0)
    assert rel[:, ok].max() <= 1e-5
