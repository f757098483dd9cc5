// ============================================================================
// mppi_oracle.cpp — the fp64 CPU ORACLE for one MPPI optimisation step.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.
// It shares NO code, header, table or constant generator with the CUDA path
// (paper_1509_01149_b200/csrc/); neither side includes or links the other.
//
// What it computes (Williams, Aldrich & Theodorou, arXiv:1509.01149 = PAPER.md):
//   * Philox4x32-10 (Random123 definition) and the fixed fp32 Box-Muller
//     sequence "BM32" of SURVEY.md Appendix B: epsilon ~ N(0,1)
//   * delta_u = sqrt(nu) * L * eps, L = chol(Sigma_u)
//   * Euler rollouts x_{t+1} = x_t + F(x_t, U_t + du_t) dt
//   * augmented cost  q~ = q(x_{t+1}) + (1-1/nu)/2 du'R du + U'R du + 1/2 U'R U
//
//   * S_min, w_k = exp(-(S_k - S_min)/lambda), eta = sum w,
//     U_t += sum_k w_k du_{t,k} / eta
//   * shift U_i = U_{i+1}, U_{N-1} = u_init
// Plants: cart-pole (PAPER.md:395 + SURVEY A10), race car (PAPER.md:398 + SURVEY A11,
// Appendix A), quadrotor (PAPER.md:422, :431-433 + SURVEY A12/A13, Appendix A),
// linear test plant.
//
// Everything is plain: loops in the paper's order, fp64, no blocking, no fusion.
// The only fp32 arithmetic on the reference path is BM32, whose contract *is*
// an fp32 operation sequence.  The "conditioning twins" (mode 1/2)
// re-run the same plant/cost code in fp32 to flag ill-conditioned samples
// (SURVEY A19); they are diagnostics, never references.
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fopenmp -shared -fPIC
// (no -ffast-math: IEEE semantics are part of the contract).
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// ---------------------------------------------------------------------------
// Philox4x32-10, Random123 definition.
// round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
//        c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0);  key bumped by the
// Weyl constants before rounds 2..10.
// ---------------------------------------------------------------------------
const uint32_t PHILOX_M0 = 0xD2511F53u;
const uint32_t PHILOX_M1 = 0xCD9E8D57u;
const uint32_t PHILOX_W0 = 0x9E3779B9u;
const uint32_t PHILOX_W1 = 0xBB67AE85u;

void philox_round(uint32_t c[4], const uint32_t k[2]) {
    uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c[0];
    uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

void philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    philox_round(c, k);
    for (int r = 1; r < 10; ++r) {
        k[0] += PHILOX_W0;
        k[1] += PHILOX_W1;
        philox_round(c, k);
    }
    for (int i = 0; i < 4; ++i) out[i] = c[i];
}

// ---------------------------------------------------------------------------
// BM32: the fixed fp32 Box-Muller sequence of SURVEY Appendix B.  Every
// operation is one IEEE binary32 round-to-nearest operation; fmaf is a fused
// multiply-add; the file is compiled with -ffp-contract=off so the compiler
// cannot fuse anything else.
// ---------------------------------------------------------------------------
float f32(double v) { return (float)v; }  // fp32 rounding of a written fraction

// ln u1 with u1 = (2*(w>>9)+1) * 2^-24   (Appendix B "Radius", steps 1-6)
float bm_ln_u1(uint32_t w) {
    uint32_t N = 2u * (w >> 9) + 1u;                 // odd, < 2^24: u1 = N * 2^-24 exactly
    int e0 = 31 - __builtin_clz(N);                  // N = f0 * 2^e0, f0 in [1,2)
    float f0 = std::ldexp((float)N, -e0);            // exact: N has <= 24 significant bits
    int e;
    float f;
    const float SQRT2_F = 0x1.6a09e6p+0f;            // fp32 nearest sqrt(2), bits 0x3FB504F3
    if (f0 >= SQRT2_F) { e = e0 + 1; f = f0 * 0.5f; } else { e = e0; f = f0; }
    float k = (float)(e - 24);                       // u1 = f * 2^k
    float s = (f - 1.0f) / (f + 1.0f);               // f-1 exact (Sterbenz); IEEE divide
    float s2 = s * s;
    float p = f32(2.0 / 11.0);                       // Horner in s^2: 2/11, 2/9, 2/7, 2/5, 2/3
    p = std::fmaf(p, s2, f32(2.0 / 9.0));
    p = std::fmaf(p, s2, f32(2.0 / 7.0));
    p = std::fmaf(p, s2, f32(2.0 / 5.0));
    p = std::fmaf(p, s2, f32(2.0 / 3.0));
    float lnf = std::fmaf(s * s2, p, 2.0f * s);      // ln f = 2s + s^3 p(s^2)
    const float LN2_HI = 0.693145751953125f;         // bits 0x3F317200: k*LN2_HI exact
    const float LN2_LO = f32(1.428606820309417232e-06);
    return std::fmaf(k, LN2_HI, std::fmaf(k, LN2_LO, lnf));
}

// Radius r(w) = sqrt(-2 ln u1)   (Appendix B "Radius", step 7)
float bm_radius(uint32_t w) {
    return std::sqrt(-2.0f * bm_ln_u1(w));           // IEEE sqrt (correctly rounded)
}

// Angle theta(w) = 2*pi*(w>>8)/2^24; returns (sin theta, cos theta)   (Appendix B "Angle")
void bm_angle(uint32_t w, float* sin_out, float* cos_out) {
    uint32_t n = w >> 8;                             // 24-bit angle index
    uint32_t o = n >> 21;                            // octant 0..7
    uint32_t rho = n & ((1u << 21) - 1u);
    if (o & 1u) rho = (1u << 21) - rho;              // reflect inside odd octants
    float x = (float)rho * f32(M_PI / 8388608.0);    // pi/2^23 per index step; x in [0, pi/4]
    float x2 = x * x;
    float ps = f32(1.0 / 362880.0);                  // sin: Horner 1/9!, -1/7!, 1/5!, -1/3!
    ps = std::fmaf(ps, x2, f32(-1.0 / 5040.0));
    ps = std::fmaf(ps, x2, f32(1.0 / 120.0));
    ps = std::fmaf(ps, x2, f32(-1.0 / 6.0));
    float s = std::fmaf(x * x2, ps, x);
    float pc = f32(-1.0 / 3628800.0);                // cos: -1/10!, 1/8!, -1/6!, 1/4!, -1/2!
    pc = std::fmaf(pc, x2, f32(1.0 / 40320.0));
    pc = std::fmaf(pc, x2, f32(-1.0 / 720.0));
    pc = std::fmaf(pc, x2, f32(1.0 / 24.0));
    pc = std::fmaf(pc, x2, f32(-1.0 / 2.0));
    float c = std::fmaf(x2, pc, 1.0f);
    float sn, cs;
    switch (o) {                                     // octant map, Appendix B step 6
        case 0: sn = s;  cs = c;  break;
        case 1: sn = c;  cs = s;  break;
        case 2: sn = c;  cs = -s; break;
        case 3: sn = s;  cs = -c; break;
        case 4: sn = -s; cs = -c; break;
        case 5: sn = -c; cs = -s; break;
        case 6: sn = -c; cs = s;  break;
        default: sn = -s; cs = c; break;
    }
    *sin_out = sn;
    *cos_out = cs;
}

// z0 = r(w0) cos th(w1), z1 = r(w0) sin th(w1), z2 = r(w2) cos th(w3), z3 = r(w2) sin th(w3)
void bm_normals(const uint32_t w[4], float z[4]) {
    float s, c;
    float r0 = bm_radius(w[0]);
    bm_angle(w[1], &s, &c);
    z[0] = r0 * c;
    z[1] = r0 * s;
    float r1 = bm_radius(w[2]);
    bm_angle(w[3], &s, &c);
    z[2] = r1 * c;
    z[3] = r1 * s;
}

// eps[t][k][j] = z_j of Philox(ctr=(k_global, t, step_lo, step_hi), key=(seed_lo, seed_hi))
void noise_one(uint64_t seed, uint64_t step, uint32_t t, uint32_t k, float z[4]) {
    uint32_t ctr[4] = {k, t, (uint32_t)step, (uint32_t)(step >> 32)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t w[4];
    philox4x32_10(ctr, key, w);
    bm_normals(w, z);
}

// ---------------------------------------------------------------------------
// Scalar math used by the plants.  MathD = the fp64 reference; MathF and
// MathFviaD are the two fp32 conditioning twins.
// ---------------------------------------------------------------------------
struct MathD {
    typedef double S;
    static constexpr bool kFma = false;
    static S sin(S x) { return std::sin(x); }
    static S cos(S x) { return std::cos(x); }
    static S atan(S x) { return std::atan(x); }
    static S exp(S x) { return std::exp(x); }
    static S sqrt(S x) { return std::sqrt(x); }
};
struct MathF {  // twin 1: fp32 libm, plain operations (no contraction: -ffp-contract=off)
    typedef float S;
    static constexpr bool kFma = false;
    static S sin(S x) { return std::sin(x); }
    static S cos(S x) { return std::cos(x); }
    static S atan(S x) { return std::atan(x); }
    static S exp(S x) { return std::exp(x); }
    static S sqrt(S x) { return std::sqrt(x); }
};
// twin 2: fp32 state, transcendentals evaluated in fp64 then rounded, and
// explicit fmaf in the Euler and cost updates (kFma) -- a rounding sequence independent of
// twin 1's, so that the two twins sample the fp32 divergence of a rollout twice
struct MathFviaD {
    typedef float S;
    static constexpr bool kFma = true;
    static S sin(S x) { return (float)std::sin((double)x); }
    static S cos(S x) { return (float)std::cos((double)x); }
    static S atan(S x) { return (float)std::atan((double)x); }
    static S exp(S x) { return (float)std::exp((double)x); }
    static S sqrt(S x) { return std::sqrt(x); }
};

template <class S> S clampv(S v, S lo, S hi) { return v < lo ? lo : (v > hi ? hi : v); }

// a b + c: one fused rounding in twin 2 (M::kFma), the plain two roundings otherwise (the fp64
// reference and twin 1 keep their original operation sequence bit for bit)
template <class M>
typename M::S mad(typename M::S a, typename M::S b, typename M::S c) {
    if constexpr (M::kFma) return std::fma(a, b, c);
    else return a * b + c;
}

enum { PLANT_CARTPOLE = 1, PLANT_RACECAR = 2, PLANT_QUADROTOR = 3, PLANT_LINEAR = 4 };

}  // namespace

// Problem description shared with oracle.py (ctypes).  Parameter layouts per plant
// are documented in oracle.py (paper_params) and in oracle/README.md.
extern "C" typedef struct {
    int32_t plant;
    int32_t n;
    int32_t m;
    int32_t T;
    double dt;
    double lambda;
    double nu;
    const double* Sigma;      // m*m row-major, natural covariance of delta_u
    const double* R;          // m*m row-major control-cost matrix
    const double* params;     // plant + cost parameters (layout per plant)
    int32_t n_params;
    int32_t n_obstacles;
    const double* obstacles;  // n_obstacles*2 (x, y) cylinder centres (quadrotor)
    double penalty;           // cost of a non-finite rollout
    const double* At;         // optional [T][m][m] sampling transforms A_t (NEXT-3); null: sqrt(nu) I
} oracle_problem;

namespace {

// ---------------------------------------------------------------------------
// Plants.  deriv() returns F(x, v) = f + G v of the Euler step.
// ---------------------------------------------------------------------------

// Cart-pole.  PAPER.md:395: p'' = 10 (u - p'); pole per SURVEY A10 / SPEC.md:344:
// th'' = -(g/l) sin th - (p''/l) cos th, th = 0 hanging.
// params: [g, l, kv, w_p, w_theta, w_thetadot, w_pdot]
template <class M>
void cartpole_deriv(const double* P, const typename M::S* x, const typename M::S* v,
                    typename M::S* xd) {
    typedef typename M::S S;
    S g = (S)P[0], l = (S)P[1], kv = (S)P[2];
    S pdot = x[1], th = x[2], thdot = x[3];
    S pdd = kv * (v[0] - pdot);
    S thdd = -(g / l) * M::sin(th) - (pdd / l) * M::cos(th);
    xd[0] = pdot;
    xd[1] = pdd;
    xd[2] = thdot;
    xd[3] = thdd;
}
// q = p^2 + 500 (1 + cos th)^2 + th'^2 + p'^2
template <class M>
typename M::S cartpole_cost(const double* P, const typename M::S* x) {
    typedef typename M::S S;
    S c = (S)1 + M::cos(x[2]);
    if constexpr (M::kFma)
        return mad<M>((S)P[6] * x[1], x[1], mad<M>((S)P[5] * x[3], x[3], mad<M>((S)P[4] * c, c, (S)P[3] * x[0] * x[0])));
    return (S)P[3] * x[0] * x[0] + (S)P[4] * c * c + (S)P[5] * x[3] * x[3] +
           (S)P[6] * x[1] * x[1];
}

// Race car, single-track with Pacejka lateral tires.
// state [X, Y, psi, vx, vy, r]; control [delta, tau]
// params: [mass, Iz, lf, lr, B, C, mu, Cm, Cr, Cd, vmin, g, steer_max, thr_min, thr_max,
//          track_a, track_b, w_track, w_speed, v_ref]
template <class M>
void racecar_deriv(const double* P, const typename M::S* x, const typename M::S* v,
                   typename M::S* xd) {
    typedef typename M::S S;
    S mass = (S)P[0], Iz = (S)P[1], lf = (S)P[2], lr = (S)P[3], B = (S)P[4], C = (S)P[5];
    S mu = (S)P[6], Cm = (S)P[7], Cr = (S)P[8], Cd = (S)P[9], vmin = (S)P[10], g = (S)P[11];
    S delta = clampv<S>(v[0], -(S)P[12], (S)P[12]);
    S tau = clampv<S>(v[1], (S)P[13], (S)P[14]);
    S psi = x[2], vx = x[3], vy = x[4], r = x[5];
    S Df = mu * mass * g * lr / (lf + lr);
    S Dr = mu * mass * g * lf / (lf + lr);
    S vbar = vx > vmin ? vx : vmin;
    S alpha_f = delta - M::atan((vy + lf * r) / vbar);
    S alpha_r = -M::atan((vy - lr * r) / vbar);
    S Fyf = Df * M::sin(C * M::atan(B * alpha_f));
    S Fyr = Dr * M::sin(C * M::atan(B * alpha_r));
    S Fx = Cm * tau - Cr * vx - Cd * vx * std::fabs(vx);
    S cpsi = M::cos(psi), spsi = M::sin(psi);
    S cd = M::cos(delta), sd = M::sin(delta);
    xd[0] = vx * cpsi - vy * spsi;
    xd[1] = vx * spsi + vy * cpsi;
    xd[2] = r;
    xd[3] = (Fx - Fyf * sd) / mass + vy * r;
    xd[4] = (Fyr + Fyf * cd) / mass - vx * r;
    xd[5] = (lf * Fyf * cd - lr * Fyr) / Iz;
}
// q = 100 d^2 + (vx - 7)^2, d = |(x/13)^2 + (y/6)^2 - 1|
template <class M>
typename M::S racecar_cost(const double* P, const typename M::S* x) {
    typedef typename M::S S;
    S a = (S)P[15], b = (S)P[16];
    S ex = x[0] / a, ey = x[1] / b;
    S dv = x[3] - (S)P[19];
    if constexpr (M::kFma) {
        S d = std::fabs(mad<M>(ex, ex, mad<M>(ey, ey, -(S)1)));
        return mad<M>((S)P[18] * dv, dv, (S)P[17] * d * d);
    }
    S d = std::fabs(ex * ex + ey * ey - (S)1);
    return (S)P[17] * d * d + (S)P[18] * dv * dv;
}

// Quadrotor, GRASP structure.
// state [px,py,pz, vx,vy,vz, phi,theta,psi, p,q,r, F1..F4]; control: 4 thrust commands
// params: [mass, arm, Ixx, Iyy, Izz, gamma, km, g, umin, umax, cphi_min,
//          gx, gy, gz, w_xy, w_z, w_yaw, w_vel, w_obs, obs_len, w_crash, ground_z, radius]
template <class M>
void quad_deriv(const double* P, const typename M::S* x, const typename M::S* v,
                typename M::S* xd) {
    typedef typename M::S S;
    S mass = (S)P[0], L = (S)P[1], Ixx = (S)P[2], Iyy = (S)P[3], Izz = (S)P[4];
    S gam = (S)P[5], km = (S)P[6], g = (S)P[7], umin = (S)P[8], umax = (S)P[9];
    S cmin = (S)P[10];
    S phi = x[6], th = x[7], psi = x[8];
    S p = x[9], q = x[10], r = x[11];
    S F1 = x[12], F2 = x[13], F3 = x[14], F4 = x[15];
    S sph = M::sin(phi), cph = M::cos(phi);
    S sth = M::sin(th), cth = M::cos(th);
    S sps = M::sin(psi), cps = M::cos(psi);
    S a = (F1 + F2 + F3 + F4) / mass;
    xd[0] = x[3];
    xd[1] = x[4];
    xd[2] = x[5];
    // v' = (sum F / m) * R e3 - g e3, R = Rz(psi) Rx(phi) Ry(theta) (ZXY)
    xd[3] = a * (cps * sth + cth * sph * sps);
    xd[4] = a * (sps * sth - cps * cth * sph);
    xd[5] = a * (cph * cth) - g;
    // Euler-angle rates from body rates (ZXY), guarded |cos phi| >= cmin
    S chat = std::fabs(cph) > cmin ? std::fabs(cph) : cmin;
    chat = std::copysign(chat, cph);
    S psidot = (-sth * p + cth * r) / chat;
    xd[6] = cth * p + sth * r;
    xd[7] = q - sph * psidot;
    xd[8] = psidot;
    // I w' = tau - w x I w
    xd[9] = (L * (F2 - F4) - q * r * (Izz - Iyy)) / Ixx;
    xd[10] = (L * (F3 - F1) - r * p * (Ixx - Izz)) / Iyy;
    xd[11] = (gam * (F1 - F2 + F3 - F4) - p * q * (Iyy - Ixx)) / Izz;
    // rotor lag F_i' = km (u_i - F_i), u_i saturated to [umin, umax]
    for (int i = 0; i < 4; ++i) xd[12 + i] = km * (clampv<S>(v[i], umin, umax) - x[12 + i]);
}
// distance from (px, py) to the nearest cylinder surface, floored at 0
template <class M>
typename M::S quad_obstacle_distance(const oracle_problem* pb, const typename M::S* x) {
    typedef typename M::S S;
    S radius = (S)pb->params[22];
    S best = std::numeric_limits<S>::infinity();
    for (int j = 0; j < pb->n_obstacles; ++j) {
        S dx = x[0] - (S)pb->obstacles[2 * j];
        S dy = x[1] - (S)pb->obstacles[2 * j + 1];
        S d = M::sqrt(dx * dx + dy * dy) - radius;
        if (d < (S)0) d = (S)0;
        if (d < best) best = d;
    }
    return best;
}
// q = 2.5 dx^2 + 2.5 dy^2 + 150 dz^2 + 50 psi^2 + |v|^2 + 350 exp(-d/12) + 1000 C
template <class M>
typename M::S quad_cost(const double* P, const typename M::S* x, typename M::S d, int crashed) {
    typedef typename M::S S;
    S ex = x[0] - (S)P[11], ey = x[1] - (S)P[12], ez = x[2] - (S)P[13];
    if constexpr (M::kFma) {
        S q = mad<M>((S)P[15] * ez, ez, mad<M>((S)P[14] * ey, ey, (S)P[14] * ex * ex));
        q = mad<M>((S)P[16] * x[8], x[8], q);
        q = mad<M>((S)P[17], mad<M>(x[3], x[3], mad<M>(x[4], x[4], x[5] * x[5])), q);
        q = mad<M>((S)P[18], M::exp(-d / (S)P[19]), q);
        return q + (S)P[20] * (S)(crashed ? 1 : 0);
    }
    S q = (S)P[14] * ex * ex + (S)P[14] * ey * ey + (S)P[15] * ez * ez;
    q += (S)P[16] * x[8] * x[8];
    q += (S)P[17] * (x[3] * x[3] + x[4] * x[4] + x[5] * x[5]);
    q += (S)P[18] * M::exp(-d / (S)P[19]);
    q += (S)P[20] * (S)(crashed ? 1 : 0);
    return q;
}

// Linear test plant x' = A x + B v, q = x'Qx.  params: [A(nxn), B(nxm), Q(nxn)]
template <class M>
void linear_deriv(const oracle_problem* pb, const typename M::S* x, const typename M::S* v,
                  typename M::S* xd) {
    typedef typename M::S S;
    int n = pb->n, m = pb->m;
    const double* A = pb->params;
    const double* B = pb->params + n * n;
    for (int i = 0; i < n; ++i) {
        S acc = 0;
        for (int j = 0; j < n; ++j) acc += (S)A[i * n + j] * x[j];
        for (int j = 0; j < m; ++j) acc += (S)B[i * m + j] * v[j];
        xd[i] = acc;
    }
}
template <class M>
typename M::S linear_cost(const oracle_problem* pb, const typename M::S* x) {
    typedef typename M::S S;
    int n = pb->n;
    const double* Q = pb->params + n * n + n * pb->m;
    S acc = 0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) acc += x[i] * (S)Q[i * n + j] * x[j];
    return acc;
}

// One Euler step of the plant including the quadrotor crash freeze.
// Returns the state cost q(x_{t+1}).
template <class M>
typename M::S plant_step(const oracle_problem* pb, typename M::S* x, const typename M::S* v,
                         int* crashed) {
    typedef typename M::S S;
    S xd[16];
    S dt = (S)pb->dt;
    int n = pb->n;
    switch (pb->plant) {
        case PLANT_CARTPOLE:
            cartpole_deriv<M>(pb->params, x, v, xd);
            for (int i = 0; i < n; ++i) x[i] = mad<M>(xd[i], dt, x[i]);   // x + F dt
            return cartpole_cost<M>(pb->params, x);
        case PLANT_RACECAR:
            racecar_deriv<M>(pb->params, x, v, xd);
            for (int i = 0; i < n; ++i) x[i] = mad<M>(xd[i], dt, x[i]);   // x + F dt
            return racecar_cost<M>(pb->params, x);
        case PLANT_QUADROTOR: {
            if (!*crashed) {  // "the rollout stops simulating the dynamics" once C = 1
                quad_deriv<M>(pb->params, x, v, xd);
                for (int i = 0; i < n; ++i) x[i] = mad<M>(xd[i], dt, x[i]);   // x + F dt
            }
            S d = quad_obstacle_distance<M>(pb, x);
            if (x[2] <= (S)pb->params[21] || d <= (S)0) *crashed = 1;  // sticky
            return quad_cost<M>(pb->params, x, d, *crashed);
        }
        case PLANT_LINEAR:
        default:
            linear_deriv<M>(pb, x, v, xd);
            for (int i = 0; i < n; ++i) x[i] = mad<M>(xd[i], dt, x[i]);   // x + F dt
            return linear_cost<M>(pb, x);
    }
}

// Cholesky of an m x m SPD matrix (fp64).  Returns false if not SPD.
bool cholesky(const double* A, int m, double* L) {
    for (int i = 0; i < m * m; ++i) L[i] = 0.0;
    for (int j = 0; j < m; ++j) {
        double d = A[j * m + j];
        for (int k = 0; k < j; ++k) d -= L[j * m + k] * L[j * m + k];
        if (!(d > 0.0)) return false;
        L[j * m + j] = std::sqrt(d);
        for (int i = j + 1; i < m; ++i) {
            double s = A[i * m + j];
            for (int k = 0; k < j; ++k) s -= L[i * m + k] * L[j * m + k];
            L[i * m + j] = s / L[j * m + j];
        }
    }
    return true;
}

// Gauss-Jordan inverse of an m x m matrix (fp64, partial pivoting).  false if singular.
bool invert(const double* A, int m, double* Ai) {
    double a[16], b[16];
    for (int i = 0; i < m * m; ++i) { a[i] = A[i]; b[i] = 0.0; }
    for (int i = 0; i < m; ++i) b[i * m + i] = 1.0;
    for (int c = 0; c < m; ++c) {
        int p = c;
        for (int r = c + 1; r < m; ++r)
            if (std::fabs(a[r * m + c]) > std::fabs(a[p * m + c])) p = r;
        if (a[p * m + c] == 0.0) return false;
        for (int j = 0; j < m; ++j) { std::swap(a[c * m + j], a[p * m + j]); std::swap(b[c * m + j], b[p * m + j]); }
        const double d = a[c * m + c];
        for (int j = 0; j < m; ++j) { a[c * m + j] /= d; b[c * m + j] /= d; }
        for (int r = 0; r < m; ++r) {
            if (r == c) continue;
            const double f = a[r * m + c];
            for (int j = 0; j < m; ++j) { a[r * m + j] -= f * a[c * m + j]; b[r * m + j] -= f * b[c * m + j]; }
        }
    }
    for (int i = 0; i < m * m; ++i) Ai[i] = b[i];
    return true;
}

// Per-step sampling factor and importance-sampling matrix (NEXT-3, Theorem 1, PAPER.md:177-201,
// :271-284 in control coordinates with Eq. 7: Sigma~ = R^{-1}, Lambda~_t = A_t R^{-1} A_t^T):
//   du_t = F_t eps,  F_t = A_t L              (default A_t = sqrt(nu) I: F = sqrt(nu) L)
//   Gamma~_t^{-1} = R - A_t^{-T} R A_t^{-1}    (default: (1 - 1/nu) R)
bool step_matrices(const oracle_problem* pb, int t, const double* L, double* F, double* Gi) {
    const int m = pb->m;
    if (!pb->At) {
        const double s = std::sqrt(pb->nu);
        for (int i = 0; i < m * m; ++i) { F[i] = s * L[i]; Gi[i] = (1.0 - 1.0 / pb->nu) * pb->R[i]; }
        return true;
    }
    const double* A = pb->At + (size_t)t * m * m;
    double Ai[16];
    if (!invert(A, m, Ai)) return false;
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) {
            double f = 0.0;
            for (int k = 0; k < m; ++k) f += A[i * m + k] * L[k * m + j];
            F[i * m + j] = f;
            double g = 0.0;                       // (A^{-T} R A^{-1})_{ij}
            for (int k = 0; k < m; ++k)
                for (int l = 0; l < m; ++l) g += Ai[k * m + i] * pb->R[k * m + l] * Ai[l * m + j];
            Gi[i * m + j] = pb->R[i * m + j] - g;
        }
    return true;
}

// Neumaier-compensated running sum (for the k-ordered reductions of PAPER.md:320)
struct NeumaierSum {
    double s = 0.0, c = 0.0;
    void add(double v) {
        double t = s + v;
        if (std::fabs(s) >= std::fabs(v)) c += (s - t) + v; else c += (v - t) + s;
        s = t;
    }
    double value() const { return s + c; }
};

// One rollout of sample k.  eps row layout [T][K][m].  Returns S~_k.
template <class M>
double rollout_one(const oracle_problem* pb, const double* Lsc /* L = chol(Sigma_u) */,
                   const double* x0, const double* U, const float* eps, int64_t K, int64_t k,
                   int* crashed_out, double* qstep = nullptr /* [T]: q~ of each step, or null */) {
    typedef typename M::S S;
    const int n = pb->n, m = pb->m, T = pb->T;
    S x[16];
    for (int i = 0; i < n; ++i) x[i] = (S)x0[i];
    S Rt[16];
    for (int i = 0; i < m * m; ++i) Rt[i] = (S)pb->R[i];
    int crashed = 0;
    S Stilde = 0;
    for (int t = 0; t < T; ++t) {
        // F_t = A_t L, Gi_t = Gamma~_t^{-1}; special case A = sqrt(nu) I: F = sqrt(nu) L and
        // Gi = (1 - 1/nu) R, whose half is the (1 - 1/nu)/2 of PAPER.md:330
        double Fd[16], Gd[16];
        step_matrices(pb, t, Lsc, Fd, Gd);
        S Ft[16], Gt[16];
        for (int i = 0; i < m * m; ++i) { Ft[i] = (S)Fd[i]; Gt[i] = (S)Gd[i]; }
        const float* e = eps + ((int64_t)t * K + k) * m;
        S du[4], u[4], v[4];
        for (int i = 0; i < m; ++i) {                 // du = A_t L eps
            S acc = 0;
            for (int j = 0; j < m; ++j) acc = mad<M>(Ft[i * m + j], (S)e[j], acc);
            du[i] = acc;
            u[i] = (S)U[t * m + i];
            v[i] = u[i] + du[i];                      // u_i + du_{i,k}
        }
        S q = plant_step<M>(pb, x, v, &crashed);      // x_{t+1}, q(x_{t+1})
        S duGdu = 0, uRdu = 0, uRu = 0;
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) {
                duGdu = mad<M>(du[i] * Gt[i * m + j], du[j], duGdu);
                uRdu = mad<M>(u[i] * Rt[i * m + j], du[j], uRdu);
                uRu = mad<M>(u[i] * Rt[i * m + j], u[j], uRu);
            }
        // q~ = q + 1/2 du'Gamma~^{-1} du + u'R du + 1/2 u'R u
        S qt = q + (S)0.5 * duGdu + uRdu + (S)0.5 * uRu;
        Stilde += qt;                                 // S~ += q~  (no dt: A2)
        if (qstep) qstep[t] = (double)qt;
    }
    // phi(x_T) = 0 for all three tasks
    if (crashed_out) *crashed_out = crashed;
    double out = (double)Stilde;
    if (!std::isfinite(out)) out = pb->penalty;
    return out;
}

bool problem_ok(const oracle_problem* pb) {
    if (!pb || pb->n < 1 || pb->n > 16 || pb->m < 1 || pb->m > 4 || pb->T < 1) return false;
    if (!(pb->dt > 0) || !(pb->lambda > 0) || !(pb->nu >= 1)) return false;
    return true;
}

}  // namespace

// ============================================================================
// extern "C" entry points (ctypes, oracle/oracle.py)
// ============================================================================
extern "C" {

void oracle_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
    philox4x32_10(ctr, key, out);
}

float oracle_bm_radius(uint32_t w) { return bm_radius(w); }

void oracle_bm_angle(uint32_t w, float* s, float* c) { bm_angle(w, s, c); }

void oracle_bm_normals(const uint32_t* w, float* z) { bm_normals(w, z); }

// The same two functions over arrays of input words (for the exhaustive GPU comparison).
void oracle_bm_radius_words(const uint32_t* w, int64_t n, float* r) {
    for (int64_t i = 0; i < n; ++i) r[i] = bm_radius(w[i]);
}

void oracle_bm_angle_words(const uint32_t* w, int64_t n, float* s, float* c) {
    for (int64_t i = 0; i < n; ++i) bm_angle(w[i], &s[i], &c[i]);
}

// Exhaustive BM32 accuracy sweep (pin P2).  Over all 2^23 radius inputs: max ulp error
// of ln u1 and of r against fp64 libm; over all 2^24 angles: max |sin err|, |cos err|.
void oracle_bm_accuracy(double* max_ln_ulp, double* max_r_ulp, double* max_sin_err,
                        double* max_cos_err, double* max_abs_z) {
    double mln = 0, mr = 0, ms = 0, mc = 0, mz = 0;
    for (uint32_t i = 0; i < (1u << 23); ++i) {
        uint32_t w = i << 9;
        double u1 = (double)(2u * i + 1u) / 16777216.0;
        double lnu_ref = std::log(u1);
        double r_ref = std::sqrt(-2.0 * lnu_ref);
        float lnu = bm_ln_u1(w);
        float r = bm_radius(w);
        mln = std::max(mln, std::fabs((double)lnu - lnu_ref) /
                                std::ldexp(1.0, std::ilogb(lnu_ref) - 23));
        mr = std::max(mr, std::fabs((double)r - r_ref) / std::ldexp(1.0, std::ilogb(r_ref) - 23));
        mz = std::max(mz, (double)r);
    }
    for (uint32_t n = 0; n < (1u << 24); ++n) {
        float s, c;
        bm_angle(n << 8, &s, &c);
        double th = 2.0 * M_PI * (double)n / 16777216.0;
        ms = std::max(ms, std::fabs((double)s - std::sin(th)));
        mc = std::max(mc, std::fabs((double)c - std::cos(th)));
    }
    *max_ln_ulp = mln; *max_r_ulp = mr; *max_sin_err = ms; *max_cos_err = mc; *max_abs_z = mz;
}

// eps [T][Kn][m] for global samples k in [k0, k0+Kn) at (seed, step).  m <= 4.
int oracle_noise(uint64_t seed, uint64_t step, int32_t T, int64_t k0, int64_t Kn, int32_t m,
                 float* out) {
    if (T < 1 || Kn < 0 || m < 1 || m > 4 || !out) return 1;
    for (int32_t t = 0; t < T; ++t)
        for (int64_t kk = 0; kk < Kn; ++kk) {
            float z[4];
            noise_one(seed, step, (uint32_t)t, (uint32_t)(k0 + kk), z);
            for (int j = 0; j < m; ++j) out[((int64_t)t * Kn + kk) * m + j] = z[j];
        }
    return 0;
}

// F(x, v) of the plant (one call, fp64).  For tests of the plant equations.
int oracle_deriv(const oracle_problem* pb, const double* x, const double* v, double* xd) {
    if (!problem_ok(pb)) return 1;
    switch (pb->plant) {
        case PLANT_CARTPOLE: cartpole_deriv<MathD>(pb->params, x, v, xd); break;
        case PLANT_RACECAR: racecar_deriv<MathD>(pb->params, x, v, xd); break;
        case PLANT_QUADROTOR: quad_deriv<MathD>(pb->params, x, v, xd); break;
        default: linear_deriv<MathD>(pb, x, v, xd); break;
    }
    return 0;
}

// q(x) of the plant (fp64).  For the quadrotor, `crashed` is the indicator C.
double oracle_state_cost(const oracle_problem* pb, const double* x, int32_t crashed) {
    switch (pb->plant) {
        case PLANT_CARTPOLE: return cartpole_cost<MathD>(pb->params, x);
        case PLANT_RACECAR: return racecar_cost<MathD>(pb->params, x);
        case PLANT_QUADROTOR:
            return quad_cost<MathD>(pb->params, x, quad_obstacle_distance<MathD>(pb, x), crashed);
        default: return linear_cost<MathD>(pb, x);
    }
}

double oracle_obstacle_distance(const oracle_problem* pb, const double* x) {
    return quad_obstacle_distance<MathD>(pb, x);
}

// One Euler step x <- x + F(x, v) dt (quadrotor: crash freeze + sticky flag).  Returns q(x').
double oracle_plant_step(const oracle_problem* pb, double* x, const double* v, int32_t* crashed) {
    int c = crashed ? *crashed : 0;
    double q = plant_step<MathD>(pb, x, v, &c);
    if (crashed) *crashed = c;
    return q;
}

// Per-sample augmented costs S~_k for samples k in [0, K) of eps [T][K][m].
// mode 0 = fp64 reference; 1 = fp32 twin (libm float); 2 = fp32 twin (fp64 transcendentals).
// nthreads <= 0: all OpenMP threads.  Returns 0 ok, 1 bad problem, 2 Sigma not SPD.
int oracle_rollout_costs(const oracle_problem* pb, const double* x0, const double* U,
                         const float* eps, int64_t K, int32_t mode, int32_t nthreads,
                         double* costs, int32_t* crashed) {
    if (!problem_ok(pb) || K < 0) return 1;
    double L[16];
    if (!cholesky(pb->Sigma, pb->m, L)) return 2;
    if (pb->At) {
        double F[16], G[16];
        for (int t = 0; t < pb->T; ++t)
            if (!step_matrices(pb, t, L, F, G)) return 3;       // singular A_t
    }
    const double* Lsc = L;
#ifdef _OPENMP
    int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel for num_threads(nt) schedule(static)
#endif
    for (int64_t k = 0; k < K; ++k) {
        int c = 0;
        double Sk;
        if (mode == 1) Sk = rollout_one<MathF>(pb, Lsc, x0, U, eps, K, k, &c);
        else if (mode == 2) Sk = rollout_one<MathFviaD>(pb, Lsc, x0, U, eps, K, k, &c);
        else Sk = rollout_one<MathD>(pb, Lsc, x0, U, eps, K, k, &c);
        costs[k] = Sk;
        if (crashed) crashed[k] = c;
    }
    return 0;
}

// The reduction and update of PAPER.md:318-321 / Alg. 1 :366-368, given costs S~_k.
//   S_min = min_k S~_k, k* = smallest k attaining it; w_k = exp(-(S~_k - S_min)/lambda);
//   eta = sum_k w_k; U_t += sum_k w_k du_{t,k} / eta with du = sqrt(nu) L eps.
// Sums run in increasing k with Neumaier compensation.  weights_out (optional, K) gets w_k.
int oracle_update(const oracle_problem* pb, const double* costs, const float* eps, int64_t K,
                  double* U, int64_t* kstar_out, double* smin_out, double* eta_out,
                  double* weights_out) {
    if (!problem_ok(pb) || K < 1) return 1;
    const int m = pb->m, T = pb->T;
    double L[16];
    if (!cholesky(pb->Sigma, m, L)) return 2;
    double smin = costs[0];
    int64_t kstar = 0;
    for (int64_t k = 1; k < K; ++k)
        if (costs[k] < smin) { smin = costs[k]; kstar = k; }
    std::vector<double> w(K);
    NeumaierSum eta;
    for (int64_t k = 0; k < K; ++k) {
        w[k] = std::exp(-(costs[k] - smin) / pb->lambda);
        eta.add(w[k]);
    }
    const double etav = eta.value();
    for (int t = 0; t < T; ++t) {
        double F[16], G[16];
        step_matrices(pb, t, L, F, G);
        for (int i = 0; i < m; ++i) {
            NeumaierSum num;
            for (int64_t k = 0; k < K; ++k) {
                const float* e = eps + ((int64_t)t * K + k) * m;
                double du = 0.0;                       // du = A_t L eps (default sqrt(nu) L eps)
                for (int j = 0; j < m; ++j) du += F[i * m + j] * (double)e[j];
                num.add(w[k] * du);
            }
            U[t * m + i] += num.value() / etav;
        }
    }
    if (kstar_out) *kstar_out = kstar;
    if (smin_out) *smin_out = smin;
    if (eta_out) *eta_out = etav;
    if (weights_out) for (int64_t k = 0; k < K; ++k) weights_out[k] = w[k];
    return 0;
}

// Per-step augmented costs q~_{t,k} (fp64), out[k*T + t].  For the cost-to-go weighting.
int oracle_rollout_stepcosts(const oracle_problem* pb, const double* x0, const double* U,
                             const float* eps, int64_t K, int32_t nthreads, double* out, int32_t mode) {
    if (!problem_ok(pb) || K < 0) return 1;
    double L[16];
    if (!cholesky(pb->Sigma, pb->m, L)) return 2;
    const double* Lsc = L;
#ifdef _OPENMP
    int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel for num_threads(nt) schedule(static)
#endif
    for (int64_t k = 0; k < K; ++k) {
        int c = 0;   // mode as oracle_rollout_costs: 0 fp64, 1 / 2 the fp32 conditioning twins
        if (mode == 1) rollout_one<MathF>(pb, Lsc, x0, U, eps, K, k, &c, out + k * pb->T);
        else if (mode == 2) rollout_one<MathFviaD>(pb, Lsc, x0, U, eps, K, k, &c, out + k * pb->T);
        else rollout_one<MathD>(pb, Lsc, x0, U, eps, K, k, &c, out + k * pb->T);
    }
    return 0;
}

// PAPER.md:320 / Alg. 1 :367 literally: per timestep i the weights use the cost-to-go
//   S~(tau_{i,k}) = sum_{j >= i} q~_{j,k}      ("from time t_i onward"; phi = 0)
//   w_{i,k} = exp(-(S~_{i,k} - min_k S~_{i,k}) / lambda),  eta_i = sum_k w_{i,k},
//   U_i += sum_k w_{i,k} du_{i,k} / eta_i.
// stepcosts[k*T + t] = q~_{t,k}; a non-finite cost-to-go is charged the penalty.
// smin_out (optional, T) and eta_out (optional, T).  Sums in increasing k, Neumaier.
int oracle_update_ctg(const oracle_problem* pb, const double* stepcosts, const float* eps,
                      int64_t K, double* U, double* smin_out, double* eta_out) {
    if (!problem_ok(pb) || K < 1) return 1;
    const int m = pb->m, T = pb->T;
    double L[16];
    if (!cholesky(pb->Sigma, m, L)) return 2;
    std::vector<double> ctg((size_t)K * T);
    for (int64_t k = 0; k < K; ++k) {
        NeumaierSum acc;
        for (int t = T - 1; t >= 0; --t) {
            acc.add(stepcosts[k * T + t]);
            double v = acc.value();
            ctg[(size_t)k * T + t] = std::isfinite(v) ? v : pb->penalty;
        }
    }
    for (int t = 0; t < T; ++t) {
        double smin = ctg[t];
        for (int64_t k = 1; k < K; ++k) smin = std::min(smin, ctg[(size_t)k * T + t]);
        std::vector<double> w(K);
        NeumaierSum eta;
        for (int64_t k = 0; k < K; ++k) {
            w[k] = std::exp(-(ctg[(size_t)k * T + t] - smin) / pb->lambda);
            eta.add(w[k]);
        }
        double F[16], G[16];
        step_matrices(pb, t, L, F, G);
        for (int i = 0; i < m; ++i) {
            NeumaierSum num;
            for (int64_t k = 0; k < K; ++k) {
                const float* e = eps + ((int64_t)t * K + k) * m;
                double du = 0.0;
                for (int j = 0; j < m; ++j) du += F[i * m + j] * (double)e[j];
                num.add(w[k] * du);
            }
            U[t * m + i] += num.value() / eta.value();
        }
        if (smin_out) smin_out[t] = smin;
        if (eta_out) eta_out[t] = eta.value();
    }
    return 0;
}

// Full step: costs then update (fp64 reference).
int oracle_optimize(const oracle_problem* pb, const double* x0, double* U, const float* eps,
                    int64_t K, int32_t nthreads, double* costs, int64_t* kstar, double* eta) {
    int rc = oracle_rollout_costs(pb, x0, U, eps, K, 0, nthreads, costs, nullptr);
    if (rc) return rc;
    return oracle_update(pb, costs, eps, K, U, kstar, nullptr, eta, nullptr);
}

// Alg. 1 shift: u_i = u_{i+1} for i < N-1, u_{N-1} = u_init.
void oracle_shift(double* U, int32_t T, int32_t m, const double* u_init) {
    for (int t = 0; t + 1 < T; ++t)
        for (int i = 0; i < m; ++i) U[t * m + i] = U[(t + 1) * m + i];
    for (int i = 0; i < m; ++i) U[(T - 1) * m + i] = u_init[i];
}

// Decision margins of each sample (conditioning filter): the fp64 rollout of sample k; at every
// step up to and including the first crash (C = 1 once the vehicle touches the
// ground or a cylinder), the distance of a decision from its threshold.  mode 0 (crash, DESIGN.md
// reading A19'): min(|z - ground_z|, |surface distance to the nearest cylinder|) -- a sample whose
// margin is below the fp32 trajectory error can legitimately crash one step earlier or later in
// an fp32 rollout; mode 1 (Euler guard, A19''): |cos phi|.  Plants other than the quadrotor:
// +inf.  Returns 0 ok.
static int decision_margin(const oracle_problem* pb, const double* x0, const double* U,
                           const float* eps, int64_t K, int32_t nthreads, double* margin, int mode) {
    if (!problem_ok(pb) || K < 0) return 1;
    double L[16];
    if (!cholesky(pb->Sigma, pb->m, L)) return 2;
#ifdef _OPENMP
    int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel for num_threads(nt) schedule(static)
#endif
    for (int64_t k = 0; k < K; ++k) {
        double mk = std::numeric_limits<double>::infinity();
        if (pb->plant == PLANT_QUADROTOR) {
            const int n = pb->n, m = pb->m;
            double x[16];
            for (int i = 0; i < n; ++i) x[i] = x0[i];
            int crashed = 0;
            for (int t = 0; t < pb->T && !crashed; ++t) {
                const float* e = eps + ((int64_t)t * K + k) * m;
                double F[16], G[16];
                step_matrices(pb, t, L, F, G);
                double v[4];
                for (int i = 0; i < m; ++i) {
                    double du = 0;
                    for (int j = 0; j < m; ++j) du += F[i * m + j] * (double)e[j];
                    v[i] = U[t * m + i] + du;
                }
                plant_step<MathD>(pb, x, v, &crashed);
                double mt = std::fabs(x[2] - pb->params[21]);
                for (int j = 0; j < pb->n_obstacles; ++j) {
                    const double dx = x[0] - pb->obstacles[2 * j], dy = x[1] - pb->obstacles[2 * j + 1];
                    mt = std::min(mt, std::fabs(std::sqrt(dx * dx + dy * dy) - pb->params[22]));
                }
                if (mode == 1) mt = std::fabs(std::cos(x[6]));   // Euler-guard margin (A19'')
                if (!std::isfinite(mt)) mt = 0.0;          // a diverged state: no margin
                mk = std::min(mk, mt);
            }
        }
        margin[k] = mk;
    }
    return 0;
}

int oracle_crash_margin(const oracle_problem* pb, const double* x0, const double* U,
                        const float* eps, int64_t K, int32_t nthreads, double* margin) {
    return decision_margin(pb, x0, U, eps, K, nthreads, margin, 0);
}

// Euler-guard margin of each sample (conditioning filter, reading A19''): the ZXY
// Euler-angle rate psi' = (-sin th p + cos th r) / cos phi is singular at cos phi = 0 (gimbal
// lock); reading A12 guards the divisor as sign(cos phi) max(|cos phi|, cphi_min), so inside the
// band |cos phi| < cphi_min the rate is decided by the SIGN of cos phi (a discontinuity) and the
// trajectory chatters across it.  Returns, per sample, min over the steps up to and including
// the first crash of |cos phi_{t+1}| of the fp64 rollout (+inf for the other plants).
int oracle_euler_margin(const oracle_problem* pb, const double* x0, const double* U,
                        const float* eps, int64_t K, int32_t nthreads, double* margin) {
    return decision_margin(pb, x0, U, eps, K, nthreads, margin, 1);
}

// States of one rollout (for plots/debugging): xs [T+1][n], with the sample's eps column.
int oracle_trajectory(const oracle_problem* pb, const double* x0, const double* U,
                      const float* eps, int64_t K, int64_t k, double* xs) {
    if (!problem_ok(pb)) return 1;
    double L[16];
    if (!cholesky(pb->Sigma, pb->m, L)) return 2;
    const int n = pb->n, m = pb->m;
    double x[16];
    for (int i = 0; i < n; ++i) { x[i] = x0[i]; xs[i] = x[i]; }
    int crashed = 0;
    for (int t = 0; t < pb->T; ++t) {
        const float* e = eps + ((int64_t)t * K + k) * m;
        double F[16], G[16];
        step_matrices(pb, t, L, F, G);
        double v[4];
        for (int i = 0; i < m; ++i) {
            double du = 0;
            for (int j = 0; j < m; ++j) du += F[i * m + j] * (double)e[j];
            v[i] = U[t * m + i] + du;
        }
        plant_step<MathD>(pb, x, v, &crashed);
        for (int i = 0; i < n; ++i) xs[(t + 1) * n + i] = x[i];
    }
    return 0;
}

}  // extern "C"
