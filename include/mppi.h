/*
 * mppi.h — C ABI of libmppi_b200.so: one Model Predictive Path Integral (MPPI)
 * optimisation step on an NVIDIA B200 (sm_100a), after
 *   G. Williams, A. Aldrich, E. Theodorou, "Model Predictive Path Integral Control
 *   using Covariance Variable Importance Sampling", arXiv:1509.01149.
 *
 * The step (Algorithm 1; update law Eq. App_PI, :318-321):
 *   1. draw eps[t][k] ~ N(0, I_m)
 *   2. du[t][k] = sqrt(nu) * L * eps[t][k], L = chol(Sigma) (PAPER.md:308 A = sqrt(nu) I, :312)
 *   3. roll out x_{t+1} = x_t + F(x_t, U_t + du_t) * dt
 *      accumulating S~_k = sum_t q~ with
 *      q~ = q(x_{t+1}) + (1 - 1/nu)/2 du'R du + U_t'R du + 1/2 U_t'R U_t
 *   4. S_min = min_k S~_k, w_k = exp(-(S~_k - S_min)/lambda), eta = sum_k w_k
 *   5. U_t += sum_k w_k du[t][k] / eta
 *
 * Conventions for every entry point:
 *   - Device pointers are CUDA global-memory addresses on the context's device; host
 *     pointers are ordinary CPU memory.  Each argument says which.
 *   - Every call is ASYNCHRONOUS on the context's stream unless stated otherwise:
 *     MPPI_OK means "validated and enqueued".  Errors of kernels already enqueued
 *     surface as MPPI_ERR_CUDA on a later call.
 *   - A context is single-owner and not thread-safe: one call at a time.
 *   - Floating-point buffers are fp32, row-major, densely packed.
 *   - Layouts: U is [T][m]; eps (noise) is [T][K_loc][m] (sample-contiguous rows so that
 *     per-timestep reads across samples coalesce); costs is [K_loc].
 *   - On error the call returns a non-zero status, enqueues nothing, and
 *     mppi_last_error() returns a thread-local description.
 *   - There is no CPU fallback: without a usable CUDA device mppi_create fails with
 *     MPPI_ERR_CUDA.
 */
#ifndef MPPI_B200_H
#define MPPI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPPI_ABI_VERSION 1

typedef enum {
    MPPI_OK = 0,
    MPPI_ERR_INVALID_ARG = 1,  /* bad size, pointer, non-finite or out-of-range scalar */
    MPPI_ERR_NOT_SPD = 2,      /* Sigma or R is not symmetric positive definite (fp64 Cholesky) */
    MPPI_ERR_OOM = 3,          /* device or pinned-host allocation failed */
    MPPI_ERR_CUDA = 4,         /* CUDA runtime error (no device, launch failure, async fault) */
    MPPI_ERR_NCCL = 5,         /* NCCL unavailable or a collective failed */
    MPPI_ERR_UNSUPPORTED = 6   /* valid request outside what this build implements */
} mppi_status_t;

typedef enum {
    MPPI_PLANT_CARTPOLE = 1,   /* PAPER.md:395 (§V-A); n = 4, m = 1 */
    MPPI_PLANT_RACECAR = 2,    /* PAPER.md:398 (§V-B); n = 6, m = 2 */
    MPPI_PLANT_QUADROTOR = 3,  /* PAPER.md:422, :431-433 (§V-C); n = 16, m = 4 */
    MPPI_PLANT_LINEAR = 4      /* linear test plant x' = A x + B v, q = x'Qx; n <= 8, m <= 4 */
} mppi_plant_t;

/* ---------------------------------------------------------------- dynamics (F of the Euler step) */

/* Cart-pole, state [p, p', theta, theta'], control u = desired cart velocity.
 * p'' = vel_gain (u - p')                            (vel_gain = 10)
 * theta'' = -(g/l) sin theta - (p''/l) cos theta,  theta = 0 hanging */
typedef struct {
    float g;             /* 9.81 */
    float pole_length;   /* 1.0 */
    float vel_gain;      /* 10.0 */
} mppi_cartpole_dynamics_t;

/* Race car, state [X, Y, psi, vx, vy, r], control [delta (steer, rad), tau (throttle)].
 * Single-track model with Pacejka lateral tires (the paper's
 * [HindThesis] model is unavailable).  delta and tau saturate inside F.
 *   D_f = mu m g lr/(lf+lr), D_r = mu m g lf/(lf+lr), vbar = max(vx, v_min)
 *   alpha_f = delta - atan((vy + lf r)/vbar), alpha_r = -atan((vy - lr r)/vbar)
 *   F_yf = D_f sin(C atan(B alpha_f)), F_yr = D_r sin(C atan(B alpha_r))
 *   F_x  = Cm tau - Cr vx - Cd vx|vx|
 *   X' = vx cos psi - vy sin psi, Y' = vx sin psi + vy cos psi, psi' = r
 *   vx' = (F_x - F_yf sin delta)/m + vy r, vy' = (F_yr + F_yf cos delta)/m - vx r
 *   r'  = (lf F_yf cos delta - lr F_yr)/Iz */
typedef struct {
    float mass, Iz, lf, lr;
    float tire_B, tire_C, mu;
    float Cm, Cr, Cd;
    float v_min, g;
    float steer_max;                 /* |delta| <= steer_max */
    float throttle_min, throttle_max;
} mppi_racecar_dynamics_t;

/* Quadrotor, state [p(3), v(3), phi, theta, psi (ZXY Euler), p, q, r (body rates),
 * F1..F4 (rotor thrusts)], control = 4 thrust commands saturated to [thrust_min, thrust_max].
 * GRASP structure:
 *   v' = (sum F / mass) R(phi,theta,psi) e3 - g e3,  R = Rz(psi) Rx(phi) Ry(theta)
 *   phi' = c_th p + s_th r;  psi' = (-s_th p + c_th r)/chat, chat = copysign(max(|c_phi|, cos_phi_min), c_phi)
 *   theta' = q - s_phi psi'
 *   I w' = [arm (F2 - F4), arm (F3 - F1), yaw_coeff (F1 - F2 + F3 - F4)] - w x I w
 *   F_i' = motor_gain (sat(u_i) - F_i) */
typedef struct {
    float mass, arm;
    float Ixx, Iyy, Izz;
    float yaw_coeff, motor_gain, g;
    float thrust_min, thrust_max;
    float cos_phi_min;
} mppi_quadrotor_dynamics_t;

/* Linear test plant: x' = A x + B v, A [n][n], B [n][m] row-major. */
typedef struct {
    int32_t n;           /* 1..8 */
    float A[64];
    float B[32];
} mppi_linear_dynamics_t;

typedef struct {
    uint32_t struct_size;            /* sizeof(mppi_dynamics_t) */
    mppi_plant_t plant;
    union {
        mppi_cartpole_dynamics_t cartpole;
        mppi_racecar_dynamics_t racecar;
        mppi_quadrotor_dynamics_t quadrotor;
        mppi_linear_dynamics_t linear;
    } p;
} mppi_dynamics_t;

/* ---------------------------------------------------------------- state cost q(x) */

/* q = w_p p^2 + w_theta (1 + cos theta)^2 + w_thetadot theta'^2 + w_pdot p'^2
 * (paper: 1, 500, 1, 1) */
typedef struct {
    float w_p, w_theta, w_thetadot, w_pdot;
} mppi_cartpole_cost_t;

/* q = w_track d^2 + w_speed (vx - v_ref)^2, d = |(X/a)^2 + (Y/b)^2 - 1|
 * (paper: 100, 1, v_ref = 7, a = 13, b = 6) */
typedef struct {
    float track_a, track_b;
    float w_track, w_speed, v_ref;
} mppi_racecar_cost_t;

/* q = w_xy((px-gx)^2 + (py-gy)^2) + w_z (pz-gz)^2 + w_yaw psi^2 + w_vel |v|^2
 *                 + w_obs exp(-d / obs_length) + w_crash C
 * (paper: 2.5, 150, 50, 1, 350, 12, 1000).  d = distance from (px, py) to the nearest
 * cylinder surface, max(0, |p - c_j| - obstacle_radius); d = +inf with no
 * obstacles.  C = 1 once pz <= ground_z or d <= 0; C is sticky and freezes the state for the
 * rest of the rollout; the frozen state keeps being charged every step.
 * w_xy and w_z must be >= 0 (INVALID_ARG otherwise: the rollout folds sqrt(w) into the
 * position differences). */
typedef struct {
    float goal[3];
    float w_xy, w_z, w_yaw, w_vel;
    float w_obs, obs_length, w_crash;
    float ground_z;
    float obstacle_radius;           /* one radius for every cylinder */
    int32_t n_obstacles;             /* 0..MPPI_MAX_OBSTACLES */
    const float* obstacles_xy;       /* HOST [n_obstacles][2] cylinder centres; copied at create */
} mppi_quadrotor_cost_t;

#define MPPI_MAX_OBSTACLES 4096

/* Linear test plant: q = x'Q x, Q [n][n] row-major. */
typedef struct {
    float Q[64];
} mppi_linear_cost_t;

typedef struct {
    uint32_t struct_size;            /* sizeof(mppi_cost_t) */
    float penalty;                   /* S~_k of a rollout whose cost is not finite; e.g. 1e30 */
    union {
        mppi_cartpole_cost_t cartpole;
        mppi_racecar_cost_t racecar;
        mppi_quadrotor_cost_t quadrotor;
        mppi_linear_cost_t linear;
    } p;
} mppi_cost_t;

/* ---------------------------------------------------------------- sharding across GPUs */

/* K is split into world contiguous shards; rank r owns global samples
 * [r*K/world, (r+1)*K/world).  Noise counters use the GLOBAL sample index, so the union of
 * the shards' noise equals the single-GPU noise bit for bit.  The two
 * cross-rank reductions (MIN of the cost key, SUM of [eta, A]) are done by the caller
 * between the split-phase calls below (e.g. NCCL allreduce via torch.distributed). */
typedef struct {
    int32_t rank;
    int32_t world;
} mppi_dist_t;

typedef struct mppi_ctx mppi_ctx;

typedef struct {
    int32_t n, m, T;
    int32_t plant;
    int64_t K;                       /* global sample count */
    int64_t K_loc;                   /* samples of this rank */
    int64_t k_offset;                /* first global sample of this rank */
    int32_t n_chunks;                /* K-chunks of the weighted-noise reduction (partials rows) */
    int32_t reserved;
    size_t workspace_bytes;          /* device memory owned by the context */
} mppi_info_t;

/* Host-readable summary of the last completed step (see mppi_get_stats). */
typedef struct {
    int64_t k_star;                  /* global index of the minimum-cost sample (ties: smallest k) */
    float s_min;                     /* S_min = S~_{k*} */
    float eta;                       /* normaliser sum_k exp(-(S~_k - S_min)/lambda) (global after apply) */
} mppi_stats_t;

/* ---------------------------------------------------------------- lifecycle */

/* mppi_create — Alg. 1 "Given" block.
 *   dynamics, cost : HOST structs, copied (obstacles too).  cost->penalty must be finite.
 *   K              : global number of samples, >= 1; K_loc = K/world must be an integer
 *                    multiple of 4 (16-byte aligned noise rows).
 *   T              : horizon steps, 1..4096 (a non-diagonal Sigma or R keeps two m x m matrices
 *                    per step in shared memory: INVALID_ARG when they no longer fit, T > ~1200
 *                    at m = 4).
 *   dt             : Euler step > 0.
 *   lambda         : temperature > 0.
 *   nu             : exploration variance scale >= 1 (PAPER.md:308; Gamma invertible, :197).
 *   m              : control dimension; must equal the plant's (1, 2, 4, or 1..4 for LINEAR).
 *   Sigma          : HOST fp64 [m][m], the natural covariance of delta-u (PAPER.md:312:
 *                    du = eps/(sqrt(rho) sqrt(dt)) -> Sigma = I/(rho dt) in the special case).
 *                    The sampling covariance is nu*Sigma.  Factored in fp64 (Cholesky), used as fp32.
 *   R              : HOST fp64 [m][m] SPD control-cost matrix.
 *   dist           : HOST, NULL for a single GPU.
 *   cuda_stream    : cudaStream_t (NULL = legacy default stream) on the current device; all
 *                    work of this context is enqueued on it.
 *   out            : receives the context.
 * Synchronous.  Allocates the workspace (noise [T][K_loc][m], costs, reduction partials).
 * Errors: INVALID_ARG, NOT_SPD, OOM, CUDA. */
mppi_status_t mppi_create(const mppi_dynamics_t* dynamics, const mppi_cost_t* cost, int64_t K,
                          int32_t T, float dt, float lambda, float nu, int32_t m,
                          const double* Sigma, const double* R, const mppi_dist_t* dist,
                          void* cuda_stream, mppi_ctx** out);

/* Frees the context after synchronising its stream.  NULL is a no-op. */
void mppi_destroy(mppi_ctx* ctx);

mppi_status_t mppi_info(const mppi_ctx* ctx, mppi_info_t* out /* HOST */);

/* Changes the stream later calls enqueue on (e.g. torch's current stream). */
mppi_status_t mppi_set_stream(mppi_ctx* ctx, void* cuda_stream);

/* ---------------------------------------------------------------- the step */

/* mppi_optimize — one full MPPI step.  world == 1, or world > 1 with a communicator attached by
 * mppi_nccl_attach (else UNSUPPORTED; the split-phase calls below work without one):
 *   noise -> rollout -> min -> weights + weighted noise sum -> U update.
 * Kernels: K1 noise (or drawn inside K2, MPPI_OPTION_FUSED_NOISE), K2 rollout (+ CTA min and
 * int64 atomicMin of the (cost, k) key), K3 weights + weighted noise sum per chunk, K4 fixed-order
 * chunk sum and update; with a communicator the two allreduces sit between K2/K3 and K3/K4.
 *   x0    : HOST float [n], the current state x_{t0}; read before return (passed by value).
 *   U     : DEVICE float [T][m], the nominal control sequence, updated in place.
 *   seed, step : Philox key and counter words; eps[t][k][j] = j-th normal of
 *           Philox4x32-10(ctr = (k, t, step_lo, step_hi), key = (seed_lo, seed_hi)) transformed
 *           by the fixed fp32 Box-Muller sequence of SURVEY.md Appendix B.
 *   noise : NULL -> generate eps as above into the context; otherwise DEVICE float [T][K][m]
 *           of N(0,1) samples supplied by the caller (seed/step ignored), read-only.
 * Errors: INVALID_ARG (NULL U, non-finite x0), UNSUPPORTED (world > 1 without a communicator),
 * NCCL, CUDA. */
mppi_status_t mppi_optimize(mppi_ctx* ctx, const float* x0, float* U, uint64_t seed,
                            uint64_t step, const float* noise);

/* mppi_use_graph — mppi_optimize replays the step as one CUDA graph (default: enabled): built on
 * the first call of each noise mode, later calls only update the kernel-node arguments (x0,
 * seed, step, U, noise).  Results are identical to direct launches.  While per-kernel profiling
 * is enabled (mppi_profile_enable) kernels are launched directly. */
mppi_status_t mppi_use_graph(mppi_ctx* ctx, int32_t enable);

typedef enum {
    MPPI_OPTION_CUDA_GRAPH = 1,        /* same as mppi_use_graph (default 1) */
    MPPI_OPTION_PACKED_SAMPLES = 2,    /* quadrotor, K_loc >= 65536: two samples per thread with FP32x2
                                          arithmetic (diagonal or general Sigma / A_t; the general
                                          variant needs the obstacle grid) (default 1); bitwise
                                          identical results */
    MPPI_OPTION_FUSED_NOISE = 3,       /* when the library draws the noise and K_loc >= 65536: the
                                          rollout kernel draws it itself (same counters,
                                          bit-identical values, still written to the context's noise
                                          buffer for the reduction) instead of a separate noise
                                          pass (default 1) */
    MPPI_OPTION_OBSTACLE_GRID = 4,     /* quadrotor: the nearest cylinder is searched among a per-cell
                                          candidate list (host-built at create, see
                                          mppi_obstacle_grid) instead of all cylinders, when the
                                          grid fits in shared memory beside the horizon's per-step
                                          records; bitwise identical results (default 1) */
    MPPI_OPTION_BULK_REDUCTION = 5,    /* K_loc >= 65536: the weighted-noise reductions (trajectory and
                                          cost-to-go weights) stream their tiles through a shared-
                                          memory ring filled by bulk copies (cp.async.bulk +
                                          mbarrier) instead of per-thread loads; identical results
                                          (default 1) */
    MPPI_OPTION_PDL = 6,               /* the step's CUDA graph links its kernels with programmatic
                                          (dependent-launch) edges: a kernel's CTAs launch as the
                                          previous kernel's last CTAs exit and wait
                                          (griddepcontrol.wait) for its results; identical results.
                                          Default 0: on B200 it saves 1.3-1.5 us of p50 latency at
                                          C1-C3 but adds 1-5 us at p99 (profiles/r2_ab_latency_pdl.txt,
                                          scripts/ab_latency.py, 4 x 200 calls per setting) */
    MPPI_OPTION_SPARSE_REDUCTION = 7,  /* with the bulk-copy reduction (K_loc >= 65536, trajectory
                                          weights): a pass over the costs flags the 256-column
                                          blocks holding a nonzero fp32 weight and the
                                          weighted noise sum streams only those (zero weights add
                                          exact zeros: identical results).  With small lambda the
                                          weights are nearly one-hot (C1-C5: one nonzero weight), and
                                          the reduction then reads kilobytes instead of 4 T K m bytes.
                                          Default 0: bench.py measures the dense GEMV the north_star
                                          defines and reports this mode beside it */
    MPPI_OPTION_FUSED_REDUCTION = 8,   /* packed quadrotor path (K_loc >= 65536, diagonal or general
                                          Sigma / A_t, obstacle grid, in-kernel noise, trajectory
                                          weights; mppi_last_kernels shows whether it ran): every rollout CTA
                                          weights its samples against its own minimum and forms its
                                          partial weighted noise sums from its noise tile right after
                                          the rollouts, so that HBM read overlaps the other CTAs'
                                          rollouts; a small kernel rescales the partials by
                                          exp(-(m_c - S_min)/lambda) in CTA order.  Costs, noise and
                                          k* identical; U equal up to rounding.  With cost-to-go
                                          weights the same kernels run the suffix-sum pass (S~_{t,k},
                                          bit-identical to the separate pass, and the per-t CTA
                                          minima) and the per-(CTA, t) weighted sums in their
                                          epilogue, rescaled to S_min,t afterwards (default 1) */
    MPPI_OPTION_GATHER_COMBINE = 9,    /* sharded step with the library's communicator, trajectory
                                          weights: ONE collective instead of two -- every rank forms
                                          its weighted sums against its own minimum, an ncclAllGather
                                          exchanges the [key, eta_r, A_r] records, and every rank
                                          rescales them by exp(-(S_r - S_min)/lambda) in rank order
                                          (PAPER.md:320 is invariant to the shift).  k* and S_min
                                          identical, U equal to rounding (single rank: bitwise)
                                          (default 1) */
    MPPI_OPTION_NOISE_AHEAD = 10       /* K_loc < 65536 (the noise is its own pass), CUDA-graph
                                          path, one GPU: after the step's graph, the noise of
                                          (seed, step + 1) is drawn into a second buffer on a
                                          library-owned side stream, and a following call with
                                          exactly that (seed, step) skips its noise kernel (it
                                          waits on the side stream's event instead) -- the noise
                                          leaves the control update's critical path (U is
                                          complete on the context stream without it).  Noise is
                                          a pure function of (seed, step, k), so results are
                                          bitwise identical; any other call that rewrites the
                                          context's noise buffer discards the drawn-ahead noise.
                                          Default 0: a synchronous control loop at C3 (race car,
                                          K = 16384, T = 150) gains 8 us of its 67 us p50, but
                                          back-to-back steps lose 5 us and C1/C2 gain nothing
                                          (+9 us of host enqueue for the side launch;
                                          profiles/r2_ab_noise_ahead_latency.txt) */
} mppi_option_t;

/* mppi_set_option — execution options that never change results (FUSED_REDUCTION: U to rounding). */
mppi_status_t mppi_set_option(mppi_ctx* ctx, mppi_option_t option, int32_t value);

/* mppi_optimize_host — the same step end to end from HOST buffers: copies x0 and U in,
 * runs mppi_optimize on the context's device copy of U, copies the updated U back.
 * SYNCHRONOUS (returns after U is in host memory).  U: HOST float [T][m] in/out. */
mppi_status_t mppi_optimize_host(mppi_ctx* ctx, const float* x0, float* U, uint64_t seed,
                                 uint64_t step);

/* ---------------------------------------------------------------- NCCL (multi-GPU, row e) */

#define MPPI_NCCL_ID_BYTES 128

/* mppi_nccl_unique_id — a fresh NCCL unique id (HOST uint8 [128]); call on one rank and hand the
 * bytes to every rank (e.g. torch.distributed broadcast).  NCCL is the libnccl.so.2 the process
 * already loaded (torch's), resolved at run time.  Errors: NCCL. */
mppi_status_t mppi_nccl_unique_id(uint8_t* id);

/* mppi_nccl_attach — COLLECTIVE over the context's world (every rank calls it with the same id;
 * blocks until all joined): creates the communicator the library uses from then on, so that
 * mppi_optimize runs the whole K-sharded step on the context stream:
 *   rollouts of this rank's K/world samples -> ncclAllReduce(MIN) of the int64 (cost, k) key
 *   (8 B) -> local weights and weighted noise sums -> ncclAllReduce(SUM) of [eta, A] ((1+T m) fp32)
 *   -> the same U update on every rank (U stays a bit-identical replica).
 * A single-rank communicator (world == 1) is allowed (the collectives are identities).
 * With MPPI_WEIGHTS_COST_TO_GO the collectives are MIN over the T per-step minima of the
 * cost-to-go and SUM over [eta_t (T), A (T m)] instead. */
mppi_status_t mppi_nccl_attach(mppi_ctx* ctx, const uint8_t* id);

/* ---------------------------------------------------------------- split phase (multi-GPU) */

/* mppi_rollout_costs — noise (unless supplied) and rollouts of this rank's K_loc samples.
 *   costs   : DEVICE float [K_loc] or NULL; receives S~_k (penalty where non-finite).
 *   min_key : DEVICE int64 [1] or NULL; receives this rank's minimum key
 *             key = (int64)ord32(S_min) << 32 | k_global, ord32 the order-preserving signed
 *             map of the fp32 bits (b >= 0 ? b : b ^ 0x7fffffff).  The smallest key is the
 *             smallest cost, ties to the smallest global k; combine ranks with a signed MIN.
 * The context keeps its own copy of the costs and the key for mppi_accumulate. */
mppi_status_t mppi_rollout_costs(mppi_ctx* ctx, const float* x0, const float* U, uint64_t seed,
                                 uint64_t step, const float* noise, float* costs,
                                 int64_t* min_key);

/* mppi_accumulate — weights and weighted noise sum over this rank's samples.
 *   global_min_key : DEVICE int64 [1], the MIN over ranks of the keys (NULL: this rank's key).
 *   buf            : DEVICE float [1 + T*m] receiving [eta_r, A_r[0][0..m), ..., A_r[T-1][..]]
 *                    with eta_r = sum_k w_k and A_r[t][j] = sum_k w_k eps[t][k][j] over this
 *                    rank's k in a fixed order (deterministic).  SUM it over ranks, then apply. */
mppi_status_t mppi_accumulate(mppi_ctx* ctx, const int64_t* global_min_key, float* buf);

/* mppi_apply — U_t += sqrt(nu) L A[t] / eta with [eta, A] = buf (DEVICE, read-only),
 * U DEVICE [T][m] in place.  Per entry: d_i = sum_{j<=i} fl(sL[i][j]*A[t][j]) accumulated in
 * order j = 0..i, U[t][i] = fl(U[t][i] + fl(d_i / eta)). */
mppi_status_t mppi_apply(mppi_ctx* ctx, float* U, const float* buf);

/* The split phase of the one-collective combine (MPPI_OPTION_GATHER_COMBINE), for callers that
 * run their own collective (or emulate ranks):
 *   mppi_gather_record_len — floats per record: 2 (the int64 (cost, k) key) + 1 (eta) + T*m (A)
 *                            + padding to an even count; -1 for a NULL ctx.
 *   mppi_accumulate_record — after mppi_rollout_costs: this rank's weights w_k =
 *                            exp(-(S_k - S_min,r)/lambda) against its OWN minimum S_min,r, its
 *                            eta_r and A_r, written with its key as one record.
 *                            record : DEVICE float [mppi_gather_record_len].  Asynchronous.
 *   mppi_apply_gathered    — n_records records concatenated (DEVICE [n][len], e.g. an all-gather
 *                            in rank order): S_min = min of the keys, eta = sum_r c_r eta_r,
 *                            A = sum_r c_r A_r with c_r = exp(-(S_min,r - S_min)/lambda) in record
 *                            order, then U_t += s L A_t / eta as mppi_apply.
 *                            Every rank that applies the same records gets the same bits.
 *                            U : DEVICE [T][m] in/out.  Asynchronous.
 * INVALID_ARG for NULL pointers or n_records < 1; UNSUPPORTED with cost-to-go weights. */
int64_t mppi_gather_record_len(const mppi_ctx* ctx);
mppi_status_t mppi_accumulate_record(mppi_ctx* ctx, float* record);
mppi_status_t mppi_apply_gathered(mppi_ctx* ctx, float* U, const float* records, int32_t n_records);

/* ---------------------------------------------------------------- general variance transform (NEXT-3) */

/* mppi_set_sampling_transform — per-step variance transforms A_t of Theorem 1 (PAPER.md:177-201,
 * B_E = A_t B_c), replacing the special case A = sqrt(nu) I.  With Eq. 7 in control
 * coordinates (Sigma~ = R^{-1}, Lambda~_t = A_t R^{-1} A_t^T) the step samples
 *   du_t = A_t L eps,  L = chol(Sigma)
 * and charges  q~ = q + 1/2 du'(R - A_t^{-T} R A_t^{-1}) du + U_t'R du + 1/2 U_t'R U_t
 * (for A_t = sqrt(nu) I exactly the (1 - 1/nu)/2 of PAPER.md:330); the update is
 * U_t += A_t L A[t] / eta.  nu is then unused.
 *   A : HOST fp64 [T][m][m] row-major, each A_t invertible (else INVALID_ARG); copied.  NULL
 *       restores A_t = sqrt(nu) I.
 * Synchronises the stream.  Uses the general (dense m x m) rollout path. */
mppi_status_t mppi_set_sampling_transform(mppi_ctx* ctx, const double* A);

/* ---------------------------------------------------------------- cost-to-go weights (NEXT-1) */

typedef enum {
    MPPI_WEIGHTS_TRAJECTORY = 0,  /* w_k from the whole-horizon S~_k for every u_t (default) */
    MPPI_WEIGHTS_COST_TO_GO = 1   /* PAPER.md:320-322 / Alg. 1 :367 literally: u_t weighted by
                                     w_{t,k} = exp(-(S~_{t,k} - min_k S~_{t,k})/lambda) with the cost-to-go
                                     S~_{t,k} = sum_{j >= t} q~_{j,k}; eta_t per timestep.  u_0 equals
                                     the trajectory weighting's (S~_{0,k} = S~_k) up to rounding. */
} mppi_weighting_t;

/* mppi_set_weighting — selects the estimator of the update (synchronises the stream).  The
 * cost-to-go mode allocates a [T][K_loc] fp32 buffer of per-step costs on first use, adds 8 B
 * of HBM traffic per sample-step and a per-(t,k) exp.  Sharded (world > 1) it runs through
 * mppi_nccl_attach + mppi_optimize: allreduce MIN over the T per-step minima, then SUM over
 * [eta_t (T), A (T m)]; the split-phase calls refuse it (UNSUPPORTED). */
mppi_status_t mppi_set_weighting(mppi_ctx* ctx, mppi_weighting_t mode);

/* mppi_cost_to_go — copies S~_{t,k} of the last cost-to-go step into `out` (DEVICE float
 * [T][K_loc]).  Asynchronous.  INVALID_ARG unless the cost-to-go weighting is enabled. */
mppi_status_t mppi_cost_to_go(mppi_ctx* ctx, float* out);

/* ---------------------------------------------------------------- on-device MPC loop (NEXT-2) */

/* mppi_closed_loop — Algorithm 1's while-loop for n_steps receding-horizon
 * steps entirely on the device, as one CUDA graph: per step i
 *   optimise U from the device state x (noise counter step0 + i),
 *   send u_0 to the plant: x <- x + F(x, u_0) dt with this context's model, noise-free
 *   (the plant's accurate path), then shift U (u_j = u_{j+1},
 *   u_{T-1} = u_init).
 *   x      : DEVICE float [n], the plant state, in/out.
 *   U      : DEVICE float [T][m], in/out.
 *   u_init : HOST float [m].
 *   reset_crash : nonzero clears the device plant's crash flag (quadrotor) first.
 *   x_log  : DEVICE float [n_steps + 1][n] (x_0 .. x_N) or NULL;  u_log: DEVICE [n_steps][m] (the
 *            executed u_0) or NULL;  q_log: DEVICE [n_steps] (q(x_{i+1})) or NULL.
 * Sharded (world > 1, after mppi_nccl_attach): each step runs with the library's collectives and
 * every rank advances its own replica of the plant with the same all-reduced u_0 (enqueued step by
 * step instead of one graph).
 * SYNCHRONOUS (returns after the loop ran).  plant != LINEAR, and world == 1 or a communicator,
 * else UNSUPPORTED. */
mppi_status_t mppi_closed_loop(mppi_ctx* ctx, float* x, float* U, uint64_t seed, uint64_t step0,
                               int32_t n_steps, const float* u_init, int32_t reset_crash,
                               float* x_log, float* u_log, float* q_log);

/* ---------------------------------------------------------------- path-integral estimate (NEXT-4) */

/* mppi_feynman_kac — the Feynman-Kac path integral Psi(x0) = E_P[exp(-S(tau)/lambda)]
 * (discrete form :78): K rollouts of this context's plant from x0 with U = 0 under
 * the natural noise (the context must have nu == 1, so every importance-sampling term of q~
 * vanishes and S~ = S = sum_t q(x_{t+1})), then, in a fixed-order reduction,
 *   log Psi-hat = -S_min/lambda + log( (1/K) sum_k w_k ),  w_k = exp(-(S_k - S_min)/lambda),
 *   se         = std_k(w_k) / (sqrt(K) mean_k(w_k))     (delta-method std. error of log Psi-hat).
 * V(x0) = -lambda log Psi(x0) is the value function of PAPER.md:56.
 *   x0  : HOST float [n];  seed, step : as mppi_optimize.
 *   out : HOST double [3] = {log_psi, se_log_psi, s_min}.
 * Sharded (world > 1, after mppi_nccl_attach): every rank rolls out its K/G samples, an NCCL
 * MIN of the (cost, k) key gives the global S_min, an NCCL SUM adds the fp64 partial sums, and
 * every rank returns the same estimate over all K samples.
 * SYNCHRONOUS.  world > 1 without a communicator -> UNSUPPORTED; nu != 1 -> UNSUPPORTED. */
mppi_status_t mppi_feynman_kac(mppi_ctx* ctx, const float* x0, uint64_t seed, uint64_t step,
                               double* out);

/* ---------------------------------------------------------------- helpers around the step */

/* mppi_shift — Alg. 1: U_i = U_{i+1}, U_{T-1} = u_init.
 *   U DEVICE [T][m] in place; u_init HOST float [m]. */
mppi_status_t mppi_shift(mppi_ctx* ctx, float* U, const float* u_init);

/* mppi_noise — writes this rank's eps [T][K_loc][m] for (seed, step) into `out` (DEVICE). */
mppi_status_t mppi_noise(mppi_ctx* ctx, uint64_t seed, uint64_t step, float* out);

/* mppi_plant_step — advances the plant one Euler step on the HOST with the same fp32 plant
 * code the rollout kernel runs (environment simulation for closed-loop MPC, Alg. 1 :377).
 *   x HOST float [n] in/out; u HOST float [m]; crashed HOST int32 in/out (quadrotor C flag,
 *   may be NULL); q_out HOST float or NULL receives q(x').  Synchronous; touches no device. */
mppi_status_t mppi_plant_step(mppi_ctx* ctx, float* x, const float* u, int32_t* crashed,
                              float* q_out);

/* mppi_obstacle_grid — HOST only (no device, no context): the nearest-cylinder candidate grid
 * mppi_create builds for the quadrotor, for inspection and tests.
 *   xy     : HOST float [n][2] cylinder centres, 2 <= n <= 127 (else UNSUPPORTED: no grid).
 *   words  : HOST uint32 [capacity] or NULL; receives the [ny][nx] cell words (four 7-bit centre
 *            indices, unused slots repeating the first, 3-bit count in bits 28..30, 0 = no list).
 *   geom   : HOST float [6] = (nx, ny, ox, oy, inv_h, band): a point p lies in cell
 *            (floor(p.x * inv_h + ox), floor(p.y * inv_h + oy)) (fp32 fma), border cells
 *            extending `band` cells outward.
 * Errors: INVALID_ARG (NULL xy / geom, capacity < nx * ny with words != NULL), UNSUPPORTED. */
mppi_status_t mppi_obstacle_grid(const float* xy, int32_t n, uint32_t* words, int64_t capacity,
                                 float* geom);

/* mppi_get_stats — SYNCHRONOUS: waits for the stream, then reads the last step's k*, S_min
 * and eta (eta is this rank's local sum unless mppi_apply ran with a summed buffer). */
mppi_status_t mppi_get_stats(mppi_ctx* ctx, mppi_stats_t* out /* HOST */);

/* mppi_replay_count — SYNCHRONOUS: waits for the stream, then returns in *out (HOST) the number
 * of rollouts this context has re-run since creation (cumulative, one per sample on the
 * one-sample kernels, one per sample pair on the packed quadrotor kernel).  A rollout is re-run
 * from x0 after its step loop, with the per-step accurate fallbacks, when an angle left the fast
 * sin/cos range or a position left the obstacle grid's band or met an overflowing cell (DESIGN.md
 * §6); results are identical either way, only the time differs.  Telemetry for that slow path.
 * Errors: INVALID_ARG (NULL out), CUDA. */
mppi_status_t mppi_replay_count(mppi_ctx* ctx, int64_t* out);

/* Number of kernels the last mppi_optimize / split-phase call enqueued (for launch accounting). */
int32_t mppi_last_launch_count(const mppi_ctx* ctx);

/* mppi_last_kernels — the kernels the last mppi_optimize / split-phase call enqueued, in launch
 * order, as their (mangled) device-function names separated by ',' (which kernel variant the
 * dispatch chose: packed / fused noise / obstacle grid / fused reduction ...).
 *   buf : HOST char [len], receives a NUL-terminated string, truncated to len - 1 characters.
 * Returns the full length needed (excluding the NUL), or -1 for NULL ctx / buf or len < 1. */
int64_t mppi_last_kernels(const mppi_ctx* ctx, char* buf, int64_t len);

/* ---------------------------------------------------------------- per-kernel device time */

typedef enum {
    MPPI_KERNEL_NOISE = 0,     /* K1 noise_kernel */
    MPPI_KERNEL_ROLLOUT = 1,   /* K2 rollout_kernel / rollout_kernel_x2 (incl. in-kernel noise) */
    MPPI_KERNEL_WSUM = 2,      /* K3 wsum (weights + weighted noise sum; cost-to-go: also the
                                  suffix-sum and per-step minimum passes) */
    MPPI_KERNEL_FINALIZE = 3,  /* K4 finalize (partials -> [eta, A] -> U) */
    MPPI_KERNEL_SHIFT = 4,     /* K5 shift_kernel */
    MPPI_KERNEL_COLLECTIVE = 5, /* the NCCL all-reduces of a sharded step (MIN key, SUM [eta, A];
                                   NCCL's kernels on the context stream, not this library's) */
    MPPI_KERNEL_KINDS = 6
} mppi_kernel_kind_t;

typedef struct {
    double total_ms[MPPI_KERNEL_KINDS];  /* summed CUDA-event time of the launches of each kind */
    int64_t launches[MPPI_KERNEL_KINDS];
} mppi_kernel_times_t;

/* mppi_profile_enable — while enabled, every kernel launch of this context is bracketed by two
 * CUDA events recorded on the context stream (the stream the kernel runs on). */
mppi_status_t mppi_profile_enable(mppi_ctx* ctx, int32_t enable);

/* mppi_profile_read — SYNCHRONOUS: waits for the stream, returns the accumulated per-kind times
 * since the last read (or enable), and resets them.  out: HOST. */
mppi_status_t mppi_profile_read(mppi_ctx* ctx, mppi_kernel_times_t* out);

const char* mppi_last_error(void);           /* thread-local, never NULL */
const char* mppi_status_string(mppi_status_t s);
int32_t mppi_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MPPI_B200_H */
