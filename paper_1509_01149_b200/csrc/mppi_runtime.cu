// mppi_runtime.cu — host runtime behind include/mppi.h: validation, fp64 Cholesky of Sigma,
// parameter digestion, workspace sizing/allocation and the enqueue sequences of the step.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <new>
#include <string>

#include "mppi_internal.h"
#include "nvtx3/nvToolsExt.h"   // header-only NVTX v3: named ranges for nsys/ncu (no-ops without a tool)

using namespace mppi;

namespace {

// an NVTX range for the duration of one public call (the host-side enqueue of its work)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

thread_local std::string g_err;

mppi_status_t fail(mppi_status_t s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

mppi_status_t cuda_fail(cudaError_t e, const char* what) {
    return fail(MPPI_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define MPPI_CUDA(call, what)                          \
    do {                                               \
        cudaError_t e_ = (call);                       \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

bool is_fin(double v) { return std::isfinite(v); }

// fp64 Cholesky A = L L^T (lower); false if A is not symmetric positive definite.
bool cholesky64(const double* A, int m, double* L) {
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j)
            if (!is_fin(A[i * m + j]) || fabs(A[i * m + j] - A[j * m + i]) > 1e-12 * (fabs(A[i * m + j]) + 1e-300))
                return false;
    for (int i = 0; i < m * m; ++i) L[i] = 0.0;
    for (int j = 0; j < m; ++j) {
        double d = A[j * m + j];
        for (int k = 0; k < j; ++k) d -= L[j * m + k] * L[j * m + k];
        if (!(d > 0.0)) return false;
        L[j * m + j] = sqrt(d);
        for (int i = j + 1; i < m; ++i) {
            double s = A[i * m + j];
            for (int k = 0; k < j; ++k) s -= L[i * m + k] * L[j * m + k];
            L[i * m + j] = s / L[j * m + j];
        }
    }
    return true;
}

int plant_state_dim(int plant) {
    switch (plant) {
        case MPPI_PLANT_CARTPOLE: return 4;
        case MPPI_PLANT_RACECAR: return 6;
        case MPPI_PLANT_QUADROTOR: return 16;
        default: return 0;
    }
}
int plant_control_dim(int plant) {
    switch (plant) {
        case MPPI_PLANT_CARTPOLE: return 1;
        case MPPI_PLANT_RACECAR: return 2;
        case MPPI_PLANT_QUADROTOR: return 4;
        default: return 0;
    }
}

bool all_finite_d(const double* p, int n) {
    for (int i = 0; i < n; ++i)
        if (!std::isfinite(p[i])) return false;
    return true;
}

bool all_finite(const float* p, int n) {
    for (int i = 0; i < n; ++i)
        if (!isfinite(p[i])) return false;
    return true;
}

// Nearest-cylinder candidate grid for the packed quadrotor rollout (the obstacle term needs
// min_j |p - c_j|^2).  Cells of side h tile the forest's bounding box plus a border;
// a cell lists every centre j that no single other centre i beats over the whole cell:
//   j is dropped iff some i has |p - c_i|^2 < |p - c_j|^2 - margin at all four corners of the cell
//   grown by `slack` (the difference is affine in p, so the corners decide).
// Every centre that can be the fp32 minimum for a point the kernel assigns to the cell is
// therefore listed (slack >> the cell-assignment rounding, margin >> the fp32 error of d^2 over
// the cell), and the minimum over the list equals the minimum over all centres bit for bit.
// Border cells also cover a band of 30 spacings outside the grid (their rectangles are grown
// outward; an affine difference still peaks at a corner).  Cells with more than kCellMaxCand
// candidates, and points beyond the band, take the full loop.
void build_cell_grid(Ctx& c, const float* xy, int n) {
    c.cells_host.clear();
    c.cent_host.clear();
    c.cell_nx = c.cell_ny = 0;
    if (n < 2 || n > (1 << kCellIdxBits)) return;
    double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
    for (int j = 0; j < n; ++j) {
        xmin = fmin(xmin, xy[2 * j]); xmax = fmax(xmax, xy[2 * j]);
        ymin = fmin(ymin, xy[2 * j + 1]); ymax = fmax(ymax, xy[2 * j + 1]);
    }
    std::vector<double> nn(n, 1e300);   // nearest-neighbour spacing sets the cell size
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i)
            if (i != j) nn[j] = fmin(nn[j], hypot((double)xy[2 * i] - xy[2 * j], (double)xy[2 * i + 1] - xy[2 * j + 1]));
    std::vector<double> sorted = nn;
    std::sort(sorted.begin(), sorted.end());
    const double spacing = sorted[n / 2];
    if (!(spacing > 1e-6) || !std::isfinite(xmax - xmin) || !std::isfinite(ymax - ymin)) return;
    const double pad = 3.0 * spacing;
    double h = 0.2 * spacing;
    const double W = (xmax - xmin) + 2 * pad, H = (ymax - ymin) + 2 * pad;
    const double kMaxCells = 8192.0;
    if (W * H / (h * h) > kMaxCells) h = sqrt(W * H / kMaxCells);
    const float inv_h = (float)(1.0 / h);
    h = 1.0 / (double)inv_h;                                   // the cell size the kernel sees
    const int nx = (int)ceil(W / h), ny = (int)ceil(H / h);
    const double gx0 = (float)(xmin - pad), gy0 = (float)(ymin - pad);   // representable origin
    // the kernel's fp32 cell assignment floor(fma(p, 1/h, -g0/h)) is off by < 1e-4 cells
    // cells; beyond it: full search (replay).  30 spacings: a border cell's strip is short enough
    // that no cell of the configs' forests needs more than kCellMaxCand candidates (at 100
    // spacings six top-border strips overflowed, and once U has converged -- trajectories
    // reaching 8-20 m past the forest -- 6 % of the packed rollout's warps replayed a pair:
    // C4 241 -> 435 us per step; profiles/r2_grid_band.txt), while sampled quadrotors stay far
    // inside it (<= 20 m past the grid in 8192 fp64 rollouts)
    const double band = ceil(30.0 * spacing / h);
    const double slack = 1e-3 * h + 1e-6 * (fabs(gx0) + fabs(gy0) + W + H + 2 * band * h);
    std::vector<uint32_t> words((size_t)nx * ny);
    std::vector<double> d2(4 * (size_t)n);
    std::vector<int> cand;
    for (int iy = 0; iy < ny; ++iy)
        for (int ix = 0; ix < nx; ++ix) {
            // border cells also stand for the band of `band` cells outside the grid
            const double x0 = gx0 + (ix == 0 ? -band : ix) * h - slack;
            const double x1 = gx0 + (ix == nx - 1 ? nx + band : ix + 1) * h + slack;
            const double y0 = gy0 + (iy == 0 ? -band : iy) * h - slack;
            const double y1 = gy0 + (iy == ny - 1 ? ny + band : iy + 1) * h + slack;
            const double px[4] = {x0, x0, x1, x1}, py[4] = {y0, y1, y0, y1};
            for (int j = 0; j < n; ++j)
                for (int k = 0; k < 4; ++k) {
                    const double dx = px[k] - xy[2 * j], dy = py[k] - xy[2 * j + 1];
                    d2[4 * j + k] = dx * dx + dy * dy;
                }
            cand.clear();
            for (int j = 0; j < n; ++j) {
                double mx = 0.0;
                for (int k = 0; k < 4; ++k) mx = fmax(mx, d2[4 * j + k]);
                const double margin = 1e-5 * mx + 1e-6;
                bool dominated = false;
                for (int i = 0; i < n && !dominated; ++i) {
                    if (i == j) continue;
                    bool all = true;
                    for (int k = 0; k < 4 && all; ++k) all = d2[4 * i + k] < d2[4 * j + k] - margin;
                    dominated = all;
                }
                if (!dominated) cand.push_back(j);
            }
            uint32_t w = 0;
            if (!cand.empty() && (int)cand.size() <= kCellMaxCand) {
                for (int s = 0; s < kCellMaxCand; ++s)
                    w |= (uint32_t)cand[s < (int)cand.size() ? s : 0] << (kCellIdxBits * s);
                w |= (uint32_t)cand.size() << 28;
            }
            words[(size_t)iy * nx + ix] = w;
        }
    words.resize((words.size() + 3) & ~size_t(3), 0u);   // whole 16-byte groups (vector staging)
    c.cells_host.swap(words);
    c.cent_host.resize(n);
    for (int j = 0; j < n; ++j) c.cent_host[j] = make_float2(-xy[2 * j], -xy[2 * j + 1]);
    c.cell_nx = nx;
    c.cell_ny = ny;
    c.cell_ox = (float)(-gx0 * (double)inv_h);
    c.cell_oy = (float)(-gy0 * (double)inv_h);
    c.cell_inv_h = inv_h;
    c.cell_band = (float)band;
}

mppi_status_t digest_params(Ctx& c, const mppi_dynamics_t* d, const mppi_cost_t* q) {
    memset(&c.params, 0, sizeof(c.params));
    switch (c.plant) {
        case MPPI_PLANT_CARTPOLE: {
            const mppi_cartpole_dynamics_t& D = d->p.cartpole;
            const mppi_cartpole_cost_t& Q = q->p.cartpole;
            if (!(D.pole_length > 0) || !all_finite(&D.g, 3) || !all_finite(&Q.w_p, 4))
                return fail(MPPI_ERR_INVALID_ARG, "cartpole: parameters must be finite, pole_length > 0");
            CartpoleParams& P = c.params.cartpole;
            P.g_over_l = (float)((double)D.g / D.pole_length);
            P.inv_l = (float)(1.0 / D.pole_length);
            P.kv = D.vel_gain;
            P.w_p = Q.w_p; P.w_theta = Q.w_theta; P.w_thetadot = Q.w_thetadot; P.w_pdot = Q.w_pdot;
            return MPPI_OK;
        }
        case MPPI_PLANT_RACECAR: {
            const mppi_racecar_dynamics_t& D = d->p.racecar;
            const mppi_racecar_cost_t& Q = q->p.racecar;
            if (!all_finite(&D.mass, 15) || !all_finite(&Q.track_a, 5) || !(D.mass > 0) ||
                !(D.Iz > 0) || !(D.lf + D.lr > 0) || !(D.v_min > 0) || !(Q.track_a > 0) ||
                !(Q.track_b > 0) || D.throttle_min > D.throttle_max || D.steer_max < 0)
                return fail(MPPI_ERR_INVALID_ARG, "racecar: invalid parameters");
            RacecarParams& P = c.params.racecar;
            const double L = (double)D.lf + D.lr;
            P.inv_mass = (float)(1.0 / D.mass);
            P.inv_Iz = (float)(1.0 / D.Iz);
            P.lf = D.lf; P.lr = D.lr;
            P.tire_B = D.tire_B; P.tire_C = D.tire_C;
            P.Df = (float)((double)D.mu * D.mass * D.g * D.lr / L);
            P.Dr = (float)((double)D.mu * D.mass * D.g * D.lf / L);
            P.Cm = D.Cm; P.Cr = D.Cr; P.Cd = D.Cd; P.v_min = D.v_min;
            P.steer_max = D.steer_max; P.throttle_min = D.throttle_min; P.throttle_max = D.throttle_max;
            P.inv_a = (float)(1.0 / Q.track_a); P.inv_b = (float)(1.0 / Q.track_b);
            P.w_track = Q.w_track; P.w_speed = Q.w_speed; P.v_ref = Q.v_ref;
            return MPPI_OK;
        }
        case MPPI_PLANT_QUADROTOR: {
            const mppi_quadrotor_dynamics_t& D = d->p.quadrotor;
            const mppi_quadrotor_cost_t& Q = q->p.quadrotor;
            if (!all_finite(&D.mass, 11) || !all_finite(Q.goal, 3) || !all_finite(&Q.w_xy, 9) ||
                !(D.mass > 0) || !(D.Ixx > 0) || !(D.Iyy > 0) || !(D.Izz > 0) ||
                !(D.cos_phi_min > 0) || !(Q.obs_length > 0) || Q.obstacle_radius < 0 ||
                D.thrust_min > D.thrust_max)
                return fail(MPPI_ERR_INVALID_ARG, "quadrotor: invalid parameters");
            if (Q.n_obstacles < 0 || Q.n_obstacles > MPPI_MAX_OBSTACLES ||
                (Q.n_obstacles > 0 && !Q.obstacles_xy))
                return fail(MPPI_ERR_INVALID_ARG, "quadrotor: n_obstacles must be in [0, %d] with a host array",
                            MPPI_MAX_OBSTACLES);
            if (Q.n_obstacles > 0 && !all_finite(Q.obstacles_xy, 2 * Q.n_obstacles))
                return fail(MPPI_ERR_INVALID_ARG, "quadrotor: obstacle centres must be finite");
            QuadrotorParams& P = c.params.quadrotor;
            P.inv_mass = (float)(1.0 / D.mass);
            P.arm = D.arm;
            P.inv_Ixx = (float)(1.0 / D.Ixx); P.inv_Iyy = (float)(1.0 / D.Iyy); P.inv_Izz = (float)(1.0 / D.Izz);
            P.gyro_x = (float)((double)D.Izz - D.Iyy);
            P.gyro_y = (float)((double)D.Ixx - D.Izz);
            P.gyro_z = (float)((double)D.Iyy - D.Ixx);
            P.yaw_coeff = D.yaw_coeff; P.motor_gain = D.motor_gain; P.g = D.g;
            P.thrust_min = D.thrust_min; P.thrust_max = D.thrust_max; P.cos_phi_min = D.cos_phi_min;
            P.gx = Q.goal[0]; P.gy = Q.goal[1]; P.gz = Q.goal[2];
            P.w_xy = Q.w_xy; P.w_z = Q.w_z; P.w_yaw = Q.w_yaw; P.w_vel = Q.w_vel;
            P.w_obs = Q.w_obs; P.inv_obs_length = (float)(1.0 / Q.obs_length); P.w_crash = Q.w_crash;
            P.ground_z = Q.ground_z; P.radius = Q.obstacle_radius;
            if (!(Q.w_xy >= 0) || !(Q.w_z >= 0))
                return fail(MPPI_ERR_INVALID_ARG, "quadrotor: w_xy and w_z must be >= 0");
            P.gyro_xi = (float)(((double)D.Izz - D.Iyy) / D.Ixx);       // folded constants (plants.cuh)
            P.gyro_yi = (float)(((double)D.Ixx - D.Izz) / D.Iyy);
            P.gyro_zi = (float)(((double)D.Iyy - D.Ixx) / D.Izz);
            P.arm_xi = (float)((double)D.arm / D.Ixx);
            P.arm_yi = (float)((double)D.arm / D.Iyy);
            P.yaw_zi = (float)((double)D.yaw_coeff / D.Izz);
            P.sw_xy = (float)sqrt((double)Q.w_xy);
            P.sgx = (float)((double)Q.goal[0] * sqrt((double)Q.w_xy));
            P.sgy = (float)((double)Q.goal[1] * sqrt((double)Q.w_xy));
            P.sw_z = (float)sqrt((double)Q.w_z);
            P.sgz = (float)((double)Q.goal[2] * sqrt((double)Q.w_z));
            P.obs_k2 = (float)(1.4426950408889634 / (double)Q.obs_length);
            P.obs_rk2 = (float)((double)Q.obstacle_radius * 1.4426950408889634 / (double)Q.obs_length);
            {   // the largest float x with sqrtf(x) <= radius (IEEE sqrt is monotone)
                float x = (float)((double)P.radius * (double)P.radius);
                while (sqrtf(x) > P.radius) x = nextafterf(x, 0.0f);
                while (sqrtf(nextafterf(x, INFINITY)) <= P.radius) x = nextafterf(x, INFINITY);
                P.crash_d2 = x;
            }
            const int n = Q.n_obstacles;
            c.n_obs_pairs = (n + 1) / 2;
            c.obs_host.assign(c.n_obs_pairs, make_float4(-1e15f, -1e15f, -1e15f, -1e15f));
            for (int j = 0; j < n; ++j) {
                float4& p = c.obs_host[j / 2];
                if (j % 2 == 0) { p.x = -Q.obstacles_xy[2 * j]; p.z = -Q.obstacles_xy[2 * j + 1]; }
                else            { p.y = -Q.obstacles_xy[2 * j]; p.w = -Q.obstacles_xy[2 * j + 1]; }
            }
            build_cell_grid(c, Q.obstacles_xy, n);
            return MPPI_OK;
        }
        case MPPI_PLANT_LINEAR: {
            const mppi_linear_dynamics_t& D = d->p.linear;
            const int n = D.n, m = c.m;
            if (n < 1 || n > 8) return fail(MPPI_ERR_INVALID_ARG, "linear: n must be in 1..8");
            if (!all_finite(D.A, n * n) || !all_finite(D.B, n * m) || !all_finite(q->p.linear.Q, n * n))
                return fail(MPPI_ERR_INVALID_ARG, "linear: A, B, Q must be finite");
            LinearParams& P = c.params.linear;
            P.n = n;
            P.m = m;
            for (int i = 0; i < n; ++i) {
                for (int j = 0; j < n; ++j) {
                    P.A[i * 8 + j] = D.A[i * n + j];
                    P.Q[i * 8 + j] = q->p.linear.Q[i * n + j];
                }
                for (int j = 0; j < m; ++j) P.B[i * 4 + j] = D.B[i * m + j];
            }
            c.n = n;
            return MPPI_OK;
        }
        default:
            return fail(MPPI_ERR_INVALID_ARG, "unknown plant %d", c.plant);
    }
}

void free_graph(GraphState& G) {
    if (G.exec) cudaGraphExecDestroy(G.exec);
    if (G.graph) cudaGraphDestroy(G.graph);
    G.exec = nullptr;
    G.graph = nullptr;
    G.nodes.clear();
    G.funcs.clear();
    G.last.clear();
}

void free_graphs(Ctx& c) {
    for (GraphState& G : c.graphs) free_graph(G);
    free_graph(c.loop_graph);
}

void free_ctx(Ctx& c) {
    if (c.side_stream) cudaStreamSynchronize(c.side_stream);   // a noise drawn ahead may still write
    free_graphs(c);
    nccl_detach(c);
    cudaFree(c.d_commbuf);
    cudaFree(c.d_grec);
    cudaFree(c.d_gather);
    for (auto& p : c.ev_pending) { cudaEventDestroy(p.second.first); cudaEventDestroy(p.second.second); }
    for (auto e : c.ev_pool) cudaEventDestroy(e);
    c.ev_pending.clear();
    c.ev_pool.clear();
    cudaFree(c.d_obs);
    cudaFree(c.d_cells);
    cudaFree(c.d_cent);
    cudaFree(c.d_flags);
    cudaFree(c.d_epi);
    cudaFree(c.d_eps);
    cudaFree(c.d_eps2);
    if (c.ev_chain_done) cudaEventDestroy(c.ev_chain_done);
    if (c.ev_side_done) cudaEventDestroy(c.ev_side_done);
    if (c.side_stream) cudaStreamDestroy(c.side_stream);
    c.side_stream = nullptr;
    c.ev_chain_done = c.ev_side_done = nullptr;
    cudaFree(c.d_costs);
    cudaFree(c.d_key_init);
    cudaFree(c.d_part);
    cudaFree(c.d_eta_part);
    cudaFree(c.d_stats);
    cudaFree(c.d_U);
    cudaFree(c.d_fk);
    cudaFree(c.d_ctg);
    cudaFree(c.d_mats);
    cudaFree(c.d_ctg_partmin);
    cudaFree(c.d_ctg_smin);
    cudaFree(c.d_ctg_eta);
    if (c.h_U_pinned) cudaFreeHost(c.h_U_pinned);
}

template <class T>
mppi_status_t dalloc(Ctx& c, T** p, size_t count, const char* what) {
    const size_t bytes = count * sizeof(T);
    cudaError_t e = cudaMalloc((void**)p, bytes > 0 ? bytes : 16);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return fail(MPPI_ERR_OOM, "cudaMalloc(%zu bytes) for %s failed", bytes, what);
    }
    if (e != cudaSuccess) return cuda_fail(e, what);
    c.workspace_bytes += bytes;
    return MPPI_OK;
}

mppi_status_t check_ctx(const mppi_ctx* ctx) {
    if (!ctx) return fail(MPPI_ERR_INVALID_ARG, "ctx is NULL");
    return MPPI_OK;
}

// Surface asynchronous faults of earlier work before enqueuing more (CUDA, and an attached NCCL
// communicator's asynchronous error state).
mppi_status_t sticky_check(Ctx& c) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "earlier CUDA error");
    e = cudaStreamQuery(c.stream);
    if (e != cudaSuccess && e != cudaErrorNotReady) return cuda_fail(e, "stream fault");
    if (const int r = nccl_async_error(c))
        return fail(MPPI_ERR_NCCL, "NCCL communicator error: %s", nccl_error(r));
    return MPPI_OK;
}

mppi_status_t do_rollout(Ctx& c, const float* x0, const float* U, uint64_t seed, uint64_t step,
                         const float* noise, float* costs_out, const float** eps_used) {
    if (!x0 || !U) return fail(MPPI_ERR_INVALID_ARG, "x0 and U must be non-NULL");
    // (a device-resident x0 -- the closed loop's plant state -- is not readable here)
    if (!c.x0_on_device && !all_finite(x0, c.n)) return fail(MPPI_ERR_INVALID_ARG, "x0 must be finite");
    mppi_status_t s = sticky_check(c);
    if (s) return s;
    c.ahead_ok = false;   // d_eps is rewritten below: a noise drawn ahead may be clobbered
    if (c.side_pending) {   // ... and must not still be writing it
        MPPI_CUDA(cudaStreamWaitEvent(c.stream, c.ev_side_done, 0), "wait for the noise drawn ahead");
        c.side_pending = false;
    }
    const float* eps = noise;
    const bool fused = !noise && fused_noise_applies(c);
    if (!noise && !fused) {
        MPPI_CUDA(launch_noise(c, seed, step, c.d_eps, true), "noise_kernel launch");
        eps = c.d_eps;
    } else {
        MPPI_CUDA(cudaMemcpyAsync(&c.d_stats->min_key, c.d_key_init, sizeof(long long),
                                  cudaMemcpyDeviceToDevice, c.stream), "min-key reset");
    }
    if (fused) {   // the rollout draws eps itself and writes it to d_eps for the reduction
        c.gen_eps = c.d_eps;
        c.gen_seed = seed;
        c.gen_step = step;
        eps = c.d_eps;
    }
    const cudaError_t e = launch_rollout(c, x0, U, eps, costs_out);
    c.gen_eps = nullptr;
    MPPI_CUDA(e, "rollout_kernel launch");
    *eps_used = eps;
    return MPPI_OK;
}

}  // namespace

extern "C" {

int32_t mppi_abi_version(void) { return MPPI_ABI_VERSION; }

const char* mppi_last_error(void) { return g_err.c_str(); }

const char* mppi_status_string(mppi_status_t s) {
    switch (s) {
        case MPPI_OK: return "MPPI_OK";
        case MPPI_ERR_INVALID_ARG: return "MPPI_ERR_INVALID_ARG";
        case MPPI_ERR_NOT_SPD: return "MPPI_ERR_NOT_SPD";
        case MPPI_ERR_OOM: return "MPPI_ERR_OOM";
        case MPPI_ERR_CUDA: return "MPPI_ERR_CUDA";
        case MPPI_ERR_UNSUPPORTED: return "MPPI_ERR_UNSUPPORTED";
        case MPPI_ERR_NCCL: return "MPPI_ERR_NCCL";
        default: return "MPPI_ERR_UNKNOWN";
    }
}

mppi_status_t mppi_create(const mppi_dynamics_t* dynamics, const mppi_cost_t* cost, int64_t K,
                          int32_t T, float dt, float lambda, float nu, int32_t m,
                          const double* Sigma, const double* R, const mppi_dist_t* dist,
                          void* cuda_stream, mppi_ctx** out) {
    g_err.clear();
    if (!out) return fail(MPPI_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!dynamics || !cost || !Sigma || !R)
        return fail(MPPI_ERR_INVALID_ARG, "dynamics, cost, Sigma and R must be non-NULL");
    if (dynamics->struct_size != sizeof(mppi_dynamics_t) || cost->struct_size != sizeof(mppi_cost_t))
        return fail(MPPI_ERR_INVALID_ARG, "struct_size mismatch (dynamics %u vs %zu, cost %u vs %zu)",
                    dynamics->struct_size, sizeof(mppi_dynamics_t), cost->struct_size, sizeof(mppi_cost_t));
    const int plant = (int)dynamics->plant;
    if (plant < MPPI_PLANT_CARTPOLE || plant > MPPI_PLANT_LINEAR)
        return fail(MPPI_ERR_INVALID_ARG, "unknown plant %d", plant);
    if (plant == MPPI_PLANT_LINEAR) {
        if (m != 1 && m != 2 && m != 4) return fail(MPPI_ERR_INVALID_ARG, "linear plant: m must be 1, 2 or 4");
    } else if (m != plant_control_dim(plant)) {
        return fail(MPPI_ERR_INVALID_ARG, "m = %d but the plant has %d controls", m, plant_control_dim(plant));
    }
    if (K < 1 || K > INT_MAX) return fail(MPPI_ERR_INVALID_ARG, "K must be in [1, 2^31)");
    if (T < 1 || T > 4096) return fail(MPPI_ERR_INVALID_ARG, "T must be in [1, 4096]");
    if (!is_fin(dt) || !(dt > 0)) return fail(MPPI_ERR_INVALID_ARG, "dt must be finite and > 0");
    if (!is_fin(lambda) || !(lambda > 0)) return fail(MPPI_ERR_INVALID_ARG, "lambda must be finite and > 0");
    if (!is_fin(nu) || !(nu >= 1)) return fail(MPPI_ERR_INVALID_ARG, "nu must be finite and >= 1");
    if (!is_fin(cost->penalty)) return fail(MPPI_ERR_INVALID_ARG, "penalty must be finite");
    int rank = 0, world = 1;
    if (dist) {
        rank = dist->rank;
        world = dist->world;
        if (world < 1 || rank < 0 || rank >= world)
            return fail(MPPI_ERR_INVALID_ARG, "dist: need 0 <= rank < world");
    }
    if (K % world) return fail(MPPI_ERR_INVALID_ARG, "K = %lld not divisible by world = %d", (long long)K, world);
    const int64_t K_loc = K / world;
    if (K_loc % 4) return fail(MPPI_ERR_INVALID_ARG, "K/world = %lld must be a multiple of 4", (long long)K_loc);
    double L[16], LR[16];
    if (!cholesky64(Sigma, m, L)) return fail(MPPI_ERR_NOT_SPD, "Sigma is not symmetric positive definite");
    if (!cholesky64(R, m, LR)) return fail(MPPI_ERR_NOT_SPD, "R is not symmetric positive definite");

    mppi_ctx* ctx = new (std::nothrow) mppi_ctx();
    if (!ctx) return fail(MPPI_ERR_OOM, "host allocation failed");
    Ctx& c = ctx->c;
    c.plant = plant;
    c.n = plant_state_dim(plant);
    c.m = m;
    c.T = T;
    c.K = K;
    c.K_loc = K_loc;
    c.rank = rank;
    c.world = world;
    c.k_offset = (int64_t)rank * K_loc;
    c.dt = dt;
    c.lambda = lambda;
    c.nu = nu;
    c.c1 = (float)(0.5 * (1.0 - 1.0 / (double)nu));   // (1 - 1/nu)/2
    c.penalty = cost->penalty;
    c.stream = (cudaStream_t)cuda_stream;
    const double s = sqrt((double)nu);
    bool diag = true;
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) {
            c.sL[i * m + j] = (float)(s * L[i * m + j]);
            c.R[i * m + j] = (float)R[i * m + j];
            if (i != j && (L[i * m + j] != 0.0 || R[i * m + j] != 0.0)) diag = false;
        }
    c.diag = diag;
    c.diag0 = diag;
    for (int i = 0; i < m * m; ++i) c.L64[i] = L[i];
    for (int i = 0; i < m; ++i)   // IS_t = K_t + sum_i e_i (a_i e_i + b_ti) on the diagonal path
        c.ad[i] = (float)(0.5 * (1.0 - 1.0 / (double)nu) * R[i * m + i] * (s * L[i * m + i]) * (s * L[i * m + i]));
    mppi_status_t st = digest_params(c, dynamics, cost);
    if (st) { delete ctx; return st; }

    cudaError_t e = cudaGetDevice(&c.device);
    if (e != cudaSuccess) { delete ctx; return cuda_fail(e, "cudaGetDevice (no CUDA device?)"); }
    if (rollout_smem_bytes(c, false) + kRolloutStaticSmem > smem_optin_bytes()) {
        const size_t need = rollout_smem_bytes(c, false) + kRolloutStaticSmem;
        delete ctx;
        return fail(MPPI_ERR_INVALID_ARG, "T = %d needs %zu B of shared memory per rollout CTA (limit %zu)", T,
                    need, smem_optin_bytes());
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    // weighted-noise reduction grid (n_chunks x t-tiles CTAs): a whole number of waves of the
    // resident CTA slots (just under, so the last wave is full), about 4 waves, at least 256
    // float4 columns per chunk
    const int64_t ncols = K_loc * m / 4;
    const int ttiles = (T + kWsumTT - 1) / kWsumTT;
    const int64_t slots = (int64_t)sms * wsum_blocks_per_sm(m);
    const int64_t max_ch = (ncols + kWsumThreads - 1) / kWsumThreads;
    int64_t nch = (4 * slots) / ttiles;
    if (nch > max_ch) nch = max_ch;
    if (nch < 1) nch = 1;
    c.cols_per_chunk = (ncols + nch - 1) / nch;
    // whole 256-column blocks: every bulk copy of the reduction kernels starts 16-B aligned
    c.cols_per_chunk = (c.cols_per_chunk + kWsumThreads - 1) / kWsumThreads * kWsumThreads;
    c.n_chunks = (int)((ncols + c.cols_per_chunk - 1) / c.cols_per_chunk);

    // fused reduction (packed quadrotor): per-CTA partials, combined in chunks of <= 256 CTAs
    if (plant == MPPI_PLANT_QUADROTOR && m == 4 && K_loc >= kPackedMinK) {
        const int64_t nblk = (K_loc / 2 + kRolloutThreads - 1) / kRolloutThreads;
        if ((nblk + c.n_chunks - 1) / c.n_chunks <= 256) c.epi_nblk = (int)nblk;
    }
    mppi_status_t a;
    if ((a = dalloc(c, &c.d_eps, (size_t)T * K_loc * m, "noise")) ||
        (a = dalloc(c, &c.d_costs, (size_t)K_loc, "costs")) ||
        (a = dalloc(c, &c.d_key_init, 1, "key init")) ||
        (a = dalloc(c, &c.d_part, (size_t)c.n_chunks * T * m, "partials")) ||
        (a = dalloc(c, &c.d_eta_part, (size_t)c.n_chunks, "eta partials")) ||
        (a = dalloc(c, &c.d_stats, 1, "stats")) ||
        (a = dalloc(c, &c.d_U, (size_t)T * m, "U staging")) ||
        (a = dalloc(c, &c.d_obs, (size_t)(c.n_obs_pairs > 0 ? c.n_obs_pairs : 1), "obstacles")) ||
        (a = dalloc(c, &c.d_flags, (size_t)((ncols + kWsumThreads - 1) / kWsumThreads), "weight block flags")) ||
        (c.epi_nblk > 0 && (a = dalloc(c, &c.d_epi, (size_t)c.epi_nblk * ((size_t)T * m + std::max<size_t>(4, 2 * (size_t)T)),
                                         "fused-reduction partials"))) ||   // trajectory: T m + 4; cost-to-go: T (m + 2)
        (!c.cells_host.empty() &&
         ((a = dalloc(c, &c.d_cells, c.cells_host.size(), "obstacle grid")) ||
          (a = dalloc(c, &c.d_cent, c.cent_host.size(), "obstacle centres"))))) {
        free_ctx(c);
        delete ctx;
        return a;
    }
    e = cudaMallocHost((void**)&c.h_U_pinned, (size_t)T * m * sizeof(float));
    if (e != cudaSuccess) { free_ctx(c); delete ctx; return fail(MPPI_ERR_OOM, "pinned staging"); }
    const long long kinit = LLONG_MAX;
    DeviceStats st0;
    st0.min_key = LLONG_MAX;
    st0.eta = 0.0f;
    st0.plant_crashed = 0;
    st0.replays = 0;
    if ((e = cudaMemcpy(c.d_key_init, &kinit, sizeof(kinit), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(c.d_stats, &st0, sizeof(st0), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (c.n_obs_pairs > 0 &&
         (e = cudaMemcpy(c.d_obs, c.obs_host.data(), c.n_obs_pairs * sizeof(float4), cudaMemcpyHostToDevice)) != cudaSuccess) ||
        (!c.cells_host.empty() &&
         ((e = cudaMemcpy(c.d_cells, c.cells_host.data(), c.cells_host.size() * sizeof(uint32_t),
                          cudaMemcpyHostToDevice)) != cudaSuccess ||
          (e = cudaMemcpy(c.d_cent, c.cent_host.data(), c.cent_host.size() * sizeof(float2),
                          cudaMemcpyHostToDevice)) != cudaSuccess))) {
        free_ctx(c);
        delete ctx;
        return cuda_fail(e, "workspace init");
    }
    *out = ctx;
    return MPPI_OK;
}

void mppi_destroy(mppi_ctx* ctx) {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->c.stream);
    free_ctx(ctx->c);
    delete ctx;
}

mppi_status_t mppi_info(const mppi_ctx* ctx, mppi_info_t* out) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    if (!out) return fail(MPPI_ERR_INVALID_ARG, "out is NULL");
    const Ctx& c = ctx->c;
    out->n = c.n;
    out->m = c.m;
    out->T = c.T;
    out->plant = c.plant;
    out->K = c.K;
    out->K_loc = c.K_loc;
    out->k_offset = c.k_offset;
    out->n_chunks = c.n_chunks;
    out->reserved = 0;
    out->workspace_bytes = c.workspace_bytes;
    return MPPI_OK;
}

mppi_status_t mppi_set_stream(mppi_ctx* ctx, void* cuda_stream) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    ctx->c.stream = (cudaStream_t)cuda_stream;
    return MPPI_OK;
}

// the update after the rollout: trajectory weights (K3 + K4) or per-timestep cost-to-go weights
static cudaError_t launch_reduce_update(Ctx& c, const float* eps, float* U) {
    cudaError_t e;
    if (c.ctg) {
        if ((e = launch_ctg(c)) != cudaSuccess) return e;
        if ((e = launch_wsum_ctg(c, eps)) != cudaSuccess) return e;
        return launch_finalize_ctg(c, U);
    }
    if (c.epi_active) {   // the rollout formed per-CTA sums: rescale, then K4
        if ((e = launch_epi_combine(c, &c.d_stats->min_key)) != cudaSuccess) return e;
        return launch_finalize(c, nullptr, nullptr, U);
    }
    if ((e = launch_wsum(c, eps, &c.d_stats->min_key)) != cudaSuccess) return e;
    return launch_finalize(c, nullptr, nullptr, U);
}

static cudaKernelNodeParams node_params(KLaunch& L) {
    cudaKernelNodeParams p = {};
    p.func = const_cast<void*>(L.func);
    p.gridDim = L.grid;
    p.blockDim = L.block;
    p.sharedMemBytes = (unsigned)L.smem;
    L.argp[0] = L.args;
    p.kernelParams = L.argp;
    p.extra = nullptr;
    return p;
}

// mppi_optimize through a CUDA graph: the launchers collect their launches (same arguments as
// the direct path), the graph is built once per context and noise mode, later calls only update
// the kernel-node parameters (x0, seed, step, U and noise pointers) and replay it.
static mppi_status_t optimize_graph(Ctx& c, const float* x0, float* U, uint64_t seed, uint64_t step,
                                    const float* noise) {
    if (!x0 || !U) return fail(MPPI_ERR_INVALID_ARG, "x0 and U must be non-NULL");
    if (!all_finite(x0, c.n)) return fail(MPPI_ERR_INVALID_ARG, "x0 must be finite");
    if (mppi_status_t s = sticky_check(c)) return s;
    c.last_launches = 0;
    c.last_funcs.clear();
    c.pending.clear();
    c.collect = true;
    const float* eps = noise ? noise : c.d_eps;
    const bool fused = !noise && fused_noise_applies(c);
    c.epi_active = !noise && epi_applies(c);
    // noise ahead: the separate-noise path draws (seed, step + 1) beside this step's chain
    const bool ahead = !noise && !fused && c.noise_ahead && c.world == 1 && c.d_eps2 && c.side_stream;
    const bool hit = ahead && c.ahead_ok && c.ahead_seed == seed && c.ahead_step == step;
    if (hit) eps = c.ahead_buf;
    float* next = ahead ? (eps == c.d_eps ? c.d_eps2 : c.d_eps) : nullptr;
    cudaError_t e = cudaSuccess;
    if (!noise && !fused && !hit) e = launch_noise(c, seed, step, c.d_eps, true);
    if (fused) {
        c.gen_eps = c.d_eps;
        c.gen_seed = seed;
        c.gen_step = step;
    }
    if (e == cudaSuccess) e = launch_rollout(c, x0, U, eps, nullptr);
    c.gen_eps = nullptr;
    if (e == cudaSuccess) e = launch_reduce_update(c, eps, U);
    c.epi_active = false;
    c.collect = false;
    if (e != cudaSuccess) return cuda_fail(e, "collecting the step's launches");
    GraphState& G = c.graphs[noise ? 1 : hit ? 2 : 0];
    bool same = G.exec && G.funcs.size() == c.pending.size();
    for (size_t i = 0; same && i < c.pending.size(); ++i) same = G.funcs[i] == c.pending[i].func;
    if (!same) {
        if (G.exec) cudaGraphExecDestroy(G.exec);
        if (G.graph) cudaGraphDestroy(G.graph);
        G = GraphState();
        MPPI_CUDA(cudaGraphCreate(&G.graph, 0), "cudaGraphCreate");
        cudaGraphNode_t prev = nullptr;
        if (noise || fused || hit) {   // no K1 on the chain: the min key is reset by a copy node
            MPPI_CUDA(cudaGraphAddMemcpyNode1D(&prev, G.graph, nullptr, 0, &c.d_stats->min_key, c.d_key_init,
                                               sizeof(long long), cudaMemcpyDeviceToDevice), "memcpy node");
        }
        bool prev_is_kernel = false;
        for (size_t li = 0; li < c.pending.size(); ++li) {
            KLaunch& L = c.pending[li];
            cudaKernelNodeParams p = node_params(L);
            cudaGraphNode_t node;
            MPPI_CUDA(cudaGraphAddKernelNode(&node, G.graph, nullptr, 0, &p), "cudaGraphAddKernelNode");
            if (prev) {
                // kernel -> kernel: programmatic edge (the successor starts while the predecessor
                // drains and waits in griddepcontrol.wait before touching its outputs)
                cudaGraphEdgeData ed;
                memset(&ed, 0, sizeof(ed));
                if (prev_is_kernel && c.use_pdl) {
                    ed.from_port = cudaGraphKernelNodePortProgrammatic;
                    ed.type = cudaGraphDependencyTypeProgrammatic;
                }
                MPPI_CUDA(cudaGraphAddDependencies_v2(G.graph, &prev, &node, &ed, 1), "graph edge");
            }
            G.nodes.push_back(node);
            G.funcs.push_back(L.func);
            G.last.push_back(L);
            prev = node;
            prev_is_kernel = true;
        }
        MPPI_CUDA(cudaGraphInstantiate(&G.exec, G.graph, 0), "cudaGraphInstantiate");
    } else {
        for (size_t i = 0; i < c.pending.size(); ++i) {
            KLaunch& L = c.pending[i];
            const KLaunch& O = G.last[i];
            // most calls change only x0 / seed / step: skip the nodes whose arguments are unchanged
            if (L.nargs == O.nargs && memcmp(L.args, O.args, L.nargs) == 0 && L.smem == O.smem &&
                L.grid.x == O.grid.x && L.grid.y == O.grid.y && L.grid.z == O.grid.z && L.block.x == O.block.x)
                continue;
            cudaKernelNodeParams p = node_params(L);
            MPPI_CUDA(cudaGraphExecKernelNodeSetParams(G.exec, G.nodes[i], &p), "graph node update");
            G.last[i] = L;
        }
    }
    // the noise drawn ahead by the previous call (side stream) must be complete before this
    // step reads it -- or, on a miss, before this step rewrites a buffer it may still be writing
    if (c.side_pending) {
        MPPI_CUDA(cudaStreamWaitEvent(c.stream, c.ev_side_done, 0), "wait for the noise drawn ahead");
        c.side_pending = false;
    }
    MPPI_CUDA(cudaGraphLaunch(G.exec, c.stream), "cudaGraphLaunch");
    c.last_eps = eps;
    c.ahead_ok = false;
    if (ahead) {
        // draw (seed, step + 1) on the side stream once this step's chain is done (its buffer was
        // read by the previous step, which precedes this chain on the context stream): the update
        // U is complete without waiting for it, and the next call waits for ev_side_done
        MPPI_CUDA(cudaEventRecord(c.ev_chain_done, c.stream), "event record");
        MPPI_CUDA(cudaStreamWaitEvent(c.side_stream, c.ev_chain_done, 0), "side stream wait");
        cudaStream_t main = c.stream;
        c.stream = c.side_stream;
        const cudaError_t en = launch_noise(c, seed, step + 1, next, false);
        c.stream = main;
        MPPI_CUDA(en, "noise_kernel launch (ahead)");
        MPPI_CUDA(cudaEventRecord(c.ev_side_done, c.side_stream), "event record");
        c.side_pending = true;
        c.ahead_ok = true;
        c.ahead_buf = next;
        c.ahead_seed = seed;
        c.ahead_step = step + 1;
    }
    return MPPI_OK;
}

mppi_status_t mppi_use_graph(mppi_ctx* ctx, int32_t enable) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    ctx->c.use_graph = enable != 0;
    return MPPI_OK;
}

mppi_status_t mppi_set_option(mppi_ctx* ctx, mppi_option_t option, int32_t value) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    switch (option) {
        case MPPI_OPTION_CUDA_GRAPH: ctx->c.use_graph = value != 0; return MPPI_OK;
        case MPPI_OPTION_PACKED_SAMPLES: ctx->c.pack2 = value != 0; return MPPI_OK;
        case MPPI_OPTION_FUSED_NOISE: ctx->c.fuse_noise = value != 0; return MPPI_OK;
        case MPPI_OPTION_OBSTACLE_GRID: ctx->c.use_cells = value != 0; return MPPI_OK;
        case MPPI_OPTION_BULK_REDUCTION: ctx->c.tma_wsum = value != 0; return MPPI_OK;
        case MPPI_OPTION_SPARSE_REDUCTION: ctx->c.sparse_wsum = value != 0; return MPPI_OK;
        case MPPI_OPTION_FUSED_REDUCTION: ctx->c.epi = value != 0; return MPPI_OK;
        case MPPI_OPTION_GATHER_COMBINE: ctx->c.gather_combine = value != 0; return MPPI_OK;
        case MPPI_OPTION_NOISE_AHEAD: {
            Ctx& c = ctx->c;
            c.ahead_ok = false;
            c.noise_ahead = value != 0;
            // below the in-kernel-noise threshold the noise is its own pass: a second buffer, a
            // side stream and the two events that order it (allocated once, on first enable)
            if (c.noise_ahead && c.K_loc < kPackedMinK && !c.d_eps2) {
                if (mppi_status_t a = dalloc(c, &c.d_eps2, (size_t)c.T * c.K_loc * c.m, "noise (ahead)")) return a;
                if (cudaStreamCreateWithFlags(&c.side_stream, cudaStreamNonBlocking) != cudaSuccess ||
                    cudaEventCreateWithFlags(&c.ev_chain_done, cudaEventDisableTiming) != cudaSuccess ||
                    cudaEventCreateWithFlags(&c.ev_side_done, cudaEventDisableTiming) != cudaSuccess)
                    return fail(MPPI_ERR_CUDA, "side stream / events for the noise drawn ahead");
            }
            return MPPI_OK;
        }
        case MPPI_OPTION_PDL:
            MPPI_CUDA(cudaStreamSynchronize(ctx->c.stream), "stream sync");
            ctx->c.use_pdl = value != 0;
            free_graphs(ctx->c);   // the edges are baked into the graph
            return MPPI_OK;
        default: return fail(MPPI_ERR_INVALID_ARG, "unknown option %d", (int)option);
    }
}

// The K-sharded step with the library's communicator (row e): rollouts -> allreduce MIN of the
// key -> local weights and weighted noise sums -> allreduce SUM of [eta, A] -> identical update
// on every rank.  All on the context stream; direct launches.
static mppi_status_t optimize_nccl(Ctx& c, const float* x0, float* U, uint64_t seed, uint64_t step,
                                   const float* noise) {
    c.last_launches = 0;
    c.last_funcs.clear();
    const float* eps = nullptr;
    const bool epi = !noise && epi_applies(c);
    c.epi_active = epi;
    mppi_status_t rs = do_rollout(c, x0, U, seed, step, noise, nullptr, &eps);
    c.epi_active = false;
    if (rs) return rs;
    int r;
    if (!c.ctg && c.gather_combine && c.d_gather) {
        // one collective: every rank sums its samples against its OWN minimum (the rollout's
        // key), all-gathers [key, eta_r, A_r], and rescales the records by
        // exp(-(S_r - S_min)/lambda) in rank order -- identical inputs, identical U on every rank
        if (epi) {
            MPPI_CUDA(launch_epi_combine(c, &c.d_stats->min_key), "fused-reduction combine launch");
        } else {
            MPPI_CUDA(launch_wsum(c, eps, &c.d_stats->min_key), "wsum_kernel launch");
        }
        MPPI_CUDA(launch_finalize_record(c, c.d_grec), "finalize (record) launch");
        { NvtxRange nv_("nccl collective"); ProfScope p(c, MPPI_KERNEL_COLLECTIVE); r = nccl_all_gather(c, c.d_grec, c.d_gather, (size_t)gather_record_len(c)); }
        if (r) return fail(MPPI_ERR_NCCL, "ncclAllGather(records): %s", nccl_error(r));
        MPPI_CUDA(launch_finalize_gathered(c, c.d_gather, c.world, U), "finalize (gathered) launch");
        c.last_eps = eps;
        return MPPI_OK;
    }
    { NvtxRange nv_("nccl collective"); ProfScope p(c, MPPI_KERNEL_COLLECTIVE); r = nccl_min_key(c, &c.d_stats->min_key); }
    if (r) return fail(MPPI_ERR_NCCL, "ncclAllReduce(MIN key): %s", nccl_error(r));
    if (c.ctg) {
        // NEXT-1 sharded: local suffix sums and per-t minima -> MIN over the T
        // minima -> per-(t, k) weights and local sums -> SUM of [eta_t (T), A (T m)] -> update
        MPPI_CUDA(launch_ctg(c), "cost-to-go launch");
        { NvtxRange nv_("nccl collective"); ProfScope p(c, MPPI_KERNEL_COLLECTIVE); r = nccl_min_f32(c, c.d_ctg_smin, (size_t)c.T); }
        if (r) return fail(MPPI_ERR_NCCL, "ncclAllReduce(MIN S_t): %s", nccl_error(r));
        MPPI_CUDA(launch_wsum_ctg(c, eps), "wsum_ctg launch");
        MPPI_CUDA(launch_finalize_ctg(c, nullptr, nullptr, c.d_commbuf), "finalize_ctg (partials) launch");
        { NvtxRange nv_("nccl collective"); ProfScope p(c, MPPI_KERNEL_COLLECTIVE); r = nccl_sum_buf(c, c.d_commbuf, (size_t)c.T + (size_t)c.T * c.m); }
        if (r) return fail(MPPI_ERR_NCCL, "ncclAllReduce(SUM [eta_t, A]): %s", nccl_error(r));
        MPPI_CUDA(launch_finalize_ctg(c, U, c.d_commbuf, nullptr), "finalize_ctg (apply) launch");
        c.last_eps = eps;
        return MPPI_OK;
    }
    if (epi) {
        MPPI_CUDA(launch_epi_combine(c, &c.d_stats->min_key), "fused-reduction combine launch");
    } else {
        MPPI_CUDA(launch_wsum(c, eps, &c.d_stats->min_key), "wsum_kernel launch");
    }
    MPPI_CUDA(launch_finalize(c, nullptr, c.d_commbuf, nullptr), "finalize (partials) launch");
    { NvtxRange nv_("nccl collective"); ProfScope p(c, MPPI_KERNEL_COLLECTIVE); r = nccl_sum_buf(c, c.d_commbuf, (size_t)1 + (size_t)c.T * c.m); }
    if (r) return fail(MPPI_ERR_NCCL, "ncclAllReduce(SUM [eta, A]): %s", nccl_error(r));
    MPPI_CUDA(launch_finalize(c, c.d_commbuf, nullptr, U), "finalize (apply) launch");
    c.last_eps = eps;
    return MPPI_OK;
}

mppi_status_t mppi_nccl_unique_id(uint8_t* id) {
    if (!id) return fail(MPPI_ERR_INVALID_ARG, "id is NULL");
    const int r = nccl_unique_id(id);
    if (r) return fail(MPPI_ERR_NCCL, "ncclGetUniqueId: %s", nccl_error(r));
    return MPPI_OK;
}

mppi_status_t mppi_nccl_attach(mppi_ctx* ctx, const uint8_t* id) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (!id) return fail(MPPI_ERR_INVALID_ARG, "id is NULL");
    if (c.nccl) return fail(MPPI_ERR_INVALID_ARG, "a communicator is already attached");
    if (!c.d_commbuf)
        if (mppi_status_t a = dalloc(c, &c.d_commbuf, (size_t)c.T + (size_t)c.T * c.m, "comm buffer")) return a;
    if (!c.d_grec)
        if (mppi_status_t a = dalloc(c, &c.d_grec, (size_t)gather_record_len(c), "gather record")) return a;
    if (!c.d_gather)
        if (mppi_status_t a = dalloc(c, &c.d_gather, (size_t)c.world * gather_record_len(c), "gather buffer")) return a;
    const int r = nccl_attach(c, id);
    if (r) return fail(MPPI_ERR_NCCL, "ncclCommInitRank(world %d, rank %d): %s", c.world, c.rank, nccl_error(r));
    free_graphs(c);
    return MPPI_OK;
}

mppi_status_t mppi_optimize(mppi_ctx* ctx, const float* x0, float* U, uint64_t seed, uint64_t step,
                            const float* noise) {
    NvtxRange nvtx_("mppi_optimize");
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (c.nccl) return optimize_nccl(c, x0, U, seed, step, noise);
    if (c.world != 1) return fail(MPPI_ERR_UNSUPPORTED, "mppi_optimize with world > 1 needs mppi_nccl_attach "
                                  "(or use the split-phase calls)");
    if (c.use_graph && !c.prof) return optimize_graph(c, x0, U, seed, step, noise);
    c.last_launches = 0;
    c.last_funcs.clear();
    const float* eps = nullptr;
    c.epi_active = !noise && epi_applies(c);
    mppi_status_t s = do_rollout(c, x0, U, seed, step, noise, nullptr, &eps);
    const cudaError_t e = s ? cudaSuccess : launch_reduce_update(c, eps, U);
    c.epi_active = false;
    if (s) return s;
    MPPI_CUDA(e, "reduction/update launch");
    return MPPI_OK;
}

mppi_status_t mppi_set_weighting(mppi_ctx* ctx, mppi_weighting_t mode) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (mode != MPPI_WEIGHTS_TRAJECTORY && mode != MPPI_WEIGHTS_COST_TO_GO)
        return fail(MPPI_ERR_INVALID_ARG, "unknown weighting %d", (int)mode);
    if (mode == MPPI_WEIGHTS_COST_TO_GO && !c.d_ctg) {
        const int64_t nblk = (c.K_loc + 255) / 256;
        mppi_status_t a;
        if ((a = dalloc(c, &c.d_ctg, (size_t)c.T * c.K_loc, "cost-to-go")) ||
            (a = dalloc(c, &c.d_ctg_partmin, (size_t)c.T * nblk, "cost-to-go minima")) ||
            (a = dalloc(c, &c.d_ctg_smin, (size_t)c.T, "cost-to-go smin")) ||
            (a = dalloc(c, &c.d_ctg_eta, (size_t)c.n_chunks * c.T, "cost-to-go eta")))
            return a;
    }
    MPPI_CUDA(cudaStreamSynchronize(c.stream), "stream sync");
    c.ctg = mode == MPPI_WEIGHTS_COST_TO_GO;
    free_graphs(c);     // the step's kernel sequence changed
    return MPPI_OK;
}

// fp64 Gauss-Jordan inverse (partial pivoting); false if singular
static bool invert64(const double* A, int m, double* Ai) {
    double a[16], b[16];
    for (int i = 0; i < m * m; ++i) { a[i] = A[i]; b[i] = 0.0; }
    for (int i = 0; i < m; ++i) b[i * m + i] = 1.0;
    for (int col = 0; col < m; ++col) {
        int p = col;
        for (int r = col + 1; r < m; ++r)
            if (fabs(a[r * m + col]) > fabs(a[p * m + col])) p = r;
        if (!(fabs(a[p * m + col]) > 0.0)) return false;
        for (int j = 0; j < m; ++j) {
            double tmp = a[col * m + j]; a[col * m + j] = a[p * m + j]; a[p * m + j] = tmp;
            tmp = b[col * m + j]; b[col * m + j] = b[p * m + j]; b[p * m + j] = tmp;
        }
        const double d = a[col * m + col];
        for (int j = 0; j < m; ++j) { a[col * m + j] /= d; b[col * m + j] /= d; }
        for (int r = 0; r < m; ++r) {
            if (r == col) continue;
            const double f = a[r * m + col];
            for (int j = 0; j < m; ++j) { a[r * m + j] -= f * a[col * m + j]; b[r * m + j] -= f * b[col * m + j]; }
        }
    }
    for (int i = 0; i < m * m; ++i) Ai[i] = b[i];
    return true;
}

mppi_status_t mppi_set_sampling_transform(mppi_ctx* ctx, const double* A) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    MPPI_CUDA(cudaStreamSynchronize(c.stream), "stream sync");
    free_graphs(c);     // the step's kernels change
    if (!A) {
        c.per_t = false;
        c.diag = c.diag0;
        return MPPI_OK;
    }
    const int m = c.m;
    std::vector<float> mats((size_t)c.T * 32, 0.0f);
    double Rd[16];
    for (int i = 0; i < m * m; ++i) Rd[i] = (double)c.R[i];
    for (int t = 0; t < c.T; ++t) {
        const double* At = A + (size_t)t * m * m;
        if (!all_finite_d(At, m * m)) return fail(MPPI_ERR_INVALID_ARG, "A_%d must be finite", t);
        double Ai[16];
        if (!invert64(At, m, Ai)) return fail(MPPI_ERR_INVALID_ARG, "A_%d is singular (Theorem 1 needs A_t invertible)", t);
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) {
                double f = 0.0, g = 0.0;
                for (int k = 0; k < m; ++k) f += At[i * m + k] * c.L64[k * m + j];
                for (int k = 0; k < m; ++k)
                    for (int l = 0; l < m; ++l) g += Ai[k * m + i] * Rd[k * m + l] * Ai[l * m + j];
                mats[(size_t)t * 32 + i * m + j] = (float)f;
                mats[(size_t)t * 32 + 16 + i * m + j] = (float)(0.5 * (Rd[i * m + j] - g));
            }
    }
    if (!c.d_mats) {
        if (mppi_status_t a = dalloc(c, &c.d_mats, (size_t)c.T * 32, "sampling transforms")) return a;
    }
    MPPI_CUDA(cudaMemcpy(c.d_mats, mats.data(), mats.size() * sizeof(float), cudaMemcpyHostToDevice), "A_t upload");
    const bool diag_before = c.diag;
    c.diag = false;
    if (rollout_smem_bytes(c, false) + kRolloutStaticSmem > smem_optin_bytes()) {
        c.diag = diag_before;
        return fail(MPPI_ERR_INVALID_ARG, "per-step transforms at T = %d need %zu B of shared memory per rollout CTA",
                    c.T, rollout_smem_bytes(c, false));
    }
    c.per_t = true;
    return MPPI_OK;
}

mppi_status_t mppi_cost_to_go(mppi_ctx* ctx, float* out) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (!out) return fail(MPPI_ERR_INVALID_ARG, "out is NULL");
    if (!c.ctg) return fail(MPPI_ERR_INVALID_ARG, "cost-to-go weighting is not enabled");
    MPPI_CUDA(cudaMemcpyAsync(out, c.d_ctg, (size_t)c.T * c.K_loc * sizeof(float), cudaMemcpyDeviceToDevice,
                              c.stream), "cost-to-go copy");
    return MPPI_OK;
}

mppi_status_t mppi_optimize_host(mppi_ctx* ctx, const float* x0, float* U, uint64_t seed, uint64_t step) {
    NvtxRange nvtx_("mppi_optimize_host");
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (!U) return fail(MPPI_ERR_INVALID_ARG, "U is NULL");
    const size_t bytes = (size_t)c.T * c.m * sizeof(float);
    memcpy(c.h_U_pinned, U, bytes);
    MPPI_CUDA(cudaMemcpyAsync(c.d_U, c.h_U_pinned, bytes, cudaMemcpyHostToDevice, c.stream), "U H2D");
    if (mppi_status_t s = mppi_optimize(ctx, x0, c.d_U, seed, step, nullptr)) return s;
    MPPI_CUDA(cudaMemcpyAsync(c.h_U_pinned, c.d_U, bytes, cudaMemcpyDeviceToHost, c.stream), "U D2H");
    MPPI_CUDA(cudaStreamSynchronize(c.stream), "stream sync");
    memcpy(U, c.h_U_pinned, bytes);
    return MPPI_OK;
}

mppi_status_t mppi_rollout_costs(mppi_ctx* ctx, const float* x0, const float* U, uint64_t seed,
                                 uint64_t step, const float* noise, float* costs, int64_t* min_key) {
    NvtxRange nvtx_("mppi_rollout_costs");
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    c.last_launches = 0;
    c.last_funcs.clear();
    const float* eps = nullptr;
    if (mppi_status_t s = do_rollout(c, x0, U, seed, step, noise, costs, &eps)) return s;
    c.last_eps = eps;  // mppi_accumulate reads the same noise again
    if (min_key)
        MPPI_CUDA(cudaMemcpyAsync(min_key, &c.d_stats->min_key, sizeof(long long),
                                  cudaMemcpyDeviceToDevice, c.stream), "min key copy");
    return MPPI_OK;
}

mppi_status_t mppi_accumulate(mppi_ctx* ctx, const int64_t* global_min_key, float* buf) {
    NvtxRange nvtx_("mppi_accumulate");
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (!buf) return fail(MPPI_ERR_INVALID_ARG, "buf is NULL");
    if (c.ctg) return fail(MPPI_ERR_UNSUPPORTED, "the split phase uses trajectory weights; with cost-to-go "
                           "weighting shard through mppi_nccl_attach + mppi_optimize");
    if (mppi_status_t s = sticky_check(c)) return s;
    c.last_launches = 0;
    c.last_funcs.clear();
    const long long* key = global_min_key ? (const long long*)global_min_key : &c.d_stats->min_key;
    MPPI_CUDA(launch_wsum(c, c.last_eps ? c.last_eps : c.d_eps, key), "wsum_kernel launch");
    MPPI_CUDA(launch_finalize(c, nullptr, buf, nullptr), "finalize_kernel launch");
    if (global_min_key)
        MPPI_CUDA(cudaMemcpyAsync(&c.d_stats->min_key, key, sizeof(long long),
                                  cudaMemcpyDeviceToDevice, c.stream), "global key copy");
    return MPPI_OK;
}

int64_t mppi_gather_record_len(const mppi_ctx* ctx) { return ctx ? gather_record_len(ctx->c) : -1; }

mppi_status_t mppi_accumulate_record(mppi_ctx* ctx, float* record) {
    NvtxRange nvtx_("mppi_accumulate_record");
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (!record) return fail(MPPI_ERR_INVALID_ARG, "record is NULL");
    if (c.ctg) return fail(MPPI_ERR_UNSUPPORTED, "the split phase uses trajectory weights");
    if (mppi_status_t s = sticky_check(c)) return s;
    c.last_launches = 0;
    c.last_funcs.clear();
    // the weights against this rank's own minimum (the key mppi_rollout_costs left in the context)
    MPPI_CUDA(launch_wsum(c, c.last_eps ? c.last_eps : c.d_eps, &c.d_stats->min_key), "wsum_kernel launch");
    MPPI_CUDA(launch_finalize_record(c, record), "finalize (record) launch");
    return MPPI_OK;
}

mppi_status_t mppi_apply_gathered(mppi_ctx* ctx, float* U, const float* records, int32_t n_records) {
    NvtxRange nvtx_("mppi_apply_gathered");
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (!U || !records || n_records < 1) return fail(MPPI_ERR_INVALID_ARG, "U, records non-NULL and n_records >= 1");
    if (mppi_status_t s = sticky_check(c)) return s;
    c.last_launches = 0;
    c.last_funcs.clear();
    MPPI_CUDA(launch_finalize_gathered(c, records, n_records, U), "finalize (gathered) launch");
    return MPPI_OK;
}

mppi_status_t mppi_apply(mppi_ctx* ctx, float* U, const float* buf) {
    NvtxRange nvtx_("mppi_apply");
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (!U || !buf) return fail(MPPI_ERR_INVALID_ARG, "U and buf must be non-NULL");
    if (mppi_status_t s = sticky_check(c)) return s;
    c.last_launches = 0;
    c.last_funcs.clear();
    MPPI_CUDA(launch_finalize(c, buf, nullptr, U), "finalize_kernel launch");
    return MPPI_OK;
}

mppi_status_t mppi_shift(mppi_ctx* ctx, float* U, const float* u_init) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (!U || !u_init) return fail(MPPI_ERR_INVALID_ARG, "U and u_init must be non-NULL");
    if (!all_finite(u_init, c.m)) return fail(MPPI_ERR_INVALID_ARG, "u_init must be finite");
    if (mppi_status_t s = sticky_check(c)) return s;
    c.last_launches = 0;
    c.last_funcs.clear();
    MPPI_CUDA(launch_shift(c, U, u_init), "shift_kernel launch");
    return MPPI_OK;
}

mppi_status_t mppi_noise(mppi_ctx* ctx, uint64_t seed, uint64_t step, float* out) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (!out) return fail(MPPI_ERR_INVALID_ARG, "out is NULL");
    if (mppi_status_t s = sticky_check(c)) return s;
    c.last_launches = 0;
    c.last_funcs.clear();
    MPPI_CUDA(launch_noise(c, seed, step, out, false), "noise_kernel launch");
    return MPPI_OK;
}

mppi_status_t mppi_plant_step(mppi_ctx* ctx, float* x, const float* u, int32_t* crashed, float* q_out) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (!x || !u) return fail(MPPI_ERR_INVALID_ARG, "x and u must be non-NULL");
    const float q = host_plant_step(c, x, u, crashed);
    if (q_out) *q_out = q;
    return MPPI_OK;
}

mppi_status_t mppi_obstacle_grid(const float* xy, int32_t n, uint32_t* words, int64_t capacity, float* geom) {
    if (!xy || !geom) return fail(MPPI_ERR_INVALID_ARG, "xy and geom must be non-NULL");
    if (n < 2 || n > (1 << kCellIdxBits)) return fail(MPPI_ERR_UNSUPPORTED, "no grid for %d obstacles", n);
    if (!all_finite(xy, 2 * n)) return fail(MPPI_ERR_INVALID_ARG, "obstacle centres must be finite");
    Ctx c;
    build_cell_grid(c, xy, n);
    if (c.cell_nx == 0) return fail(MPPI_ERR_UNSUPPORTED, "degenerate obstacle layout: no grid");
    geom[0] = (float)c.cell_nx;
    geom[1] = (float)c.cell_ny;
    geom[2] = c.cell_ox;
    geom[3] = c.cell_oy;
    geom[4] = c.cell_inv_h;
    geom[5] = c.cell_band;
    if (words) {
        const int64_t ncell = (int64_t)c.cell_nx * c.cell_ny;   // (the device copy is padded past it)
        if (capacity < ncell) return fail(MPPI_ERR_INVALID_ARG, "capacity below nx * ny");
        memcpy(words, c.cells_host.data(), (size_t)ncell * sizeof(uint32_t));
    }
    return MPPI_OK;
}

mppi_status_t mppi_get_stats(mppi_ctx* ctx, mppi_stats_t* out) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    if (!out) return fail(MPPI_ERR_INVALID_ARG, "out is NULL");
    Ctx& c = ctx->c;
    MPPI_CUDA(cudaStreamSynchronize(c.stream), "stream sync");
    DeviceStats h;
    MPPI_CUDA(cudaMemcpy(&h, c.d_stats, sizeof(h), cudaMemcpyDeviceToHost), "stats D2H");
    int b = (int)(h.min_key >> 32);
    b = b >= 0 ? b : (b ^ 0x7fffffff);
    float smin;
    memcpy(&smin, &b, sizeof(smin));
    out->k_star = (int64_t)(uint32_t)(h.min_key & 0xffffffffLL);
    out->s_min = smin;
    out->eta = h.eta;
    return MPPI_OK;
}

mppi_status_t mppi_replay_count(mppi_ctx* ctx, int64_t* out) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    if (!out) return fail(MPPI_ERR_INVALID_ARG, "out is NULL");
    Ctx& c = ctx->c;
    MPPI_CUDA(cudaStreamSynchronize(c.stream), "stream sync");
    unsigned long long n = 0;
    MPPI_CUDA(cudaMemcpy(&n, &c.d_stats->replays, sizeof(n), cudaMemcpyDeviceToHost), "replay count D2H");
    *out = (int64_t)n;
    return MPPI_OK;
}

int32_t mppi_last_launch_count(const mppi_ctx* ctx) { return ctx ? ctx->c.last_launches : 0; }

int64_t mppi_last_kernels(const mppi_ctx* ctx, char* buf, int64_t len) {
    if (!ctx || !buf || len < 1) return -1;
    std::string names;
    for (const void* f : ctx->c.last_funcs) {
        const char* nm = nullptr;
        if (cudaFuncGetName(&nm, f) != cudaSuccess || !nm) nm = "?";
        if (!names.empty()) names += ',';
        names += nm;
    }
    const size_t n = std::min((size_t)(len - 1), names.size());
    memcpy(buf, names.data(), n);
    buf[n] = '\0';
    return (int64_t)names.size();
}

mppi_status_t mppi_closed_loop(mppi_ctx* ctx, float* x, float* U, uint64_t seed, uint64_t step0,
                               int32_t n_steps, const float* u_init, int32_t reset_crash,
                               float* x_log, float* u_log, float* q_log) {
    NvtxRange nvtx_("mppi_closed_loop");
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    c.ahead_ok = false;   // the loop's graph rewrites the noise buffer
    if (c.side_pending) {
        MPPI_CUDA(cudaStreamWaitEvent(c.stream, c.ev_side_done, 0), "wait for the noise drawn ahead");
        c.side_pending = false;
    }
    if (c.world != 1 && !c.nccl)
        return fail(MPPI_ERR_UNSUPPORTED, "mppi_closed_loop with world > 1 needs mppi_nccl_attach");
    if (c.plant == MPPI_PLANT_LINEAR) return fail(MPPI_ERR_UNSUPPORTED, "mppi_closed_loop: linear test plant");
    if (!x || !U || !u_init || n_steps < 1) return fail(MPPI_ERR_INVALID_ARG, "x, U, u_init non-NULL, n_steps >= 1");
    if (!all_finite(u_init, c.m)) return fail(MPPI_ERR_INVALID_ARG, "u_init must be finite");
    if (mppi_status_t s = sticky_check(c)) return s;
    if (reset_crash)
        MPPI_CUDA(cudaMemsetAsync(&c.d_stats->plant_crashed, 0, sizeof(int), c.stream), "crash reset");
    if (c.nccl) {
        // sharded: every rank runs the step with the library's collectives and advances its own
        // replica of the plant with the same (all-reduced, hence identical) u_0 -- the replicas
        // stay bitwise equal.  Enqueued step by step (the collectives sit between the kernels).
        if (x_log) MPPI_CUDA(cudaMemcpyAsync(x_log, x, (size_t)c.n * sizeof(float), cudaMemcpyDeviceToDevice, c.stream), "x_log[0]");
        int launches = 0;
        for (int i = 0; i < n_steps; ++i) {
            c.x0_on_device = true;
            mppi_status_t s = optimize_nccl(c, x, U, seed, step0 + (uint64_t)i, nullptr);
            c.x0_on_device = false;
            if (s) return s;
            launches += c.last_launches;
            MPPI_CUDA(launch_advance(c, x, U, u_init, x_log ? x_log + (size_t)(i + 1) * c.n : nullptr,
                                     u_log ? u_log + (size_t)i * c.m : nullptr, q_log ? q_log + i : nullptr),
                      "closed-loop advance");
        }
        c.last_launches = launches + n_steps;
        MPPI_CUDA(cudaStreamSynchronize(c.stream), "stream sync");
        return MPPI_OK;
    }
    // collect n_steps x [noise, rollout (x0 from device), wsum, finalize, advance] into one graph
    c.last_launches = 0;
    c.last_funcs.clear();
    c.pending.clear();
    c.collect = true;
    c.x0_on_device = true;
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < n_steps && e == cudaSuccess; ++i) {
        e = launch_noise(c, seed, step0 + (uint64_t)i, c.d_eps, true);
        if (e == cudaSuccess) e = launch_rollout(c, x, U, c.d_eps, nullptr);
        if (e == cudaSuccess) e = launch_reduce_update(c, c.d_eps, U);
        if (e == cudaSuccess)
            e = launch_advance(c, x, U, u_init, x_log ? x_log + (size_t)(i + 1) * c.n : nullptr,
                               u_log ? u_log + (size_t)i * c.m : nullptr, q_log ? q_log + i : nullptr);
    }
    c.collect = false;
    c.x0_on_device = false;
    if (e != cudaSuccess) return cuda_fail(e, "collecting the closed loop");
    if (x_log) MPPI_CUDA(cudaMemcpyAsync(x_log, x, (size_t)c.n * sizeof(float), cudaMemcpyDeviceToDevice, c.stream), "x_log[0]");
    // the instantiated loop graph is kept: a later call with the same kernel sequence (same
    // n_steps and variants) only updates the nodes whose arguments changed (seed, step, pointers)
    GraphState& G = c.loop_graph;
    bool same = G.exec && G.funcs.size() == c.pending.size();
    for (size_t i = 0; same && i < c.pending.size(); ++i) same = G.funcs[i] == c.pending[i].func;
    if (!same) {
        free_graph(G);
        MPPI_CUDA(cudaGraphCreate(&G.graph, 0), "cudaGraphCreate");
        cudaGraphNode_t prev = nullptr;
        for (KLaunch& L : c.pending) {
            cudaKernelNodeParams p = node_params(L);
            cudaGraphNode_t node;
            cudaError_t ee = cudaGraphAddKernelNode(&node, G.graph, prev ? &prev : nullptr, prev ? 1 : 0, &p);
            if (ee != cudaSuccess) { free_graph(G); return cuda_fail(ee, "closed-loop graph"); }
            G.nodes.push_back(node);
            G.funcs.push_back(L.func);
            G.last.push_back(L);
            prev = node;
        }
        e = cudaGraphInstantiate(&G.exec, G.graph, 0);
        if (e != cudaSuccess) { free_graph(G); return cuda_fail(e, "closed-loop graph instantiate"); }
    } else {
        for (size_t i = 0; i < c.pending.size(); ++i) {
            KLaunch& L = c.pending[i];
            const KLaunch& O = G.last[i];
            if (L.nargs == O.nargs && memcmp(L.args, O.args, L.nargs) == 0 && L.smem == O.smem &&
                L.grid.x == O.grid.x && L.grid.y == O.grid.y && L.grid.z == O.grid.z && L.block.x == O.block.x)
                continue;
            cudaKernelNodeParams p = node_params(L);
            MPPI_CUDA(cudaGraphExecKernelNodeSetParams(G.exec, G.nodes[i], &p), "closed-loop graph node update");
            G.last[i] = L;
        }
    }
    e = cudaGraphLaunch(G.exec, c.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
    if (e != cudaSuccess) return cuda_fail(e, "closed-loop graph launch");
    return MPPI_OK;
}

mppi_status_t mppi_feynman_kac(mppi_ctx* ctx, const float* x0, uint64_t seed, uint64_t step, double* out) {
    NvtxRange nvtx_("mppi_feynman_kac");
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    if (!out) return fail(MPPI_ERR_INVALID_ARG, "out is NULL");
    if (c.world != 1 && !c.nccl)
        return fail(MPPI_ERR_UNSUPPORTED, "mppi_feynman_kac with world > 1 needs mppi_nccl_attach");
    if (c.nu != 1.0f) return fail(MPPI_ERR_UNSUPPORTED, "mppi_feynman_kac samples the uncontrolled "
                                  "dynamics P: create the context with nu == 1");
    c.last_launches = 0;
    c.last_funcs.clear();
    // U = 0 (uncontrolled dynamics) in the context's staging buffer
    MPPI_CUDA(cudaMemsetAsync(c.d_U, 0, (size_t)c.T * c.m * sizeof(float), c.stream), "U = 0");
    const float* eps = nullptr;
    if (mppi_status_t s = do_rollout(c, x0, c.d_U, seed, step, nullptr, nullptr, &eps)) return s;
    const int nblk = 148;
    if (!c.d_fk) MPPI_CUDA(cudaMalloc((void**)&c.d_fk, 2 * nblk * sizeof(double)), "fk partials");
    if (c.nccl) {   // sharded: the global S_min, then the sums of exp(-(S - S_min)/lambda) over ranks
        int r = nccl_min_key(c, &c.d_stats->min_key);
        if (r) return fail(MPPI_ERR_NCCL, "ncclAllReduce(MIN key): %s", nccl_error(r));
    }
    MPPI_CUDA(launch_fk_reduce(c, c.d_fk, nblk), "fk_reduce launch");
    if (c.nccl) {
        int r = nccl_sum_f64(c, c.d_fk, (size_t)2 * nblk);
        if (r) return fail(MPPI_ERR_NCCL, "ncclAllReduce(SUM fk partials): %s", nccl_error(r));
    }
    double part[2 * 148];
    long long key = 0;
    MPPI_CUDA(cudaMemcpyAsync(part, c.d_fk, sizeof(part), cudaMemcpyDeviceToHost, c.stream), "fk D2H");
    MPPI_CUDA(cudaMemcpyAsync(&key, &c.d_stats->min_key, sizeof(key), cudaMemcpyDeviceToHost, c.stream), "key D2H");
    MPPI_CUDA(cudaStreamSynchronize(c.stream), "stream sync");
    double s1 = 0.0, s2 = 0.0;
    for (int i = 0; i < nblk; ++i) { s1 += part[2 * i]; s2 += part[2 * i + 1]; }
    int b = (int)(key >> 32);
    b = b >= 0 ? b : (b ^ 0x7fffffff);
    float smin;
    memcpy(&smin, &b, sizeof(smin));
    const double K = (double)(c.nccl ? c.K : c.K_loc);   // the sums cover every rank's samples
    const double mean = s1 / K;
    const double var = K > 1 ? (s2 / K - mean * mean) * K / (K - 1) : 0.0;
    out[0] = -(double)smin / (double)c.lambda + log(mean);
    out[1] = sqrt(var > 0 ? var : 0.0) / sqrt(K) / mean;
    out[2] = (double)smin;
    return MPPI_OK;
}

static mppi_status_t drain_profile(Ctx& c) {
    for (auto& p : c.ev_pending) {
        float ms = 0.0f;
        cudaError_t e = cudaEventElapsedTime(&ms, p.second.first, p.second.second);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
        c.prof_ms[p.first] += ms;
        c.prof_n[p.first] += 1;
        c.ev_pool.push_back(p.second.first);
        c.ev_pool.push_back(p.second.second);
    }
    c.ev_pending.clear();
    return MPPI_OK;
}

mppi_status_t mppi_profile_enable(mppi_ctx* ctx, int32_t enable) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    Ctx& c = ctx->c;
    MPPI_CUDA(cudaStreamSynchronize(c.stream), "stream sync");
    if (mppi_status_t s = drain_profile(c)) return s;
    for (int i = 0; i < MPPI_KERNEL_KINDS; ++i) { c.prof_ms[i] = 0.0; c.prof_n[i] = 0; }
    c.prof = enable != 0;
    return MPPI_OK;
}

mppi_status_t mppi_profile_read(mppi_ctx* ctx, mppi_kernel_times_t* out) {
    if (mppi_status_t s = check_ctx(ctx)) return s;
    if (!out) return fail(MPPI_ERR_INVALID_ARG, "out is NULL");
    Ctx& c = ctx->c;
    MPPI_CUDA(cudaStreamSynchronize(c.stream), "stream sync");
    if (mppi_status_t s = drain_profile(c)) return s;
    for (int i = 0; i < MPPI_KERNEL_KINDS; ++i) {
        out->total_ms[i] = c.prof_ms[i];
        out->launches[i] = c.prof_n[i];
        c.prof_ms[i] = 0.0;
        c.prof_n[i] = 0;
    }
    return MPPI_OK;
}

}  // extern "C"
