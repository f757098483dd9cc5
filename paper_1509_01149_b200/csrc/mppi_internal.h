// mppi_internal.h — context layout and kernel launchers shared by mppi_kernels.cu and
// mppi_runtime.cu (internal; the public boundary is include/mppi.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "mppi.h"
#include "noise.cuh"
#include "plants.cuh"

namespace mppi {

constexpr int kRolloutThreads = 128;
// upper bound of the rollout kernels' static shared memory (candidate-grid centres, block minima)
constexpr size_t kRolloutStaticSmem = 2304;
constexpr int kWsumThreads = 256;
#ifndef MPPI_X2_MINB
// packed rollout: 3 resident CTAs per SM (register cap 168; 155 used, no spills).  Measured
// against 4 CTAs / 128 registers: -0.25 % at K = 2^22 ... -2.6 % at 2^16, 5 CTAs (96 registers,
// spills) +3.5 %, 2 CTAs +6.5 % (profiles/r2_ab_occupancy.txt): the step loop is bound by the
// FMA-heavy pipe and issue, not by the number of warps hiding latency
#define MPPI_X2_MINB 3
#endif
#ifndef MPPI_EPI_ROWS
#define MPPI_EPI_ROWS 2      // fused-reduction epilogue: noise rows per warp pass (8 float4 loads each)
#endif
constexpr int kWsumTT = 8;                      // timestep rows per reduction CTA
#ifndef MPPI_WSUM_STAGES
#define MPPI_WSUM_STAGES 2
#endif
constexpr int kWsumStages = MPPI_WSUM_STAGES;   // bulk-copy ring depth of wsum_tma_kernel
constexpr size_t kWsumTmaSmem = (size_t)kWsumStages * kWsumTT * kWsumThreads * 16;   // 64 KB: 3 CTAs / SM
constexpr int kWsumCtgStages = 2;               // wsum_ctg_tma_kernel ring depth (eps + cost-to-go tiles)
// eps float4 + (4/m) cost-to-go floats per column: 80 KB (m = 4) .. 128 KB (m = 1)
constexpr size_t wsum_ctg_tma_smem(int m) { return (size_t)kWsumCtgStages * kWsumTT * kWsumThreads * (16 + 16 / m); }
constexpr int kEpsStages = 4;                   // one-sample rollout's cp.async ring depth
constexpr int kNoiseTT = 8;  // timesteps per noise thread
constexpr int kMaxStaticPairs = 32;
// the two-samples-per-thread quadrotor kernel is used from this many samples per GPU on (below
// it the one-sample kernel fills the 148 SMs better: scripts/compare_pack.py on B200)
constexpr int64_t kPackedMinK = 65536;  // quadrotor: obstacle pairs compiled as a constant up to here

// per-timestep constants of the rollout staged in shared memory (one 48-byte record per t)
struct StepRec {
    float4 u;  // U_t (zero padded to 4)
    float4 b;  // diagonal path: s_i (R U_t)_i; general path: (R U_t)_i
    float4 k;  // .x = U_t'R U_t / 2
};  // timesteps per weighted-noise tile (register accumulators = 8 * m)

union PlantParamsU {
    CartpoleParams cartpole;
    RacecarParams racecar;
    QuadrotorParams quadrotor;
    LinearParams linear;
};

// One kernel launch: the kernel takes a single by-value parameter struct, copied here so the
// launch can go to the stream directly or become (or update) a node of the context's CUDA graph.
struct KLaunch {
    const void* func = nullptr;
    dim3 grid, block;
    size_t smem = 0;
    int kind = 0;
    size_t nargs = 0;
    alignas(16) unsigned char args[2048];
    void* argp[1];
};

struct GraphState {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<cudaGraphNode_t> nodes;   // kernel nodes in launch order
    std::vector<const void*> funcs;
    std::vector<KLaunch> last;            // the arguments each node was last set to
};

// Device-side per-step results readable by mppi_get_stats.
struct DeviceStats {
    long long min_key;
    float eta;
    int plant_crashed;   // crash flag of the device-resident plant (mppi_closed_loop)
    unsigned long long replays;   // cumulative: rollouts re-run after the loop (mppi_replay_count)
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int plant = 0, n = 0, m = 0, T = 0;
    int64_t K = 0, K_loc = 0, k_offset = 0;
    int rank = 0, world = 1;
    float dt = 0, lambda = 0, nu = 1, c1 = 0, penalty = 1e30f;
    bool diag = true;               // L and R both diagonal -> diagonal fast path (and no A_t)
    bool diag0 = true;              // the create-time value (restored when A_t is cleared)
    bool per_t = false;             // NEXT-3: per-step transforms A_t set
    float* d_mats = nullptr;        // [T][2][16] F_t = A_t L, G_t = (R - A_t^-T R A_t^-1) / 2
    double L64[16] = {0};           // chol(Sigma) fp64
    bool pack2 = true;              // quadrotor (diagonal): two samples per thread, FP32x2
    bool fuse_noise = true;         // packed rollout draws its own noise (no K1 pass)
    bool tma_wsum = true;           // K3 streams eps with bulk copies (MPPI_OPTION_BULK_REDUCTION)
    bool use_pdl = false;           // programmatic kernel->kernel edges in the step graph (MPPI_OPTION_PDL, default 0)
    bool sparse_wsum = false;       // K3 skips all-zero-weight column blocks (MPPI_OPTION_SPARSE_REDUCTION)
    bool epi = true;                // packed rollout forms the weighted sums itself (MPPI_OPTION_FUSED_REDUCTION)
    bool epi_active = false;        // set around one optimize step that uses it
    float* d_epi = nullptr;         // [epi_nblk][T m + 4] per-CTA partials
    int epi_nblk = 0;
    uint8_t* d_flags = nullptr;     // [ceil(K_loc m / 4 / 256)] nonzero-weight block flags
    // set around a fused launch: the rollout writes the noise it draws here (else nullptr)
    float* gen_eps = nullptr;
    uint64_t gen_seed = 0, gen_step = 0;
    float sL[16] = {0};             // sqrt(nu) * chol(Sigma), fp32, row-major m x m
    float R[16] = {0};              // control cost, fp32
    float ad[4] = {0};              // diagonal path: (1 - 1/nu)/2 R_ii (sqrt(nu) L_ii)^2
    PlantParamsU params;            // pre-digested plant/cost parameters
    std::vector<float4> obs_host;   // negated obstacle pairs (host copy, for mppi_plant_step)
    int n_obs_pairs = 0;
    // nearest-cylinder candidate grid (quadrotor): cell words + negated centres, see build_cell_grid
    std::vector<uint32_t> cells_host;
    std::vector<float2> cent_host;
    uint32_t* d_cells = nullptr;
    float2* d_cent = nullptr;
    int cell_nx = 0, cell_ny = 0;
    float cell_ox = 0.0f, cell_oy = 0.0f, cell_inv_h = 0.0f;   // cell coord = p / h + o
    bool use_cells = true;          // MPPI_OPTION_OBSTACLE_GRID (when a grid was built)
    float cell_band = 0.0f;         // border cells extend this many cells outward
    // device workspace
    float4* d_obs = nullptr;
    float* d_eps = nullptr;         // [T][K_loc][m]
    float* d_costs = nullptr;       // [K_loc]
    long long* d_key_init = nullptr;  // constant INT64_MAX (reset source)
    float* d_part = nullptr;        // [n_chunks][T*m]
    float* d_eta_part = nullptr;    // [n_chunks]
    DeviceStats* d_stats = nullptr;
    float* d_U = nullptr;           // [T][m] for mppi_optimize_host / mppi_feynman_kac
    double* d_fk = nullptr;         // Feynman-Kac partial sums (lazy)
    // NEXT-1 per-timestep cost-to-go weighting (lazy workspace)
    bool ctg = false;
    bool ctg_fused = false;         // the last rollout launch ran the fused cost-to-go pass
    float* d_ctg = nullptr;         // [T][K_loc] q~ then S~_{t,k}
    float* d_ctg_partmin = nullptr; // [T][ceil(K_loc/256)]
    float* d_ctg_smin = nullptr;    // [T]
    float* d_ctg_eta = nullptr;     // [n_chunks][T]
    float* h_U_pinned = nullptr;    // pinned staging for mppi_optimize_host
    int n_chunks = 1;
    int64_t cols_per_chunk = 0;     // float4 columns of a noise row per chunk
    size_t workspace_bytes = 0;
    int last_launches = 0;
    std::vector<const void*> last_funcs;  // device functions of the last call's launches
    const float* last_eps = nullptr;  // noise read by the last rollout (ctx or caller buffer)
    // per-kernel CUDA-event timing (mppi_profile_enable)
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;                       // free events
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_pending;
    double prof_ms[MPPI_KERNEL_KINDS] = {0};
    int64_t prof_n[MPPI_KERNEL_KINDS] = {0};
    // CUDA-graph replay of mppi_optimize (world == 1): [0] generated noise, [1] supplied noise
    bool use_graph = true;
    bool collect = false;                 // launchers append to `pending` instead of launching
    bool x0_on_device = false;            // launch_rollout's x0 is a device pointer (closed loop)
    std::vector<KLaunch> pending;
    // CUDA-graph replay: [0] generated noise, [1] supplied noise, [2] noise drawn ahead (this
    // step's noise came from the previous call's side branch)
    GraphState graphs[3];
    // noise ahead (MPPI_OPTION_NOISE_AHEAD): after a separate-noise step's graph, the NEXT
    // step's noise (seed, step + 1) is drawn on a side stream into the other of two buffers; the
    // next call with that (seed, step) skips its noise kernel (and waits for ev_side_done)
    bool noise_ahead = false;             // default 0 (profiles/r2_ab_noise_ahead_latency.txt)
    float* d_eps2 = nullptr;              // [T][K_loc][m] (K_loc < kPackedMinK only)
    cudaStream_t side_stream = nullptr;
    cudaEvent_t ev_chain_done = nullptr, ev_side_done = nullptr;
    bool side_pending = false;            // a side launch may still be running
    bool ahead_ok = false;
    const float* ahead_buf = nullptr;
    uint64_t ahead_seed = 0, ahead_step = 0;
    GraphState loop_graph;                // mppi_closed_loop's n-step graph, reused while its kernel sequence is unchanged
    // row (e): a communicator the library drives itself (mppi_nccl_attach)
    void* nccl = nullptr;                 // ncclComm_t
    float* d_commbuf = nullptr;           // [T + T*m]: [eta, A] (trajectory: 1 + T*m used) all-reduced across ranks
    float* d_grec = nullptr;              // one-collective combine: this rank's record [gather_record_len]
    float* d_gather = nullptr;            // and every rank's, [world][gather_record_len]
    bool gather_combine = true;           // MPPI_OPTION_GATHER_COMBINE
};

// Launch (or collect, see Ctx::collect) one kernel whose single parameter is `args`.
cudaError_t emit(Ctx& c, const void* func, dim3 grid, dim3 block, size_t smem, const void* args,
                 size_t size, int kind);

// Brackets one kernel launch with CUDA events when profiling is on.
struct ProfScope {
    Ctx& c;
    int kind;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(Ctx& c_, int kind_);
    ~ProfScope();
};

// launchers (mppi_kernels.cu); each returns the CUDA error of the launch
cudaError_t launch_noise(Ctx& c, uint64_t seed, uint64_t step, float* out, bool reset_key);
cudaError_t launch_rollout(Ctx& c, const float* x0, const float* U, const float* eps,
                           float* costs_out);
cudaError_t launch_wsum(Ctx& c, const float* eps, const long long* key);
cudaError_t launch_finalize(Ctx& c, const float* buf_in, float* buf_out, float* U);
cudaError_t launch_shift(Ctx& c, float* U, const float* u_init);
int wsum_blocks_per_sm(int m);  // resident wsum CTAs per SM (occupancy API)
bool fused_noise_applies(const Ctx& c);  // the rollout kernel for c can draw its own noise
size_t rollout_smem_bytes(const Ctx& c, bool cells);   // dynamic smem of the rollout kernels
size_t smem_optin_bytes();                             // the device's per-block opt-in limit
bool grid_on(const Ctx& c);              // the obstacle candidate grid is in use
bool epi_applies(const Ctx& c);          // the packed rollout can run the fused reduction
cudaError_t launch_epi_combine(Ctx& c, const long long* key);
// one-collective combine (MPPI_OPTION_GATHER_COMBINE): record = [key (2 words), eta, A[T*m], pad]
inline int64_t gather_record_len(const Ctx& c) { return 2 + (((int64_t)c.T * c.m + 1 + 1) & ~(int64_t)1); }
cudaError_t launch_finalize_record(Ctx& c, float* rec_out);
cudaError_t launch_finalize_gathered(Ctx& c, const float* gathered, int n_rec, float* U);
// NCCL (mppi_nccl.cu): runtime-resolved, 0 on success, >0 ncclResult_t, -1 unavailable
bool nccl_available();
int nccl_unique_id(unsigned char* out);
int nccl_attach(Ctx& c, const unsigned char* id_bytes);
void nccl_detach(Ctx& c);
const char* nccl_error(int r);
int nccl_min_key(Ctx& c, long long* key);
int nccl_min_f32(Ctx& c, float* buf, size_t count);
int nccl_sum_buf(Ctx& c, float* buf, size_t count);
int nccl_all_gather(Ctx& c, const float* send, float* recv, size_t count);   // recv: [world][count]
int nccl_async_error(Ctx& c);             // nonzero: the communicator reported an asynchronous error
int nccl_sum_f64(Ctx& c, double* buf, size_t count);
cudaError_t launch_fk_reduce(Ctx& c, double* part, int nblk);   // Feynman-Kac partial sums
cudaError_t launch_ctg(Ctx& c);                                  // cost-to-go + per-t minima
cudaError_t launch_wsum_ctg(Ctx& c, const float* eps);
// buf_out: write [eta_t, A] (partials for the SUM allreduce); buf_in: apply from the summed buffer
cudaError_t launch_finalize_ctg(Ctx& c, float* U, const float* buf_in = nullptr, float* buf_out = nullptr);
cudaError_t launch_advance(Ctx& c, float* x, float* U, const float* u_init, float* x_log,
                           float* u_log, float* q_log);             // closed-loop plant step + shift

// host plant step (mppi_runtime.cu uses it for mppi_plant_step)
float host_plant_step(const Ctx& c, float* x, const float* u, int32_t* crashed);

}  // namespace mppi

struct mppi_ctx {
    mppi::Ctx c;
};
