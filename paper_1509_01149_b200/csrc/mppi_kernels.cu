// mppi_kernels.cu — the sm_100a kernels of one MPPI step (Alg. 1, :356-368).
//
//   K1 noise_kernel       eps[t][k][0..m) from Philox4x32-10 + BM32       (HBM write / int ALU)
//   K2 rollout_kernel     one sample per thread, state in registers, T Euler steps accumulating
//                         S~_k = sum_t q~; block min -> atomicMin key
//      rollout_kernel_x2  the quadrotor two samples per thread in packed FP32x2 (the C5 path);
//                         both can draw eps themselves (GEN: K1's values, written for K3), find
//                         the nearest cylinder through the candidate grid, and keep the step
//                         loop one basic block (rare fallbacks replay the sample)   (issue bound)
//   K3 wsum_tma_kernel    w_k = exp(-(S~_k - S_min)/lambda) and A[t][j] = sum_k w_k eps[t][k][j]:
//      wsum_kernel        the memory-bound K x (T m) GEMV, per-chunk partials; the tma variant
//                         streams eps through a bulk-copy ring (K_loc >= 65536) (HBM read bound)
//   K4 finalize_kernel    fixed-order sum of partials, U_t += sqrt(nu) L A_t / eta
//   K5 shift_kernel       U_i = U_{i+1}, U_{T-1} = u_init
//   NEXT rows: ctg_* (cost-to-go weights), advance_kernel (on-device closed loop),
//   fk_reduce_kernel (Feynman-Kac), general A_t through the !DIAG rollout path.
//
// No float atomics anywhere: every reduction has a fixed order, so a step is bitwise
// reproducible run to run.  The only atomic is an integer atomicMin on the
// 64-bit (cost, k) key, which is order independent.
#include <climits>
#include <cstring>
#include <type_traits>

#include "mppi_internal.h"

namespace mppi {

// ------------------------------------------------------------------------------ helpers
template <int M>
__device__ __forceinline__ void store_eps(float* p, const float* z) {
    if constexpr (M == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(z[0], z[1], z[2], z[3]);
    } else if constexpr (M == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(z[0], z[1]);
    } else {
        *p = z[0];
    }
}

// Programmatic dependent launch (MPPI_OPTION_PDL: the step graph's kernel->kernel edges are
// programmatic): a kernel's CTAs may be launched as its predecessor's last CTAs exit; pdl_wait()
// blocks until the predecessor grid has completed and its memory is visible (a no-op for an
// ordinary launch).  No kernel triggers its successor early: measured on B200, early triggers
// let waiting reduction CTAs crowd the rollout (C2 42 -> 118 us).  Every kernel waits before it
// reads anything a predecessor writes.  Only the rollout kernels read before the wait, and only
// inputs no kernel of a step graph writes: U, R, the per-step matrices, obstacles and the cell
// grid (U is written by finalize, the LAST node of the step graph; the closed-loop graph, where
// advance writes U before the next step's rollout, uses ordinary edges).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Per-thread asynchronous copy of one noise element group (4m bytes) into shared memory
// (LDGSTS: cp.async, non-blocking, no register tied to the load).  dst: shared-window address.
template <int M>
__device__ __forceinline__ void cp_async_eps(unsigned dst, const float* gsrc) {
    if constexpr (M == 4) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(gsrc) : "memory");
    } else if constexpr (M == 2) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(gsrc) : "memory");
    } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(gsrc) : "memory");
    }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int M>
__device__ __forceinline__ void load_shared_eps(unsigned src, float* e) {
    if constexpr (M == 4) {
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                     : "=f"(e[0]), "=f"(e[1]), "=f"(e[2]), "=f"(e[3]) : "r"(src) : "memory");
    } else if constexpr (M == 2) {
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(e[0]), "=f"(e[1]) : "r"(src) : "memory");
    } else {
        asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(e[0]) : "r"(src) : "memory");
    }
}

// Order-preserving signed map of fp32 bits, then (cost, k) packed so that signed int64 MIN
// picks the smallest cost and, among ties, the smallest global k.
__device__ __forceinline__ long long cost_key(float s, unsigned k) {
    int b = __float_as_int(s);
    b = b >= 0 ? b : (b ^ 0x7fffffff);
    return (long long)(((unsigned long long)(unsigned)b << 32) | (unsigned long long)k);
}

__device__ __forceinline__ float key_cost(long long key) {
    int b = (int)(key >> 32);
    b = b >= 0 ? b : (b ^ 0x7fffffff);
    return __int_as_float(b);
}

__device__ __forceinline__ long long warp_min_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------------------------ K1 noise
// Grid (ceil(K_loc/256), ceil(T/kNoiseTT)): each thread owns one sample k and kNoiseTT timesteps
// (independent Philox calls, unrolled by two for ILP), so the per-thread setup is amortised.
// Block (0,0) also resets the min key for the rollout that follows on the same stream.
struct NoiseArgs {
    float* eps;
    int K_loc, T;
    unsigned k_offset, step_lo, step_hi;
    PhiloxKeys keys;
    long long* key_reset;   // min key to reset (block (0,0)) or nullptr
};

template <int M>
__global__ void __launch_bounds__(256) noise_kernel(const NoiseArgs a) {
    pdl_wait();                        // (first node of a step graph today; waits if ever chained)
    const int k = blockIdx.x * 256 + threadIdx.x;
    const int t0 = blockIdx.y * kNoiseTT;
    if (a.key_reset && k == 0 && t0 == 0) *a.key_reset = LLONG_MAX;
    if (k >= a.K_loc) return;
    const unsigned kg = a.k_offset + (unsigned)k;
    const int t1 = min(t0 + kNoiseTT, a.T);
    const size_t row = (size_t)a.K_loc * M;
    float* p = a.eps + ((size_t)t0 * a.K_loc + k) * M;
    int t = t0;
    // two timesteps per iteration: their Box-Muller transforms run as packed FP32x2 (each lane
    // of FFMA2/FMUL2/FADD2 is the same IEEE operation as the scalar sequence)
    for (; t + 1 < t1; t += 2, p += 2 * row) {
        const uint4 wa = philox4x32_10_dev(kg, (unsigned)t, a.step_lo, a.step_hi, a.keys);
        const uint4 wb = philox4x32_10_dev(kg, (unsigned)(t + 1), a.step_lo, a.step_hi, a.keys);
        float za[M], zb[M];
        bm32_normals_x2<M>(wa, wb, za, zb);
        store_eps<M>(p, za);
        store_eps<M>(p + row, zb);
    }
    if (t < t1) {
        const uint4 w = philox4x32_10_dev(kg, (unsigned)t, a.step_lo, a.step_hi, a.keys);
        float z[M];
        bm32_normals<M>(w, z);
        store_eps<M>(p, z);
    }
}

// ------------------------------------------------------------------------------ K2 rollout
template <class PP>
struct RolloutArgs {
    const float* eps;       // [T][K_loc][M]
    const float* U;         // [T][M]
    float* costs;           // [K_loc] (context copy)
    float* costs_out;       // [K_loc] caller copy or nullptr
    long long* min_key;     // reset to INT64_MAX before launch
    unsigned long long* replays;   // cumulative count of replayed rollouts (one per sample / pair)
    const float4* obs;      // negated obstacle pairs
    int n_obs_pairs;
    int T;
    int K_loc;
    unsigned k_offset;
    float dt, c1, penalty;
    float sL[16];           // sqrt(nu) chol(Sigma), row-major M x M
    float R[16];
    float sd[4];            // diagonal path: s_i = sL[i][i]
    float ad[4];            // diagonal path: a_i = (1 - 1/nu)/2 R_ii s_i^2
    float x0[16];
    const float* x0_dev;    // device-resident x0 (closed loop) or nullptr: use x0[]
    float* qstep;           // [T][K_loc] per-step q~_{t,k} (cost-to-go weighting) or nullptr
    const float* mats;      // general path: [T][2][16] = (F_t = A_t L, G_t = (R - A^-T R A^-1)/2) or nullptr
    PP P;
    float4 obs_k[kMaxStaticPairs];  // negated obstacle pairs again, in the parameter constant bank
    // nearest-cylinder candidate grid (NP == kCellGrid): staged into shared memory per CTA
    const uint32_t* cells;
    const float2* cent;
    int cell_nx, cell_ny, n_cent;
    float cell_ox, cell_oy, cell_inv_h, cell_band;
    // fused reduction (EPI): per-CTA [A_c[T][M], m_c, eta_c, pad, pad] against the CTA's minimum
    float* epi_part;
    // fused cost-to-go pass (QSTEP && EPI): per-t CTA minima of S~_{t,k}, [T][gridDim.x]
    float* ctg_partmin;
    float lambda;
    // fused noise (GEN kernels): eps[t][k] drawn in-kernel with the K1 counters and written here
    float* eps_out;
    unsigned step_lo, step_hi;
    PhiloxKeys keys;
};

// Per-thread stream of eps[t][k] (M floats) for t = 0..T-1 through a kEpsStages-slot shared
// memory ring (sRing: [kEpsStages][blockDim][M]) filled by cp.async: the copy for step
// t + kEpsStages - 1 is issued before step t is consumed, so at small K (a step shorter than an
// L2 round trip) the step loop does not wait on memory.  f(t, e) consumes step t.
template <int M, class F>
__device__ __forceinline__ void eps_ring_loop(const float* eps, size_t row, int T, int k, float* sRing, F&& f) {
    constexpr int S = kEpsStages;
    const unsigned slot0 = (unsigned)__cvta_generic_to_shared(sRing + threadIdx.x * M);
    const unsigned slot_stride = blockDim.x * M * (unsigned)sizeof(float);
    const float* gp = eps + (size_t)k * M;                             // next step to issue
#pragma unroll
    for (int j = 0; j < S - 1; ++j) {
        if (j < T) cp_async_eps<M>(slot0 + j * slot_stride, gp + j * row);
        cp_async_commit();
    }
    gp += (size_t)(S - 1) * row;
    int slot_issue = S - 1, slot_use = 0;
    for (int t = 0; t < T; ++t) {
        if (t + S - 1 < T) cp_async_eps<M>(slot0 + slot_issue * slot_stride, gp);
        cp_async_commit();
        gp += row;
        slot_issue = slot_issue + 1 == S ? 0 : slot_issue + 1;
        cp_async_wait<S - 1>();                                        // step t has landed
        float e[M];
        load_shared_eps<M>(slot0 + slot_use * slot_stride, e);
        slot_use = slot_use + 1 == S ? 0 : slot_use + 1;
        f(t, e);
    }
}

// One sample's rollout state and its step t for the one-sample kernels.
// sMat: per-t F_t, G_t of the general path (!DIAG).
template <class Plant, bool DIAG, int NP, bool QSTEP = false>
struct ScalarRollout {
    static constexpr int M = Plant::M;
    const RolloutArgs<typename Plant::Params>& a;
    const ObstacleView& ob;
    const float* sMat;
    int k;
    Plant st;
    float S = 0.0f;
    float is_prev = 0.0f;                                              // IS term of step t-1
    bool slow = false;                                                 // a fast-path range miss

    __device__ __forceinline__ ScalarRollout(const RolloutArgs<typename Plant::Params>& a_, const ObstacleView& ob_,
                                             const float* sMat_, int k_)
        : a(a_), ob(ob_), sMat(sMat_), k(k_) {
        reset();
    }

    __device__ __forceinline__ void reset() {
        st.load(a.x0_dev ? a.x0_dev : a.x0, 0);
        S = 0.0f;
        is_prev = 0.0f;
    }

    // SAFE = false (the hot loop): the fast transcendental path only, recording in `slow`
    // whether an argument left its range (no branch in the step body); SAFE = true (replay()):
    // the per-step accurate fallback.
    template <bool SAFE = false>
    __device__ __forceinline__ void step(const StepRec* rec, const float* e, bool first, int t) {
        const float4 u4 = rec->u;
        const float4 b4 = rec->b;
        const float uu[4] = {u4.x, u4.y, u4.z, u4.w};
        const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
        float v[M];
        float is = rec->k.x;
        if (DIAG) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                v[i] = fmaf(a.sd[i], e[i], uu[i]);                     // U_t + s_i eps_i
                is = fmaf(e[i], fmaf(a.ad[i], e[i], bb[i]), is);       // IS_t
            }
        } else {
            // du = F_t eps (F_t = A_t L, NEXT-3; default sqrt(nu) L), IS_t = du'G_t du + (R U_t).du + K_t
            const float* F = sMat + t * 2 * M * M;
            const float* G = F + M * M;
            float du[M];
#pragma unroll
            for (int i = 0; i < M; ++i) {
                float d = 0.0f;
#pragma unroll
                for (int j = 0; j < M; ++j) d = fmaf(F[i * M + j], e[j], d);
                du[i] = d;
                v[i] = uu[i] + d;
            }
            float duGdu = 0.0f, uRdu = 0.0f;
#pragma unroll
            for (int i = 0; i < M; ++i) {   // du'G du over the staged upper triangle
                float in = du[i] * G[i * M + i];
#pragma unroll
                for (int j = i + 1; j < M; ++j) in = fmaf(G[i * M + j], du[j], in);
                duGdu = fmaf(du[i], in, duGdu);
                uRdu = fmaf(bb[i], du[i], uRdu);
            }
            is = duGdu + (uRdu + is);
        }
        // rotated step: q(x_t) (the cost of step t-1, 0 at t = 0) and F(x_t, v_t) only need
        // x_t, so they share one basic block; then x_{t+1} = x_t + F dt
        const float q = st.template state_cost<NP, SAFE>(first, a.P, ob);
        float xd[Plant::N];
        if constexpr (SAFE) {
            if (st.deriv_fast(v, a.P, xd)) st.deriv_accurate(v, a.P, xd);   // |angle| > 105615: rare
        } else {
            slow |= st.deriv_fast(v, a.P, xd);
        }
        st.update(xd, a.P, a.dt);
        S += q + is;                                                   // S~ += q~
        if constexpr (QSTEP) {                                         // q~_{t-1} = q(x_t) + IS_{t-1}
            if (!first) a.qstep[(size_t)(t - 1) * a.K_loc + k] = q + is_prev;
            is_prev = is;
        }
    }

    // the trajectory again from x0 with the per-step accurate fallback, reading back the noise
    // the hot loop used (eps: the rows it read or wrote): the inline-fallback semantics
    __device__ __forceinline__ void replay(const float* eps, const StepRec* rec) {
        reset();
        const size_t row = (size_t)a.K_loc * M;
        const float* ep = eps + (size_t)k * M;
        for (int t = 0; t < a.T; ++t, ++rec, ep += row) {
            float e[M];
#pragma unroll
            for (int i = 0; i < M; ++i) e[i] = ep[i];
            step<true>(rec, e, t == 0, t);
        }
    }

    // + q(x_T) (the cost of step T-1); non-finite -> penalty
    __device__ __forceinline__ float finish() {
        const float qT = st.template state_cost<NP, true>(false, a.P, ob);
        S += qT;
        if constexpr (QSTEP) a.qstep[(size_t)(a.T - 1) * a.K_loc + k] = qT + is_prev;
        if (!isfinite(S)) S = a.penalty;
        return S;
    }
};

// Stage the per-t constants U_t, s_i (R U_t)_i, U_t'R U_t / 2 (and, !DIAG, F_t, G_t), the
// obstacle pairs and (NP == kCellGrid) nothing else: callers add their own tables.
template <int M, bool DIAG, class PP>
__device__ __forceinline__ void stage_step_constants(const RolloutArgs<PP>& a, float4* sObs, StepRec* sRec, float* sMat) {
    const int tid = threadIdx.x;
    for (int i = tid; i < a.n_obs_pairs; i += blockDim.x) sObs[i] = a.obs[i];
    if (!DIAG) {
        for (int o = tid; o < a.T * 2 * M * M; o += blockDim.x) {
            const int t = o / (2 * M * M), r = o % (2 * M * M), which = r / (M * M), ij = r % (M * M);
            // default transform A = sqrt(nu) I: F = sqrt(nu) L, G = (1 - 1/nu)/2 R.  G is staged for
            // the quadratic form du'G du = sum_i du_i (G_ii du_i + sum_{j>i} (G_ij + G_ji) du_j):
            // its strict upper triangle holds G_ij + G_ji (the lower one is not read)
            auto g = [&](int q) { return a.mats ? a.mats[t * 32 + 16 + q] : a.c1 * a.R[q]; };
            const int i = ij / M, j = ij % M;
            sMat[o] = which == 0 ? (a.mats ? a.mats[t * 32 + ij] : a.sL[ij])
                                 : (j > i ? g(i * M + j) + g(j * M + i) : g(ij));
        }
    }
    for (int t = tid; t < a.T; t += blockDim.x) {
        float u[4] = {0.0f, 0.0f, 0.0f, 0.0f}, bq[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int i = 0; i < M; ++i) u[i] = a.U[t * M + i];
        float kk = 0.0f;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            float ru = 0.0f;
#pragma unroll
            for (int j = 0; j < M; ++j) ru = fmaf(a.R[i * M + j], u[j], ru);
            kk = fmaf(u[i], ru, kk);
            bq[i] = DIAG ? a.sd[i] * ru : ru;
        }
        StepRec r;
        r.u = make_float4(u[0], u[1], u[2], u[3]);
        r.b = make_float4(bq[0], bq[1], bq[2], bq[3]);
        r.k = make_float4(0.5f * kk, 0.0f, 0.0f, 0.0f);
        sRec[t] = r;
    }
}

// One sample per thread.  Per step t:
//   v = U_t + du,  du = sqrt(nu) L eps[t][k]
//   x <- x + F(x, v) dt,  S~ += q(x) + IS_t
//   IS_t = (1 - 1/nu)/2 du'R du + U_t'R du + U_t'R U_t/2
// With diagonal L and R (every shipped config) IS_t is evaluated as
//   IS_t = K_t + sum_i e_i (a_i e_i + b_ti),  b_ti = s_i (R U_t)_i,  K_t = U_t'R U_t/2,
// the same polynomial in eps with the per-t constants staged in shared memory.
// eps[t][k] reaches the thread through a kEpsStages-deep shared-memory ring filled by per-thread
// cp.async two steps ahead, so the HBM latency is hidden without tying up registers.
//
// GEN (diagonal Sigma and R, plants other than the quadrotor, whose large-K path is the packed
// kernel): eps[t][k] is drawn in step t with K1's counters and transform and written to eps_out.
// resident CTAs per SM the one-sample kernel is compiled for: the quadrotor (16 states, the
// obstacle search) needs up to 128 registers; the small plants fit 64
template <class Plant>
constexpr int rollout_min_blocks() { return std::is_same<Plant, Quadrotor>::value ? 4 : 8; }

// QSTEP: the per-step costs are stored for the cost-to-go weighting (a compile-time switch: a
// per-step runtime test would split the latency-bound step loop into two basic blocks).
template <class Plant, bool DIAG, int NP, bool GEN = false, bool QSTEP = false>
__global__ void __launch_bounds__(kRolloutThreads, rollout_min_blocks<Plant>())
    rollout_kernel(const __grid_constant__ RolloutArgs<typename Plant::Params> a) {
    constexpr int M = Plant::M;
    extern __shared__ float4 smem4[];
    float4* sObs = smem4;
    StepRec* sRec = reinterpret_cast<StepRec*>(smem4 + a.n_obs_pairs);   // per-t constants [T]
    float* sRing = reinterpret_cast<float*>(sRec + a.T);               // eps ring [kEpsStages][blockDim][M]
    // general path: per-t sampling factor F_t and IS matrix G_t after the ring ([T][2][M*M])
    float* sMat = sRing + (GEN ? 0 : kEpsStages * blockDim.x * M);
    // candidate grid (NP == kCellGrid, diagonal path only): centres and cell words
    float2* sCent = reinterpret_cast<float2*>(sMat + (DIAG ? 0 : a.T * 2 * M * M));
    // the cell table starts 16-byte aligned (the centre count rounded up to even; the smem size
    // reserves it) and the device table is padded to whole 16-byte groups (build_cell_grid)
    uint32_t* sCells = reinterpret_cast<uint32_t*>(sCent + ((a.n_cent + 1) & ~1));
    // candidate-grid centres in static shared memory (compile-time address: each lane's candidate
    // load is one LDS with an immediate base, no address arithmetic)
    __shared__ float sCentXY[NP == kCellGrid ? 2 * kCellMaxCent : 1];
    const int tid = threadIdx.x;
    stage_step_constants<M, DIAG>(a, sObs, sRec, sMat);
    if constexpr (NP == kCellGrid) {
        for (int i = tid; i < a.n_cent; i += blockDim.x) {   // SoA: [-x_j], then [-y_j]
            const float2 c = a.cent[i];
            sCentXY[i] = c.x;
            sCentXY[kCellMaxCent + i] = c.y;
        }
        const int nc = a.cell_nx * a.cell_ny;
        for (int i = tid; i < nc; i += blockDim.x) sCells[i] = a.cells[i];
    }
    __syncthreads();
    pdl_wait();                        // eps and the min-key reset of the noise pass

    const int k = blockIdx.x * blockDim.x + tid;
    long long key = LLONG_MAX;
    if (k < a.K_loc) {
        // compile-time pair count: read the forest from the kernel-parameter constant bank
        // (uniform-register operands, no per-thread registers); else shared memory
        ObstacleView ob{NP >= 0 ? a.obs_k : sObs, a.n_obs_pairs};
        if constexpr (NP == kCellGrid) {
            ob.cells = sCells;
            ob.cx = sCentXY;
            ob.cy = sCentXY + kCellMaxCent;
            ob.nx = a.cell_nx;
            ob.ny = a.cell_ny;
            ob.ox = a.cell_ox;
            ob.oy = a.cell_oy;
            ob.inv_h = a.cell_inv_h;
            ob.band = a.cell_band;
        }
        ScalarRollout<Plant, DIAG, NP, QSTEP> ro(a, ob, sMat, k);
        const size_t row = (size_t)a.K_loc * M;
        const StepRec* rec = sRec;
        if constexpr (GEN) {
            const unsigned kg = a.k_offset + (unsigned)k;
            float* op = a.eps_out + (size_t)k * M;
            for (int t = 0; t < a.T; ++t, ++rec, op += row) {
                float e[M];
                bm32_normals<M>(philox4x32_10_dev(kg, (unsigned)t, a.step_lo, a.step_hi, a.keys), e);
                store_eps<M>(op, e);
                ro.step(rec, e, t == 0, t);
            }
        } else {
            eps_ring_loop<M>(a.eps, row, a.T, k, sRing, [&](int t, const float* e) { ro.step(rec++, e, t == 0, t); });
        }
        if (__builtin_expect(ro.slow, 0)) {
            atomicAdd(a.replays, 1ull);
            ro.replay(GEN ? a.eps_out : a.eps, sRec);
        }
        const float S = ro.finish();
        a.costs[k] = S;
        if (a.costs_out) a.costs_out[k] = S;
        key = cost_key(S, a.k_offset + (unsigned)k);
    }
    key = warp_min_ll(key);
    __shared__ long long wmin[kRolloutThreads / 32];
    if ((tid & 31) == 0) wmin[tid >> 5] = key;
    __syncthreads();
    if (tid < 32) {
        long long v = tid < (int)(blockDim.x >> 5) ? wmin[tid] : LLONG_MAX;
        v = warp_min_ll(v);
        if (tid == 0 && v != LLONG_MAX) atomicMin(a.min_key, v);
    }
}

// ------------------------------------------------------------------------------ K2 rollout, x2
// Quadrotor with diagonal L and R: two adjacent samples per thread (k = 2j, 2j+1), every FP32
// operation packed as FP32x2 (QuadrotorX2), the obstacle-pair loads shared by both samples.
// Same per-step arithmetic and the same (cost, k) key as rollout_kernel.
//
// GEN: the kernel draws eps[t][k], eps[t][k+1] itself (Philox counters (k_global, t, step), the
// same packed Box-Muller as K1, so the values are bit-identical to K1's) in step t, and writes
// them to eps_out for K3; the noise pass and its HBM round trip disappear and the integer/MUFU
// noise arithmetic interleaves with the FMA-heavy dynamics of the same step.
// QSTEP: per-step costs stored for the cost-to-go weighting (compile-time: 2.4 % at C5).
//
// DIAG = false (correlated Sigma, per-step A_t of NEXT-3): du = F_t eps and the full quadratic
// IS_t with the per-t matrices staged in shared memory, lane-wise the one-sample kernel's order.
//
// EPI: the weighted-noise sums start inside this kernel.  After its samples are rolled out, a
// CTA weights them against ITS minimum, w = exp(-(S - m_c)/lambda), and re-reads its own noise
// tile (written moments ago) to form eta_c and A_c[t][j]; the HBM stream of that read overlaps
// the other CTAs' ALU-bound rollouts instead of running as a separate pass.  epi_combine_kernel
// rescales by exp(-(m_c - S_min)/lambda) (the online-softmax identity) in a fixed order.
template <int NP, bool GEN, bool QSTEP = false, bool DIAG = true, bool EPI = false>
__global__ void __launch_bounds__(kRolloutThreads, MPPI_X2_MINB)
    rollout_kernel_x2(const __grid_constant__ RolloutArgs<QuadrotorParams> a) {
    constexpr int M = 4;
    extern __shared__ float4 smem4[];
    float4* sObs = smem4;
    StepRec* sRec = reinterpret_cast<StepRec*>(smem4 + a.n_obs_pairs);
    float* sRing = reinterpret_cast<float*>(sRec + a.T);               // [2][blockDim][2 samples][4]
    float* sMat = sRing + (GEN ? 0 : 2 * kRolloutThreads * 2 * 4);     // !DIAG: [T][2][M*M]
    float2* sCent = reinterpret_cast<float2*>(sMat + (DIAG ? 0 : a.T * 2 * M * M));
    // the cell table starts 16-byte aligned (the centre count rounded up to even; the smem size
    // reserves it) and the device table is padded to whole 16-byte groups (build_cell_grid)
    uint32_t* sCells = reinterpret_cast<uint32_t*>(sCent + ((a.n_cent + 1) & ~1));
    // candidate-grid centres in static shared memory (compile-time address: each lane's candidate
    // load is one LDS with an immediate base, no address arithmetic)
    __shared__ float sCentXY[NP == kCellGrid ? 2 * kCellMaxCent : 1];
    const int tid = threadIdx.x;
    // (DIAG keeps its own staging, in this order: the shared helper, or another order, costs
    // the hot loop 4 % through ptxas' register allocation)
    if constexpr (DIAG) {
        for (int i = tid; i < a.n_obs_pairs; i += blockDim.x) sObs[i] = a.obs[i];
    }
    if constexpr (NP == kCellGrid) {
        for (int i = tid; i < a.n_cent; i += blockDim.x) {   // SoA: [-x_j], then [-y_j]
            const float2 c = a.cent[i];
            sCentXY[i] = c.x;
            sCentXY[kCellMaxCent + i] = c.y;
        }
        // 16-byte loads, eight in flight per thread, no alignment test or tail: the 22 KB table
        // arrives in a few L2 round trips instead of ~45 dependent load/store pairs per thread,
        // and the step loop's register allocation comes out faster too (C5 -1.4 %, K = 2^16..2^20
        // -1.6..2 %; profiles/r2_ab_cell_staging.txt)
        const uint4* src = reinterpret_cast<const uint4*>(a.cells);
        uint4* dst = reinterpret_cast<uint4*>(sCells);
        const int n4 = (a.cell_nx * a.cell_ny + 3) >> 2;
#pragma unroll 8   // (4: +0.2 % at C5, profiles/r2_ab_cell_staging.txt)
        for (int i = tid; i < n4; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    if constexpr (DIAG) {
        for (int t = tid; t < a.T; t += blockDim.x) {
            float u[4], bq[4];
            float kk = 0.0f;
#pragma unroll
            for (int i = 0; i < M; ++i) u[i] = a.U[t * M + i];
#pragma unroll
            for (int i = 0; i < M; ++i) {
                float ru = 0.0f;
#pragma unroll
                for (int j = 0; j < M; ++j) ru = fmaf(a.R[i * M + j], u[j], ru);
                kk = fmaf(u[i], ru, kk);
                bq[i] = a.sd[i] * ru;
            }
            StepRec r;
            r.u = make_float4(u[0], u[1], u[2], u[3]);
            r.b = make_float4(bq[0], bq[1], bq[2], bq[3]);
            r.k = make_float4(0.5f * kk, 0.0f, 0.0f, 0.0f);
            sRec[t] = r;
        }
    } else {
        stage_step_constants<M, DIAG>(a, sObs, sRec, sMat);
    }
    __syncthreads();
    pdl_wait();

    const int k = 2 * (blockIdx.x * blockDim.x + tid);                 // samples k, k+1
    long long key = LLONG_MAX;
    float cost_a = 0.0f, cost_b = 0.0f;                                // (EPI)
    if (k < a.K_loc) {
        QuadrotorX2 st;
        st.load(a.x0_dev ? a.x0_dev : a.x0);
        ObstacleView ob{NP >= 0 ? a.obs_k : sObs, a.n_obs_pairs};
        if constexpr (NP == kCellGrid) {
            ob.cells = sCells;
            ob.cx = sCentXY;
            ob.cy = sCentXY + kCellMaxCent;
            ob.nx = a.cell_nx;
            ob.ny = a.cell_ny;
            ob.ox = a.cell_ox;
            ob.oy = a.cell_oy;
            ob.inv_h = a.cell_inv_h;
            ob.band = a.cell_band;
        }
        const size_t row = (size_t)a.K_loc * M;
        V2 S = vb(0.0f);
        V2 is_prev = vb(0.0f);
        const float* gp = a.eps + (size_t)k * M;                       // 32 contiguous bytes
        const unsigned slot0 = (unsigned)__cvta_generic_to_shared(sRing + tid * 2 * M);
        const unsigned slot_sum = 2u * slot0 + blockDim.x * 2 * M * (unsigned)sizeof(float);
        unsigned cur = slot0;
        const unsigned kg = a.k_offset + (unsigned)k;
        float4* op = GEN ? reinterpret_cast<float4*>(a.eps_out + (size_t)k * M) : nullptr;
        if constexpr (!GEN) {
            cp_async_eps<4>(cur, gp);
            cp_async_eps<4>(cur + 16, gp + 4);
            cp_async_commit();
        }
        // one step t of both samples: v = U_t + s eps, IS_t, q(x_t), x <- x + F(x, v) dt, S~ += q~.
        // SAFE: per-step accurate fallback; else the fast path, tracking max |angle| in amax.
        float amax = 0.0f;
        auto body = [&](auto SAFE, int t, const StepRec* rc, const float* ea, const float* eb) {
            const float4 u4 = rc->u, b4 = rc->b;
            const float uu[4] = {u4.x, u4.y, u4.z, u4.w};
            const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
            V2 v[M];
            V2 is = vb(rc->k.x);
            if constexpr (DIAG) {
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    const V2 e = vp(ea[i], eb[i]);
                    v[i] = fma2(vb(a.sd[i]), e, vb(uu[i]));                    // U_t + s_i eps_i
                    is = fma2(e, fma2(vb(a.ad[i]), e, vb(bb[i])), is);        // IS_t
                }
            } else {
                // du = F_t eps, IS_t = du'G_t du + (R U_t).du + K_t (as ScalarRollout, lane-wise).
                // F_t is addressed from the shared-memory base, not a captured pointer: the DIAG
                // instantiation must not carry one more live value through the loop
                const float* F = reinterpret_cast<const float*>(smem4 + a.n_obs_pairs) + a.T * (sizeof(StepRec) / 4) +
                                 (GEN ? 0 : 2 * kRolloutThreads * 2 * 4) + t * 2 * M * M;
                const float* G = F + M * M;
                V2 du[M];
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    V2 d = vb(0.0f);
#pragma unroll
                    for (int j = 0; j < M; ++j) d = fma2(vb(F[i * M + j]), vp(ea[j], eb[j]), d);
                    du[i] = d;
                    v[i] = vb(uu[i]) + d;
                }
                V2 duGdu = vb(0.0f), uRdu = vb(0.0f);
#pragma unroll
                for (int i = 0; i < M; ++i) {   // du'G du over the staged upper triangle (as above)
                    V2 in = du[i] * vb(G[i * M + i]);
#pragma unroll
                    for (int j = i + 1; j < M; ++j) in = fma2(vb(G[i * M + j]), du[j], in);
                    duGdu = fma2(du[i], in, duGdu);
                    uRdu = fma2(vb(bb[i]), du[i], uRdu);
                }
                is = duGdu + (uRdu + is);
            }
            const V2 q = st.template state_cost<NP, decltype(SAFE)::value>(t == 0, a.P, ob);   // q(x_t): step t-1
            V2 xd[16];
            if constexpr (decltype(SAFE)::value) {
                if (st.deriv_fast(v, a.P, xd)) st.deriv_accurate(v, a.P, xd);
            } else {
                amax = fmaxf(amax, st.angle_absmax());
                st.deriv_fast_unchecked(v, a.P, xd);
            }
            st.update(xd, a.P, a.dt);
            S = S + (q + is);                                              // S~ += q~
            if constexpr (QSTEP) {
                if (t > 0) *reinterpret_cast<float2*>(a.qstep + (size_t)(t - 1) * a.K_loc + k) = (q + is_prev).v;
                is_prev = is;
            }
        };
        const StepRec* rec = sRec;
#ifndef MPPI_X2_UNROLL
#define MPPI_X2_UNROLL 2   // two steps per iteration: more scheduling freedom across the step boundary (-1 %)
#endif
#define MPPI_PRAGMA_(x) _Pragma(#x)
#define MPPI_UNROLL_(n) MPPI_PRAGMA_(unroll n)
        MPPI_UNROLL_(MPPI_X2_UNROLL)
        for (int t = 0; t < a.T; ++t, ++rec) {
            float ea[4], eb[4];
            if constexpr (GEN) {
                // eps_t enters only the motor-lag derivative and IS_t, late in the step, so it is
                // drawn in the same iteration and the scheduler overlaps it with the dynamics
                bm32_normals_x2<4>(philox4x32_10_dev(kg, (unsigned)t, a.step_lo, a.step_hi, a.keys),
                                   philox4x32_10_dev(kg + 1u, (unsigned)t, a.step_lo, a.step_hi, a.keys), ea, eb);
                op[0] = make_float4(ea[0], ea[1], ea[2], ea[3]);
                op[1] = make_float4(eb[0], eb[1], eb[2], eb[3]);
                op += row / 4;
            } else {
                gp += row;
                if (t + 1 < a.T) {
                    cp_async_eps<4>(slot_sum - cur, gp);
                    cp_async_eps<4>(slot_sum - cur + 16, gp + 4);
                }
                cp_async_commit();
                cp_async_wait<1>();
                load_shared_eps<4>(cur, ea);
                load_shared_eps<4>(cur + 16, eb);
            }
            body(std::false_type(), t, rec, ea, eb);
            cur = slot_sum - cur;
        }
        if (__builtin_expect(!(amax <= kSinCosFastMax) || st.miss, 0)) {
            atomicAdd(a.replays, 1ull);   // one per replayed pair
            // An angle left the fast sin/cos range, or a position left the obstacle grid's band
            // (or hit an overflow cell), somewhere on this pair's trajectories: replay both from
            // x0 with the per-step accurate fallbacks (the inline-fallback semantics), reading
            // back the noise this pass used.  Rare, and keeping the branches out of the hot loop
            // lets the step body schedule as one block.
            st.load(a.x0_dev ? a.x0_dev : a.x0);
            S = vb(0.0f);
            is_prev = vb(0.0f);
            const float* ep = (GEN ? a.eps_out : a.eps) + (size_t)k * M;
            rec = sRec;
            for (int t = 0; t < a.T; ++t, ++rec, ep += row) {
                const float4 e0 = *reinterpret_cast<const float4*>(ep);
                const float4 e1 = *reinterpret_cast<const float4*>(ep + 4);
                const float ea[4] = {e0.x, e0.y, e0.z, e0.w}, eb[4] = {e1.x, e1.y, e1.z, e1.w};
                body(std::true_type(), t, rec, ea, eb);
            }
        }
        const V2 qT = st.template state_cost<NP, true>(false, a.P, ob);   // q(x_T)
        S = S + qT;
        if constexpr (QSTEP) *reinterpret_cast<float2*>(a.qstep + (size_t)(a.T - 1) * a.K_loc + k) = (qT + is_prev).v;
        float sa = S.v.x, sb = S.v.y;
        if (!isfinite(sa)) sa = a.penalty;
        if (!isfinite(sb)) sb = a.penalty;
        *reinterpret_cast<float2*>(a.costs + k) = make_float2(sa, sb);
        if (a.costs_out) *reinterpret_cast<float2*>(a.costs_out + k) = make_float2(sa, sb);
        const long long ka = cost_key(sa, a.k_offset + (unsigned)k);
        const long long kb = cost_key(sb, a.k_offset + (unsigned)k + 1u);
        key = ka < kb ? ka : kb;
        cost_a = sa;
        cost_b = sb;
    }
    key = warp_min_ll(key);
    __shared__ long long wmin[kRolloutThreads / 32];
    __shared__ long long sBlockKey;
    if ((tid & 31) == 0) wmin[tid >> 5] = key;
    __syncthreads();
    if (tid < 32) {
        long long v = tid < (int)(blockDim.x >> 5) ? wmin[tid] : LLONG_MAX;
        v = warp_min_ll(v);
        if (tid == 0 && v != LLONG_MAX) atomicMin(a.min_key, v);
        if (tid == 0) sBlockKey = v;
    }
    if constexpr (QSTEP && EPI) {
        // fused cost-to-go pass (NEXT-1): ctg_kernel's arithmetic on this CTA's 256 samples --
        // each thread suffix-sums the q~ rows of its own two samples (it wrote them: program
        // order makes them visible), stores S~_{t,k} (non-finite -> penalty) in place and the
        // per-t CTA minimum goes to ctg_partmin[t][blockIdx.x]; ctg_min_kernel finishes S_min,t.
        // Same per-lane operations and order as ctg_kernel: bit-identical S~ and minima.
        constexpr int NW = kRolloutThreads / 32;
        const int lane = tid & 31, warp = tid >> 5;
        float* wmin_t = reinterpret_cast<float*>(smem4);   // [NW][T]: the staged records are dead
        const bool valid = k < a.K_loc;                     // (past the __syncthreads above)
        float2 sacc = make_float2(0.0f, 0.0f);
        constexpr int B = 8;                                // rows loaded ahead of the serial chain
        for (int t1 = a.T - 1; t1 >= 0; t1 -= B) {
            float2 q[B];
#pragma unroll
            for (int i = 0; i < B; ++i)
                q[i] = (valid && t1 - i >= 0) ? *reinterpret_cast<const float2*>(a.qstep + (size_t)(t1 - i) * a.K_loc + k)
                                              : make_float2(0.0f, 0.0f);
#pragma unroll
            for (int i = 0; i < B; ++i) {
                const int t = t1 - i;
                if (t < 0) break;
                float v = INFINITY;
                if (valid) {
                    sacc = __fadd2_rn(sacc, q[i]);
                    const float va = isfinite(sacc.x) ? sacc.x : a.penalty;
                    const float vb2 = isfinite(sacc.y) ? sacc.y : a.penalty;
                    *reinterpret_cast<float2*>(a.qstep + (size_t)t * a.K_loc + k) = make_float2(va, vb2);
                    v = fminf(va, vb2);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
                if (lane == 0) wmin_t[warp * a.T + t] = v;
            }
        }
        __syncthreads();
        for (int t = tid; t < a.T; t += blockDim.x) {
            float v = wmin_t[t];
#pragma unroll
            for (int w2 = 1; w2 < NW; ++w2) v = fminf(v, wmin_t[w2 * a.T + t]);
            a.ctg_partmin[(size_t)t * gridDim.x + blockIdx.x] = v;
            wmin_t[t] = v;                                  // m_{c,t} (only this thread reads column t)
        }
        __syncthreads();                                    // S~ rows of the whole CTA + m_{c,t}
        // fused cost-to-go reduction: per row t, w_{t,k} = exp((S~_{t,k} - m_{c,t}) (-1/lambda))
        // against the CTA's own per-t minimum, A_c[t][j] = sum_k w eps[t][k][j], eta_c[t] = sum_k w;
        // epi_combine_ctg_kernel rescales by exp((m_{c,t} - S_min,t) (-1/lambda)).  Warps take
        // rows, lanes 8 samples each (loads predicated, all in flight), as the trajectory epilogue.
        const int k0 = 2 * blockIdx.x * blockDim.x;
        const int nk = min(2 * (int)blockDim.x, a.K_loc - k0);
        float* part = a.epi_part + (size_t)blockIdx.x * ((size_t)a.T * (M + 2));   // [A (T M)][eta (T)][m (T)]
        const float* eps_src = GEN ? a.eps_out : a.eps;
        constexpr int J = 2 * kRolloutThreads / 32;
        for (int t = warp; t < a.T; t += NW) {
            const float mct = wmin_t[t];
            const float* srow = a.qstep + (size_t)t * a.K_loc + k0;
            const float4* row4 = reinterpret_cast<const float4*>(eps_src + ((size_t)t * a.K_loc + k0) * M);
            float sv[J];
            float4 e[J];
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int s2 = lane + 32 * j;
                sv[j] = s2 < nk ? srow[s2] : INFINITY;
                e[j] = s2 < nk ? __ldcs(row4 + s2) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            }
            float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            float wsum = 0.0f;
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const float w = lane + 32 * j < nk ? expf(__fmul_rn(sv[j] - mct, a.lambda)) : 0.0f;
                acc.x = fmaf(w, e[j].x, acc.x);
                acc.y = fmaf(w, e[j].y, acc.y);
                acc.z = fmaf(w, e[j].z, acc.z);
                acc.w = fmaf(w, e[j].w, acc.w);
                wsum += w;
            }
            const bool up = lane & 16, up2 = lane & 8;
            float c0 = up ? acc.z : acc.x, c1 = up ? acc.w : acc.y;
            c0 += __shfl_xor_sync(0xffffffffu, up ? acc.x : acc.z, 16);
            c1 += __shfl_xor_sync(0xffffffffu, up ? acc.y : acc.w, 16);
            float kk = up2 ? c1 : c0;
            kk += __shfl_xor_sync(0xffffffffu, up2 ? c0 : c1, 8);
            kk += __shfl_xor_sync(0xffffffffu, kk, 4);
            kk += __shfl_xor_sync(0xffffffffu, kk, 2);
            kk += __shfl_xor_sync(0xffffffffu, kk, 1);
            if ((lane & 7) == 0) part[t * M + (lane >> 3)] = kk;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
            if (lane == 0) {
                part[(size_t)a.T * M + t] = wsum;
                part[(size_t)a.T * (M + 1) + t] = mct;
            }
        }
    }
    if constexpr (EPI && !QSTEP) {
        constexpr int NW = kRolloutThreads / 32;
        __shared__ float sW[2 * kRolloutThreads];
        __shared__ float sEta[NW];
        const int lane = tid & 31, warp = tid >> 5;
        __syncthreads();                                              // sBlockKey; own eps rows
        const long long bk = sBlockKey;
        if (bk == LLONG_MAX) return;                                  // no sample in this CTA
        const float mc = key_cost(bk);
        const bool va = k < a.K_loc;
        const float wa = va ? expf(-__fdiv_rn(cost_a - mc, a.lambda)) : 0.0f;
        const float wb = va ? expf(-__fdiv_rn(cost_b - mc, a.lambda)) : 0.0f;
        sW[2 * tid] = wa;
        sW[2 * tid + 1] = wb;
        const float ew = warp_sum(wa + wb);
        if (lane == 0) sEta[warp] = ew;
        __syncthreads();
        const int k0 = 2 * blockIdx.x * blockDim.x;
        const int nk = min(2 * (int)blockDim.x, a.K_loc - k0);
        float* part = a.epi_part + (size_t)blockIdx.x * (a.T * M + 4);   // [A (T M)][m_c, eta_c, -, -]
        const float* eps_src = GEN ? a.eps_out : a.eps;
        // four sums across the warp in 6 shuffles (transpose-reduce, fixed order): after the
        // offset-16 and offset-8 exchanges lane l holds component 2*(l>>4 & 1) + (l>>3 & 1)
        auto reduce_store = [&](const float4 acc, int t) {
            const bool up = lane & 16, up2 = lane & 8;
            float k0 = up ? acc.z : acc.x, k1 = up ? acc.w : acc.y;
            k0 += __shfl_xor_sync(0xffffffffu, up ? acc.x : acc.z, 16);
            k1 += __shfl_xor_sync(0xffffffffu, up ? acc.y : acc.w, 16);
            float kk = up2 ? k1 : k0;
            kk += __shfl_xor_sync(0xffffffffu, up2 ? k0 : k1, 8);
            kk += __shfl_xor_sync(0xffffffffu, kk, 4);
            kk += __shfl_xor_sync(0xffffffffu, kk, 2);
            kk += __shfl_xor_sync(0xffffffffu, kk, 1);
            if ((lane & 7) == 0) part[t * M + (lane >> 3)] = kk;   // lanes 0, 8, 16, 24: j = 0..3
        };
        auto fma4 = [](float4& acc, float w, const float4 e) {   // two FFMA2 (same per-lane fma)
            const float2 ww = make_float2(w, w);
            const float2 lo = __ffma2_rn(ww, make_float2(e.x, e.y), make_float2(acc.x, acc.y));
            const float2 hi = __ffma2_rn(ww, make_float2(e.z, e.w), make_float2(acc.z, acc.w));
            acc = make_float4(lo.x, lo.y, hi.x, hi.y);
        };
        if (nk == 2 * kRolloutThreads) {
            // full CTA: the lane's 8 weights in registers, MPPI_EPI_ROWS rows (8 independent 16-byte
            // loads each) in flight per lane -- the re-read comes from HBM, so the epilogue is
            // latency-bound on how many loads a warp has outstanding.  Same summation order as
            // the loop below.
            constexpr int J = 2 * kRolloutThreads / 32;
            float wr[J];
#pragma unroll
            for (int j = 0; j < J; ++j) wr[j] = sW[lane + 32 * j];
            auto rows = [&](auto RN, int t) {
                constexpr int R = decltype(RN)::value;
                const float4* r0 = reinterpret_cast<const float4*>(eps_src + ((size_t)t * a.K_loc + k0) * M);
                float4 e[R][J];
#pragma unroll
                for (int j = 0; j < J; ++j)
#pragma unroll
                    for (int r = 0; r < R; ++r) e[r][j] = __ldcs(r0 + (size_t)r * NW * a.K_loc + lane + 32 * j);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
                    for (int j = 0; j < J; ++j) fma4(acc, wr[j], e[r][j]);
                    reduce_store(acc, t + r * NW);
                }
            };
            int t = warp;
            for (; t + (MPPI_EPI_ROWS - 1) * NW < a.T; t += MPPI_EPI_ROWS * NW)
                rows(std::integral_constant<int, MPPI_EPI_ROWS>(), t);
            for (; t < a.T; t += NW) rows(std::integral_constant<int, 1>(), t);
        } else {
            for (int t = warp; t < a.T; t += NW) {
                const float4* row4 = reinterpret_cast<const float4*>(eps_src + ((size_t)t * a.K_loc + k0) * M);
                float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll 4
                for (int s2 = lane; s2 < nk; s2 += 32) fma4(acc, sW[s2], row4[s2]);
                reduce_store(acc, t);
            }
        }
        if (tid == 0) {
            float eta = 0.0f;
#pragma unroll
            for (int w2 = 0; w2 < NW; ++w2) eta += sEta[w2];
            part[a.T * M] = mc;
            part[a.T * M + 1] = eta;
        }
    }
}

// EPI combine: the per-CTA partials of rollout_kernel_x2<..., EPI> rescaled to the global minimum
// S_min (the min key), exp(-(S - S_min)/l) = exp(-(S - m_c)/l) exp(-(m_c - S_min)/l), summed in
// CTA order within chunks of cpc CTAs into K4's partial layout [chunk][T][M] + [chunk] eta.
struct EpiCombineArgs {
    const float* epi_part;   // [nblk][T M + 4]
    const long long* key;
    float* part;             // [n_chunks][T M]
    float* eta_part;         // [n_chunks]
    int nblk, cpc, TM;
    float lambda;
};

__global__ void __launch_bounds__(256) epi_combine_kernel(const EpiCombineArgs a) {
    pdl_wait();
    __shared__ float sc[256];
    const int chunk = blockIdx.x;
    const int c0 = chunk * a.cpc, c1 = min(a.nblk, c0 + a.cpc);
    const size_t stride = (size_t)a.TM + 4;
    const float smin = key_cost(*a.key);
    for (int i = threadIdx.x; i < c1 - c0; i += blockDim.x)
        sc[i] = expf(-__fdiv_rn(__ldg(a.epi_part + (size_t)(c0 + i) * stride + a.TM) - smin, a.lambda));
    __syncthreads();
    const int o = blockIdx.y * blockDim.x + threadIdx.x;   // o < TM: A[o]; o == TM: eta
    if (o > a.TM) return;
    const int idx = o < a.TM ? o : a.TM + 1;
    float acc = 0.0f;
#ifndef MPPI_COMBINE_UNROLL
#define MPPI_COMBINE_UNROLL 32   // C5: 113 us (no unroll), 42 (16), 31 (32); profiles/r2_ab_combine_unroll.txt
#endif
    MPPI_UNROLL_(MPPI_COMBINE_UNROLL)   // independent loads in flight; the fma chain keeps CTA order
    for (int c = c0; c < c1; ++c) acc = fmaf(sc[c - c0], __ldg(a.epi_part + (size_t)c * stride + idx), acc);
    if (o < a.TM) a.part[(size_t)chunk * a.TM + o] = acc;
    else a.eta_part[chunk] = acc;
}

// cost-to-go version: per-(CTA, t) partials [A (T M)][eta (T)][m (T)] of the fused epilogue,
// rescaled by exp((m_{c,t} - S_min,t) (-1/lambda)) and summed in CTA order within chunks of cpc
// CTAs into wsum_ctg's layout: part [chunk][T][M], eta_part [chunk][T].
struct EpiCombineCtgArgs {
    const float* epi_part;   // [nblk][T (M + 2)]
    const float* smin;       // [T]
    float* part;             // [n_chunks][T][M]
    float* eta_part;         // [n_chunks][T]
    int nblk, cpc, T;
    float neg_inv_lambda;
};

__global__ void __launch_bounds__(256) epi_combine_ctg_kernel(const EpiCombineCtgArgs a) {
    pdl_wait();
    constexpr int M = 4;
    const int chunk = blockIdx.x;
    const int t = blockIdx.y * blockDim.x + threadIdx.x;
    if (t >= a.T) return;
    const int c0 = chunk * a.cpc, c1 = min(a.nblk, c0 + a.cpc);
    const size_t stride = (size_t)a.T * (M + 2);
    const float sm = a.smin[t];
    float acc[M] = {0.0f, 0.0f, 0.0f, 0.0f}, eta = 0.0f;
#pragma unroll 8   // independent loads in flight (65 -> 48 us at C5)
    for (int c = c0; c < c1; ++c) {
        const float* p = a.epi_part + (size_t)c * stride;
        const float f = expf(__fmul_rn(__ldg(p + (size_t)a.T * (M + 1) + t) - sm, a.neg_inv_lambda));
#pragma unroll
        for (int j = 0; j < M; ++j) acc[j] = fmaf(f, __ldg(p + (size_t)t * M + j), acc[j]);
        eta = fmaf(f, __ldg(p + (size_t)a.T * M + t), eta);
    }
#pragma unroll
    for (int j = 0; j < M; ++j) a.part[((size_t)chunk * a.T + t) * M + j] = acc[j];
    a.eta_part[(size_t)chunk * a.T + t] = eta;
}

// ------------------------------------------------------------------------------ K3 weights + GEMV
struct WsumArgs {
    const uint8_t* flags;       // wsum_tma_kernel: per 256-column block "some weight != 0", or nullptr
    const float* eps;           // [T][K_loc][M] viewed as [T][ncols] float4
    const float* costs;         // [K_loc]
    const long long* key;       // global min key
    float* part;                // [n_chunks][T][M]
    float* eta_part;            // [n_chunks]
    int T;
    long long ncols;            // K_loc * M / 4
    long long cols_per_chunk;
    float lambda;
};

// grid (n_chunks, ceil(T / TT)); each thread owns float4 columns (4/M samples each) of its
// chunk and accumulates TT x 4 partial sums in registers over the chunk, with TT independent
// 16-byte loads in flight per iteration.  w_k is computed once per sample per t-tile.
template <int M>
__global__ void __launch_bounds__(kWsumThreads) wsum_kernel(const WsumArgs a) {
    pdl_wait();
    constexpr int SPC = 4 / M;  // samples per float4 column
    constexpr int TT = kWsumTT;
    const int chunk = blockIdx.x;
    const int t0 = blockIdx.y * TT;
    const int nt = min(TT, a.T - t0);
    const float smin = key_cost(*a.key);
    const long long c_begin = (long long)chunk * a.cols_per_chunk;
    const long long c_end = min(a.ncols, c_begin + a.cols_per_chunk);
    const float4* __restrict__ eps4 = reinterpret_cast<const float4*>(a.eps);
    const bool do_eta = blockIdx.y == 0;
    float acc[TT][4];
#pragma unroll
    for (int tt = 0; tt < TT; ++tt)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[tt][c] = 0.0f;
    float eta = 0.0f;
    for (long long col = c_begin + threadIdx.x; col < c_end; col += kWsumThreads) {
        float cs[SPC];
        if constexpr (SPC == 4) {
            const float4 c = __ldg(reinterpret_cast<const float4*>(a.costs) + col);
            cs[0] = c.x; cs[1] = c.y; cs[2] = c.z; cs[3] = c.w;
        } else if constexpr (SPC == 2) {
            const float2 c = __ldg(reinterpret_cast<const float2*>(a.costs) + col);
            cs[0] = c.x; cs[1] = c.y;
        } else {
            cs[0] = __ldg(a.costs + col);
        }
        float w[SPC];
#pragma unroll
        for (int s = 0; s < SPC; ++s) {
            w[s] = expf(-__fdiv_rn(cs[s] - smin, a.lambda));  // PAPER.md:320 (min-shifted)
            if (do_eta) eta += w[s];
        }
        float4 v[TT];
#pragma unroll
        for (int tt = 0; tt < TT; ++tt)
            if (tt < nt) v[tt] = __ldcs(eps4 + (size_t)(t0 + tt) * a.ncols + col);
#pragma unroll
        for (int tt = 0; tt < TT; ++tt) {
            if (tt < nt) {
                acc[tt][0] = fmaf(w[0 / M], v[tt].x, acc[tt][0]);
                acc[tt][1] = fmaf(w[1 / M], v[tt].y, acc[tt][1]);
                acc[tt][2] = fmaf(w[2 / M], v[tt].z, acc[tt][2]);
                acc[tt][3] = fmaf(w[3 / M], v[tt].w, acc[tt][3]);
            }
        }
    }
    // fold the 4 lanes of a column onto the M control components, then block-reduce
    __shared__ float red[kWsumThreads / 32][TT * M + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int tt = 0; tt < TT; ++tt) {
#pragma unroll
        for (int j = 0; j < M; ++j) {
            float f = 0.0f;
#pragma unroll
            for (int s = 0; s < SPC; ++s) f += acc[tt][s * M + j];
            f = warp_sum(f);
            if (lane == 0) red[warp][tt * M + j] = f;
        }
    }
    eta = warp_sum(eta);
    if (lane == 0) red[warp][TT * M] = eta;
    __syncthreads();
    if (threadIdx.x < TT * M + 1) {
        float s = 0.0f;
#pragma unroll
        for (int w = 0; w < kWsumThreads / 32; ++w) s += red[w][threadIdx.x];
        if (threadIdx.x < TT * M) {
            const int tt = threadIdx.x / M, j = threadIdx.x % M;
            if (tt < nt) a.part[((size_t)chunk * a.T + t0 + tt) * M + j] = s;
        } else if (do_eta) {
            a.eta_part[chunk] = s;
        }
    }
}

// Sparse K3 (MPPI_OPTION_SPARSE_REDUCTION): flags[b] = 1 iff some sample of the 256-column block
// b has a nonzero fp32 weight exp(-(S - S_min)/lambda) (the exact expression K3 evaluates).
// With small lambda the weights are mostly exact zeros (C1-C5: one nonzero weight), and K3 then
// streams only the flagged blocks.
template <int M>
__global__ void __launch_bounds__(kWsumThreads) wsum_flags_kernel(const WsumArgs a) {
    pdl_wait();
    constexpr int SPC = 4 / M;
    const float smin = key_cost(*a.key);
    const long long col = (long long)blockIdx.x * kWsumThreads + threadIdx.x;
    int nz = 0;
    if (col < a.ncols) {
#pragma unroll
        for (int s2 = 0; s2 < SPC; ++s2)
            nz |= expf(-__fdiv_rn(__ldg(a.costs + col * SPC + s2) - smin, a.lambda)) != 0.0f;
    }
    nz = __syncthreads_or(nz);
    if (threadIdx.x == 0) const_cast<uint8_t*>(a.flags)[blockIdx.x] = (uint8_t)(nz != 0);
}

// K3 with the bulk-copy engine (sm_90+ cp.async.bulk, SASS UBLKCP): the same partial sums, but
// the eps tiles stream into a kWsumStages-deep shared-memory ring filled by one thread with 1-D
// bulk copies (one per timestep row, CW float4 columns) and mbarrier completion, so the bytes in
// flight no longer depend on registers per thread.  Thread i owns column i of each CW-column
// block of its chunk: the per-thread accumulation order over columns is the same as wsum_kernel.
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
        : "memory");
}

template <int M>
__global__ void __launch_bounds__(kWsumThreads, 3) wsum_tma_kernel(const WsumArgs a) {
    constexpr int SPC = 4 / M;
    constexpr int TT = kWsumTT;
    constexpr int CW = kWsumThreads;                 // float4 columns per block
    constexpr int S = kWsumStages;
    constexpr int NW = kWsumThreads / 32;
    extern __shared__ __align__(128) float4 sbuf[];  // [S][TT][CW]
    __shared__ __align__(8) uint64_t full[S], empty[S];
    const int tid = threadIdx.x, lane = tid & 31;
    const int chunk = blockIdx.x;
    const int t0 = blockIdx.y * TT;
    const int nt = min(TT, a.T - t0);
    const long long c_begin = (long long)chunk * a.cols_per_chunk;
    const long long c_end = min(a.ncols, c_begin + a.cols_per_chunk);
    const long long nblk = c_end > c_begin ? (c_end - c_begin + CW - 1) / CW : 0;
    const float4* __restrict__ eps4 = reinterpret_cast<const float4*>(a.eps);
    const bool do_eta = blockIdx.y == 0;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    pdl_wait();                        // costs, key and eps of the rollout
    const float smin = key_cost(*a.key);
    // sparse mode: blocks whose every weight is exactly 0 (flags[] == 0) are skipped by producer
    // and consumers alike; they would add exact zeros, so the sums are bit-identical
    const uint8_t* flags = a.flags ? a.flags + c_begin / CW : nullptr;
    auto flagged = [&](long long j) -> bool { return !flags || flags[j] != 0; };
    auto issue = [&](long long j, int st) {
        const long long c0 = c_begin + j * CW;
        const unsigned bytes = (unsigned)(min((long long)CW, c_end - c0) * sizeof(float4));
        mbar_expect_tx(&full[st], bytes * nt);
        for (int tt = 0; tt < nt; ++tt)
            bulk_g2s(sbuf + ((size_t)st * TT + tt) * CW, eps4 + (size_t)(t0 + tt) * a.ncols + c0, bytes, &full[st]);
    };
    long long jp = 0;                  // producer (thread 0): next block to look at
    if (tid == 0) {
        int n = 0;
        for (; jp < nblk && n < S; ++jp)
            if (flagged(jp)) issue(jp, n++);
    }
    float acc[TT][4];
#pragma unroll
    for (int tt = 0; tt < TT; ++tt)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[tt][c] = 0.0f;
    float eta = 0.0f;
    long long used = 0;                // ring slots consumed
    for (long long j = 0; j < nblk; ++j) {
        if (!flagged(j)) continue;
        const int st = (int)(used % S);
        const unsigned parity = (unsigned)((used / S) & 1);
        ++used;
        const long long col = c_begin + j * CW + tid;
        const bool valid = col < c_end;
        float w[SPC];
        if (valid) {
            float cs[SPC];
            if constexpr (SPC == 4) {
                const float4 c = __ldg(reinterpret_cast<const float4*>(a.costs) + col);
                cs[0] = c.x; cs[1] = c.y; cs[2] = c.z; cs[3] = c.w;
            } else if constexpr (SPC == 2) {
                const float2 c = __ldg(reinterpret_cast<const float2*>(a.costs) + col);
                cs[0] = c.x; cs[1] = c.y;
            } else {
                cs[0] = __ldg(a.costs + col);
            }
#pragma unroll
            for (int s2 = 0; s2 < SPC; ++s2) {
                w[s2] = expf(-__fdiv_rn(cs[s2] - smin, a.lambda));   // PAPER.md:320 (min-shifted)
                if (do_eta) eta += w[s2];
            }
        }
        mbar_wait(&full[st], parity);
        if (valid) {
            const float4* tile = sbuf + (size_t)st * TT * CW + tid;
#pragma unroll
            for (int tt = 0; tt < TT; ++tt) {
                if (tt < nt) {
                    const float4 v = tile[tt * CW];
                    acc[tt][0] = fmaf(w[0 / M], v.x, acc[tt][0]);
                    acc[tt][1] = fmaf(w[1 / M], v.y, acc[tt][1]);
                    acc[tt][2] = fmaf(w[2 / M], v.z, acc[tt][2]);
                    acc[tt][3] = fmaf(w[3 / M], v.w, acc[tt][3]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (tid == 0) {
            while (jp < nblk && !flagged(jp)) ++jp;
            if (jp < nblk) {
                mbar_wait(&empty[st], parity);   // every warp is done with this slot: refill it
                issue(jp++, st);
            }
        }
    }
    __shared__ float red[NW][TT * M + 1];
    const int warp = tid >> 5;
#pragma unroll
    for (int tt = 0; tt < TT; ++tt) {
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
            float f = 0.0f;
#pragma unroll
            for (int s2 = 0; s2 < SPC; ++s2) f += acc[tt][s2 * M + jj];
            f = warp_sum(f);
            if (lane == 0) red[warp][tt * M + jj] = f;
        }
    }
    eta = warp_sum(eta);
    if (lane == 0) red[warp][TT * M] = eta;
    __syncthreads();
    if (tid < TT * M + 1) {
        float sum = 0.0f;
#pragma unroll
        for (int w2 = 0; w2 < NW; ++w2) sum += red[w2][tid];
        if (tid < TT * M) {
            const int tt = tid / M, jj = tid % M;
            if (tt < nt) a.part[((size_t)chunk * a.T + t0 + tt) * M + jj] = sum;
        } else if (do_eta) {
            a.eta_part[chunk] = sum;
        }
    }
}

// ------------------------------------------------------------------------------ K4 finalize / apply
struct FinalizeArgs {
    const float* part;
    const float* eta_part;
    int n_chunks;
    const float* buf_in;   // [1 + T*M] = [eta, A] (already summed over ranks) or nullptr
    float* buf_out;        // [1 + T*M] or nullptr
    float* U;              // [T][M] updated in place, or nullptr
    DeviceStats* stats;
    int T, M;
    float sL[16];
    const float* mats;     // per-t F_t (NEXT-3) or nullptr: U_t += sL A_t / eta
    // one-collective combine (MPPI_OPTION_GATHER_COMBINE): n_rec records of rec floats each,
    // [key (int64 as two words), eta_r, A_r[T*M], pad], every rank's sums against its OWN
    // minimum; rescaled here by exp(-(S_r - S_min)/lambda) in rank order (or nullptr)
    const float* gathered;
    int n_rec, rec;
    float lambda;
    long long* key_out;    // the global (cost, k) key, or nullptr
    float* rec_out;        // this rank's record [key, eta, A] (the key from key_src), or nullptr
    const long long* key_src;
};

__global__ void __launch_bounds__(1024) finalize_kernel(const FinalizeArgs a) {
    pdl_wait();
    extern __shared__ float sA[];  // [1 + T*M]: eta, A
    const int TM = a.T * a.M;
    if (a.gathered) {
        // global minimum over the records' keys, then the online-softmax rescale of each rank's
        // sums (the epi_combine arithmetic one level up), accumulated in rank order
        long long kmin = LLONG_MAX;
        for (int r = 0; r < a.n_rec; ++r) {
            const long long kr = *reinterpret_cast<const long long*>(a.gathered + (size_t)r * a.rec);
            kmin = kr < kmin ? kr : kmin;
        }
        const float smin = key_cost(kmin);
        for (int o = threadIdx.x; o < TM + 1; o += blockDim.x) {
            float acc = 0.0f;
            for (int r = 0; r < a.n_rec; ++r) {
                const float* rr = a.gathered + (size_t)r * a.rec;
                const float sc = expf(-__fdiv_rn(key_cost(*reinterpret_cast<const long long*>(rr)) - smin, a.lambda));
                acc = fmaf(sc, rr[2 + o], acc);
            }
            sA[o] = acc;
        }
        if (a.key_out && threadIdx.x == 0) *a.key_out = kmin;
    } else if (a.buf_in) {
        for (int o = threadIdx.x; o < TM + 1; o += blockDim.x) sA[o] = a.buf_in[o];
    } else {
        for (int o = threadIdx.x; o < TM; o += blockDim.x) {
            float s = 0.0f;
            for (int c = 0; c < a.n_chunks; ++c) s += a.part[(size_t)c * TM + o];  // chunk order
            sA[1 + o] = s;
        }
        if (threadIdx.x == 0) {
            float e = 0.0f;
            for (int c = 0; c < a.n_chunks; ++c) e += a.eta_part[c];
            sA[0] = e;
        }
    }
    __syncthreads();
    if (a.buf_out)
        for (int o = threadIdx.x; o < TM + 1; o += blockDim.x) a.buf_out[o] = sA[o];
    if (a.rec_out) {
        for (int o = threadIdx.x; o < TM + 1; o += blockDim.x) a.rec_out[2 + o] = sA[o];
        if (threadIdx.x == 0) *reinterpret_cast<long long*>(a.rec_out) = *a.key_src;
    }
    if (a.stats && threadIdx.x == 0) a.stats->eta = sA[0];
    if (a.U) {
        const float eta = sA[0];
        for (int o = threadIdx.x; o < TM; o += blockDim.x) {
            const int t = o / a.M, i = o % a.M;
            float d = 0.0f;  // d_i = sum_{j<=i} sL[i][j] A[t][j], explicit rounding order
            if (a.mats) {    // general transform: d = F_t A_t (all j)
                for (int j = 0; j < a.M; ++j)
                    d = __fadd_rn(d, __fmul_rn(a.mats[t * 32 + i * a.M + j], sA[1 + t * a.M + j]));
            } else {
                for (int j = 0; j <= i; ++j) d = __fadd_rn(d, __fmul_rn(a.sL[i * a.M + j], sA[1 + t * a.M + j]));
            }
            a.U[o] = __fadd_rn(a.U[o], __fdiv_rn(d, eta));   // U_t += sum w du / eta
        }
    }
}

// ------------------------------------------------------------------------------ NEXT-1: cost-to-go
// S~(tau_{t,k}) = sum_{j >= t} q~_{j,k} ("from time t_i onward"), in place over the
// [T][K_loc] per-step costs, reverse order per sample (coalesced rows); non-finite -> penalty.
// Per CTA and t the minimum over its samples goes to partmin[t][blockIdx.x].
struct CtgArgs {
    float* ctg;          // [T][K_loc] q~ in, S~ out
    float* partmin;      // [T][nblk]
    int T, K_loc, nblk;
    float penalty;
};

__global__ void __launch_bounds__(256) ctg_kernel(const CtgArgs a) {
    pdl_wait();
    extern __shared__ float wmin_t[];   // [8 warps][T]
    const int k = blockIdx.x * 256 + threadIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float s = 0.0f;
    constexpr int B = 8;                 // rows loaded ahead: the suffix sum is a serial chain
    for (int t1 = a.T - 1; t1 >= 0; t1 -= B) {
        float q[B];
#pragma unroll
        for (int i = 0; i < B; ++i)
            q[i] = (k < a.K_loc && t1 - i >= 0) ? a.ctg[(size_t)(t1 - i) * a.K_loc + k] : 0.0f;
#pragma unroll
        for (int i = 0; i < B; ++i) {
            const int t = t1 - i;
            if (t < 0) break;
            float v = INFINITY;
            if (k < a.K_loc) {
                s += q[i];
                v = isfinite(s) ? s : a.penalty;
                a.ctg[(size_t)t * a.K_loc + k] = v;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
            if (lane == 0) wmin_t[warp * a.T + t] = v;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < a.T; t += 256) {
        float v = wmin_t[t];
#pragma unroll
        for (int w = 1; w < 8; ++w) v = fminf(v, wmin_t[w * a.T + t]);
        a.partmin[(size_t)t * a.nblk + blockIdx.x] = v;
    }
}

// smin[t] = min over CTAs of partmin[t][.]  (one CTA per t; min is exact, order-free)
struct CtgMinArgs {
    const float* partmin;
    int nblk;
    float* smin;
};

__global__ void __launch_bounds__(256) ctg_min_kernel(const CtgMinArgs a) {
    pdl_wait();
    const int t = blockIdx.x;
    float v = INFINITY;
    for (int i = threadIdx.x; i < a.nblk; i += 256) v = fminf(v, a.partmin[(size_t)t * a.nblk + i]);
    __shared__ float r[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) r[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = r[0];
        for (int w = 1; w < 8; ++w) m = fminf(m, r[w]);
        a.smin[t] = m;
    }
}

// A[t][j] = sum_k w_{t,k} eps[t][k][j], eta_t = sum_k w_{t,k}, w_{t,k} = exp(-(S~_{t,k} - smin_t)/lambda)
// (PAPER.md:320 with per-timestep weights).  Same tiling and fixed-order reduction as wsum_kernel.
struct WsumCtgArgs {
    const float* eps;
    const float* ctg;     // [T][K_loc]
    const float* smin;    // [T]
    float* part;          // [n_chunks][T][M]
    float* eta_part;      // [n_chunks][T]
    int T, K_loc;
    long long ncols, cols_per_chunk;
    float neg_inv_lambda;   // -1/lambda (fp32 of the fp64 value)
};

template <int M>
__global__ void __launch_bounds__(kWsumThreads) wsum_ctg_kernel(const WsumCtgArgs a) {
    pdl_wait();
    constexpr int SPC = 4 / M;
    constexpr int TT = kWsumTT;
    const int chunk = blockIdx.x;
    const int t0 = blockIdx.y * TT;
    const int nt = min(TT, a.T - t0);
    const long long c_begin = (long long)chunk * a.cols_per_chunk;
    const long long c_end = min(a.ncols, c_begin + a.cols_per_chunk);
    const float4* __restrict__ eps4 = reinterpret_cast<const float4*>(a.eps);
    float acc[TT][4], eta[TT];
#pragma unroll
    for (int tt = 0; tt < TT; ++tt) {
        eta[tt] = 0.0f;
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[tt][c] = 0.0f;
    }
    for (long long col = c_begin + threadIdx.x; col < c_end; col += kWsumThreads) {
#pragma unroll
        for (int tt = 0; tt < TT; ++tt) {
            if (tt < nt) {
                const int t = t0 + tt;
                const float sm = a.smin[t];
                const float* crow = a.ctg + (size_t)t * a.K_loc + col * SPC;
                float w[SPC];
#pragma unroll
                for (int s = 0; s < SPC; ++s) {
                    // exp(-(S - S_min,t)/lambda) with a precomputed -1/lambda: no division slow
                    // path in the unrolled t-tile, so all its loads issue before the arithmetic
                    w[s] = expf(__fmul_rn(crow[s] - sm, a.neg_inv_lambda));
                    eta[tt] += w[s];
                }
                const float4 v = __ldcs(eps4 + (size_t)t * a.ncols + col);
                acc[tt][0] = fmaf(w[0 / M], v.x, acc[tt][0]);
                acc[tt][1] = fmaf(w[1 / M], v.y, acc[tt][1]);
                acc[tt][2] = fmaf(w[2 / M], v.z, acc[tt][2]);
                acc[tt][3] = fmaf(w[3 / M], v.w, acc[tt][3]);
            }
        }
    }
    __shared__ float red[kWsumThreads / 32][TT * (M + 1)];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int tt = 0; tt < TT; ++tt) {
#pragma unroll
        for (int j = 0; j < M; ++j) {
            float f = 0.0f;
#pragma unroll
            for (int s = 0; s < SPC; ++s) f += acc[tt][s * M + j];
            f = warp_sum(f);
            if (lane == 0) red[warp][tt * M + j] = f;
        }
        const float e = warp_sum(eta[tt]);
        if (lane == 0) red[warp][TT * M + tt] = e;
    }
    __syncthreads();
    if (threadIdx.x < TT * (M + 1)) {
        float s = 0.0f;
#pragma unroll
        for (int w = 0; w < kWsumThreads / 32; ++w) s += red[w][threadIdx.x];
        if (threadIdx.x < TT * M) {
            const int tt = threadIdx.x / M, j = threadIdx.x % M;
            if (tt < nt) a.part[((size_t)chunk * a.T + t0 + tt) * M + j] = s;
        } else {
            const int tt = threadIdx.x - TT * M;
            if (tt < nt) a.eta_part[(size_t)chunk * a.T + t0 + tt] = s;
        }
    }
}

// wsum_ctg_kernel with the bulk-copy engine: each stage holds TT rows of CW float4 eps columns
// and the matching TT x (CW * SPC) cost-to-go values; same per-thread accumulation order.
template <int M>
__global__ void __launch_bounds__(kWsumThreads, 2) wsum_ctg_tma_kernel(const WsumCtgArgs a) {
    pdl_wait();
    constexpr int SPC = 4 / M;
    constexpr int TT = kWsumTT;
    constexpr int CW = kWsumThreads;
    constexpr int S = kWsumCtgStages;
    constexpr int NW = kWsumThreads / 32;
    extern __shared__ __align__(128) float4 sbuf[];   // [S][TT][CW] eps, then [S][TT][CW*SPC] ctg
    float* sctg = reinterpret_cast<float*>(sbuf + (size_t)S * TT * CW);
    __shared__ __align__(8) uint64_t full[S], empty[S];
    const int tid = threadIdx.x, lane = tid & 31;
    const int chunk = blockIdx.x;
    const int t0 = blockIdx.y * TT;
    const int nt = min(TT, a.T - t0);
    const long long c_begin = (long long)chunk * a.cols_per_chunk;
    const long long c_end = min(a.ncols, c_begin + a.cols_per_chunk);
    const long long nblk = c_end > c_begin ? (c_end - c_begin + CW - 1) / CW : 0;
    const float4* __restrict__ eps4 = reinterpret_cast<const float4*>(a.eps);
    if (tid == 0) {
        for (int s2 = 0; s2 < S; ++s2) {
            mbar_init(&full[s2], 1);
            mbar_init(&empty[s2], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](long long j) {
        const int st = (int)(j % S);
        const long long c0 = c_begin + j * CW;
        const long long cols = min((long long)CW, c_end - c0);
        const unsigned eb = (unsigned)(cols * sizeof(float4));
        const unsigned cb = (unsigned)(cols * SPC * sizeof(float));
        mbar_expect_tx(&full[st], (eb + cb) * nt);
        for (int tt = 0; tt < nt; ++tt) {
            bulk_g2s(sbuf + ((size_t)st * TT + tt) * CW, eps4 + (size_t)(t0 + tt) * a.ncols + c0, eb, &full[st]);
            bulk_g2s(sctg + ((size_t)st * TT + tt) * CW * SPC, a.ctg + (size_t)(t0 + tt) * a.K_loc + c0 * SPC, cb, &full[st]);
        }
    };
    if (tid == 0)
        for (long long j = 0; j < nblk && j < S; ++j) issue(j);
    float acc[TT][4], eta[TT];
#pragma unroll
    for (int tt = 0; tt < TT; ++tt) {
        eta[tt] = 0.0f;
#pragma unroll
        for (int c2 = 0; c2 < 4; ++c2) acc[tt][c2] = 0.0f;
    }
    float sm[TT];
#pragma unroll
    for (int tt = 0; tt < TT; ++tt) sm[tt] = tt < nt ? a.smin[t0 + tt] : 0.0f;
    for (long long j = 0; j < nblk; ++j) {
        const int st = (int)(j % S);
        const unsigned parity = (unsigned)((j / S) & 1);
        const bool valid = c_begin + j * CW + tid < c_end;
        mbar_wait(&full[st], parity);
        if (valid) {
            const float4* tile = sbuf + (size_t)st * TT * CW + tid;
            const float* ctile = sctg + (size_t)st * TT * CW * SPC + tid * SPC;
#pragma unroll
            for (int tt = 0; tt < TT; ++tt) {
                if (tt < nt) {
                    float w[SPC];
#pragma unroll
                    for (int s2 = 0; s2 < SPC; ++s2) {
                        w[s2] = expf(__fmul_rn(ctile[tt * CW * SPC + s2] - sm[tt], a.neg_inv_lambda));
                        eta[tt] += w[s2];
                    }
                    const float4 v = tile[tt * CW];
                    acc[tt][0] = fmaf(w[0 / M], v.x, acc[tt][0]);
                    acc[tt][1] = fmaf(w[1 / M], v.y, acc[tt][1]);
                    acc[tt][2] = fmaf(w[2 / M], v.z, acc[tt][2]);
                    acc[tt][3] = fmaf(w[3 / M], v.w, acc[tt][3]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (tid == 0 && j + S < nblk) {
            mbar_wait(&empty[st], parity);
            issue(j + S);
        }
    }
    __shared__ float red[NW][TT * (M + 1)];
    const int warp = tid >> 5;
#pragma unroll
    for (int tt = 0; tt < TT; ++tt) {
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
            float f = 0.0f;
#pragma unroll
            for (int s2 = 0; s2 < SPC; ++s2) f += acc[tt][s2 * M + jj];
            f = warp_sum(f);
            if (lane == 0) red[warp][tt * M + jj] = f;
        }
        const float e = warp_sum(eta[tt]);
        if (lane == 0) red[warp][TT * M + tt] = e;
    }
    __syncthreads();
    if (tid < TT * (M + 1)) {
        float sum = 0.0f;
#pragma unroll
        for (int w2 = 0; w2 < NW; ++w2) sum += red[w2][tid];
        if (tid < TT * M) {
            const int tt = tid / M, jj = tid % M;
            if (tt < nt) a.part[((size_t)chunk * a.T + t0 + tt) * M + jj] = sum;
        } else {
            const int tt = tid - TT * M;
            if (tt < nt) a.eta_part[(size_t)chunk * a.T + t0 + tt] = sum;
        }
    }
}

// U_t += sqrt(nu) L A_t / eta_t (per-timestep normalisers), fixed order over chunks
struct FinalizeCtgArgs {
    const float* part;
    const float* eta_part;
    int n_chunks;
    const float* buf_in;   // [T + T*M] = [eta_t, A] already summed over ranks, or nullptr
    float* buf_out;        // [T + T*M] (partials mode: no update), or nullptr
    float* U;
    DeviceStats* stats;
    int T, M;
    float sL[16];
    const float* mats;
};

// fixed-order sums over chunks, then U_t += sqrt(nu) L A_t / eta_t.  Sharded (row e): a
// partials pass writes [eta_t, A] for the SUM allreduce, an apply pass reads it back; the
// arithmetic is the same as the one-pass form, so one rank reproduces it bit for bit.
__global__ void __launch_bounds__(1024) finalize_ctg_kernel(const FinalizeCtgArgs a) {
    pdl_wait();
    const int TM = a.T * a.M;
    if (a.buf_out) {
        for (int o = threadIdx.x; o < a.T + TM; o += blockDim.x) {
            float v = 0.0f;
            if (o < a.T) {
                for (int c = 0; c < a.n_chunks; ++c) v += a.eta_part[(size_t)c * a.T + o];
            } else {
                const int tj = o - a.T, t = tj / a.M, j = tj % a.M;
                for (int c = 0; c < a.n_chunks; ++c) v += a.part[((size_t)c * a.T + t) * a.M + j];
            }
            a.buf_out[o] = v;
        }
        return;
    }
    for (int o = threadIdx.x; o < TM; o += blockDim.x) {
        const int t = o / a.M, i = o % a.M;
        float eta = 0.0f;
        if (a.buf_in) eta = a.buf_in[t];
        else for (int c = 0; c < a.n_chunks; ++c) eta += a.eta_part[(size_t)c * a.T + t];
        float d = 0.0f;
        const int jmax = a.mats ? a.M - 1 : i;
        for (int j = 0; j <= jmax; ++j) {
            float A = 0.0f;
            if (a.buf_in) A = a.buf_in[a.T + t * a.M + j];
            else for (int c = 0; c < a.n_chunks; ++c) A += a.part[((size_t)c * a.T + t) * a.M + j];
            const float f = a.mats ? a.mats[t * 32 + i * a.M + j] : a.sL[i * a.M + j];
            d = __fadd_rn(d, __fmul_rn(f, A));
        }
        a.U[o] = __fadd_rn(a.U[o], __fdiv_rn(d, eta));
        if (o == 0 && a.stats) a.stats->eta = eta;
    }
}

cudaError_t launch_ctg(Ctx& c) {
    const int nblk = (int)((c.K_loc + 255) / 256);
    if (c.ctg_fused) {   // the packed rollout already wrote S~ and the per-CTA minima
        CtgMinArgs m{c.d_ctg_partmin, nblk, c.d_ctg_smin};
        return emit(c, (const void*)ctg_min_kernel, dim3(c.T), dim3(256), 0, &m, sizeof(m), MPPI_KERNEL_WSUM);
    }
    CtgArgs a{};
    a.ctg = c.d_ctg;
    a.partmin = c.d_ctg_partmin;
    a.T = c.T;
    a.K_loc = (int)c.K_loc;
    a.nblk = nblk;
    a.penalty = c.penalty;
    const size_t smem = (size_t)8 * c.T * sizeof(float);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(ctg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = emit(c, (const void*)ctg_kernel, dim3(nblk), dim3(256), smem, &a, sizeof(a), MPPI_KERNEL_WSUM);
    if (e != cudaSuccess) return e;
    CtgMinArgs m{c.d_ctg_partmin, nblk, c.d_ctg_smin};
    return emit(c, (const void*)ctg_min_kernel, dim3(c.T), dim3(256), 0, &m, sizeof(m), MPPI_KERNEL_WSUM);
}

cudaError_t launch_wsum_ctg(Ctx& c, const float* eps) {
    if (c.ctg_fused) {   // the rollout formed per-(CTA, t) sums: rescale to S_min,t and chunk them
        EpiCombineCtgArgs e{};
        e.epi_part = c.d_epi;
        e.smin = c.d_ctg_smin;
        e.part = c.d_part;
        e.eta_part = c.d_ctg_eta;
        e.nblk = c.epi_nblk;
        e.cpc = (c.epi_nblk + c.n_chunks - 1) / c.n_chunks;
        e.T = c.T;
        e.neg_inv_lambda = (float)(-1.0 / (double)c.lambda);
        const dim3 grid((unsigned)c.n_chunks, (unsigned)((c.T + 255) / 256));
        return emit(c, (const void*)epi_combine_ctg_kernel, grid, dim3(256), 0, &e, sizeof(e), MPPI_KERNEL_WSUM);
    }
    WsumCtgArgs a{};
    a.eps = eps;
    a.ctg = c.d_ctg;
    a.smin = c.d_ctg_smin;
    a.part = c.d_part;
    a.eta_part = c.d_ctg_eta;
    a.T = c.T;
    a.K_loc = (int)c.K_loc;
    a.ncols = c.K_loc * c.m / 4;
    a.cols_per_chunk = c.cols_per_chunk;
    a.neg_inv_lambda = (float)(-1.0 / (double)c.lambda);
    const dim3 grid((unsigned)c.n_chunks, (unsigned)((c.T + kWsumTT - 1) / kWsumTT));
    if (c.tma_wsum && c.K_loc >= kPackedMinK) {   // small K: plain loads have less latency
        const void* f = c.m == 1 ? (const void*)wsum_ctg_tma_kernel<1> : c.m == 2 ? (const void*)wsum_ctg_tma_kernel<2>
                      : c.m == 4 ? (const void*)wsum_ctg_tma_kernel<4> : nullptr;
        if (!f) return cudaErrorInvalidValue;
        const size_t smem = wsum_ctg_tma_smem(c.m);
        cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        return emit(c, f, grid, dim3(kWsumThreads), smem, &a, sizeof(a), MPPI_KERNEL_WSUM);
    }
    const void* f = c.m == 1 ? (const void*)wsum_ctg_kernel<1> : c.m == 2 ? (const void*)wsum_ctg_kernel<2>
                  : c.m == 4 ? (const void*)wsum_ctg_kernel<4> : nullptr;
    if (!f) return cudaErrorInvalidValue;
    return emit(c, f, grid, dim3(kWsumThreads), 0, &a, sizeof(a), MPPI_KERNEL_WSUM);
}

cudaError_t launch_finalize_ctg(Ctx& c, float* U, const float* buf_in, float* buf_out) {
    FinalizeCtgArgs a{};
    a.part = c.d_part;
    a.eta_part = c.d_ctg_eta;
    a.n_chunks = c.n_chunks;
    a.buf_in = buf_in;
    a.buf_out = buf_out;
    a.U = U;
    a.stats = c.d_stats;
    a.T = c.T;
    a.M = c.m;
    for (int i = 0; i < 16; ++i) a.sL[i] = c.sL[i];
    a.mats = c.per_t ? c.d_mats : nullptr;
    const int n = c.T * c.m + (buf_out ? c.T : 0);
    const int threads = n >= 1024 ? 1024 : ((n + 31) / 32) * 32;
    return emit(c, (const void*)finalize_ctg_kernel, dim3(1), dim3(threads), 0, &a, sizeof(a),
                MPPI_KERNEL_FINALIZE);
}

// ------------------------------------------------------------------------------ closed-loop advance
// Alg. 1 after the update: send u_0 to the (simulated, noise-free) plant,
// x <- x + F(x, u_0) dt with the plant's accurate path, then shift U (u_i = u_{i+1}, u_{T-1} =
// u_init).  One CTA; the plant step runs on thread 0 from the shared-memory copy of U.
template <class PP>
struct AdvanceArgs {
    float* x;              // [n] device state, in/out
    float* U;              // [T][M]
    int* crashed;          // device flag (quadrotor)
    float* x_log;          // [n] row for x' or nullptr
    float* u_log;          // [M] row for u_0 or nullptr
    float* q_log;          // q(x') or nullptr
    const float4* obs;
    int n_obs_pairs;
    int T, n;
    float dt;
    float4 u_init;
    PP P;
};

template <class Plant>
__global__ void __launch_bounds__(1024) advance_kernel(const __grid_constant__ AdvanceArgs<typename Plant::Params> a) {
    pdl_wait();                        // reads U and x written by its predecessors
    constexpr int M = Plant::M;
    extern __shared__ float sUa[];
    const int TM = a.T * M;
    for (int o = threadIdx.x; o < TM; o += blockDim.x) sUa[o] = a.U[o];
    __syncthreads();
    if (threadIdx.x == 0) {
        Plant st;
        float xin[16] = {0};
        for (int i = 0; i < a.n; ++i) xin[i] = a.x[i];
        st.load(xin, *a.crashed);
        const ObstacleView ob{a.obs, a.n_obs_pairs};
        float u0[M];
#pragma unroll
        for (int i = 0; i < M; ++i) u0[i] = sUa[i];
        float xd[Plant::N];
        st.template state_cost<-1, true>(true, a.P, ob);
        st.deriv_accurate(u0, a.P, xd);
        st.update(xd, a.P, a.dt);
        const float q = st.template state_cost<-1, true>(false, a.P, ob);
        float xo[16];
        st.store(xo);
        for (int i = 0; i < a.n; ++i) {
            a.x[i] = xo[i];
            if (a.x_log) a.x_log[i] = xo[i];
        }
        if (a.u_log)
            for (int i = 0; i < M; ++i) a.u_log[i] = u0[i];
        if (a.q_log) *a.q_log = q;
        *a.crashed = st.crashed;
    }
    const float* ui = reinterpret_cast<const float*>(&a.u_init);
    for (int o = threadIdx.x; o < TM; o += blockDim.x) a.U[o] = o < TM - M ? sUa[o + M] : ui[o - (TM - M)];
}

template <class Plant>
static cudaError_t launch_advance_t(Ctx& c, const typename Plant::Params& P, float* x, float* U,
                                    const float* u_init, float* x_log, float* u_log, float* q_log) {
    AdvanceArgs<typename Plant::Params> a{};
    a.x = x;
    a.U = U;
    a.crashed = &c.d_stats->plant_crashed;
    a.x_log = x_log;
    a.u_log = u_log;
    a.q_log = q_log;
    a.obs = c.d_obs;
    a.n_obs_pairs = c.n_obs_pairs;
    a.T = c.T;
    a.n = c.n;
    a.dt = c.dt;
    float* up = reinterpret_cast<float*>(&a.u_init);
    for (int i = 0; i < 4; ++i) up[i] = i < c.m ? u_init[i] : 0.0f;
    a.P = P;
    const size_t smem = (size_t)c.T * c.m * sizeof(float);
    auto kern = advance_kernel<Plant>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int threads = c.T * c.m >= 1024 ? 1024 : ((c.T * c.m + 31) / 32) * 32;
    return emit(c, (const void*)kern, dim3(1), dim3(threads), smem, &a, sizeof(a), MPPI_KERNEL_SHIFT);
}

cudaError_t launch_advance(Ctx& c, float* x, float* U, const float* u_init, float* x_log, float* u_log,
                           float* q_log) {
    switch (c.plant) {
        case MPPI_PLANT_CARTPOLE: return launch_advance_t<Cartpole>(c, c.params.cartpole, x, U, u_init, x_log, u_log, q_log);
        case MPPI_PLANT_RACECAR: return launch_advance_t<Racecar>(c, c.params.racecar, x, U, u_init, x_log, u_log, q_log);
        case MPPI_PLANT_QUADROTOR: return launch_advance_t<Quadrotor>(c, c.params.quadrotor, x, U, u_init, x_log, u_log, q_log);
        default: return cudaErrorNotSupported;
    }
}

// ------------------------------------------------------------------------------ Feynman-Kac reduction
// partial sums of w_k = exp(-(S_k - S_min)/lambda) and w_k^2 per CTA, fp64, fixed order
struct FkArgs {
    const float* costs;
    const long long* key;
    int K_loc;
    float lambda;
    double* part;   // [gridDim.x][2]
};

__global__ void __launch_bounds__(256) fk_reduce_kernel(const FkArgs a) {
    pdl_wait();                        // costs and key of the rollout
    const float smin = key_cost(*a.key);
    double s1 = 0.0, s2 = 0.0;
    for (int k = blockIdx.x * 256 + threadIdx.x; k < a.K_loc; k += gridDim.x * 256) {
        const double w = (double)expf(-__fdiv_rn(a.costs[k] - smin, a.lambda));
        s1 += w;
        s2 += w * w;
    }
    __shared__ double r1[256], r2[256];
    r1[threadIdx.x] = s1;
    r2[threadIdx.x] = s2;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            r1[threadIdx.x] += r1[threadIdx.x + o];
            r2[threadIdx.x] += r2[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.part[2 * blockIdx.x] = r1[0];
        a.part[2 * blockIdx.x + 1] = r2[0];
    }
}

cudaError_t launch_fk_reduce(Ctx& c, double* part, int nblk) {
    FkArgs a{};
    a.costs = c.d_costs;
    a.key = &c.d_stats->min_key;
    a.K_loc = (int)c.K_loc;
    a.lambda = c.lambda;
    a.part = part;
    return emit(c, (const void*)fk_reduce_kernel, dim3(nblk), dim3(256), 0, &a, sizeof(a), MPPI_KERNEL_WSUM);
}

// ------------------------------------------------------------------------------ K5 shift
struct ShiftArgs {
    float* U;
    int T, M;
    float4 u_init;
};

__global__ void __launch_bounds__(1024) shift_kernel(const ShiftArgs a) {
    pdl_wait();                        // U of the update
    float* U = a.U;
    const int T = a.T, M = a.M;
    const float4 u_init = a.u_init;
    extern __shared__ float sU[];
    const int TM = T * M;
    for (int o = threadIdx.x; o < TM; o += blockDim.x) sU[o] = U[o];
    __syncthreads();
    for (int o = threadIdx.x; o < TM; o += blockDim.x) {
        float v;
        if (o < TM - M) {
            v = sU[o + M];
        } else {
            const int i = o - (TM - M);
            v = i == 0 ? u_init.x : (i == 1 ? u_init.y : (i == 2 ? u_init.z : u_init.w));
        }
        U[o] = v;
    }
}

// ============================================================================== launchers
static cudaEvent_t take_event(Ctx& c) {
    if (!c.ev_pool.empty()) {
        cudaEvent_t e = c.ev_pool.back();
        c.ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

cudaError_t emit(Ctx& c, const void* func, dim3 grid, dim3 block, size_t smem, const void* args,
                 size_t size, int kind) {
    if (size > sizeof(KLaunch::args)) return cudaErrorInvalidValue;
    c.last_launches++;
    c.last_funcs.push_back(func);
    if (c.collect) {
        c.pending.emplace_back();
        KLaunch& L = c.pending.back();
        L.func = func;
        L.grid = grid;
        L.block = block;
        L.smem = smem;
        L.kind = kind;
        L.nargs = size;
        memcpy(L.args, args, size);
        return cudaSuccess;
    }
    ProfScope prof(c, kind);
    void* argp[1] = {const_cast<void*>(args)};
    return cudaLaunchKernel(func, grid, block, argp, smem, c.stream);
}

ProfScope::ProfScope(Ctx& c_, int kind_) : c(c_), kind(kind_) {
    if (!c.prof) return;
    a = take_event(c);
    b = take_event(c);
    cudaEventRecord(a, c.stream);
}

ProfScope::~ProfScope() {
    if (!c.prof || !a) return;
    cudaEventRecord(b, c.stream);
    c.ev_pending.push_back(std::make_pair(kind, std::make_pair(a, b)));
}

static PhiloxKeys philox_key_schedule(uint64_t seed) {
    PhiloxKeys K;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        K.k0[r] = k0;
        K.k1[r] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return K;
}

cudaError_t launch_noise(Ctx& c, uint64_t seed, uint64_t step, float* out, bool reset_key) {
    const PhiloxKeys keys = philox_key_schedule(seed);
    const dim3 grid((unsigned)((c.K_loc + 255) / 256), (unsigned)((c.T + kNoiseTT - 1) / kNoiseTT));
    NoiseArgs a{};
    a.eps = out;
    a.K_loc = (int)c.K_loc;
    a.T = c.T;
    a.k_offset = (unsigned)c.k_offset;
    a.step_lo = (unsigned)step;
    a.step_hi = (unsigned)(step >> 32);
    a.keys = keys;
    a.key_reset = reset_key ? reinterpret_cast<long long*>(&c.d_stats->min_key) : nullptr;
    const void* f = c.m == 1 ? (const void*)noise_kernel<1> : c.m == 2 ? (const void*)noise_kernel<2>
                  : c.m == 4 ? (const void*)noise_kernel<4> : nullptr;
    if (!f) return cudaErrorInvalidValue;
    return emit(c, f, grid, dim3(256), 0, &a, sizeof(a), MPPI_KERNEL_NOISE);
}

// The rollout kernels' argument block from the context (eps: the noise read by non-GEN kernels).
template <class Plant>
static void fill_rollout_args(Ctx& c, const typename Plant::Params& P, const float* x0, const float* U,
                              const float* eps, float* costs_out, RolloutArgs<typename Plant::Params>& a) {
    a.eps = eps;
    a.eps_out = c.gen_eps;
    a.cells = c.d_cells;
    a.cent = c.d_cent;
    a.cell_nx = c.cell_nx;
    a.cell_ny = c.cell_ny;
    a.n_cent = (int)c.cent_host.size();
    a.cell_ox = c.cell_ox;
    a.cell_oy = c.cell_oy;
    a.cell_inv_h = c.cell_inv_h;
    a.cell_band = c.cell_band;
    a.step_lo = (unsigned)c.gen_step;
    a.step_hi = (unsigned)(c.gen_step >> 32);
    a.keys = philox_key_schedule(c.gen_seed);
    a.U = U;
    a.costs = c.d_costs;
    a.costs_out = costs_out;
    a.min_key = &c.d_stats->min_key;
    a.replays = &c.d_stats->replays;
    a.obs = c.d_obs;
    a.n_obs_pairs = c.n_obs_pairs;
    a.T = c.T;
    a.K_loc = (int)c.K_loc;
    a.k_offset = (unsigned)c.k_offset;
    a.dt = c.dt;
    a.c1 = c.c1;
    a.penalty = c.penalty;
    for (int i = 0; i < 16; ++i) { a.sL[i] = c.sL[i]; a.R[i] = c.R[i]; a.x0[i] = 0.0f; }
    for (int i = 0; i < 4; ++i) {
        a.sd[i] = i < c.m ? c.sL[i * c.m + i] : 0.0f;
        a.ad[i] = i < c.m ? c.ad[i] : 0.0f;
    }
    a.x0_dev = nullptr;
    a.qstep = c.ctg ? c.d_ctg : nullptr;
    a.mats = c.per_t ? c.d_mats : nullptr;
    if (c.x0_on_device) a.x0_dev = x0;
    else for (int i = 0; i < c.n && i < 16; ++i) a.x0[i] = x0[i];
    a.P = P;
    for (int i = 0; i < kMaxStaticPairs; ++i)
        a.obs_k[i] = i < c.n_obs_pairs ? c.obs_host[i] : make_float4(-1e15f, -1e15f, -1e15f, -1e15f);
}

template <class Plant, bool DIAG, int NP, bool X2 = false>
static cudaError_t launch_rollout_t(Ctx& c, const typename Plant::Params& P, const float* x0,
                                    const float* U, const float* eps, float* costs_out) {
    RolloutArgs<typename Plant::Params> a{};
    fill_rollout_args<Plant>(c, P, x0, U, eps, costs_out, a);
    const int spt = X2 ? 2 : 1;                                      // samples per thread
    const size_t smem = (size_t)c.n_obs_pairs * sizeof(float4) + (size_t)c.T * sizeof(StepRec) +
                        (c.gen_eps ? 0 : (size_t)(X2 ? 2 : kEpsStages) * kRolloutThreads * spt * Plant::M * sizeof(float)) +
                        (DIAG ? 0 : (size_t)c.T * 2 * Plant::M * Plant::M * sizeof(float)) +
                        (NP == kCellGrid ? c.cent_host.size() * sizeof(float2) + 16 + c.cells_host.size() * sizeof(uint32_t) : 0);
    const void* kern;
    if constexpr (X2 && !DIAG) {   // general Sigma / A_t: grid path only
        static_assert(NP == kCellGrid, "packed general-Sigma kernel: candidate-grid path only");
        if (c.ctg && c.gen_eps && c.epi && c.d_epi) {   // + fused cost-to-go pass and reduction
            a.ctg_partmin = c.d_ctg_partmin;
            a.epi_part = c.d_epi;
            a.lambda = (float)(-1.0 / (double)c.lambda);   // the epilogue's weights: (S - m) (-1/lambda)
            c.ctg_fused = true;
            kern = (const void*)rollout_kernel_x2<NP, true, true, false, true>;
        } else if (c.ctg) {
            kern = c.gen_eps ? (const void*)rollout_kernel_x2<NP, true, true, false> : (const void*)rollout_kernel_x2<NP, false, true, false>;
        } else if (c.epi_active && c.gen_eps) {   // fused reduction (EPI): the same sum of eps
            a.epi_part = c.d_epi;
            a.lambda = c.lambda;
            kern = (const void*)rollout_kernel_x2<NP, true, false, false, true>;
        } else {
            kern = c.gen_eps ? (const void*)rollout_kernel_x2<NP, true, false, false> : (const void*)rollout_kernel_x2<NP, false, false, false>;
        }
    } else if constexpr (X2) {
        if (c.ctg) {
            if constexpr (NP >= 0) {
                return launch_rollout_t<Plant, DIAG, -1, true>(c, P, x0, U, eps, costs_out);
            } else if constexpr (NP == kCellGrid) {
                if (c.gen_eps && c.epi && c.d_epi) {   // + fused cost-to-go pass and reduction
                    a.ctg_partmin = c.d_ctg_partmin;
                    a.epi_part = c.d_epi;
                    a.lambda = (float)(-1.0 / (double)c.lambda);   // (S - m) (-1/lambda)
                    c.ctg_fused = true;
                    kern = (const void*)rollout_kernel_x2<NP, true, true, true, true>;
                } else {
                    kern = c.gen_eps ? (const void*)rollout_kernel_x2<NP, true, true> : (const void*)rollout_kernel_x2<NP, false, true>;
                }
            } else {
                kern = c.gen_eps ? (const void*)rollout_kernel_x2<NP, true, true> : (const void*)rollout_kernel_x2<NP, false, true>;
            }
        } else {
            if constexpr (NP == kCellGrid) {
                if (c.epi_active && c.gen_eps) {    // fused reduction (EPI)
                    a.epi_part = c.d_epi;
                    a.lambda = c.lambda;
                    kern = (const void*)rollout_kernel_x2<NP, true, false, true, true>;
                } else {
                    kern = c.gen_eps ? (const void*)rollout_kernel_x2<NP, true> : (const void*)rollout_kernel_x2<NP, false>;
                }
            } else {
                kern = c.gen_eps ? (const void*)rollout_kernel_x2<NP, true> : (const void*)rollout_kernel_x2<NP, false>;
            }
        }
    } else {
        // cost-to-go weighting: the QSTEP variants exist for the runtime-count and grid obstacle
        // paths (and every other plant); exact-count quadrotor variants defer to NP = -1
        constexpr bool kQ = NP < 0 || !std::is_same<Plant, Quadrotor>::value;
        if constexpr (!kQ) {
            if (c.ctg) return launch_rollout_t<Plant, DIAG, -1>(c, P, x0, U, eps, costs_out);
        }
        if constexpr (!std::is_same<Plant, Quadrotor>::value || NP == kCellGrid) {
            if (c.ctg) kern = c.gen_eps ? (const void*)rollout_kernel<Plant, DIAG, NP, true, kQ>
                                        : (const void*)rollout_kernel<Plant, DIAG, NP, false, kQ>;
            else kern = c.gen_eps ? (const void*)rollout_kernel<Plant, DIAG, NP, true> : (const void*)rollout_kernel<Plant, DIAG, NP>;
        } else {
            if (c.gen_eps) return cudaErrorInvalidValue;   // fused_noise_applies() excludes this variant
            kern = c.ctg ? (const void*)rollout_kernel<Plant, DIAG, NP, false, kQ> : (const void*)rollout_kernel<Plant, DIAG, NP>;
        }
    }
    if (smem + kRolloutStaticSmem > 48 * 1024) {   // (static + dynamic above the default 48 KB)
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const unsigned grid = (unsigned)((c.K_loc / spt + kRolloutThreads - 1) / kRolloutThreads);
    return emit(c, (const void*)kern, dim3(grid), dim3(kRolloutThreads), smem, &a, sizeof(a),
                MPPI_KERNEL_ROLLOUT);
}

// The quadrotor's obstacle loop is compiled for the context's exact pair count when it is at
// most kMaxStaticPairs (diagonal L and R: every shipped configuration); other plants, general
// covariances and larger forests use the runtime-count loop.
template <class Plant, bool DIAG, int NP>
static cudaError_t dispatch_np(Ctx& c, const typename Plant::Params& P, const float* x0,
                               const float* U, const float* eps, float* costs_out) {
    if constexpr (NP == 0) {
        if (grid_on(c)) {
            if (c.pack2 && c.K_loc >= kPackedMinK)
                return launch_rollout_t<Plant, DIAG, kCellGrid, true>(c, P, x0, U, eps, costs_out);
            return launch_rollout_t<Plant, DIAG, kCellGrid>(c, P, x0, U, eps, costs_out);
        }
    }
    if constexpr (NP > kMaxStaticPairs) {
        if (c.pack2 && c.K_loc >= kPackedMinK) return launch_rollout_t<Plant, DIAG, -1, true>(c, P, x0, U, eps, costs_out);
        return launch_rollout_t<Plant, DIAG, -1>(c, P, x0, U, eps, costs_out);
    } else {
        if (c.n_obs_pairs == NP) {
            if (c.pack2 && c.K_loc >= kPackedMinK) return launch_rollout_t<Plant, DIAG, NP, true>(c, P, x0, U, eps, costs_out);
            return launch_rollout_t<Plant, DIAG, NP>(c, P, x0, U, eps, costs_out);
        }
        return dispatch_np<Plant, DIAG, NP + 1>(c, P, x0, U, eps, costs_out);
    }
}

template <class Plant, bool DIAG>
static cudaError_t launch_rollout_np(Ctx& c, const typename Plant::Params& P, const float* x0,
                                     const float* U, const float* eps, float* costs_out) {
    if constexpr (std::is_same<Plant, Quadrotor>::value && DIAG)
        return dispatch_np<Plant, DIAG, 0>(c, P, x0, U, eps, costs_out);
    if constexpr (std::is_same<Plant, Quadrotor>::value && !DIAG) {   // general Sigma / A_t
        if (grid_on(c)) {
            if (c.pack2 && c.K_loc >= kPackedMinK)
                return launch_rollout_t<Plant, DIAG, kCellGrid, true>(c, P, x0, U, eps, costs_out);
            return launch_rollout_t<Plant, DIAG, kCellGrid>(c, P, x0, U, eps, costs_out);
        }
    }
    return launch_rollout_t<Plant, DIAG, -1>(c, P, x0, U, eps, costs_out);
}

template <class Plant>
static cudaError_t launch_rollout_p(Ctx& c, const typename Plant::Params& P, const float* x0,
                                    const float* U, const float* eps, float* costs_out) {
    return c.diag ? launch_rollout_np<Plant, true>(c, P, x0, U, eps, costs_out)
                  : launch_rollout_np<Plant, false>(c, P, x0, U, eps, costs_out);
}

// Dynamic shared memory of the rollout kernels (obstacle pairs, per-t records, the eps ring,
// the general path's per-t matrices, the candidate grid), and the device's opt-in limit.
size_t rollout_smem_bytes(const Ctx& c, bool cells) {
    const int m = c.m;
    return (size_t)c.n_obs_pairs * sizeof(float4) + (size_t)c.T * sizeof(StepRec) +
           (size_t)kEpsStages * kRolloutThreads * m * sizeof(float) +
           (c.diag ? 0 : (size_t)c.T * 2 * m * m * sizeof(float)) +
           (cells ? c.cent_host.size() * sizeof(float2) + 16 + c.cells_host.size() * sizeof(uint32_t) : 0);
}

size_t smem_optin_bytes() {
    static size_t v = [] {
        int dev = 0, b = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&b, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || b <= 0)
            b = 227 * 1024;
        return (size_t)b;
    }();
    return v;
}

// the obstacle candidate grid is used when it was built, is enabled and fits in shared memory
// beside the horizon's per-t records (very long horizons fall back to the full search)
bool grid_on(const Ctx& c) {
    return c.use_cells && c.cell_nx > 0 && rollout_smem_bytes(c, true) + kRolloutStaticSmem <= smem_optin_bytes();
}

// the packed rollout's fused reduction (EPI): the C5-type path (packed quadrotor, diagonal,
// candidate grid, in-kernel noise, trajectory weights)
bool epi_applies(const Ctx& c) {
    // (diagonal or general Sigma / A_t: both packed variants sum the standard-normal eps)
    return c.epi && c.d_epi && c.plant == MPPI_PLANT_QUADROTOR && c.pack2 &&
           !c.ctg && c.K_loc >= kPackedMinK && grid_on(c) && fused_noise_applies(c);
}

cudaError_t launch_epi_combine(Ctx& c, const long long* key) {
    EpiCombineArgs a{};
    a.epi_part = c.d_epi;
    a.key = key;
    a.part = c.d_part;
    a.eta_part = c.d_eta_part;
    a.nblk = c.epi_nblk;
    a.cpc = (c.epi_nblk + c.n_chunks - 1) / c.n_chunks;
    a.TM = c.T * c.m;
    a.lambda = c.lambda;
    if (a.cpc > 256) return cudaErrorInvalidValue;   // sized at create so that it is not
    const dim3 grid((unsigned)c.n_chunks, (unsigned)((a.TM + 1 + 255) / 256));
    return emit(c, (const void*)epi_combine_kernel, grid, dim3(256), 0, &a, sizeof(a), MPPI_KERNEL_WSUM);
}

bool fused_noise_applies(const Ctx& c) {
    // GEN kernels only once the step is throughput-bound (measured: -2..4 % at K = 2^20 for the
    // one-sample kernel; at small K the per-thread noise lengthens the latency-bound step loop)
#ifndef MPPI_GEN_MIN_K
#define MPPI_GEN_MIN_K kPackedMinK
#endif
    if (!c.fuse_noise || c.K_loc < MPPI_GEN_MIN_K) return false;
    if (c.plant == MPPI_PLANT_QUADROTOR) {
        if (c.diag && !c.per_t && c.pack2) return true;   // packed kernel (any obstacle path)
        return grid_on(c);                                 // one-sample grid kernel (any Sigma, A_t)
    }
    return true;                                           // one-sample kernel (any Sigma, A_t)
}

cudaError_t launch_rollout(Ctx& c, const float* x0, const float* U, const float* eps,
                           float* costs_out) {
    c.ctg_fused = false;   // set by the dispatch when the packed cost-to-go rollout runs the pass
    switch (c.plant) {
        case MPPI_PLANT_CARTPOLE:
            return launch_rollout_p<Cartpole>(c, c.params.cartpole, x0, U, eps, costs_out);
        case MPPI_PLANT_RACECAR:
            return launch_rollout_p<Racecar>(c, c.params.racecar, x0, U, eps, costs_out);
        case MPPI_PLANT_QUADROTOR:
            return launch_rollout_p<Quadrotor>(c, c.params.quadrotor, x0, U, eps, costs_out);
        case MPPI_PLANT_LINEAR: {
            float xp[16] = {0};
            if (c.x0_on_device) return cudaErrorNotSupported;   // linear test plant: host x0 only
            for (int i = 0; i < c.n; ++i) xp[i] = x0[i];
            if (c.m == 1) return launch_rollout_p<Linear<1>>(c, c.params.linear, xp, U, eps, costs_out);
            if (c.m == 2) return launch_rollout_p<Linear<2>>(c, c.params.linear, xp, U, eps, costs_out);
            if (c.m == 4) return launch_rollout_p<Linear<4>>(c, c.params.linear, xp, U, eps, costs_out);
            return cudaErrorInvalidValue;
        }
        default:
            return cudaErrorInvalidValue;
    }
}

cudaError_t launch_wsum(Ctx& c, const float* eps, const long long* key) {
    WsumArgs a{};
    a.flags = nullptr;
    a.eps = eps;
    a.costs = c.d_costs;
    a.key = key;
    a.part = c.d_part;
    a.eta_part = c.d_eta_part;
    a.T = c.T;
    a.ncols = c.K_loc * c.m / 4;
    a.cols_per_chunk = c.cols_per_chunk;
    a.lambda = c.lambda;
    const dim3 grid((unsigned)c.n_chunks, (unsigned)((c.T + kWsumTT - 1) / kWsumTT));
    if (c.tma_wsum && c.K_loc >= kPackedMinK) {   // small K: plain loads have less latency
        const void* f = c.m == 1 ? (const void*)wsum_tma_kernel<1> : c.m == 2 ? (const void*)wsum_tma_kernel<2>
                      : c.m == 4 ? (const void*)wsum_tma_kernel<4> : nullptr;
        if (!f) return cudaErrorInvalidValue;
        if (c.sparse_wsum && c.d_flags && c.K_loc >= kPackedMinK) {   // (small K: the extra pass costs more)
            a.flags = c.d_flags;
            const void* ff = c.m == 1 ? (const void*)wsum_flags_kernel<1> : c.m == 2 ? (const void*)wsum_flags_kernel<2>
                           : (const void*)wsum_flags_kernel<4>;
            const unsigned nb = (unsigned)((a.ncols + kWsumThreads - 1) / kWsumThreads);
            cudaError_t e = emit(c, ff, dim3(nb), dim3(kWsumThreads), 0, &a, sizeof(a), MPPI_KERNEL_WSUM);
            if (e != cudaSuccess) return e;
        }
        const size_t smem = kWsumTmaSmem;
        cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        return emit(c, f, grid, dim3(kWsumThreads), smem, &a, sizeof(a), MPPI_KERNEL_WSUM);
    }
    const void* f = c.m == 1 ? (const void*)wsum_kernel<1> : c.m == 2 ? (const void*)wsum_kernel<2>
                  : c.m == 4 ? (const void*)wsum_kernel<4> : nullptr;
    if (!f) return cudaErrorInvalidValue;
    return emit(c, f, grid, dim3(kWsumThreads), 0, &a, sizeof(a), MPPI_KERNEL_WSUM);
}

int wsum_blocks_per_sm(int m) {
    int n = 0;
    cudaError_t e = cudaErrorInvalidValue;
    const void* f = m == 1 ? (const void*)wsum_tma_kernel<1> : m == 2 ? (const void*)wsum_tma_kernel<2>
                  : m == 4 ? (const void*)wsum_tma_kernel<4> : nullptr;
    if (f && cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWsumTmaSmem) == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, kWsumThreads, kWsumTmaSmem);
    return (e == cudaSuccess && n > 0) ? n : 1;
}

// The one-collective combine's two ends: the local record [local key, eta_r, A_r] (rec_out, sums
// against this rank's own minimum), and the rescale of n_rec gathered records + the U update.
cudaError_t launch_finalize_record(Ctx& c, float* rec_out) {
    FinalizeArgs a{};
    a.part = c.d_part;
    a.eta_part = c.d_eta_part;
    a.n_chunks = c.n_chunks;
    a.T = c.T;
    a.M = c.m;
    a.rec_out = rec_out;
    a.key_src = &c.d_stats->min_key;
    const size_t smem = (size_t)(c.T * c.m + 1) * sizeof(float);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int threads = c.T * c.m >= 1024 ? 1024 : ((c.T * c.m + 31) / 32) * 32;
    return emit(c, (const void*)finalize_kernel, dim3(1), dim3(threads), smem, &a, sizeof(a),
                MPPI_KERNEL_FINALIZE);
}

cudaError_t launch_finalize_gathered(Ctx& c, const float* gathered, int n_rec, float* U) {
    FinalizeArgs a{};
    a.n_chunks = 0;
    a.U = U;
    a.stats = c.d_stats;
    a.T = c.T;
    a.M = c.m;
    for (int i = 0; i < 16; ++i) a.sL[i] = c.sL[i];
    a.mats = c.per_t ? c.d_mats : nullptr;
    a.gathered = gathered;
    a.n_rec = n_rec;
    a.rec = (int)gather_record_len(c);
    a.lambda = c.lambda;
    a.key_out = &c.d_stats->min_key;
    const size_t smem = (size_t)(c.T * c.m + 1) * sizeof(float);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int threads = c.T * c.m >= 1024 ? 1024 : ((c.T * c.m + 31) / 32) * 32;
    return emit(c, (const void*)finalize_kernel, dim3(1), dim3(threads), smem, &a, sizeof(a),
                MPPI_KERNEL_FINALIZE);
}

cudaError_t launch_finalize(Ctx& c, const float* buf_in, float* buf_out, float* U) {
    FinalizeArgs a{};
    a.part = c.d_part;
    a.eta_part = c.d_eta_part;
    a.n_chunks = c.n_chunks;
    a.buf_in = buf_in;
    a.buf_out = buf_out;
    a.U = U;
    a.stats = c.d_stats;
    a.T = c.T;
    a.M = c.m;
    for (int i = 0; i < 16; ++i) a.sL[i] = c.sL[i];
    a.mats = c.per_t ? c.d_mats : nullptr;
    const size_t smem = (size_t)(c.T * c.m + 1) * sizeof(float);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int threads = c.T * c.m >= 1024 ? 1024 : ((c.T * c.m + 31) / 32) * 32;
    return emit(c, (const void*)finalize_kernel, dim3(1), dim3(threads), smem, &a, sizeof(a),
                MPPI_KERNEL_FINALIZE);
}

cudaError_t launch_shift(Ctx& c, float* U, const float* u_init) {
    float4 ui = make_float4(0, 0, 0, 0);
    float* up = reinterpret_cast<float*>(&ui);
    for (int i = 0; i < c.m; ++i) up[i] = u_init[i];
    const size_t smem = (size_t)c.T * c.m * sizeof(float);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(shift_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int threads = c.T * c.m >= 1024 ? 1024 : ((c.T * c.m + 31) / 32) * 32;
    ShiftArgs a{};
    a.U = U;
    a.T = c.T;
    a.M = c.m;
    a.u_init = ui;
    return emit(c, (const void*)shift_kernel, dim3(1), dim3(threads), smem, &a, sizeof(a), MPPI_KERNEL_SHIFT);
}

// ------------------------------------------------------------------------------ host plant step
template <class Plant>
static float host_step_t(const Ctx& c, const typename Plant::Params& P, float* x, const float* u,
                         int32_t* crashed) {
    Plant st;
    float xin[16] = {0};
    for (int i = 0; i < c.n && i < 16; ++i) xin[i] = x[i];
    st.load(xin, crashed ? *crashed : 0);
    const ObstacleView ob{c.obs_host.data(), c.n_obs_pairs};
    float xd[Plant::N];
    st.template state_cost<-1, true>(true, P, ob);   // cart-pole: sin/cos of the current angle
    st.deriv_accurate(u, P, xd);
    st.update(xd, P, c.dt);
    const float q = st.template state_cost<-1, true>(false, P, ob);
    float xo[16] = {0};
    st.store(xo);
    for (int i = 0; i < c.n; ++i) x[i] = xo[i];
    if (crashed) *crashed = st.crashed;
    return q;
}

float host_plant_step(const Ctx& c, float* x, const float* u, int32_t* crashed) {
    switch (c.plant) {
        case MPPI_PLANT_CARTPOLE: return host_step_t<Cartpole>(c, c.params.cartpole, x, u, crashed);
        case MPPI_PLANT_RACECAR: return host_step_t<Racecar>(c, c.params.racecar, x, u, crashed);
        case MPPI_PLANT_QUADROTOR: return host_step_t<Quadrotor>(c, c.params.quadrotor, x, u, crashed);
        default:
            if (c.m == 1) return host_step_t<Linear<1>>(c, c.params.linear, x, u, crashed);
            if (c.m == 2) return host_step_t<Linear<2>>(c, c.params.linear, x, u, crashed);
            return host_step_t<Linear<4>>(c, c.params.linear, x, u, crashed);
    }
}

}  // namespace mppi
