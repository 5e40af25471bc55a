// esom_train.cu -- online SOM / k-means ticks with the f64 working copy of
// the landmarks resident in shared memory, split across a thread-block
// cluster when it does not fit one SM (ref: som.py:44-68, graphmodel.py:87-102).
//
// A tick is a strictly sequential walk over the host-drawn samples: BMU of
// x_s over all landmarks (f64, lowest index on ties), then every landmark
// moves by alpha * h_j * (x_s - hi_j).  The latency of one sample is the
// whole cost, so the design keeps everything on chip:
//   * CTA r of a CS-CTA cluster owns landmarks [r*gs, (r+1)*gs) as f64 rows in
//     its shared memory (row stride d+1 doubles: conflict-free row walks);
//   * the sample rows are staged in shared memory SB at a time (one load
//     latency per chunk instead of one per sample);
//   * BMU: 4 threads per landmark (f64 FMA partial sums, fixed shuffle order),
//     block argmin, then the CS per-CTA candidates are exchanged through
//     distributed shared memory with ONE cluster barrier per sample
//     (candidate slots double-buffered by sample parity);
//   * update: warps walk rows (lane = dimension), h_j computed once per
//     landmark per sample.
// The summation order of |hi_j - x|^2 differs from numpy's einsum, so
// distances agree to ~1e-16 relative; BMUs differ only on exact near-ties
// (same contract as the single-CTA kernel it replaces).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "esom_common.cuh"
#include "esom_host.h"

using namespace esom;
using namespace esom_host;

namespace {

constexpr int kTickThreads = 1024;
constexpr int kTickSB = 64;          // sample rows staged per chunk
constexpr size_t kTickSmemCap = 200 * 1024;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_peer(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ double ld_peer_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ int ld_peer_s32(uint32_t addr) {
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ bool lex_less(double v, int j, double bv, int bj) { return v < bv || (v == bv && j < bj); }

template <bool SOM>
__global__ void __launch_bounds__(kTickThreads) online_tick_cluster_kernel(const float* __restrict__ X, int d,
                                                                           const int64_t* __restrict__ sample, int B,
                                                                           float* __restrict__ hi_f32,
                                                                           const float* __restrict__ lo, int g, int gs,
                                                                           double sigma, double alpha) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double cand_v[2];
    __shared__ int cand_j[2];
    __shared__ double red_v[32];
    __shared__ int red_j[32];
    __shared__ int s_bmu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t rank = cluster_rank(), cs = cluster_size();
    const int ds = d + 1;
    double* H = sm;                                    // gs x ds (f64 working copy of the owned rows)
    double* ah = H + (size_t)gs * ds;                  // gs: alpha * h_j of the current sample
    double* xs = ah + gs;                              // SB x d staged sample rows (f64 once)
    const int j0 = (int)rank * gs;
    const int gl = max(0, min(gs, g - j0));            // rows this CTA owns
    for (int e = tid; e < gl * d; e += kTickThreads) H[(e / d) * ds + e % d] = (double)hi_f32[(int64_t)j0 * d + e];
    const double denom = 2.0 * sigma * sigma;

    for (int s0 = 0; s0 < B; s0 += kTickSB) {
        const int nb = min(kTickSB, B - s0);
        __syncthreads();  // the previous chunk's rows are consumed
        for (int e = tid; e < nb * d; e += kTickThreads) xs[e] = (double)__ldg(X + sample[s0 + e / d] * d + e % d);
        __syncthreads();
        for (int s = 0; s < nb; ++s) {
            const double* x = xs + s * d;
            // ---- local BMU: 4 threads per landmark ----
            double bv = __longlong_as_double(0x7ff0000000000000ll);
            int bj = 0x7fffffff;
            const int part = tid & 3;
            for (int base = 0; base < gl; base += kTickThreads / 4) {
                const int jl = base + (tid >> 2);
                double acc = 0.0;
                if (jl < gl) {
                    const double* h = H + jl * ds;
#pragma unroll 8
                    for (int c = part; c < d; c += 4) {
                        const double t = h[c] - x[c];
                        acc = fma(t, t, acc);
                    }
                }
                acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                acc += __shfl_xor_sync(0xffffffffu, acc, 2);
                if (jl < gl && lex_less(acc, j0 + jl, bv, bj)) {
                    bv = acc;
                    bj = j0 + jl;
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                if (lex_less(ov, oj, bv, bj)) bv = ov, bj = oj;
            }
            if (lane == 0) red_v[warp] = bv, red_j[warp] = bj;
            __syncthreads();
            if (warp == 0) {
                bv = lane < kTickThreads / 32 ? red_v[lane] : __longlong_as_double(0x7ff0000000000000ll);
                bj = lane < kTickThreads / 32 ? red_j[lane] : 0x7fffffff;
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                    const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                    if (lex_less(ov, oj, bv, bj)) bv = ov, bj = oj;
                }
                if (lane == 0) {
                    cand_v[s & 1] = bv;
                    cand_j[s & 1] = bj;
                    if (cs == 1) s_bmu = bj;
                }
            }
            // ---- cluster exchange of the per-CTA candidates (DSMEM) ----
            if (cs > 1) {
                cluster_sync_all();
                if (tid == 0) {
                    double v = __longlong_as_double(0x7ff0000000000000ll);
                    int jb = 0x7fffffff;
                    for (uint32_t r = 0; r < cs; ++r) {
                        const double ov = ld_peer_f64(map_peer(&cand_v[s & 1], r));
                        const int oj = ld_peer_s32(map_peer(&cand_j[s & 1], r));
                        if (lex_less(ov, oj, v, jb)) v = ov, jb = oj;
                    }
                    s_bmu = jb;
                }
            }
            __syncthreads();
            const int b = s_bmu;
            // ---- update ----
            if (SOM) {
                const double lbx = (double)lo[2 * b], lby = (double)lo[2 * b + 1];
                for (int jl = tid; jl < gl; jl += kTickThreads) {
                    const double dx = (double)lo[2 * (j0 + jl)] - lbx, dy = (double)lo[2 * (j0 + jl) + 1] - lby;
                    const double l2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
                    ah[jl] = __dmul_rn(alpha, exp(__ddiv_rn(-l2, denom)));
                }
                __syncthreads();
                for (int jl = warp; jl < gl; jl += kTickThreads / 32) {
                    double* h = H + jl * ds;
                    const double a = ah[jl];
                    for (int c = lane; c < d; c += 32) h[c] = __dadd_rn(h[c], __dmul_rn(a, __dsub_rn(x[c], h[c])));
                }
            } else if (b >= j0 && b < j0 + gl) {
                double* h = H + (b - j0) * ds;
                for (int c = tid; c < d; c += kTickThreads)
                    h[c] = __dadd_rn(h[c], __dmul_rn(alpha, __dsub_rn(x[c], h[c])));
            }
            __syncthreads();
        }
    }
    for (int e = tid; e < gl * d; e += kTickThreads) hi_f32[(int64_t)j0 * d + e] = (float)H[(e / d) * ds + e % d];
    if (cs > 1) cluster_sync_all();  // no CTA exits while a peer may still read its candidate slots
}


// ---------------------------------------------------------------------------
// Register-resident variant (d <= 32 x Q): thread (warp w, lane l) of cluster
// CTA r holds hi[j][c] for j = r*gs + w + 32 m (m < M) and c = l + 32 q
// (q < Q) in registers -- no shared-memory traffic for the landmarks at all.
// Per sample: per-landmark warp-shuffle sums (M independent reductions),
// per-warp argmin, one __syncthreads + per-CTA argmin (every warp redundantly,
// no second barrier), one cluster barrier + CS candidates read over DSMEM
// (CS > 1), then h_j = exp(.) computed by lane m and shuffled, and the
// in-register update.  ~1 barrier pair per sample is the critical path.
// ---------------------------------------------------------------------------
template <bool SOM, int M, int Q>
__global__ void __launch_bounds__(kTickThreads) online_tick_reg_kernel(const float* __restrict__ X, int d,
                                                                       const int64_t* __restrict__ sample, int B,
                                                                       float* __restrict__ hi_f32,
                                                                       const float* __restrict__ lo, int g, int gs,
                                                                       double sigma, double alpha) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red_v[2][32];
    __shared__ int red_j[2][32];
    __shared__ double cand_v[2];
    __shared__ int cand_j[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t rank = cluster_rank(), cs = cluster_size();
    double2* LO = reinterpret_cast<double2*>(sm);       // g layout positions (f64)
    double* xs = sm + 2 * (size_t)g;                     // SB x (32 Q) staged sample rows
    constexpr int DP = 32 * Q;
    if (SOM)  // k-means has no layout (lo == nullptr)
        for (int j = tid; j < g; j += kTickThreads) LO[j] = make_double2((double)lo[2 * j], (double)lo[2 * j + 1]);
    const int j0 = (int)rank * gs;
    double h[M][Q];
    bool own[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int j = j0 + warp + 32 * m;
        own[m] = (warp + 32 * m < gs) && j < g;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int c = lane + 32 * q;
            h[m][q] = (own[m] && c < d) ? (double)hi_f32[(int64_t)j * d + c] : 0.0;
        }
    }
    const double denom = 2.0 * sigma * sigma;
    const double inf = __longlong_as_double(0x7ff0000000000000ll);

    for (int s0 = 0; s0 < B; s0 += kTickSB) {
        const int nb = min(kTickSB, B - s0);
        __syncthreads();
        for (int e = tid; e < nb * DP; e += kTickThreads) {
            const int r = e / DP, c = e % DP;
            xs[e] = c < d ? (double)__ldg(X + sample[s0 + r] * d + c) : 0.0;
        }
        __syncthreads();
        for (int s = 0; s < nb; ++s) {
            const int par = s & 1;
            double xv[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) xv[q] = xs[s * DP + lane + 32 * q];
            // distances of this warp's M landmarks (all lanes end with the sums)
            double dist[M];
#pragma unroll
            for (int m = 0; m < M; ++m) {
                double a = 0.0;
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const double t = h[m][q] - xv[q];
                    a = fma(t, t, a);
                }
                dist[m] = a;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1)
#pragma unroll
                for (int m = 0; m < M; ++m) dist[m] += __shfl_xor_sync(0xffffffffu, dist[m], o);
            double bv = inf;
            int bj = 0x7fffffff;
#pragma unroll
            for (int m = 0; m < M; ++m)
                if (own[m] && dist[m] < bv) bv = dist[m], bj = j0 + warp + 32 * m;  // m ascending: first minimum
            if (lane == 0) red_v[par][warp] = bv, red_j[par][warp] = bj;
            __syncthreads();
            // per-CTA argmin, redundantly in every warp (no second barrier)
            bv = red_v[par][lane];
            bj = red_j[par][lane];
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                if (lex_less(ov, oj, bv, bj)) bv = ov, bj = oj;
            }
            if (cs > 1) {
                if (tid == 0) cand_v[par] = bv, cand_j[par] = bj;
                cluster_sync_all();
                bv = inf;
                bj = 0x7fffffff;
                if (lane < (int)cs) {
                    bv = ld_peer_f64(map_peer(&cand_v[par], lane));
                    bj = ld_peer_s32(map_peer(&cand_j[par], lane));
                }
#pragma unroll
                for (int o = 4; o; o >>= 1) {  // cs <= 8
                    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                    const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                    if (lex_less(ov, oj, bv, bj)) bv = ov, bj = oj;
                }
            }
            const int b = __shfl_sync(0xffffffffu, bj, 0);  // lanes >= cs hold partial results
            if (SOM) {
                // lane m computes alpha * h_j for the warp's landmark m, then broadcast
                const double2 lb = LO[b];
                double ahl = 0.0;
                if (lane < M) {
                    const int j = min(j0 + warp + 32 * lane, g - 1);
                    const double2 lj = LO[j];
                    const double dx = lj.x - lb.x, dy = lj.y - lb.y;
                    const double l2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
                    ahl = __dmul_rn(alpha, exp(__ddiv_rn(-l2, denom)));
                }
#pragma unroll
                for (int m = 0; m < M; ++m) {
                    const double a = __shfl_sync(0xffffffffu, ahl, m);
#pragma unroll
                    for (int q = 0; q < Q; ++q) h[m][q] = __dadd_rn(h[m][q], __dmul_rn(a, __dsub_rn(xv[q], h[m][q])));
                }
            } else {
#pragma unroll
                for (int m = 0; m < M; ++m)
                    if (j0 + warp + 32 * m == b)
#pragma unroll
                        for (int q = 0; q < Q; ++q)
                            h[m][q] = __dadd_rn(h[m][q], __dmul_rn(alpha, __dsub_rn(xv[q], h[m][q])));
            }
        }
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int j = j0 + warp + 32 * m;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int c = lane + 32 * q;
            if (own[m] && c < d) hi_f32[(int64_t)j * d + c] = (float)h[m][q];
        }
    }
    if (cs > 1) cluster_sync_all();
}


// ---------------------------------------------------------------------------
// Row-per-thread variant (d <= 64): thread t of cluster CTA r owns landmark
// j = r*T + t with its whole f64 row in registers.  The distance is a
// per-thread f64 FMA sum (4 interleaved partial chains, no shuffles); only
// the argmin crosses lanes (5 shuffle levels per warp + W-entry CTA reduce +
// the cluster exchange); h_j is one exp per thread; the update touches only
// the thread's own registers.  The f64 work per sample (5 g d ops) is spread
// over CS SMs with T = 32 W threads each.
// ---------------------------------------------------------------------------
template <bool SOM, int DP, int W>
__global__ void __launch_bounds__(32 * W) online_tick_row_kernel(const float* __restrict__ X, int d,
                                                                 const int64_t* __restrict__ sample, int B,
                                                                 float* __restrict__ hi_f32, const float* __restrict__ lo,
                                                                 int g, double sigma, double alpha) {
    constexpr int T = 32 * W;
    constexpr int SB = 128;  // staged samples per chunk
    __shared__ __align__(16) double xs[SB * DP];
    __shared__ double red_v[2][W];
    __shared__ int red_j[2][W];
    __shared__ double cand_v[2];
    __shared__ int cand_j[2];
    extern __shared__ double2 LOs[];  // g layout positions (f64), SOM only
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t rank = cluster_rank(), cs = cluster_size();
    const int j = (int)rank * T + tid;
    const bool own = j < g;
    double h[DP];
#pragma unroll
    for (int c = 0; c < DP; ++c) h[c] = (own && c < d) ? (double)hi_f32[(int64_t)j * d + c] : 0.0;
    double2 lj = make_double2(0.0, 0.0);
    if (SOM) {
        for (int q = tid; q < g; q += T) LOs[q] = make_double2((double)lo[2 * q], (double)lo[2 * q + 1]);
        if (own) lj = make_double2((double)lo[2 * j], (double)lo[2 * j + 1]);
    }
    const double denom = 2.0 * sigma * sigma;
    const double inf = __longlong_as_double(0x7ff0000000000000ll);

    for (int s0 = 0; s0 < B; s0 += SB) {
        const int nb = min(SB, B - s0);
        __syncthreads();
        for (int e = tid; e < nb * DP; e += T) {
            const int r = e / DP, c = e % DP;
            xs[e] = c < d ? (double)__ldg(X + sample[s0 + r] * d + c) : 0.0;
        }
        __syncthreads();
        for (int s = 0; s < nb; ++s) {
            const int par = s & 1;
            const double2* x2 = reinterpret_cast<const double2*>(xs + s * DP);
            double p[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int c2 = 0; c2 < DP / 2; ++c2) {
                const double2 xv = x2[c2];  // broadcast
                const double t0 = h[2 * c2] - xv.x, t1 = h[2 * c2 + 1] - xv.y;
                p[(2 * c2) & 3] = fma(t0, t0, p[(2 * c2) & 3]);
                p[(2 * c2 + 1) & 3] = fma(t1, t1, p[(2 * c2 + 1) & 3]);
            }
            double bv = own ? (p[0] + p[1]) + (p[2] + p[3]) : inf;
            int bj = own ? j : 0x7fffffff;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                if (lex_less(ov, oj, bv, bj)) bv = ov, bj = oj;
            }
            if (lane == 0) red_v[par][warp] = bv, red_j[par][warp] = bj;
            __syncthreads();
            bv = red_v[par][0];
            bj = red_j[par][0];
#pragma unroll
            for (int w = 1; w < W; ++w)
                if (lex_less(red_v[par][w], red_j[par][w], bv, bj)) bv = red_v[par][w], bj = red_j[par][w];
            if (cs > 1) {
                if (tid == 0) cand_v[par] = bv, cand_j[par] = bj;
                cluster_sync_all();
                bv = inf;
                bj = 0x7fffffff;
                if (lane < (int)cs) {
                    bv = ld_peer_f64(map_peer(&cand_v[par], lane));
                    bj = ld_peer_s32(map_peer(&cand_j[par], lane));
                }
#pragma unroll
                for (int o = 4; o; o >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                    const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                    if (lex_less(ov, oj, bv, bj)) bv = ov, bj = oj;
                }
                bj = __shfl_sync(0xffffffffu, bj, 0);
            }
            const int b = bj;
            const double* xr = xs + s * DP;
            if (SOM) {
                const double2 lb = LOs[b];
                const double dx = lj.x - lb.x, dy = lj.y - lb.y;
                const double l2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
                const double a = __dmul_rn(alpha, exp(__ddiv_rn(-l2, denom)));
#pragma unroll
                for (int c = 0; c < DP; ++c) h[c] = __dadd_rn(h[c], __dmul_rn(a, __dsub_rn(xr[c], h[c])));
            } else if (j == b) {
#pragma unroll
                for (int c = 0; c < DP; ++c) h[c] = __dadd_rn(h[c], __dmul_rn(alpha, __dsub_rn(xr[c], h[c])));
            }
        }
    }
    if (own)
#pragma unroll
        for (int c = 0; c < DP; ++c)
            if (c < d) hi_f32[(int64_t)j * d + c] = (float)h[c];
    if (cs > 1) cluster_sync_all();
}

}  // namespace

namespace esom_host {

template <bool SOM, int DP, int W>
int launch_row(int cs, const float* X, int d, const int64_t* sample, int B, float* hi, const float* lo, int g,
               double sigma, double alpha, cudaStream_t st) {
    auto kern = online_tick_row_kernel<SOM, DP, W>;
    const size_t smem = SOM ? (size_t)g * 16 : 0;
    if (smem > 160 * 1024) return -1;
    if (smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, 1, 1);
    cfg.blockDim = dim3(32 * W, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, X, d, sample, B, hi, lo, g, sigma, alpha);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(ESOM_ERR_CUDA, "online_tick_row_kernel launch: %s", cudaGetErrorString(e));
    }
    return cuda_check("online_tick_row_kernel");
}

// W warps per CTA (landmarks per CTA = 32 W), cs = ceil(g / 32 W) <= 8
template <bool SOM, int DP>
int launch_row_w(const float* X, int d, const int64_t* sample, int B, float* hi, const float* lo, int g, double sigma,
                 double alpha, cudaStream_t st) {
    static const int wpref = getenv("ESOM_TICK_W") ? atoi(getenv("ESOM_TICK_W")) : 0;
    // measured (B200, C3/C4 shapes, 256 samples): g <= 256 one 256-thread CTA
    // (0.34 ms; a cluster barrier per sample costs more than it saves), larger g
    // the narrowest CTAs that fit 8 per cluster (g = 1024: W = 4, 0.45 ms)
    int w = wpref ? wpref : (g <= 256 ? 8 : 1);
    while (w < 8 && (g + 32 * w - 1) / (32 * w) > 8) w *= 2;
    const int cs = (g + 32 * w - 1) / (32 * w);
    if (cs > 8) return -1;
    switch (w) {
        case 1: return launch_row<SOM, DP, 1>(cs, X, d, sample, B, hi, lo, g, sigma, alpha, st);
        case 2: return launch_row<SOM, DP, 2>(cs, X, d, sample, B, hi, lo, g, sigma, alpha, st);
        case 4: return launch_row<SOM, DP, 4>(cs, X, d, sample, B, hi, lo, g, sigma, alpha, st);
        case 8: return launch_row<SOM, DP, 8>(cs, X, d, sample, B, hi, lo, g, sigma, alpha, st);
        default: return -1;
    }
}

template <bool SOM>
int launch_row_any(const float* X, int d, const int64_t* sample, int B, float* hi, const float* lo, int g,
                   double sigma, double alpha, cudaStream_t st) {
    if (d <= 8) return launch_row_w<SOM, 8>(X, d, sample, B, hi, lo, g, sigma, alpha, st);
    if (d <= 16) return launch_row_w<SOM, 16>(X, d, sample, B, hi, lo, g, sigma, alpha, st);
    if (d <= 32) return launch_row_w<SOM, 32>(X, d, sample, B, hi, lo, g, sigma, alpha, st);
    return -1;
}

template <bool SOM, int M, int Q>
int launch_reg(int cs, int gs, const float* X, int d, const int64_t* sample, int B, float* hi, const float* lo, int g,
               double sigma, double alpha, cudaStream_t st) {
    auto kern = online_tick_reg_kernel<SOM, M, Q>;
    const size_t smem = (size_t)g * 16 + (size_t)kTickSB * 32 * Q * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, 1, 1);
    cfg.blockDim = dim3(kTickThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, X, d, sample, B, hi, lo, g, gs, sigma, alpha);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(ESOM_ERR_CUDA, "online_tick_reg_kernel launch: %s", cudaGetErrorString(e));
    }
    return cuda_check("online_tick_reg_kernel");
}

template <bool SOM>
int launch_reg_any(const float* X, int d, const int64_t* sample, int B, float* hi, const float* lo, int g,
                   double sigma, double alpha, cudaStream_t st) {
    // registers per thread: M x Q doubles; CTAs per cluster cs = g / (32 M) <= 8
    static const int mpref = getenv("ESOM_TICK_M") ? atoi(getenv("ESOM_TICK_M")) : 0;
    const int Q = (d + 31) / 32;
    if (Q > 2 || (size_t)g * 16 + (size_t)kTickSB * 64 * 8 > kTickSmemCap) return -1;
    for (int M = 1; M <= 8; M *= 2) {
        if (mpref && M < mpref) continue;
        const int cs = (g + 32 * M - 1) / (32 * M);
        // measured (B200, d = 32): 4-CTA clusters balance the per-SM shuffle work
        // against the cluster barrier (g = 256: M = 2 0.54 ms/tick vs M = 1 0.68, M = 8 0.73)
        if (!mpref && cs > 4 && M < 8 && M * 2 * Q <= 8) continue;
        if (cs > 8 || M * Q > 8) continue;
        const int gs = 32 * M;
        if (Q == 1) {
            if (M == 1) return launch_reg<SOM, 1, 1>(cs, gs, X, d, sample, B, hi, lo, g, sigma, alpha, st);
            if (M == 2) return launch_reg<SOM, 2, 1>(cs, gs, X, d, sample, B, hi, lo, g, sigma, alpha, st);
            if (M == 4) return launch_reg<SOM, 4, 1>(cs, gs, X, d, sample, B, hi, lo, g, sigma, alpha, st);
            return launch_reg<SOM, 8, 1>(cs, gs, X, d, sample, B, hi, lo, g, sigma, alpha, st);
        }
        if (M == 1) return launch_reg<SOM, 1, 2>(cs, gs, X, d, sample, B, hi, lo, g, sigma, alpha, st);
        if (M == 2) return launch_reg<SOM, 2, 2>(cs, gs, X, d, sample, B, hi, lo, g, sigma, alpha, st);
        return launch_reg<SOM, 4, 2>(cs, gs, X, d, sample, B, hi, lo, g, sigma, alpha, st);
    }
    return -1;
}

// Returns ESOM_OK on launch, -1 when the shape needs the global-memory kernel
// (f64 rows do not fit 8 CTAs' shared memory), else an error code.
int launch_online_tick_cluster(bool som, const float* X, int d, const int64_t* sample, int B, float* hi,
                               const float* lo, int g, double sigma, double alpha, cudaStream_t st) {
    if (getenv("ESOM_TICK_GLOBAL")) return -1;  // A/B switches (measurement only)
    if (!getenv("ESOM_TICK_SMEM") && !getenv("ESOM_TICK_REG")) {
        const int r = som ? launch_row_any<true>(X, d, sample, B, hi, lo, g, sigma, alpha, st)
                          : launch_row_any<false>(X, d, sample, B, hi, lo, g, sigma, alpha, st);
        if (r >= 0) return r;
    }
    if (!getenv("ESOM_TICK_SMEM")) {
        const int r = som ? launch_reg_any<true>(X, d, sample, B, hi, lo, g, sigma, alpha, st)
                          : launch_reg_any<false>(X, d, sample, B, hi, lo, g, sigma, alpha, st);
        if (r >= 0) return r;
    }
    int cs = 1, gs = g;
    size_t smem = 0;
    for (cs = 1; cs <= 8; cs *= 2) {
        gs = (g + cs - 1) / cs;
        smem = ((size_t)gs * (d + 1) + gs + (size_t)kTickSB * d) * 8;
        if (smem <= kTickSmemCap) break;
    }
    if (cs > 8) return -1;
    auto kern = som ? online_tick_cluster_kernel<true> : online_tick_cluster_kernel<false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, 1, 1);
    cfg.blockDim = dim3(kTickThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, X, d, sample, B, hi, lo, g, gs, sigma, alpha);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(ESOM_ERR_CUDA, "online_tick_cluster_kernel launch: %s", cudaGetErrorString(e));
    }
    return cuda_check("online_tick_cluster_kernel");
}

}  // namespace esom_host
