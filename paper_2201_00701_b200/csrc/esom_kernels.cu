// esom_kernels.cu -- sm_100a kernels of the EmbedSOM hot path and the C ABI
// declared in include/esom.h.
//
//   pack_landmarks_kernel   hi (g×d) -> Lt[tile][c][32], padded   (prep for TMA staging)
//   pair_table_kernel       packed triangle 0.5/hd2 (faithful hd2 test)  ref: projection.py:332-340
//   knn_scan_kernel<DC,KP>  exact distance tiles + top-k (+ BMU statistics)   esom_scan.cuh
//                            ref: knn.py:65-92 / 148-184
//   project_fast_kernel<KP> scores + law-of-cosines projection              esom_project.cuh
//                            ref: projection.py:38-121; embed = scan + project (projection.py:220-245)
//   knn_sort_kernel         k > 64 fallback: block-per-point full sort    ref: knn.py:201-214
//   scores_kernel           ref: projection.py:38-65
//   project_kernel          faithful mixed-precision pair loop            ref: projection.py:68-121
//   som_tick_kernel         sequential online SOM (one CTA)               ref: som.py:44-68
//   kmeans_tick_kernel      sequential online k-means (one CTA)           ref: graphmodel.py:87-102
//   batch_update_kernel     batch-SOM landmark update (NEW)
#include <cstdarg>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "esom_common.cuh"
#include "esom_faithful.cuh"
#include "esom_host.h"
#include "esom_scan_args.h"
#include "../../include/esom.h"

using namespace esom;

namespace esom_host {

thread_local char g_err[512] = "";

int set_err(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

std::atomic<long long> g_launches{0};

int cuda_check(const char* where, int launches) {
    g_launches.fetch_add(launches, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof(g_err), "CUDA error in %s: %s", where, cudaGetErrorString(e));
        return ESOM_ERR_CUDA;
    }
    return ESOM_OK;
}

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

int max_smem_optin() {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v > 0 ? v : 227 * 1024;
}

size_t resident_limit() {
    static size_t lim = 0;
    if (!lim) {
        const char* e = getenv("ESOM_RESIDENT_KB");
        lim = (size_t)(e ? atoi(e) : 96) * 1024;
    }
    return lim;
}

}  // namespace esom_host

using namespace esom_host;

// ---------------------------------------------------------------------------
// Kernel timing (diagnostic, off by default): CUDA events recorded on the
// launching stream around the hot kernels, summed per kernel name on query.
// bench.py uses it to time the dominant kernel live (esom_timing_*).
// ---------------------------------------------------------------------------
namespace {
struct TimedLaunch {
    std::string name;
    cudaEvent_t a, b;
};
std::mutex g_tmu;
std::vector<TimedLaunch> g_tl;
bool g_timing = false;

struct KTimer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t st;
    const char* name;
    KTimer(const char* n, cudaStream_t s) : st(s), name(n) {
        if (!g_timing) return;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
    }
    ~KTimer() {
        if (!a) return;
        cudaEventRecord(b, st);
        std::lock_guard<std::mutex> lk(g_tmu);
        g_tl.push_back({name, a, b});
    }
};
}  // namespace

namespace {

int round_dp(int d) { return d <= 4 ? 4 : (d + 3) / 4 * 4; }

// ---------------------------------------------------------------------------
// Preparation kernels
// ---------------------------------------------------------------------------

// Lt[tile][c][32]: landmark j = tile*32 + lane, dim c.  Dims c >= d are 0
// (adds +0 to an exact sum -> bit-identical); rows j >= g are +inf (never
// selected: (inf, j >= g) never precedes the (inf, g) sentinel).
__global__ void pack_landmarks_kernel(const float* __restrict__ hi, int g, int d, int dp, int ntiles,
                                      float* __restrict__ Lt, int32_t* flag) {
    const int64_t total = (int64_t)ntiles * dp * kTile;
    bool bad = false;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int lane = (int)(e % kTile);
        const int c = (int)((e / kTile) % dp);
        const int t = (int)(e / ((int64_t)kTile * dp));
        const int j = t * kTile + lane;
        float v;
        if (j >= g) v = __int_as_float(0x7f800000);
        else if (c >= d) v = 0.0f;
        else {
            v = hi[(int64_t)j * d + c];
            bad |= !finite_f(v);
        }
        Lt[e] = v;
    }
    flag_nonfinite(flag, bad);
}

__global__ void check_finite_kernel(const float* __restrict__ v, int64_t count, int32_t* flag) {
    bool bad = false;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
        bad |= !finite_f(v[e]);
    flag_nonfinite(flag, bad);
}

// Packed upper triangle T[tri(u,v)] (u < v) = 0.5 / hd2(u,v) as f32 when the
// reference keeps the pair (hd2 >= 1e-12 with hd2 = sum_c (f64)(e*e), e =
// hi[v,c] - hi[u,c] in f32, ref: projection.py:332-340), else -1.  hd2 is
// symmetric (f32 subtraction is sign-symmetric), so one triangle suffices.
// *tmax (zeroed by the caller) = max kept T: the model-wide bound the
// projection uses to decide which points need f64 squared distances.
__global__ void pair_table_kernel(const float* __restrict__ hi, int g, int d, float* __restrict__ T,
                                  float* __restrict__ tmax) {
    const int64_t total = (int64_t)g * g;
    float tm = 0.0f;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int u = (int)(e / g), v = (int)(e % g);
        if (v <= u) continue;
        const float* hu = hi + (int64_t)u * d;
        const float* hv = hi + (int64_t)v * d;
        double hd2 = 0.0;
        for (int c = 0; c < d; ++c) {
            const float df = __fsub_rn(hv[c], hu[c]);
            hd2 = __dadd_rn(hd2, (double)__fmul_rn(df, df));
        }
        const float t = hd2 < kPairEps ? -1.0f : (float)(0.5 / hd2);
        T[(int64_t)u * (2 * (int64_t)g - u - 1) / 2 + (v - u - 1)] = t;
        tm = fmaxf(tm, t);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
    if ((threadIdx.x & 31) == 0 && tm > 0.0f) atomicMax(reinterpret_cast<int*>(tmax), __float_as_int(tm));
}


// Tiled form for d <= 64: a 32 x 32 block of (u, v) pairs stages its 64 rows in
// shared memory once (the row-per-pair kernel above re-reads 2 d floats per
// pair from L1/L2).  Same per-pair arithmetic and order -> identical table.
constexpr int kPairTile = 32;

__global__ void __launch_bounds__(256) pair_table_tiled_kernel(const float* __restrict__ hi, int g, int d,
                                                               float* __restrict__ T, float* __restrict__ tmax) {
    __shared__ float Ru[kPairTile][65], Rv[kPairTile][65];
    const int tu = blockIdx.y, tv = blockIdx.x;
    if (tv < tu) return;  // upper triangle of tiles
    const int u0 = tu * kPairTile, v0 = tv * kPairTile;
    for (int e = threadIdx.x; e < kPairTile * d; e += blockDim.x) {
        const int r = e / d, c = e % d;
        Ru[r][c] = u0 + r < g ? hi[(int64_t)(u0 + r) * d + c] : 0.0f;
        Rv[r][c] = v0 + r < g ? hi[(int64_t)(v0 + r) * d + c] : 0.0f;
    }
    __syncthreads();
    float tm = 0.0f;
    for (int e = threadIdx.x; e < kPairTile * kPairTile; e += blockDim.x) {
        const int ru = e / kPairTile, rv = e % kPairTile;  // lanes walk v: conflict-free rows (stride 65)
        const int u = u0 + ru, v = v0 + rv;
        if (u >= g || v >= g || v <= u) continue;
        double hd2 = 0.0;
        for (int c = 0; c < d; ++c) {
            const float df = __fsub_rn(Rv[rv][c], Ru[ru][c]);
            hd2 = __dadd_rn(hd2, (double)__fmul_rn(df, df));
        }
        const float t = hd2 < kPairEps ? -1.0f : (float)(0.5 / hd2);
        T[(int64_t)u * (2 * (int64_t)g - u - 1) / 2 + (v - u - 1)] = t;
        tm = fmaxf(tm, t);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
    if ((threadIdx.x & 31) == 0 && tm > 0.0f) atomicMax(reinterpret_cast<int*>(tmax), __float_as_int(tm));
}

// Landmark centroid c (f64 mean, rounded to f32; dims >= d are 0): the
// tensor-core screens work on x - c and l - c, whose norms (and so the error
// bounds) are several times smaller than those of x and l.
__global__ void center_kernel(const float* __restrict__ hi, int g, int d, int dpad, float* __restrict__ cen) {
    // one block per 32 dims: 32 row phases x 32 dims (1024 threads), f64
    // partial sums, 4 rows in flight per thread; any centre is valid (the
    // screens' bounds use the centred vectors actually formed), this one is
    // the rounded mean
    __shared__ double part[32][33];
    const int c = threadIdx.x & 31, r0 = threadIdx.x >> 5;
    const int c0 = blockIdx.x * 32;
    double s = 0.0;
    if (c0 + c < d) {
        int j = r0;
        for (; j + 96 < g; j += 128) {
            const float a0 = __ldg(hi + (int64_t)j * d + c0 + c), a1 = __ldg(hi + (int64_t)(j + 32) * d + c0 + c);
            const float a2 = __ldg(hi + (int64_t)(j + 64) * d + c0 + c), a3 = __ldg(hi + (int64_t)(j + 96) * d + c0 + c);
            s += ((double)a0 + (double)a1) + ((double)a2 + (double)a3);
        }
        for (; j < g; j += 32) s += (double)__ldg(hi + (int64_t)j * d + c0 + c);
    }
    part[r0][c] = s;
    __syncthreads();
    if (r0 == 0 && c0 + c < dpad) {
        double t = 0.0;
        for (int q = 0; q < 32; ++q) t += part[q][c];
        cen[c0 + c] = c0 + c < d ? (float)(t / g) : 0.0f;
    }
}

// Tensor-core operands of the landmarks (esom_tc.cuh, esom_tc2.cuh): l' =
// fl(l - c) as B = -2 l' (exact scaling: the MMA yields -2 x'.l') split into
// bf16 hi/lo in the canonical K-major layout (gpad rows x d16, zero padded),
// |l'_j|^2 (nearest f32 of the f64 sum; +inf on padding rows) and max |l'_j|,
// max |l'_j|^2 (rounded up) for the error bounds.
__global__ void tc_prepare_kernel(const float* __restrict__ hi0, int g, int d, int d16, int gpad,
                                  const int32_t* __restrict__ rowmap, const float* __restrict__ cen,
                                  uint16_t* __restrict__ Bhi, uint16_t* __restrict__ Blo, float* __restrict__ ln,
                                  float* __restrict__ lstats) {
    const int chunks = d16 / 8;
    const int64_t total = (int64_t)gpad * chunks;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int row = (int)(e / chunks), c0 = (int)(e % chunks) * 8;
        // screen row `row` holds landmark rowmap[row] (rows >= g: padding)
        const float* hi = hi0 + (row < g ? (int64_t)(__ldg(rowmap + row) - row) * d : 0);
        uint32_t hw[4], lw[4];
        for (int q = 0; q < 8; q += 2) {
            const float v0 = (row < g && c0 + q < d) ? -2.0f * (hi[(int64_t)row * d + c0 + q] - cen[c0 + q]) : 0.0f;
            const float v1 =
                (row < g && c0 + q + 1 < d) ? -2.0f * (hi[(int64_t)row * d + c0 + q + 1] - cen[c0 + q + 1]) : 0.0f;
            const uint16_t h0 = __bfloat16_as_ushort(__float2bfloat16_rn(v0));
            const uint16_t h1 = __bfloat16_as_ushort(__float2bfloat16_rn(v1));
            const uint16_t l0 = __bfloat16_as_ushort(__float2bfloat16_rn(v0 - __bfloat162float(__ushort_as_bfloat16(h0))));
            const uint16_t l1 = __bfloat16_as_ushort(__float2bfloat16_rn(v1 - __bfloat162float(__ushort_as_bfloat16(h1))));
            hw[q >> 1] = (uint32_t)h0 | ((uint32_t)h1 << 16);
            lw[q >> 1] = (uint32_t)l0 | ((uint32_t)l1 << 16);
        }
        const int64_t off = (((int64_t)(row >> 3) * chunks + (c0 >> 3)) << 6) + ((row & 7) << 3);  // in uint16
        *reinterpret_cast<uint4*>(Bhi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(Blo + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        if (c0 == 0) {
            if (row < g) {
                double s = 0.0;
                for (int c = 0; c < d; ++c) {
                    const double v = (double)(hi[(int64_t)row * d + c] - cen[c]);
                    s = fma(v, v, s);
                }
                ln[row] = (float)s;  // nearest f32 (<= 2^-24 relative, in the screens' bounds)
                atomicMax(reinterpret_cast<int*>(lstats), __float_as_int((float)(sqrt(s) * (1.0 + 1e-6))));
                atomicMax(reinterpret_cast<int*>(lstats + 1), __float_as_int((float)(s * (1.0 + 1e-6))));
            } else {
                ln[row] = __int_as_float(0x7f800000);
            }
        }
    }
}

// Exact-phase landmark rows for esom_tc2.cuh: gpad x ls f32, dims >= d and
// rows >= g zero (a +0 term leaves the reference's sequential sum unchanged;
// padding rows are never logged: their |l|^2 is +inf).
__global__ void lrow_kernel(const float* __restrict__ hi, int g, int d, int gpad, int ls,
                            const int32_t* __restrict__ rowmap, float* __restrict__ Lr) {
    const int64_t total = (int64_t)gpad * ls;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e / ls), c = (int)(e % ls);
        Lr[e] = (j < g && c < d) ? hi[(int64_t)__ldg(rowmap + j) * d + c] : 0.0f;
    }
}

// Screen-row order of the landmarks (tensor-core screens, g <= 1024).  The
// screens bound the k-th distance by the k-th smallest minimum over 32
// landmark groups (screen row mod 32), which is tight only when a point's k
// nearest landmarks fall in different groups.  A trained SOM keeps
// lattice-adjacent landmarks adjacent in hi, and with index order a 4 x 4
// lattice patch of a 32-wide map fell into 4 groups (C4 trained: 58 exact
// candidates per point).  Ordering the rows along the Morton curve of the
// LAYOUT (lo) makes any compact patch span consecutive rows, i.e. distinct
// groups (C4 trained: 19 candidates; untrained models are unaffected).  One
// CTA: min/max of lo, 2 x 10-bit Morton keys, bitonic sort of (key, index)
// (ties by index); lo == NULL or g > 1024: identity.
__device__ __forceinline__ uint32_t spread10(uint32_t v) {
    v &= 1023u;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}

__global__ void __launch_bounds__(1024) screen_order_kernel(const float* __restrict__ lo, int g, int gpad,
                                                           int32_t* __restrict__ rowmap) {
    __shared__ uint64_t key[1024];
    __shared__ float red[4][32];
    const int t = threadIdx.x;
    if (lo == nullptr || gpad > 1024) {
        for (int j = t; j < gpad; j += blockDim.x) rowmap[j] = j;
        return;
    }
    float mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (int j = t; j < g; j += blockDim.x) {
        const float x = lo[2 * j], y = lo[2 * j + 1];
        mnx = fminf(mnx, x); mny = fminf(mny, y); mxx = fmaxf(mxx, x); mxy = fmaxf(mxy, y);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mnx = fminf(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mny = fminf(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mxy = fmaxf(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
    }
    if ((t & 31) == 0) {
        red[0][t >> 5] = mnx; red[1][t >> 5] = mny; red[2][t >> 5] = mxx; red[3][t >> 5] = mxy;
    }
    __syncthreads();
    mnx = red[0][0]; mny = red[1][0]; mxx = red[2][0]; mxy = red[3][0];
    for (int w = 1; w < 32; ++w) {
        mnx = fminf(mnx, red[0][w]); mny = fminf(mny, red[1][w]);
        mxx = fmaxf(mxx, red[2][w]); mxy = fmaxf(mxy, red[3][w]);
    }
    const float span = fmaxf(fmaxf(mxx - mnx, mxy - mny), 1e-30f);
    for (int j = t; j < 1024; j += blockDim.x) {
        uint64_t kv = ~0ull;  // padding rows sort last, in index order
        if (j < g) {
            const float fx = (lo[2 * j] - mnx) / span, fy = (lo[2 * j + 1] - mny) / span;
            // non-finite layouts (rejected elsewhere) fall back to index order
            const uint32_t qx = (fx >= 0.0f && fx <= 1.0f) ? (uint32_t)(fx * 1023.0f) : 0u;
            const uint32_t qy = (fy >= 0.0f && fy <= 1.0f) ? (uint32_t)(fy * 1023.0f) : 0u;
            kv = ((uint64_t)(spread10(qx) | (spread10(qy) << 1)) << 32) | (uint32_t)j;
        } else {
            kv = (~0ull << 32) | (uint32_t)j;
        }
        key[j] = kv;
    }
    __syncthreads();
    for (int size = 2; size <= 1024; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int j = t; j < 1024; j += blockDim.x) {
                const int p = j ^ stride;
                if (p > j) {
                    const uint64_t a = key[j], b = key[p];
                    if ((a > b) == ((j & size) == 0)) {
                        key[j] = b;
                        key[p] = a;
                    }
                }
            }
            __syncthreads();
        }
    for (int j = t; j < gpad; j += blockDim.x) rowmap[j] = (int32_t)(uint32_t)key[j];
}

// BMU bucket sort of a chunk's neighbour rows (counting sort on idx[:,0]):
// the projection visits points grouped by nearest landmark, so the pair-table
// gathers of a warp coalesce when the table does not fit in shared memory.
__global__ void bmu_hist_kernel(const int32_t* __restrict__ idx, int64_t n, int k, int g, int32_t* __restrict__ cnt) {
    extern __shared__ int32_t h[];
    for (int b = threadIdx.x; b < g; b += blockDim.x) h[b] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&h[__ldg(idx + i * k)], 1);
    __syncthreads();
    for (int b = threadIdx.x; b < g; b += blockDim.x)
        if (h[b]) atomicAdd(cnt + b, h[b]);
}

__global__ void bmu_scan_kernel(int32_t* __restrict__ cnt, int g) {  // one CTA: exclusive scan in place
    // each thread sums a contiguous chunk, then a warp-shuffle block scan of the
    // chunk sums (a serial pass over 1024 partials by one thread cost ~9 us)
    __shared__ int32_t wsum[32];
    const int per = (g + blockDim.x - 1) / blockDim.x;
    const int b0 = threadIdx.x * per;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int s = 0;
    for (int b = b0; b < b0 + per && b < g; ++b) s += cnt[b];
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        int v = lane < nw ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (lane < nw) wsum[lane] = v;  // inclusive scan of the warp sums
    }
    __syncthreads();
    int acc = incl - s + (w > 0 ? wsum[w - 1] : 0);
    for (int b = b0; b < b0 + per && b < g; ++b) {
        const int v = cnt[b];
        cnt[b] = acc;
        acc += v;
    }
}

__global__ void bmu_scatter_kernel(const int32_t* __restrict__ idx, int64_t n, int k, int32_t* __restrict__ cursor,
                                   int32_t* __restrict__ perm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        perm[atomicAdd(cursor + __ldg(idx + i * k), 1)] = (int32_t)i;
}

// Scatter with CTA-local ranks: each CTA ranks its slice of points per bucket
// in shared memory, reserves one range per (CTA, bucket) with a single global
// atomic, then writes perm -- instead of one contended global atomic per point.
constexpr int kScatItems = 8;

__global__ void bmu_scatter2_kernel(const int32_t* __restrict__ idx, int64_t n, int k, int g,
                                    int32_t* __restrict__ cursor, int32_t* __restrict__ perm) {
    extern __shared__ int32_t sh[];
    int32_t* hist = sh;       // g
    int32_t* base = sh + g;   // g
    const int64_t slice = (int64_t)blockDim.x * kScatItems;
    for (int64_t s0 = blockIdx.x * slice; s0 < n; s0 += (int64_t)gridDim.x * slice) {
        for (int b = threadIdx.x; b < g; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        int bk[kScatItems], rk[kScatItems];
#pragma unroll
        for (int q = 0; q < kScatItems; ++q) {
            const int64_t i = s0 + (int64_t)q * blockDim.x + threadIdx.x;
            bk[q] = i < n ? __ldg(idx + i * k) : -1;
            rk[q] = bk[q] >= 0 ? atomicAdd(hist + bk[q], 1) : 0;
        }
        __syncthreads();
        for (int b = threadIdx.x; b < g; b += blockDim.x)
            if (hist[b]) base[b] = atomicAdd(cursor + b, hist[b]);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kScatItems; ++q) {
            const int64_t i = s0 + (int64_t)q * blockDim.x + threadIdx.x;
            if (bk[q] >= 0) perm[base[bk[q]] + rk[q]] = (int32_t)i;
        }
        __syncthreads();
    }
}

int grid_for(int64_t work, int threads);

// BMU counting sort of n neighbour rows (bucket = idx[i * k]): counts, exclusive
// scan, scatter.  Afterwards cntb[b] is the end of bucket b in perm.
int bmu_sort(const int32_t* idx, int64_t n, int k, int g, int32_t* cntb, int32_t* perm, cudaStream_t st) {
    cudaMemsetAsync(cntb, 0, (size_t)g * 4, st);
    bmu_hist_kernel<<<num_sms() * 2, 512, (size_t)g * 4, st>>>(idx, n, k, g, cntb);
    bmu_scan_kernel<<<1, 1024, 0, st>>>(cntb, g);
    if (g <= 8192) {
        const size_t smem = (size_t)g * 8;
        if (smem > 48 * 1024) cudaFuncSetAttribute(bmu_scatter2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int64_t slices = (n + 256 * kScatItems - 1) / (256 * kScatItems);
        const int64_t cap = (int64_t)num_sms() * 4;
        bmu_scatter2_kernel<<<(unsigned)(slices < cap ? (slices < 1 ? 1 : slices) : cap), 256, smem, st>>>(idx, n, k, g,
                                                                                                         cntb, perm);
    } else {
        bmu_scatter_kernel<<<grid_for(n, 256), 256, 0, st>>>(idx, n, k, cntb, perm);
    }
    return cuda_check("bmu_sort", 3);
}

// Batch-SOM statistics from a BMU-sorted order (after bmu_scatter, ends[b] is
// the end of landmark b's segment of perm): one warp per (kSegPart sorted
// positions, 32-dim slice) sums its points' fixed-point coordinates (exact
// int64) and adds one partial per segment it touches to S / C (~n/64 atomics
// per address row instead of one per point and dimension; integer sums, so
// the order of the partials does not matter).
constexpr int kSegPart = 256;

__global__ void __launch_bounds__(256, 4) bmu_segsum_kernel(const float* __restrict__ X, int d,
                                                         const int32_t* __restrict__ perm,
                                                         const int32_t* __restrict__ ends, int g, int64_t n,
                                                         acc_t* __restrict__ S, acc_t* __restrict__ C, double scale,
                                                         const int32_t* __restrict__ idx, int k) {
    // warp w sums sorted positions [w*kSegPart, (w+1)*kSegPart) (times the 32-dim
    // slices): every launched warp has work; a range crossing a BMU boundary
    // flushes one partial per segment it touches.  The first segment is the BMU
    // of the range's first point (idx[perm[p0] * k]: two dependent loads instead of
    // a 10-step binary search over ends, which dominated the short ranges)
    const int lane = threadIdx.x & 31;
    const int nsl = (d + 31) / 32;
    const int64_t nch = (n + kSegPart - 1) / kSegPart;
    const int64_t nw = nch * nsl;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nw;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int sl = (int)(w % nsl);
        const int64_t p0 = (w / nsl) * kSegPart;
        const int64_t p1 = p0 + kSegPart < n ? p0 + kSegPart : n;
        const int c = sl * 32 + lane;
        // segment of p0 = the BMU of its point (the counting sort's key)
        int b = __ldg(idx + (int64_t)__ldg(perm + p0) * k);
        int64_t pos = p0;
        while (pos < p1) {
            const int64_t e = min((int64_t)__ldg(ends + b), p1);
            acc_t acc = 0, acc1 = 0, acc2 = 0, acc3 = 0;
            if (S)
                for (int64_t base = pos; base < e; base += 32) {  // 32 perm entries per coalesced load
                    const int pe = base + lane < e ? __ldg(perm + base + lane) : 0;
                    const int nb = e - base < 32 ? (int)(e - base) : 32;
#pragma unroll
                    for (int h = 0; h < 32; h += 16) {
                        float v[16];  // 16 row loads in flight per lane (4 CTAs per SM without spills)
#pragma unroll
                        for (int q = 0; q < 16; ++q) {
                            const int r = __shfl_sync(0xffffffffu, pe, h + q);
                            v[q] = (h + q < nb && c < d) ? __ldg(X + (int64_t)r * d + c) : 0.0f;
                        }
#pragma unroll
                        for (int q = 0; q < 16; q += 4) {
                            acc += acc_fx(v[q], scale);
                            acc1 += acc_fx(v[q + 1], scale);
                            acc2 += acc_fx(v[q + 2], scale);
                            acc3 += acc_fx(v[q + 3], scale);
                        }
                    }
                }
            acc += (acc1 + acc2) + acc3;
            if (e > pos) {
                if (S && c < d) atomicAdd(S + (int64_t)b * d + c, acc);
                if (C && lane == 0 && sl == 0) atomicAdd(C + b, (acc_t)(e - pos));
            }
            pos = e;
            ++b;
        }
    }
}


// Batch-SOM statistics straight from the natural point order when the int64
// table fits one SM (d <= 32, g (d + 1) 8 B <= 200 KB; C3): X streams
// coalesced, each warp adds 8 points per step into a shared-memory fixed-point
// table (lane = dimension, 64-bit shared atomics), then one atomic per table
// entry into S / C.  No BMU sort and no row gather (the sorted-segment kernel above
// reads X in BMU order: random 128-byte rows, ncu 1.3 TB/s at C3).
constexpr int kAccThreads = 1024;

__global__ void __launch_bounds__(kAccThreads) bmu_accum_smem_kernel(const float* __restrict__ X, int64_t n, int d,
                                                                    const int32_t* __restrict__ idx, int k, int g,
                                                                    acc_t* __restrict__ S, acc_t* __restrict__ C,
                                                                    double scale) {
    extern __shared__ acc_t sS[];  // g x d, then g counts
    acc_t* sC = sS + (size_t)g * d;
    for (int e = threadIdx.x; e < g * d + g; e += kAccThreads) sS[e] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * (kAccThreads / 32) + warp;
    const int64_t nwarps = (int64_t)gridDim.x * (kAccThreads / 32);
    for (int64_t i0 = gw * 8; i0 < n; i0 += nwarps * 8) {
        float v[8];
        // lane u < 8 loads point i0 + u's BMU once (not 8 broadcast loads per lane) and
        // counts it: one count atomic instruction per 8 points
        const int bl = (lane < 8 && i0 + lane < n) ? __ldg(idx + (i0 + lane) * k) : -1;
        if (bl >= 0) atomicAdd(sC + bl, 1ull);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t i = i0 + u;
            v[u] = (i < n && lane < d) ? __ldg(X + i * d + lane) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int b = __shfl_sync(0xffffffffu, bl, u);
            if (b < 0) continue;
            if (lane < d) atomicAdd(sS + (size_t)b * d + lane, acc_fx(v[u], scale));
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < g * d; e += kAccThreads)
        if (S && sS[e] != 0) atomicAdd(S + e, sS[e]);
    for (int j = threadIdx.x; j < g; j += kAccThreads)
        if (C && sC[j] != 0) atomicAdd(C + j, sC[j]);
}

bool accum_smem_ok(int g, int d) { return d <= 32 && ((size_t)g * d + g) * 8 <= 200 * 1024; }

// ---------------------------------------------------------------------------
// Scores (ref: projection.py:38-59).  numba's float(f32) stays f32, so the
// root is sqrtf, widened; the rest is f64.  `exp` is CUDA's (<= 1 ulp from
// glibc); everything else is correctly rounded like the reference.
// ---------------------------------------------------------------------------
__global__ void scores_kernel(const float* __restrict__ sqd, int64_t n, int k, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float* row = sqd + i * k;
        score_row_dev(k, [&](int t) { return row[t]; }, out + i * k);
    }
}

__global__ void project_kernel(const float* __restrict__ X, int64_t n, int d, const float* __restrict__ hi,
                               const float* __restrict__ lo, const int32_t* __restrict__ idx,
                               const double* __restrict__ sc, int k, float* __restrict__ xy) {
    // d <= 32 with 32-byte rows: the register-resident variant (one kernel-uniform branch)
    const bool v8 = (d & 7) == 0 && rows32(hi, d) && rows32(X, d);
    const bool r32 = v8 && d <= 32;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (r32)
            project_row_faithful32(X + i * d, hi, lo, idx + i * k, sc + i * k, d, k, xy + 2 * i);
        else if (v8)
            project_row_faithful_v8(X + i * d, hi, lo, idx + i * k, sc + i * k, d, k, xy + 2 * i);
        else
            project_row_faithful(X + i * d, hi, lo, idx + i * k, sc + i * k, d, k, xy + 2 * i);
    }
}

// ---------------------------------------------------------------------------
// k > 64 (or huge d) fallback: one CTA per point, all g keys in smem,
// bitonic sort on the packed (f32 bits << 32 | j) key (monotone for s >= 0).
// ---------------------------------------------------------------------------
__global__ void knn_sort_kernel(const float* __restrict__ X, int64_t n, int d, const float* __restrict__ L, int g,
                                int gpow, int k, int32_t* __restrict__ out_idx, float* __restrict__ out_sqd,
                                int32_t* flag) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned long long* key = reinterpret_cast<unsigned long long*>(smem_raw);
    bool bad = false;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const float* x = X + i * d;
        for (int j = threadIdx.x; j < gpow; j += blockDim.x) {
            unsigned long long kk = ~0ull;
            if (j < g) {
                const float* l = L + (int64_t)j * d;
                float s = 0.0f;
                for (int c = 0; c < d; ++c) {
                    const float xv = x[c];
                    bad |= !finite_f(xv);
                    const float t = __fsub_rn(xv, l[c]);
                    s = __fadd_rn(s, __fmul_rn(t, t));
                }
                kk = ((unsigned long long)__float_as_uint(s) << 32) | (unsigned)j;
            }
            key[j] = kk;
        }
        __syncthreads();
        for (int size = 2; size <= gpow; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int t = threadIdx.x; t < gpow; t += blockDim.x) {
                    const int u = t ^ stride;
                    if (u > t) {
                        const bool asc = (t & size) == 0;
                        const unsigned long long ka = key[t], kb = key[u];
                        if ((ka > kb) == asc) {
                            key[t] = kb;
                            key[u] = ka;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int q = threadIdx.x; q < k; q += blockDim.x) {
            out_idx[i * k + q] = (int32_t)(key[q] & 0xffffffffu);
            out_sqd[i * k + q] = __uint_as_float((unsigned)(key[q] >> 32));
        }
        __syncthreads();
    }
    flag_nonfinite(flag, bad);
}

// ---------------------------------------------------------------------------
// Online trainers.  One CTA walks the host-drawn samples in order, hi in f64
// (workspace), exactly the per-element update order of numpy:
//   hi += (alpha * h_j) * (x - hi)      (ref: som.py:66-67)
// BMU = first index of the f64 minimum (ref: som.py:60-62, argmin).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void block_argmin(double v, int j, double* sv, int* sj, double& bv, int& bj) {
    // lexicographic (v, j) min across the block
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oj = __shfl_xor_sync(0xffffffffu, j, o);
        if (ov < v || (ov == v && oj < j)) {
            v = ov;
            j = oj;
        }
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        sv[w] = v;
        sj[w] = j;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < nw ? sv[threadIdx.x] : __longlong_as_double(0x7ff0000000000000ll);
        j = threadIdx.x < nw ? sj[threadIdx.x] : 0x7fffffff;
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int oj = __shfl_xor_sync(0xffffffffu, j, o);
            if (ov < v || (ov == v && oj < j)) {
                v = ov;
                j = oj;
            }
        }
        if (threadIdx.x == 0) {
            sv[0] = v;
            sj[0] = j;
        }
    }
    __syncthreads();
    bv = sv[0];
    bj = sj[0];
    __syncthreads();
}

template <bool SOM>
__global__ void __launch_bounds__(1024) online_tick_kernel(const float* __restrict__ X, int d,
                                                           const int64_t* __restrict__ sample, int B,
                                                           float* __restrict__ hi_f32, const float* __restrict__ lo,
                                                           int g, double sigma, double alpha, double* __restrict__ hi) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* x = reinterpret_cast<double*>(smem_raw);   // d
    double* ah = x + d;                                  // g  (alpha * h_j)
    __shared__ double red_v[32];
    __shared__ int red_j[32];
    const int64_t gd = (int64_t)g * d;
    for (int64_t e = threadIdx.x; e < gd; e += blockDim.x) hi[e] = (double)hi_f32[e];
    const double denom = 2.0 * sigma * sigma;
    __syncthreads();
    for (int s = 0; s < B; ++s) {
        const float* xs = X + sample[s] * d;
        for (int c = threadIdx.x; c < d; c += blockDim.x) x[c] = (double)xs[c];
        __syncthreads();
        double bv = __longlong_as_double(0x7ff0000000000000ll);
        int bj = 0x7fffffff;
        for (int j = threadIdx.x; j < g; j += blockDim.x) {
            const double* hj = hi + (int64_t)j * d;
            double acc = 0.0;
            for (int c = 0; c < d; ++c) {
                const double t = __dsub_rn(hj[c], x[c]);
                acc = __dadd_rn(acc, __dmul_rn(t, t));
            }
            if (acc < bv || (acc == bv && j < bj)) {
                bv = acc;
                bj = j;
            }
        }
        int b;
        double dummy;
        block_argmin(bv, bj, red_v, red_j, dummy, b);
        if (SOM) {
            const double lbx = (double)lo[2 * b], lby = (double)lo[2 * b + 1];
            for (int j = threadIdx.x; j < g; j += blockDim.x) {
                const double dx = __dsub_rn((double)lo[2 * j], lbx), dy = __dsub_rn((double)lo[2 * j + 1], lby);
                const double l2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
                ah[j] = __dmul_rn(alpha, exp(__ddiv_rn(-l2, denom)));
            }
            __syncthreads();
            for (int64_t e = threadIdx.x; e < gd; e += blockDim.x) {
                const int j = (int)(e / d), c = (int)(e % d);
                hi[e] = __dadd_rn(hi[e], __dmul_rn(ah[j], __dsub_rn(x[c], hi[e])));
            }
        } else {
            for (int c = threadIdx.x; c < d; c += blockDim.x) {
                double* hb = hi + (int64_t)b * d;
                hb[c] = __dadd_rn(hb[c], __dmul_rn(alpha, __dsub_rn(x[c], hb[c])));
            }
        }
        __syncthreads();
    }
    for (int64_t e = threadIdx.x; e < gd; e += blockDim.x) hi_f32[e] = (float)hi[e];
}

// ---------------------------------------------------------------------------
// Batch-SOM update (NEW).  One CTA per landmark j:
//   H_jb = exp(-|lo_j - lo_b|^2 / (2 sigma^2)),  num_j = sum_b H_jb S_b,
//   den_j = sum_b H_jb C_b;  mode 0: hi_j += (alpha/B)(num_j - den_j hi_j)
//   mode 1: hi_j = num_j / den_j (den_j > 0).
// ---------------------------------------------------------------------------
__global__ void batch_update_kernel(const acc_t* __restrict__ S, const acc_t* __restrict__ C, double inv_scale,
                                    const float* __restrict__ lo, int g, int d, double sigma, double alpha, int mode,
                                    float* __restrict__ hi) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* h = reinterpret_cast<double*>(smem_raw);  // g
    __shared__ double red[32];
    __shared__ double red2[16][32];
    const double denom = 2.0 * sigma * sigma;
    for (int j = blockIdx.x; j < g; j += gridDim.x) {
        const double ljx = lo[2 * j], ljy = lo[2 * j + 1];
        double den_p = 0.0, b_p = 0.0;
        for (int b = threadIdx.x; b < g; b += blockDim.x) {
            const double dx = ljx - (double)lo[2 * b], dy = ljy - (double)lo[2 * b + 1];
            const double cb = (double)(long long)C[b];
            const double hv = cb > 0.0 ? exp(-(dx * dx + dy * dy) / denom) : 0.0;
            h[b] = hv;
            den_p += hv * cb;
            b_p += cb;
        }
        // block reduce den, B
        for (int o = 16; o > 0; o >>= 1) {
            den_p += __shfl_xor_sync(0xffffffffu, den_p, o);
            b_p += __shfl_xor_sync(0xffffffffu, b_p, o);
        }
        const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
        if ((threadIdx.x & 31) == 0) {
            red[w] = den_p;
            red[16 + w] = b_p;
        }
        __syncthreads();
        double den = 0.0, Btot = 0.0;
        for (int q = 0; q < nw; ++q) {
            den += red[q];
            Btot += red[16 + q];
        }
        // num_j = H_j. S in 32-dim slices: lane = dimension, warps split b (coalesced S rows)
        const int lane = threadIdx.x & 31;
        for (int c0 = 0; c0 < d; c0 += 32) {
            const int c = c0 + lane;
            double num = 0.0;
            if (c < d)
                for (int b = w; b < g; b += nw)
                    num = fma(h[b], (double)(long long)S[(int64_t)b * d + c] * inv_scale, num);
            red2[w][lane] = num;
            __syncthreads();
            if (w == 0 && c < d) {
                double tot = 0.0;
                for (int q = 0; q < nw; ++q) tot += red2[q][lane];
                float* hj = hi + (int64_t)j * d + c;
                if (mode == 1) {
                    if (den > 0.0) *hj = (float)(tot / den);
                } else if (Btot > 0.0) {
                    const double h0 = (double)*hj;
                    *hj = (float)(h0 + (alpha / Btot) * (tot - den * h0));
                }
            }
            __syncthreads();
        }
    }
}

int kp_for(int k) {
    if (k <= 4) return 4;
    if (k <= 8) return 8;
    if (k <= 16) return 16;
    if (k <= 32) return 32;
    if (k <= 64) return 64;
    return 0;
}

struct Plan {
    int dp, dc, nch, ntiles, kp;
    size_t tile_bytes;
};

Plan make_plan(int d, int g, int k) {
    Plan p;
    p.dp = round_dp(d);
    if (p.dp <= 64) {
        p.dc = p.dp <= 4 ? 4 : p.dp <= 8 ? 8 : p.dp <= 16 ? 16 : p.dp <= 32 ? 32 : 64;
        p.dp = p.dc;
        p.nch = 1;
    } else {
        p.dc = 32;
        p.dp = (d + 31) / 32 * 32;
        p.nch = p.dp / 32;
    }
    p.ntiles = (g + kTile - 1) / kTile;
    p.kp = kp_for(k);
    p.tile_bytes = (size_t)p.dp * kTile * 4;
    return p;
}

int dispatch_scan(const Plan& p, ScanArgs a, cudaStream_t st) {
#define ESOM_CASE(DCV, KPV) \
    if (p.dc == DCV && p.kp == KPV) return launch_scan_t<DCV, KPV>(a, st);
#define ESOM_KPS(DCV) ESOM_CASE(DCV, 4) ESOM_CASE(DCV, 8) ESOM_CASE(DCV, 16) ESOM_CASE(DCV, 32) ESOM_CASE(DCV, 64)
    ESOM_KPS(4)
    ESOM_KPS(8)
    ESOM_KPS(16)
    ESOM_KPS(32)
    ESOM_KPS(64)
#undef ESOM_KPS
#undef ESOM_CASE
    return set_err(ESOM_ERR_UNSUPPORTED, "no scan kernel for this (d, k)%s", "");
}

int dispatch_project(int kp, ProjArgs a, cudaStream_t st) {
    switch (kp) {
        case 4: return launch_project_t<4>(a, st);
        case 8: return launch_project_t<8>(a, st);
        case 16: return launch_project_t<16>(a, st);
        case 32: return launch_project_t<32>(a, st);
        case 64: return launch_project_t<64>(a, st);
    }
    return set_err(ESOM_ERR_UNSUPPORTED, "no projection kernel for k%s", "");
}

int grid_for(int64_t work, int threads) {
    int64_t b = (work + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms() * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

// hi -> f64 (exact widening), once per model
__global__ void widen_kernel(const float* __restrict__ src, int64_t n, double* __restrict__ dst) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        dst[e] = (double)src[e];
}

// |h_j|^2 in f64 per landmark row (the far-point distances' dot-product form)
__global__ void row_norm64_kernel(const float* __restrict__ hi, int g, int d, double* __restrict__ hn) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < g; j += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < d; ++c) {
            const double v = (double)hi[(int64_t)j * d + c];
            s = fma(v, v, s);
        }
        hn[j] = s;
    }
}

struct ModelLayout {
    size_t lt, tri, bhi, blo, ln, lstats, lrow, rowmap, rec, hi64, hn64, total;
    bool has_rec;  // g x g pair records for project_reg3_kernel (k <= 16, g <= 1024)
    int d16, gpad, ls;
    // tensor-core GEMM screen for d > 32 (esom_tc3.cuh): per-model operands + per-chunk scratch
    bool t3;
    int dk, gp3;
    int64_t t3chunk;
    size_t cen3, b3hi, b3lo, ln3, ls3, a3hi, a3lo, xn3, cand3, cnt3, bmu3, perm3, hist3;
    // split tc2 screen (d <= 32, g > 256): per-chunk candidate bitmaps + info
    int64_t t2chunk;
    size_t t2bits, t2info, t2key, t2perm, t2hist;
};

size_t a256(size_t b) { return (b + 255) / 256 * 256; }

ModelLayout model_layout(int g, int d, int k, bool with_pairs) {
    const Plan p = make_plan(d, g, k < 1 ? 1 : k);
    ModelLayout m{};
    m.d16 = (d + 15) / 16 * 16;
    m.gpad = (g + 31) / 32 * 32;
    size_t o = 0;
    m.lt = o;
    o += a256((size_t)p.ntiles * p.tile_bytes);
    m.tri = o;
    if (with_pairs) o += a256((size_t)g * (g > 1 ? g - 1 : 1) / 2 * 4);
    m.has_rec = with_pairs && g <= 1024 && k <= 16;
    m.rec = o;
    if (m.has_rec) o += a256((size_t)g * g * 16);
    m.bhi = o;
    o += a256((size_t)m.gpad * m.d16 * 2);
    m.blo = o;
    o += a256((size_t)m.gpad * m.d16 * 2);
    m.ln = o;
    o += a256((size_t)m.gpad * 4);
    m.lstats = o;
    o += 256;
    m.rowmap = o;  // screen row -> landmark index of the tensor-core operands below
    o += a256((size_t)m.gpad * 4);
    m.ls = 0;
    m.lrow = o;
    if (d <= 32) {  // padded f32 rows of the pipelined tensor-core screen (esom_tc2.cuh)
        m.ls = (((m.d16 + 3) / 4) | 1) * 4;
        o += a256((size_t)m.gpad * m.ls * 4);
    }
    m.hi64 = o;  // f64 copy of hi: the far-point distances of the projection (precise_sqd)
    if (with_pairs) o += a256((size_t)g * d * 8);
    m.hn64 = o;  // |h_j|^2 in f64 (same use)
    if (with_pairs) o += a256((size_t)g * 8);
    m.t2chunk = 0;
    if (d <= 32 && m.gpad <= 1024) {
        m.t2chunk = 1 << 20;
        m.t2bits = o;  o += a256((size_t)m.t2chunk * (m.gpad / 32) * 4);
        m.t2info = o;  o += a256((size_t)m.t2chunk * 8);
        m.t2key = o;   o += a256((size_t)m.t2chunk * 4);
        m.t2perm = o;  o += a256((size_t)m.t2chunk * 4);
        m.t2hist = o;  o += a256((size_t)m.gpad * 4);
    }
    m.t3 = d > 32 && k <= 32 && g <= 65535;
    if (m.t3) {
        m.dk = (d + 31) / 32 * 32;
        m.gp3 = (g + 255) / 256 * 256;
        int64_t ch = (int64_t)(((size_t)512 << 20) / ((size_t)m.dk * 4 + 160));
        ch = ch >= (1 << 18) ? (1 << 18) : (ch < 4096 ? 4096 : ch / 256 * 256);
        m.t3chunk = ch;
        m.cen3 = o;  o += a256((size_t)m.dk * 4);
        m.b3hi = o;  o += a256((size_t)m.gp3 * m.dk * 2);
        m.b3lo = o;  o += a256((size_t)m.gp3 * m.dk * 2);
        m.ln3 = o;   o += a256((size_t)m.gp3 * 4);
        m.ls3 = o;   o += 256;
        m.a3hi = o;  o += a256((size_t)ch * m.dk * 2);
        m.a3lo = o;  o += a256((size_t)ch * m.dk * 2);
        m.xn3 = o;   o += a256((size_t)ch * 4);
        m.cand3 = o; o += a256((size_t)ch * 64 * 2);
        m.cnt3 = o;  o += a256((size_t)ch * 4);
        m.bmu3 = o;  o += a256((size_t)ch * 4);
        m.perm3 = o; o += a256((size_t)ch * 4);
        m.hist3 = o; o += a256((size_t)m.gp3 * 4);
    }
    m.total = o + 256;
    return m;
}

int32_t* g_tc_stats = nullptr;  // diagnostic: device counter of logged candidates (esom_set_tc_stats)
int32_t* tc_stats_ptr() { return g_tc_stats; }

bool tc_enabled() {  // ESOM_TC=0 forces the CUDA-core scan (read per call: tests toggle it)
    const char* e = getenv("ESOM_TC");
    return e ? atoi(e) != 0 : true;
}

// shapes the split-bf16 tensor-core screen handles (smem budget of esom_tc.cuh)
bool tc_eligible(int64_t n, int d, int g, int k) { return tc_enabled() && n >= 1024 && d <= 32 && g <= 4096 && k <= 16; }

// lo (nullable): the layout that orders the screen rows (screen_order_kernel);
// only the split tc2 screen + exact kernel read the row map, so any other
// screen that will run gets the identity order
int tc2_warpgroups();
int prepare_tc(const float* hi, const float* lo, int g, int d, int k, const ModelLayout& m, char* ws,
               cudaStream_t st, bool keep_order = false) {
    cudaMemsetAsync(ws + m.lstats, 0, 8, st);
    float* cen = reinterpret_cast<float*>(ws + m.lstats + 128);
    int32_t* rowmap = reinterpret_cast<int32_t*>(ws + m.rowmap);
    const bool ordered = lo && tc2_warpgroups() > 0 && m.ls && kp_for(k) <= 16 && m.gpad <= 1024 && m.t2chunk;
    if (!keep_order)  // (the caller's layout is unchanged since the last preparation: keep its order)
        screen_order_kernel<<<1, 1024, 0, st>>>(ordered ? lo : nullptr, g, m.gpad, rowmap);
    center_kernel<<<(m.d16 + 31) / 32, 1024, 0, st>>>(hi, g, d, m.d16, cen);
    tc_prepare_kernel<<<grid_for((int64_t)m.gpad * (m.d16 / 8), 256), 256, 0, st>>>(
        hi, g, d, m.d16, m.gpad, rowmap, cen, reinterpret_cast<uint16_t*>(ws + m.bhi),
        reinterpret_cast<uint16_t*>(ws + m.blo), reinterpret_cast<float*>(ws + m.ln),
        reinterpret_cast<float*>(ws + m.lstats));
    if (int e = cuda_check("tc_prepare_kernel", keep_order ? 2 : 3)) return e;  // (order) + center + operands
    if (m.ls) {
        lrow_kernel<<<grid_for((int64_t)m.gpad * m.ls, 256), 256, 0, st>>>(hi, g, d, m.gpad, m.ls, rowmap,
                                                                          reinterpret_cast<float*>(ws + m.lrow));
        return cuda_check("lrow_kernel");
    }
    return ESOM_OK;
}

// returns ESOM_ERR_UNSUPPORTED when the shape does not fit (caller falls back)
int tc2_warpgroups() {  // ESOM_TC2_W selects 2..4 warpgroups per CTA (default 4); 0 disables tc2
    const char* e = getenv("ESOM_TC2_W");
    return e ? atoi(e) : 4;
}

// the requested number of warpgroups, or fewer when the shared-memory carve-up does not fit
template <int KP>
int launch_tc2_w(Tc2Args a, int W, cudaStream_t st) {
    int e = ESOM_ERR_UNSUPPORTED;
    if (W >= 4) e = launch_tc2_t<KP, 4>(a, st);
    if (e == ESOM_ERR_UNSUPPORTED && W >= 3) e = launch_tc2_t<KP, 3>(a, st);
    if (e == ESOM_ERR_UNSUPPORTED) e = launch_tc2_t<KP, 2>(a, st);
    return e;
}

// pipelined screen (esom_tc2.cuh); ESOM_ERR_UNSUPPORTED when the shape does not fit
int dispatch_tc2(const Plan& p, const ModelLayout& m, const ScanArgs& s, const char* ws, cudaStream_t st,
                 const ProjArgs* fuse = nullptr, bool* fused_done = nullptr) {
    const int W = tc2_warpgroups();
    // the non-empty-word mask of the candidate bitmaps is one 32-bit word:
    // gpad <= 1024 (larger g: the round-streaming esom_tc.cuh screen; the
    // randomised parity test caught the fused kernel being picked at g = 1500)
    if (W <= 0 || !m.ls || p.kp > 16 || m.gpad > 1024) return ESOM_ERR_UNSUPPORTED;
    Tc2Args a{};
    a.X = s.X;
    a.n = s.n;
    a.d = s.d;
    a.d16 = m.d16;
    a.g = s.g;
    a.gpad = m.gpad;
    a.k = s.k;
    a.Bhi = reinterpret_cast<const uint16_t*>(ws + m.bhi);
    a.Blo = reinterpret_cast<const uint16_t*>(ws + m.blo);
    a.ln = reinterpret_cast<const float*>(ws + m.ln);
    a.Lrow = reinterpret_cast<const float*>(ws + m.lrow);
    a.rowmap = reinterpret_cast<const int32_t*>(ws + m.rowmap);
    a.ls = m.ls;
    a.L = s.L;
    a.lstats = reinterpret_cast<const float*>(ws + m.lstats);
    a.center = reinterpret_cast<const float*>(ws + m.lstats + 128);
    a.out_idx = s.out_idx;
    a.out_sqd = s.out_sqd;
    a.bmu = s.bmu;
    a.accS = s.accS;
    a.accC = s.accC;
    a.acc_scale = s.acc_scale;
    a.qe_sum = s.qe_sum;
    a.flag = s.flag;
    a.stats = tc_stats_ptr();
    // screen-only kernel + separate exact kernel (default; ESOM_TC2_FUSED=1 keeps the fused kernel)
    const bool split = m.t2chunk && !getenv("ESOM_TC2_FUSED");
    if (split) {
        const int Ws = getenv("ESOM_TC2_W") ? W : (m.gpad > 256 ? 3 : 4);  // measured best (C4 / C2)
        // g > 256: screen-only kernel (more warpgroups: no bitmaps / rows in its smem) writes
        // candidate bitmaps; knn_exact_bits_kernel re-evaluates them with the rows in smem
        char* w = const_cast<char*>(ws);
        for (int64_t s0 = 0; s0 < s.n; s0 += m.t2chunk) {
            Tc2Args c = a;
            c.n = s.n - s0 < m.t2chunk ? s.n - s0 : m.t2chunk;
            c.X = s.X + s0 * s.d;
            c.out_idx = s.out_idx ? s.out_idx + s0 * s.k : nullptr;
            c.out_sqd = s.out_sqd ? s.out_sqd + s0 * s.k : nullptr;
            c.bmu = s.bmu ? s.bmu + s0 : nullptr;
            c.cbits = reinterpret_cast<uint32_t*>(w + m.t2bits);
            c.cinfo = reinterpret_cast<int2*>(w + m.t2info);
            const bool lsort = c.n >= 4096;
            c.ckey = lsort ? reinterpret_cast<int32_t*>(w + m.t2key) : nullptr;
            int e;
            {
                KTimer tm("knn_tc2_kernel", st);
                e = p.kp == 4 ? launch_tc2_w<4>(c, Ws, st) : p.kp == 8 ? launch_tc2_w<8>(c, Ws, st)
                                                                        : launch_tc2_w<16>(c, Ws, st);
            }
            if (e) return e;
            if (lsort) {
                c.perm = reinterpret_cast<int32_t*>(w + m.t2perm);
                if (int e2 = bmu_sort(c.ckey, c.n, 1, s.g, reinterpret_cast<int32_t*>(w + m.t2hist),
                                      const_cast<int32_t*>(c.perm), st))
                    return e2;
            }
            if (fuse && p.kp == 16) {  // embed: exact phase + projection in one kernel
                ProjArgs q = *fuse;
                q.n = c.n;
                q.X = fuse->X + s0 * s.d;
                q.xy = fuse->xy + 2 * s0;
                q.idx = fuse->idx + s0 * s.k;
                q.sqd = fuse->sqd + s0 * s.k;
                c.out_idx = nullptr;
                c.out_sqd = nullptr;
                KTimer tmf("embed_fused_kernel", st);
                e = launch_embed_fused_c(c, q, st);
                if (e == ESOM_OK) {
                    if (fused_done) *fused_done = true;
                    continue;
                }
                if (e != ESOM_ERR_UNSUPPORTED) return e;
                g_err[0] = 0;
                c.out_idx = s.out_idx ? s.out_idx + s0 * s.k : nullptr;
                c.out_sqd = s.out_sqd ? s.out_sqd + s0 * s.k : nullptr;
            }
            if (fused_done) *fused_done = false;
            KTimer tm2("knn_exact_bits_kernel", st);
            e = p.kp == 4 ? launch_exact_bits_t<4>(c, st) : p.kp == 8 ? launch_exact_bits_t<8>(c, st)
                                                                      : launch_exact_bits_t<16>(c, st);
            if (e) return e;
        }
        return ESOM_OK;
    }
    KTimer tm("knn_tc2_kernel", st);
    switch (p.kp) {
        case 4: return launch_tc2_w<4>(a, W, st);
        case 8: return launch_tc2_w<8>(a, W, st);
        case 16: return launch_tc2_w<16>(a, W, st);
    }
    return ESOM_ERR_UNSUPPORTED;
}

int dispatch_tc(const Plan& p, const ModelLayout& m, const ScanArgs& s, const char* ws, cudaStream_t st,
                const ProjArgs* fuse = nullptr, bool* fused_done = nullptr) {
    {
        const int e = dispatch_tc2(p, m, s, ws, st, fuse, fused_done);
        if (e != ESOM_ERR_UNSUPPORTED) return e;
        g_err[0] = 0;
    }
    TcArgs a{};
    a.X = s.X;
    a.n = s.n;
    a.d = s.d;
    a.d16 = m.d16;
    a.dp = p.dp;
    a.g = s.g;
    a.gpad = m.gpad;
    a.k = s.k;
    a.Bhi = reinterpret_cast<const uint16_t*>(ws + m.bhi);
    a.Blo = reinterpret_cast<const uint16_t*>(ws + m.blo);
    a.ln = reinterpret_cast<const float*>(ws + m.ln);
    a.Lt = m.gpad <= 256 ? reinterpret_cast<const float*>(ws + m.lt) : nullptr;  // resident exact tiles
    a.L = s.L;
    a.lstats = reinterpret_cast<const float*>(ws + m.lstats);
    a.center = reinterpret_cast<const float*>(ws + m.lstats + 128);
    a.out_idx = s.out_idx;
    a.out_sqd = s.out_sqd;
    a.bmu = s.bmu;
    a.accS = s.accS;
    a.accC = s.accC;
    a.acc_scale = s.acc_scale;
    a.qe_sum = s.qe_sum;
    a.flag = s.flag;
    a.stats = tc_stats_ptr();
    switch (p.kp) {
        case 4: return launch_tc_t<4>(a, st);
        case 8: return launch_tc_t<8>(a, st);
        case 16: return launch_tc_t<16>(a, st);
    }
    return set_err(ESOM_ERR_UNSUPPORTED, "no tensor-core kernel for k%s", "");
}

// per-model operands of the d > 32 GEMM screen: centroid, B = -2 (l - c) split tiles, norms
int prepare_tc3(const float* hi, int g, int d, const ModelLayout& m, char* ws, int32_t* flag, cudaStream_t st) {
    if (!m.t3) return ESOM_OK;
    cudaMemsetAsync(ws + m.ls3, 0, 8, st);
    float* cen = reinterpret_cast<float*>(ws + m.cen3);
    center_kernel<<<(m.dk + 31) / 32, 1024, 0, st>>>(hi, g, d, m.dk, cen);
    if (int e = cuda_check("center_kernel")) return e;
    return t3_split(hi, g, m.gp3, d, m.dk, cen, -2.0f, 256, reinterpret_cast<uint16_t*>(ws + m.b3hi),
                    reinterpret_cast<uint16_t*>(ws + m.b3lo), reinterpret_cast<float*>(ws + m.ln3), 1,
                    reinterpret_cast<float*>(ws + m.ls3), flag, st);
}

bool t3_enabled() {  // ESOM_TC3=0 forces the CUDA-core scan for d > 32
    const char* e = getenv("ESOM_TC3");
    return tc_enabled() && (e ? atoi(e) != 0 : true);
}

// d > 32: split points -> tcgen05 GEMM screen -> approximate-BMU sort -> warp-exact re-evaluation,
// in chunks of m.t3chunk points (the chunk scratch lives in the model workspace)
int run_t3(const ModelLayout& m, const ScanArgs& a, const char* wsc, cudaStream_t st) {
    char* ws = const_cast<char*>(wsc);
    for (int64_t s = 0; s < a.n; s += m.t3chunk) {
        const int64_t cn = a.n - s < m.t3chunk ? a.n - s : m.t3chunk;
        const int64_t cpad = (cn + 255) / 256 * 256;
        const float* X = a.X + s * a.d;
        if (int e = t3_split(X, cn, cpad, a.d, m.dk, reinterpret_cast<const float*>(ws + m.cen3), 1.0f, 128,
                             reinterpret_cast<uint16_t*>(ws + m.a3hi), reinterpret_cast<uint16_t*>(ws + m.a3lo),
                             reinterpret_cast<float*>(ws + m.xn3), 0, nullptr, a.flag, st))
            return e;
        Tc3Args t{};
        t.Ahi = reinterpret_cast<const uint16_t*>(ws + m.a3hi);
        t.Alo = reinterpret_cast<const uint16_t*>(ws + m.a3lo);
        t.xnorm = reinterpret_cast<const float*>(ws + m.xn3);
        t.n = cn;
        t.d = a.d;
        t.dk = m.dk;
        t.gpad = m.gp3;
        t.k = a.k;
        t.Bhi = reinterpret_cast<const uint16_t*>(ws + m.b3hi);
        t.Blo = reinterpret_cast<const uint16_t*>(ws + m.b3lo);
        t.ln = reinterpret_cast<const float*>(ws + m.ln3);
        t.lstats = reinterpret_cast<const float*>(ws + m.ls3);
        t.cand = reinterpret_cast<uint16_t*>(ws + m.cand3);
        t.ccount = reinterpret_cast<int32_t*>(ws + m.cnt3);
        t.bmu_approx = reinterpret_cast<int32_t*>(ws + m.bmu3);
        t.stats = tc_stats_ptr();
        const int kp = kp_for(a.k);
        int e;
        {
            KTimer tm("knn_gemm_kernel", st);
            e = kp == 4 ? launch_gemm_t<4>(t, st) : kp == 8 ? launch_gemm_t<8>(t, st)
              : kp == 16 ? launch_gemm_t<16>(t, st) : launch_gemm_t<32>(t, st);
        }
        if (e) return e;
        // visit points grouped by approximate nearest landmark: a CTA's candidate rows repeat (L1 hits)
        int32_t* cntb = reinterpret_cast<int32_t*>(ws + m.hist3);
        int32_t* perm = reinterpret_cast<int32_t*>(ws + m.perm3);
        if (int e2 = bmu_sort(t.bmu_approx, cn, 1, a.g, cntb, perm, st)) return e2;
        T3ExactArgs x{};
        x.X = X;
        x.n = cn;
        x.d = a.d;
        x.dpad = (a.d + 3) / 4 * 4;
        x.g = a.g;
        x.k = a.k;
        x.L = a.L;
        x.cand = t.cand;
        x.ccount = t.ccount;
        x.perm = perm;
        x.out_idx = a.out_idx ? a.out_idx + s * a.k : nullptr;
        x.out_sqd = a.out_sqd ? a.out_sqd + s * a.k : nullptr;
        x.bmu = a.bmu ? a.bmu + s : nullptr;
        x.qe_sum = a.qe_sum;
        x.accS = a.accS;
        x.accC = a.accC;
        x.acc_scale = a.acc_scale;
        x.stats = tc_stats_ptr();
        {
            KTimer tm("knn_exact_group_kernel", st);
            if (int e3 = launch_exact_warp_t<32>(x, st)) return e3;
        }
    }
    return ESOM_OK;
}

// k-NN over a prepared model workspace: tensor-core screen when eligible, else the CUDA-core scan
// fuse (embed only): when the split tc2 path runs, the projection is fused into the
// exact phase (*fused_done = true: the caller skips its projection launch)
int run_knn(const Plan& p, const ModelLayout& m, ScanArgs a, const char* ws, cudaStream_t st,
            const ProjArgs* fuse = nullptr, bool* fused_done = nullptr) {
    if (fused_done) *fused_done = false;
    if (tc_eligible(a.n, a.d, a.g, a.k)) {
        const int e = dispatch_tc(p, m, a, ws, st, fuse, fused_done);
        if (e != ESOM_ERR_UNSUPPORTED) return e;
    }
    if (m.t3 && t3_enabled() && a.n >= 256 && a.d <= 1536) return run_t3(m, a, ws, st);
    return dispatch_scan(p, a, st);
}


}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int esom_version(void) { return ESOM_ABI_VERSION; }

void esom_set_tc_stats(int32_t* counter) { g_tc_stats = counter; }

int64_t esom_launch_count(void) { return (int64_t)g_launches.load(std::memory_order_relaxed); }

void esom_timing_begin(int32_t on) {
    std::lock_guard<std::mutex> lk(g_tmu);
    for (auto& t : g_tl) {
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    g_tl.clear();
    g_timing = on != 0;
}

double esom_timing_query(const char* name, int32_t* launches) {
    std::lock_guard<std::mutex> lk(g_tmu);
    double ms = 0.0;
    int n = 0;
    for (auto& t : g_tl) {
        if (t.name != name) continue;
        cudaEventSynchronize(t.b);
        float v = 0.0f;
        cudaEventElapsedTime(&v, t.a, t.b);
        ms += v;
        ++n;
    }
    if (launches) *launches = n;
    return ms;
}

const char* esom_last_error(void) { return g_err; }

static size_t align256(size_t b) { return (b + 255) / 256 * 256; }

size_t esom_workspace_bytes(int32_t g, int32_t d, int32_t k, int32_t with_pairs) {
    return model_layout(g, d, k, with_pairs != 0).total;
}

// points per embed chunk.  One launch per kernel over as many points as
// possible beats L2-sized chunks (measured: C2 0.817 -> 0.744 ms per frame):
// the neighbour rows round-trip through HBM (8k B per point, ~20 us per 2^20
// points) but tail effects and launch gaps disappear.  For the d > 32 GEMM
// screen the chunk is the screen's own scratch chunk.
static bool t3_shape(int32_t d, int32_t k) { return d > 32 && d <= 1536 && k <= 32; }

static int64_t embed_chunk(int32_t d, int32_t k) {
    const char* e = getenv("ESOM_EMBED_CHUNK");
    if (e) {
        const int64_t c = atoll(e);
        return c < 1024 ? 1024 : c;
    }
    if (t3_shape(d, k)) return model_layout(1, d, k, false).t3chunk;
    const int64_t c = (int64_t)(512u << 20) / (8 * (int64_t)k);  // <= 512 MB of neighbour rows
    return c < 1024 ? 1024 : c;
}

size_t esom_point_workspace_bytes(int64_t n, int32_t d, int32_t k) {
    const int64_t c = n < embed_chunk(d, k) ? n : embed_chunk(d, k);
    const size_t rows = align256((size_t)(c > 0 ? c : 1) * k * 4) * 2;
    return rows + align256((size_t)(c > 0 ? c : 1) * 4) + align256(65536 * 4) + 256;  // + perm + bucket counts
}

static ScanArgs scan_args(const Plan& p, const float* X, int64_t n, int32_t d, const float* L, int32_t g, int32_t k,
                          const float* Lt, int32_t* flag) {
    ScanArgs a{};
    a.X = X;
    a.n = n;
    a.d = d;
    a.dp = p.dp;
    a.nch = p.nch;
    a.Lt = Lt;
    a.L = L;
    a.g = g;
    a.ntiles = p.ntiles;
    a.k = k;
    a.flag = flag;
    a.nz = -0.0f;
    return a;
}

int esom_knn(const float* X, int64_t n, int32_t d, const float* L, int32_t g, int32_t k, int32_t* idx,
             float* sqd, int32_t* nonfinite_flag, void* workspace, size_t ws_bytes, cudaStream_t stream) {
    if (n < 0 || d < 1 || g < 1) return set_err(ESOM_ERR_PARAM, "bad shape n=%lld d=%lld", (long long)n, (long long)d);
    if (k < 1 || k > g) return set_err(ESOM_ERR_PARAM, "k=%lld violates 1 <= k <= g=%lld", (long long)k, (long long)g);
    if (n == 0) return ESOM_OK;
    if (k > 64 || d > 2048) {
        int gpow = 1;
        while (gpow < g) gpow <<= 1;
        const size_t smem = (size_t)gpow * 8;
        if (smem > (size_t)max_smem_optin()) return set_err(ESOM_ERR_UNSUPPORTED, "g too large for k > 64%s", "");
        cudaFuncSetAttribute(knn_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int grid = (int)(n < (int64_t)num_sms() * 8 ? n : (int64_t)num_sms() * 8);
        knn_sort_kernel<<<grid, 256, smem, stream>>>(X, n, d, L, g, gpow, k, idx, sqd, nonfinite_flag);
        if (int e = cuda_check("knn_sort_kernel")) return e;
        check_finite_kernel<<<grid_for((int64_t)g * d, 256), 256, 0, stream>>>(L, (int64_t)g * d, nonfinite_flag);
        return cuda_check("check_finite");
    }
    const Plan p = make_plan(d, g, k);
    const ModelLayout m = model_layout(g, d, k, false);
    if (ws_bytes < m.total) return set_err(ESOM_ERR_PARAM, "workspace too small%s", "");
    char* ws = reinterpret_cast<char*>(workspace);
    float* Lt = reinterpret_cast<float*>(ws + m.lt);
    pack_landmarks_kernel<<<grid_for((int64_t)p.ntiles * p.dp * kTile, 256), 256, 0, stream>>>(L, g, d, p.dp, p.ntiles,
                                                                                                   Lt, nonfinite_flag);
    if (int e = cuda_check("pack_landmarks")) return e;
    if (tc_eligible(n, d, g, k))
        if (int e = prepare_tc(L, nullptr, g, d, k, m, ws, stream)) return e;
    if (m.t3 && t3_enabled())
        if (int e = prepare_tc3(L, g, d, m, ws, nonfinite_flag, stream)) return e;
    ScanArgs a = scan_args(p, X, n, d, L, g, k, Lt, nonfinite_flag);
    a.out_idx = idx;
    a.out_sqd = sqd;
    return run_knn(p, m, a, ws, stream);
}

int esom_scores(const float* sqd, int64_t n, int32_t k, double* out, cudaStream_t stream) {
    if (k < 1) return set_err(ESOM_ERR_PARAM, "k must be >= 1%s", "");
    if (n == 0) return ESOM_OK;
    scores_kernel<<<grid_for(n, 128), 128, 0, stream>>>(sqd, n, k, out);
    return cuda_check("scores_kernel");
}

int esom_project(const float* X, int64_t n, int32_t d, const float* hi, const float* lo, int32_t g,
                 const int32_t* idx, const double* scores, int32_t k, float* xy, cudaStream_t stream) {
    (void)g;
    if (k < 1 || d < 1) return set_err(ESOM_ERR_PARAM, "bad k/d%s", "");
    if (n == 0) return ESOM_OK;
    project_kernel<<<grid_for(n, 128), 128, 0, stream>>>(X, n, d, hi, lo, idx, scores, k, xy);
    return cuda_check("project_kernel");
}

int esom_prepare_model(const float* hi, const float* lo, int32_t g, int32_t d, int32_t k, int32_t flags, void* workspace,
                       size_t ws_bytes,
                       int32_t* nonfinite_flag, cudaStream_t stream) {
    if (k > 64) return set_err(ESOM_ERR_UNSUPPORTED, "fused embed supports k <= 64 (got %lld)", (long long)k);
    const Plan p = make_plan(d, g, k);
    const ModelLayout m = model_layout(g, d, k, true);
    if (ws_bytes < m.total) return set_err(ESOM_ERR_PARAM, "workspace too small%s", "");
    char* ws = reinterpret_cast<char*>(workspace);
    float* Lt = reinterpret_cast<float*>(ws + m.lt);
    float* T = reinterpret_cast<float*>(ws + m.tri);
    pack_landmarks_kernel<<<grid_for((int64_t)p.ntiles * p.dp * kTile, 256), 256, 0, stream>>>(hi, g, d, p.dp, p.ntiles,
                                                                                                   Lt, nonfinite_flag);
    if (int e = cuda_check("pack_landmarks")) return e;
    float* tmax = reinterpret_cast<float*>(ws + m.lstats) + 2;
    cudaMemsetAsync(tmax, 0, 4, stream);
    if (d <= 64) {
        const int nt = (g + kPairTile - 1) / kPairTile;
        pair_table_tiled_kernel<<<dim3(nt, nt), 256, 0, stream>>>(hi, g, d, T, tmax);
    } else {
        pair_table_kernel<<<grid_for((int64_t)g * g, 256), 256, 0, stream>>>(hi, g, d, T, tmax);
    }
    if (int e = cuda_check("pair_table")) return e;
    widen_kernel<<<grid_for((int64_t)g * d, 256), 256, 0, stream>>>(hi, (int64_t)g * d,
                                                                    reinterpret_cast<double*>(ws + m.hi64));
    if (int e = cuda_check("widen_hi")) return e;
    row_norm64_kernel<<<grid_for(g, 128), 128, 0, stream>>>(hi, g, d, reinterpret_cast<double*>(ws + m.hn64));
    if (int e = cuda_check("row_norm64")) return e;
    if (tc_eligible(1 << 20, d, g, k))
        if (int e = prepare_tc(hi, lo, g, d, k, m, ws, stream, (flags & ESOM_PREPARE_KEEP_ORDER) != 0)) return e;
    if (m.t3 && t3_enabled())
        if (int e = prepare_tc3(hi, g, d, m, ws, nonfinite_flag, stream)) return e;
    return ESOM_OK;
}

int esom_embed_prepared(const float* X, int64_t n, int32_t d, const float* hi, const float* lo, int32_t g, int32_t k,
                        const void* model_ws, void* point_ws, size_t point_ws_bytes, float* xy, int32_t* bmu,
                        int64_t* acc_S, int64_t* acc_C, int32_t acc_fx_bits, double* qe_sum, int32_t* nonfinite_flag,
                        cudaStream_t stream) {
    return esom_embed_prepared_ex(X, n, d, hi, lo, g, k, model_ws, point_ws, point_ws_bytes, xy, bmu, acc_S, acc_C,
                                  acc_fx_bits, qe_sum, nonfinite_flag, 0, nullptr, stream);
}

int esom_embed_prepared_ex(const float* X, int64_t n, int32_t d, const float* hi, const float* lo, int32_t g,
                           int32_t k, const void* model_ws, void* point_ws, size_t point_ws_bytes, float* xy,
                           int32_t* bmu, int64_t* acc_S_, int64_t* acc_C_, int32_t acc_fx_bits, double* qe_sum,
                           int32_t* nonfinite_flag, int32_t flags, int32_t* far_count, cudaStream_t stream) {
    const bool bmu_order = (flags & ESOM_EMBED_BMU_ORDER) != 0;
    acc_t* acc_S = reinterpret_cast<acc_t*>(acc_S_);
    acc_t* acc_C = reinterpret_cast<acc_t*>(acc_C_);
    if ((acc_S || acc_C) && (acc_fx_bits < 0 || acc_fx_bits > 60))
        return set_err(ESOM_ERR_PARAM, "acc_fx_bits=%d outside [0, 60]", (int)acc_fx_bits);
    const double acc_scale = ldexp(1.0, acc_fx_bits);
    if (k < 1 || k > g) return set_err(ESOM_ERR_PARAM, "k=%lld violates 1 <= k <= g=%lld", (long long)k, (long long)g);
    if (k > 64) return set_err(ESOM_ERR_UNSUPPORTED, "fused embed supports k <= 64%s", "");
    if (n == 0) return ESOM_OK;
    if (point_ws_bytes < esom_point_workspace_bytes(n, d, k))
        return set_err(ESOM_ERR_PARAM, "point workspace too small%s", "");
    const Plan p = make_plan(d, g, k);
    const ModelLayout ml = model_layout(g, d, k, true);
    const char* mws = reinterpret_cast<const char*>(model_ws);
    const float* Lt = reinterpret_cast<const float*>(mws + ml.lt);
    const float* T = reinterpret_cast<const float*>(mws + ml.tri);
    const int64_t chunk = n < embed_chunk(d, k) ? n : embed_chunk(d, k);
    // pair records {T, g, g.lo_u} for this call's layout (project_reg3_kernel)
    // (g <= 256: the triangle table sits in shared memory and v2 is as fast without the record build)
    const bool use_rec = ml.has_rec && g > 256;
    float4* rec = reinterpret_cast<float4*>(const_cast<char*>(mws) + ml.rec);
    if (use_rec)
        if (int e = launch_pair_records(T, lo, g, rec, stream)) return e;
    int32_t* idx = reinterpret_cast<int32_t*>(point_ws);
    float* sqd = reinterpret_cast<float*>(reinterpret_cast<char*>(point_ws) + align256((size_t)chunk * k * 4));
    for (int64_t s = 0; s < n; s += chunk) {
        const int64_t m = n - s < chunk ? n - s : chunk;
        ScanArgs a = scan_args(p, X + s * d, m, d, hi, g, k, Lt, nonfinite_flag);
        a.out_idx = idx;
        a.out_sqd = sqd;
        a.bmu = bmu ? bmu + s : nullptr;
        a.qe_sum = qe_sum;  // batch-SOM sums come from the BMU-sorted order below (no atomics)
        const size_t tbytes = (size_t)g * (g - 1) / 2 * 4;
        const bool l2_table = tbytes + (size_t)g * 12 + 1024 > (size_t)max_smem_optin() && m >= 4096 && g <= 8192;
        ProjArgs q{};
        q.idx = idx;
        q.sqd = sqd;
        q.n = m;
        q.k = k;
        q.g = g;
        q.lo = lo;
        q.T = T;
        q.tmax = reinterpret_cast<const float*>(mws + ml.lstats) + 2;
        q.prec_count = far_count;
        q.far_heavy = bmu_order ? 1 : 0;
        q.store_bmu = (acc_S || acc_C) ? 1 : 0;
        q.xy = xy + 2 * s;
        q.X = X + s * d;
        q.hi = hi;
        q.hi64 = reinterpret_cast<const double*>(mws + ml.hi64);
        q.hn64 = reinterpret_cast<const double*>(mws + ml.hn64);
        q.d = d;
        q.rec = use_rec ? rec : nullptr;
        // the exact phase and the projection in one kernel when the pair triangle sits in
        // shared memory (the fused kernel visits the exact phase's locality order and
        // reads far points' landmark rows from the exact phase's shared copy)
        const bool try_fuse = p.kp == 16 && k == 16 && !l2_table && !use_rec;
        bool fused = false;
        if (int e = run_knn(p, ml, a, mws, stream, try_fuse ? &q : nullptr, &fused)) return e;
        const bool need_perm = !fused && (l2_table || ((use_rec || bmu_order) && m >= 4096));
        const bool acc_smem = (acc_S || acc_C) && !need_perm && accum_smem_ok(g, d);
        if (acc_smem) {
            const size_t smem = ((size_t)g * d + g) * 8;
            cudaFuncSetAttribute(bmu_accum_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            bmu_accum_smem_kernel<<<num_sms(), kAccThreads, smem, stream>>>(X + s * d, m, d, idx, k, g, acc_S, acc_C,
                                                                             acc_scale);
            if (int e = cuda_check("bmu_accum_smem_kernel")) return e;
        }
        if (need_perm || ((acc_S || acc_C) && !acc_smem)) {
            // BMU counting sort of the chunk (BMU = idx[:, 0]): the projection visits
            // points grouped by BMU (pair-table reads coalesce when the table is in
            // L2) and the batch-SOM sums are segment sums over the same order
            char* base = reinterpret_cast<char*>(point_ws) + 2 * align256((size_t)chunk * k * 4);
            int32_t* perm = reinterpret_cast<int32_t*>(base);
            int32_t* cntb = reinterpret_cast<int32_t*>(base + align256((size_t)chunk * 4));
            if (int e = bmu_sort(idx, m, k, g, cntb, perm, stream)) return e;
            if ((acc_S || acc_C) && !acc_smem) {
                const int64_t warps = (m + kSegPart - 1) / kSegPart * ((d + 31) / 32);
                bmu_segsum_kernel<<<grid_for(warps * 32, 256), 256, 0, stream>>>(X + s * d, d, perm, cntb, g, m,
                                                                                  acc_S, acc_C, acc_scale, idx, k);
                if (int e = cuda_check("bmu_segsum_kernel")) return e;
            }
            if (l2_table || use_rec || bmu_order) q.perm = perm;
        }
        if (!fused) {
            KTimer tm("project_kernel", stream);
            if (int e = dispatch_project(p.kp, q, stream)) return e;
        }
    }
    return ESOM_OK;
}

int32_t esom_embed_launches(int64_t n, int32_t g, int32_t d, int32_t k) {
    // kernels launched by one esom_embed_prepared call, per embed chunk: the
    // k-NN (tensor-core screen, CUDA-core scan, or for d > 32 per screen chunk
    // split + GEMM + 3 BMU-sort + exact) and the projection (+ 3 BMU-sort
    // kernels when the pair table lives in L2)
    if (n <= 0) return 0;
    const int64_t chunk = n < embed_chunk(d, k) ? n : embed_chunk(d, k);
    const size_t tbytes = (size_t)g * (g - 1) / 2 * 4;
    const bool sorted = tbytes + (size_t)g * 12 + 1024 > (size_t)max_smem_optin() && g <= 8192;
    const ModelLayout m = model_layout(g, d, k, true);
    int64_t total = 0;
    for (int64_t s = 0; s < n; s += chunk) {
        const int64_t cm = n - s < chunk ? n - s : chunk;
        int64_t knn = 1;
        if (m.t3 && t3_enabled() && cm >= 256 && d <= 1536) knn = 6 * ((cm + m.t3chunk - 1) / m.t3chunk);
        total += knn + 1 + ((sorted && cm >= 4096) ? 3 : 0);
    }
    return (int32_t)total;
}

size_t esom_embed_workspace_bytes(int64_t n, int32_t g, int32_t d, int32_t k) {
    return esom_workspace_bytes(g, d, k, 1) + esom_point_workspace_bytes(n, d, k);
}

int esom_embed(const float* X, int64_t n, int32_t d, const float* hi, const float* lo, int32_t g, int32_t k,
               void* workspace, size_t ws_bytes, float* xy, int32_t* bmu, int64_t* acc_S, int64_t* acc_C,
               int32_t acc_fx_bits, double* qe_sum, int32_t* nonfinite_flag, cudaStream_t stream) {
    if (k < 1 || k > g) return set_err(ESOM_ERR_PARAM, "k=%lld violates 1 <= k <= g=%lld", (long long)k, (long long)g);
    const size_t mb = esom_workspace_bytes(g, d, k, 1);
    if (ws_bytes < esom_embed_workspace_bytes(n, g, d, k)) return set_err(ESOM_ERR_PARAM, "workspace too small%s", "");
    if (int e = esom_prepare_model(hi, lo, g, d, k, 0, workspace, mb, nonfinite_flag, stream)) return e;
    return esom_embed_prepared(X, n, d, hi, lo, g, k, workspace, reinterpret_cast<char*>(workspace) + mb,
                               ws_bytes - mb, xy, bmu, acc_S, acc_C, acc_fx_bits, qe_sum, nonfinite_flag, stream);
}

int esom_bmu_accumulate(const float* X, int64_t n, int32_t d, const float* hi, int32_t g, void* workspace,
                        size_t ws_bytes, int32_t* bmu, int64_t* acc_S, int64_t* acc_C, int32_t acc_fx_bits,
                        double* qe_sum, int32_t* nonfinite_flag, cudaStream_t stream) {
    if (n < 0 || d < 1 || g < 1) return set_err(ESOM_ERR_PARAM, "bad shape%s", "");
    if ((acc_S || acc_C) && (acc_fx_bits < 0 || acc_fx_bits > 60))
        return set_err(ESOM_ERR_PARAM, "acc_fx_bits=%d outside [0, 60]", (int)acc_fx_bits);
    if (n == 0) return ESOM_OK;
    const Plan p = make_plan(d, g, 1);
    const ModelLayout m = model_layout(g, d, 1, false);
    if (ws_bytes < m.total) return set_err(ESOM_ERR_PARAM, "workspace too small%s", "");
    char* ws = reinterpret_cast<char*>(workspace);
    float* Lt = reinterpret_cast<float*>(ws + m.lt);
    pack_landmarks_kernel<<<grid_for((int64_t)p.ntiles * p.dp * kTile, 256), 256, 0, stream>>>(hi, g, d, p.dp, p.ntiles,
                                                                                                   Lt, nonfinite_flag);
    if (int e = cuda_check("pack_landmarks")) return e;
    if (tc_eligible(n, d, g, 1))
        if (int e = prepare_tc(hi, nullptr, g, d, 1, m, ws, stream)) return e;
    if (m.t3 && t3_enabled())
        if (int e = prepare_tc3(hi, g, d, m, ws, nonfinite_flag, stream)) return e;
    ScanArgs a = scan_args(p, X, n, d, hi, g, 1, Lt, nonfinite_flag);
    a.bmu = bmu;
    a.accS = reinterpret_cast<acc_t*>(acc_S);
    a.accC = reinterpret_cast<acc_t*>(acc_C);
    a.acc_scale = ldexp(1.0, acc_fx_bits);
    a.qe_sum = qe_sum;
    return run_knn(p, m, a, ws, stream);
}

size_t esom_tick_workspace_bytes(int32_t g, int32_t d) { return (size_t)g * d * 8 + 256; }

static int online_tick(bool som, const float* X, int32_t d, const int64_t* sample_idx, int32_t B, float* hi_inout,
                       const float* lo, int32_t g, double sigma, double alpha, void* ws, size_t ws_bytes,
                       cudaStream_t stream) {
    if (B < 0 || g < 1 || d < 1) return set_err(ESOM_ERR_PARAM, "bad tick shape%s", "");
    if (ws_bytes < esom_tick_workspace_bytes(g, d)) return set_err(ESOM_ERR_PARAM, "workspace too small%s", "");
    if (B == 0) return ESOM_OK;
    {
        const int r = launch_online_tick_cluster(som, X, d, sample_idx, B, hi_inout, lo, g, sigma, alpha, stream);
        if (r >= 0) return r;
    }
    const size_t smem = ((size_t)d + g) * 8;
    if (smem > (size_t)max_smem_optin()) return set_err(ESOM_ERR_UNSUPPORTED, "g + d too large%s", "");
    auto kern = som ? online_tick_kernel<true> : online_tick_kernel<false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<1, 1024, smem, stream>>>(X, d, sample_idx, B, hi_inout, lo, g, sigma, alpha, reinterpret_cast<double*>(ws));
    return cuda_check("online_tick_kernel");
}

int esom_som_tick(const float* X, int32_t d, const int64_t* sample_idx, int32_t B, float* hi_inout, const float* lo,
                  int32_t g, double sigma, double alpha, void* ws, size_t ws_bytes, cudaStream_t stream) {
    if (!(sigma > 0)) return set_err(ESOM_ERR_PARAM, "sigma must be > 0%s", "");
    return online_tick(true, X, d, sample_idx, B, hi_inout, lo, g, sigma, alpha, ws, ws_bytes, stream);
}

int esom_kmeans_tick(const float* X, int32_t d, const int64_t* sample_idx, int32_t B, float* hi_inout, int32_t g,
                     double alpha_km, void* ws, size_t ws_bytes, cudaStream_t stream) {
    return online_tick(false, X, d, sample_idx, B, hi_inout, nullptr, g, 1.0, alpha_km, ws, ws_bytes, stream);
}

int esom_batch_som_update(const int64_t* acc_S, const int64_t* acc_C, int32_t acc_fx_bits, const float* lo, int32_t g,
                          int32_t d, double sigma, double alpha, int32_t mode, float* hi_inout, cudaStream_t stream) {
    if (!(sigma > 0)) return set_err(ESOM_ERR_PARAM, "sigma must be > 0%s", "");
    if (acc_fx_bits < 0 || acc_fx_bits > 60) return set_err(ESOM_ERR_PARAM, "acc_fx_bits=%d outside [0, 60]", (int)acc_fx_bits);
    const size_t smem = (size_t)g * 8;
    if (smem > (size_t)max_smem_optin()) return set_err(ESOM_ERR_UNSUPPORTED, "g too large%s", "");
    cudaFuncSetAttribute(batch_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int threads = 256;
    batch_update_kernel<<<g < num_sms() * 4 ? g : num_sms() * 4, threads, smem, stream>>>(
        reinterpret_cast<const acc_t*>(acc_S), reinterpret_cast<const acc_t*>(acc_C), ldexp(1.0, -acc_fx_bits), lo, g, d,
        sigma, alpha, mode, hi_inout);
    return cuda_check("batch_update_kernel");
}

// Page-lock a caller-owned host range in place (the numpy-input pipeline of
// embed pins arrays it sees repeatedly).  A failure is reported and cleared,
// so it cannot surface later as a kernel launch error.
int esom_host_register(void* p, size_t bytes) {
    if (cudaHostRegister(p, bytes, cudaHostRegisterDefault) != cudaSuccess) {
        const cudaError_t e = cudaGetLastError();
        return set_err(ESOM_ERR_CUDA, "cudaHostRegister: %s", cudaGetErrorString(e));
    }
    return ESOM_OK;
}

int esom_host_unregister(void* p) {
    if (cudaHostUnregister(p) != cudaSuccess) {
        const cudaError_t e = cudaGetLastError();
        return set_err(ESOM_ERR_CUDA, "cudaHostUnregister: %s", cudaGetErrorString(e));
    }
    return ESOM_OK;
}

}  // extern "C"
