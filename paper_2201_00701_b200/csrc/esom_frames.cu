// esom_frames.cu -- the data formats either side of the embed path
// (SURVEY.md §8f rows 1, 3, 4): frame colours, the FramePoints wire record,
// FCS DATA-segment decoding, per-dimension statistics and the dataset
// transforms.  All of it is byte/elementwise work bound by HBM (or by PCIe
// when the output is mapped pinned host memory), so the kernels are plain
// grid-stride streams with 16-byte accesses and grids sized in multiples of
// the SM count; nothing here is GEMM-shaped.
//
// Exactness: the colour quantisation, the transforms and the decoding repeat
// the reference's f64 operations one IEEE op at a time (__d*_rn: no FMA
// contraction), so they are bit-exact given the same statistics.  The
// statistics are a deterministic blocked f64 sum (fixed partition, fixed
// order); numpy's axis-0 reduction is one sequential sum per column, so mean
// and sd agree to ~1e-15 relative, not bit for bit.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "esom_common.cuh"
#include "esom_host.h"
#include "../../include/esom.h"

using namespace esom;
using namespace esom_host;

namespace {

constexpr uint8_t kTagFramePoints = 0x31;  // ref: protocol.py:33

int stream_grid(int64_t work, int threads) {
    const int64_t blocks = (work + threads - 1) / threads;
    const int64_t cap = (int64_t)num_sms() * 8;
    return (int)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

// ---------------------------------------------------------------------------
// Colour channel (ref: engine.py:144-153):
//   rint((x[:, c] - lo) / span * 255.0).astype(uint8), span <= 0 -> 128.
// ---------------------------------------------------------------------------
__global__ void color_channel_kernel(const float* __restrict__ X, int64_t n, int d, int c, double lo, double span,
                                     uint8_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint8_t v = 128;
        if (span > 0.0) {
            const double x = (double)__ldg(X + i * d + c);
            double q = rint(__dmul_rn(__ddiv_rn(__dsub_rn(x, lo), span), 255.0));
            q = fmin(fmax(q, 0.0), 255.0);  // in range whenever lo/span are the column's min/max
            v = (uint8_t)q;
        }
        out[i] = v;
    }
}

// ---------------------------------------------------------------------------
// FramePoints wire record (ref: protocol.py:205-210 + encode, :216-218):
//   <u32 1 + len(payload)> <u8 0x31> <u32 frame_id> <u32 n> <n x 2 f32 LE> <n u8>
// = 13 + 9n bytes.  The body after the 13-byte header is the byte stream
// S = xy || colours shifted by 13 bytes (1 mod 4), so every aligned output
// word is one __byte_perm of two consecutive aligned words of S.  Each thread
// writes 16 aligned bytes; `out` may be mapped pinned host memory (the frame
// goes straight to the websocket buffer over PCIe, no device staging).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t stream_word(const uint32_t* __restrict__ xyw, const uint8_t* __restrict__ col,
                                                int64_t n, int64_t u) {
    // word u of S = xy bytes (8n) followed by colour bytes (n)
    if (u < 2 * n) return __ldg(xyw + u);
    const int64_t b = (u - 2 * n) * 4;  // first colour byte of the word
    if (b + 4 <= n && (((uintptr_t)col) & 3) == 0) return __ldg(reinterpret_cast<const uint32_t*>(col + b));
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (b + j < n) w |= (uint32_t)__ldg(col + b + j) << (8 * j);
    return w;
}

__global__ void frame_points_pack_kernel(const float* __restrict__ xy, const uint8_t* __restrict__ col, int64_t n,
                                         uint32_t frame_id, uint8_t* __restrict__ out) {
    const int64_t total = 13 + 9 * n;
    const int64_t nchunks = (total + 15) / 16;
    const uint32_t* xyw = reinterpret_cast<const uint32_t*>(xy);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nchunks; t += (int64_t)gridDim.x * blockDim.x) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t wi = 4 * t + q;  // output word: bytes [4wi, 4wi + 4)
            if (wi == 0) {
                w[q] = (uint32_t)(9 + 9 * n);  // 1 + len(payload), little endian
            } else if (wi == 1) {
                w[q] = (uint32_t)kTagFramePoints | (frame_id << 8);
            } else if (wi == 2) {
                w[q] = (frame_id >> 24) | ((uint32_t)n << 8);
            } else if (wi == 3) {
                w[q] = ((uint32_t)n >> 24) | (n > 0 ? stream_word(xyw, col, n, 0) << 8 : 0u);
            } else {
                // out byte 4wi + j = S byte 4(wi - 4) + 3 + j
                const int64_t u = wi - 4;
                const uint32_t a = stream_word(xyw, col, n, u);
                const uint32_t b = (4 * (u + 1) < 9 * n) ? stream_word(xyw, col, n, u + 1) : 0u;
                w[q] = __byte_perm(a, b, 0x6543);
            }
        }
        const int64_t o = 16 * t;
        if (o + 16 <= total) {
            *reinterpret_cast<uint4*>(out + o) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
            for (int64_t b = o; b < total; ++b) out[b] = (uint8_t)(w[(b - o) >> 2] >> (8 * ((b - o) & 3)));
        }
    }
}

// ---------------------------------------------------------------------------
// FCS DATA segment (ref: io.py:113-126): n*d f32 in $BYTEORD order ("1,2,3,4"
// little or "4,3,2,1" big endian) -> native f32, plus the finiteness check
// Dataset.from_points performs (ref: core.py:38-40, 85).
// ---------------------------------------------------------------------------
__global__ void fcs_decode_kernel(const uint32_t* __restrict__ raw, int64_t count, int big_endian,
                                  float* __restrict__ out, int32_t* flag) {
    bool bad = false;
    const int64_t nvec = count / 4;
    const uint4* rv = reinterpret_cast<const uint4*>(raw);
    uint4* ov = reinterpret_cast<uint4*>(out);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nvec; e += stride) {
        uint4 v = __ldg(rv + e);
        if (big_endian) {
            v.x = __byte_perm(v.x, 0, 0x0123);
            v.y = __byte_perm(v.y, 0, 0x0123);
            v.z = __byte_perm(v.z, 0, 0x0123);
            v.w = __byte_perm(v.w, 0, 0x0123);
        }
        bad |= !finite_f(__uint_as_float(v.x)) | !finite_f(__uint_as_float(v.y)) | !finite_f(__uint_as_float(v.z)) |
               !finite_f(__uint_as_float(v.w));
        ov[e] = v;
    }
    for (int64_t e = 4 * nvec + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += stride) {
        uint32_t v = __ldg(raw + e);
        if (big_endian) v = __byte_perm(v, 0, 0x0123);
        bad |= !finite_f(__uint_as_float(v));
        out[e] = __uint_as_float(v);
    }
    flag_nonfinite(flag, bad);
}

// ---------------------------------------------------------------------------
// Per-dimension statistics (ref: core.py:57-69 compute_dim_stats: f64 min,
// max, mean, population sd).  Block b owns rows [b*R, (b+1)*R); inside it warp
// w takes rows r = w, w + 8, ... and lane l column c0 + l (one 128-byte row
// slice per warp load); the 8 warp partials are combined in warp order, the
// block partials by one thread per column in block order.  Pass 1: min, max,
// sum.  Pass 2 (given the mean): sum of squared deviations.
// ---------------------------------------------------------------------------
constexpr int kStatThreads = 256;
constexpr int kStatWarps = kStatThreads / 32;

template <bool DEV>
__global__ void __launch_bounds__(kStatThreads) dim_partial_kernel(const float* __restrict__ X, int64_t n, int d,
                                                                   int64_t rows_per_block,
                                                                   const double* __restrict__ mean,
                                                                   double* __restrict__ part) {
    __shared__ double s_a[kStatWarps][32], s_b[kStatWarps][32], s_c[kStatWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = blockIdx.x * rows_per_block;
    const int64_t r1 = min(n, r0 + rows_per_block);
    for (int c0 = 0; c0 < d; c0 += 32) {
        const int c = c0 + lane;
        const bool on = c < d;
        const double mu = (DEV && on) ? mean[c] : 0.0;
        double s = 0.0, mn = INFINITY, mx = -INFINITY;
#pragma unroll 8
        for (int64_t r = r0 + warp; on && r < r1; r += kStatWarps) {
            const double x = (double)__ldg(X + r * d + c);
            if (DEV) {
                const double t = __dsub_rn(x, mu);
                s = __dadd_rn(s, __dmul_rn(t, t));
            } else {
                s = __dadd_rn(s, x);
                mn = fmin(mn, x);
                mx = fmax(mx, x);
            }
        }
        s_a[warp][lane] = s;
        s_b[warp][lane] = mn;
        s_c[warp][lane] = mx;
        __syncthreads();
        if (warp == 0 && on) {
            double ts = s_a[0][lane], tmn = s_b[0][lane], tmx = s_c[0][lane];
            for (int w = 1; w < kStatWarps; ++w) {
                ts = __dadd_rn(ts, s_a[w][lane]);
                tmn = fmin(tmn, s_b[w][lane]);
                tmx = fmax(tmx, s_c[w][lane]);
            }
            double* p = part + (int64_t)blockIdx.x * 3 * d;
            p[c] = ts;
            p[d + c] = tmn;
            p[2 * d + c] = tmx;
        }
        __syncthreads();
    }
}


// Vectorised form for d in {4, 8, 16, 32, 64, 128}: a thread owns 4 adjacent
// columns (one 16-byte load per row), tpr = d/4 threads cover a row, so a warp
// streams 32/tpr whole rows per load (512 contiguous bytes) and every thread
// carries 4 independent f64 chains.  Same fixed combination order
// (row slot, then block) -> deterministic.
template <bool DEV>
__global__ void __launch_bounds__(kStatThreads) dim_partial4_kernel(const float* __restrict__ X, int64_t n, int d,
                                                                    int64_t rows_per_block,
                                                                    const double* __restrict__ mean,
                                                                    double* __restrict__ part) {
    extern __shared__ double sp[];  // 3 x RB x d
    const int tpr = d >> 2, RB = kStatThreads / tpr;
    const int t = threadIdx.x, g4 = t % tpr, rs = t / tpr;
    const int c = 4 * g4;
    const int64_t r0 = blockIdx.x * rows_per_block;
    const int64_t r1 = min(n, r0 + rows_per_block);
    double s[4] = {0.0, 0.0, 0.0, 0.0}, mn[4], mx[4], mu[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        mn[q] = INFINITY;
        mx[q] = -INFINITY;
        mu[q] = DEV ? mean[c + q] : 0.0;
    }
#pragma unroll 4
    for (int64_t r = r0 + rs; r < r1; r += RB) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(X + r * d + c));
        const double x[4] = {(double)v.x, (double)v.y, (double)v.z, (double)v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (DEV) {
                const double u = __dsub_rn(x[q], mu[q]);
                s[q] = __dadd_rn(s[q], __dmul_rn(u, u));
            } else {
                s[q] = __dadd_rn(s[q], x[q]);
                mn[q] = fmin(mn[q], x[q]);
                mx[q] = fmax(mx[q], x[q]);
            }
        }
    }
    double* S = sp;
    double* A = sp + RB * d;
    double* Z = sp + 2 * RB * d;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        S[rs * d + c + q] = s[q];
        A[rs * d + c + q] = mn[q];
        Z[rs * d + c + q] = mx[q];
    }
    __syncthreads();
    for (int cc = t; cc < d; cc += kStatThreads) {
        double ts = S[cc], ta = A[cc], tz = Z[cc];
        for (int q = 1; q < RB; ++q) {
            ts = __dadd_rn(ts, S[q * d + cc]);
            ta = fmin(ta, A[q * d + cc]);
            tz = fmax(tz, Z[q * d + cc]);
        }
        double* p = part + (int64_t)blockIdx.x * 3 * d;
        p[cc] = ts;
        p[d + cc] = ta;
        p[2 * d + cc] = tz;
    }
}

bool stats_vec4(int d) { return d == 4 || d == 8 || d == 16 || d == 32 || d == 64 || d == 128; }

// one thread per column: combine the block partials in block order.
// one warp per column: lane l combines block partials l, l + 32, ... in order,
// then a fixed xor-shuffle tree (deterministic; the earlier one-thread-per-
// column loop over all block partials was a latency chain of nblocks loads)
template <bool DEV>
__global__ void dim_final_kernel(const double* __restrict__ part, int nblocks, int64_t n, int d, double* mn,
                                 double* mx, double* mean, double* sd) {
    const int c = blockIdx.x;
    const int lane = threadIdx.x;
    double s = 0.0, a = INFINITY, b = -INFINITY;
    for (int q = lane; q < nblocks; q += 32) {
        const double* p = part + (int64_t)q * 3 * d;
        s = __dadd_rn(s, p[c]);
        if (!DEV) {
            a = fmin(a, p[d + c]);
            b = fmax(b, p[2 * d + c]);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
        a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane) return;
    if (DEV) {
        sd[c] = __dsqrt_rn(__ddiv_rn(s, (double)n));
    } else {
        mn[c] = a;
        mx[c] = b;
        mean[c] = __ddiv_rn(s, (double)n);
    }
}

int stat_blocks(int64_t n) {
    int64_t b = (int64_t)num_sms() * 4;  // (8 per SM measured slower: 0.60 vs 0.55 ms at 10M x 32)
    const int64_t min_rows = 1024;  // keep a block's rows long enough to stream
    if (b * min_rows > n) b = (n + min_rows - 1) / min_rows;
    return (int)(b < 1 ? 1 : b);
}

// ---------------------------------------------------------------------------
// Dataset transforms (ref: io.py:200-225 apply_transform), elementwise in f64:
//   none: x;  minmax: 0.5 if span <= 0 else (x - min) / span;
//   zscore: 0 if sd <= 0 else (x - mean) / sd;  affine: a * x + b (no FMA)
// then astype(float32) (round to nearest).  Per-column parameters in smem.
// ---------------------------------------------------------------------------
struct ColXf {
    int32_t kind;
    double p, q;  // minmax: (min, span); zscore: (mean, sd); affine: (a, b)
};

__device__ __forceinline__ float xform1(const ColXf& t, float xf) {
    const double x = (double)xf;
    double y;
    if (t.kind == 0) y = x;
    else if (t.kind == 1) y = t.q <= 0.0 ? 0.5 : __ddiv_rn(__dsub_rn(x, t.p), t.q);
    else if (t.kind == 2) y = t.q <= 0.0 ? 0.0 : __ddiv_rn(__dsub_rn(x, t.p), t.q);
    else y = __dadd_rn(__dmul_rn(t.p, x), t.q);
    return __double2float_rn(y);
}

// d % 4 == 0: one float4 (4 adjacent columns of one row) per thread-step
__global__ void transform4_kernel(const float4* __restrict__ X, int64_t n4, int d, const int32_t* __restrict__ kind,
                                  const double* __restrict__ pa, const double* __restrict__ pb,
                                  const double* __restrict__ mn, const double* __restrict__ mx,
                                  const double* __restrict__ mean, const double* __restrict__ sd,
                                  float4* __restrict__ out, int32_t* flag);

__global__ void transform_kernel(const float* __restrict__ X, int64_t n, int d, const int32_t* __restrict__ kind,
                                 const double* __restrict__ pa, const double* __restrict__ pb,
                                 const double* __restrict__ mn, const double* __restrict__ mx,
                                 const double* __restrict__ mean, const double* __restrict__ sd,
                                 float* __restrict__ out, int32_t* flag) {
    extern __shared__ ColXf cx[];
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        ColXf t;
        t.kind = kind[c];
        if (t.kind == 1) {
            t.p = mn[c];
            t.q = __dsub_rn(mx[c], mn[c]);
        } else if (t.kind == 2) {
            t.p = mean[c];
            t.q = sd[c];
        } else {
            t.p = pa ? pa[c] : 1.0;
            t.q = pb ? pb[c] : 0.0;
        }
        cx[c] = t;
    }
    __syncthreads();
    bool bad = false;
    const int64_t total = n * d;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int cstep = (int)(stride % d);
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int c = (int)(e % d);  // column of e, advanced incrementally (one division per thread)
    for (; e < total; e += stride, c = (c + cstep >= d) ? c + cstep - d : c + cstep) {
        const ColXf t = cx[c];
        const double x = (double)__ldg(X + e);
        double y;
        if (t.kind == 0) y = x;
        else if (t.kind == 1) y = t.q <= 0.0 ? 0.5 : __ddiv_rn(__dsub_rn(x, t.p), t.q);
        else if (t.kind == 2) y = t.q <= 0.0 ? 0.0 : __ddiv_rn(__dsub_rn(x, t.p), t.q);
        else y = __dadd_rn(__dmul_rn(t.p, x), t.q);
        const float f = __double2float_rn(y);
        bad |= !finite_f(f);
        out[e] = f;
    }
    flag_nonfinite(flag, bad);
}


// ---------------------------------------------------------------------------
// Landmark-side graph ops, g-sized f64 work.
//
// layout_tick (ref: graphmodel.py:138-192): F_i = sum of Hooke pulls over the
// edges touching i (the edges where i is the first endpoint in edge order,
// then those where it is the second -- np.add.at's order) + the softened
// all-pairs repulsion sum_j rep (p_i - p_j) / (|p_i - p_j|^2 + eps)^1.5 (j
// ascending); then v <- damping (v + dt F), p <- p + dt v, pinned rows keep
// p and get v = 0.  One warp per landmark: lanes stride j, a fixed-order
// shuffle tree reduces (deterministic); the edges arrive as a host-built
// CSR (node -> signed edge list).
// ---------------------------------------------------------------------------
__global__ void layout_tick_kernel(const float* __restrict__ lo, int g, const int32_t* __restrict__ pairs,
                                   const float* __restrict__ rest, const int32_t* __restrict__ csr_ptr,
                                   const int32_t* __restrict__ csr_edge, const uint8_t* __restrict__ pinned,
                                   double stiffness, double repulsion, double eps, double damping, double dt,
                                   double* __restrict__ vel, float* __restrict__ lo_out,
                                   double* __restrict__ forces) {
    const int lane = threadIdx.x & 31;
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= g) return;
    const double px = (double)lo[2 * i], py = (double)lo[2 * i + 1];
    double rx = 0.0, ry = 0.0;
    for (int j = lane; j < g; j += 32) {
        if (j == i) continue;  // np.fill_diagonal(inv, 0)
        const double dx = __dsub_rn(px, (double)lo[2 * j]), dy = __dsub_rn(py, (double)lo[2 * j + 1]);
        const double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
        const double q = __dadd_rn(r2, eps);
        const double inv = __ddiv_rn(repulsion, __dmul_rn(q, __dsqrt_rn(q)));  // q^1.5 (numpy: pow; ~1 ulp apart)
        rx = __dadd_rn(rx, __dmul_rn(inv, dx));
        ry = __dadd_rn(ry, __dmul_rn(inv, dy));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        rx = __dadd_rn(rx, __shfl_down_sync(0xffffffffu, rx, o));
        ry = __dadd_rn(ry, __shfl_down_sync(0xffffffffu, ry, o));
    }
    if (lane) return;
    double fx = 0.0, fy = 0.0;
    for (int q = csr_ptr[i]; q < csr_ptr[i + 1]; ++q) {
        const int s = csr_edge[q];
        const int e = s >= 0 ? s : -s - 1;  // s < 0: i is the edge's second endpoint
        const int a = pairs[2 * e], b = pairs[2 * e + 1];
        const double dx = __dsub_rn((double)lo[2 * b], (double)lo[2 * a]);
        const double dy = __dsub_rn((double)lo[2 * b + 1], (double)lo[2 * a + 1]);
        const double dist = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
        if (!(dist > 0.0)) continue;
        const double k = __ddiv_rn(__dmul_rn(stiffness, __dsub_rn(dist, (double)rest[e])), dist);
        const double ux = __dmul_rn(k, dx), uy = __dmul_rn(k, dy);
        fx = s >= 0 ? __dadd_rn(fx, ux) : __dsub_rn(fx, ux);
        fy = s >= 0 ? __dadd_rn(fy, uy) : __dsub_rn(fy, uy);
    }
    fx = __dadd_rn(fx, rx);
    fy = __dadd_rn(fy, ry);
    if (forces) {
        forces[2 * i] = fx;
        forces[2 * i + 1] = fy;
    }
    double vx = __dmul_rn(damping, __dadd_rn(vel[2 * i], __dmul_rn(dt, fx)));
    double vy = __dmul_rn(damping, __dadd_rn(vel[2 * i + 1], __dmul_rn(dt, fy)));
    float ox = __double2float_rn(__dadd_rn(px, __dmul_rn(dt, vx)));
    float oy = __double2float_rn(__dadd_rn(py, __dmul_rn(dt, vy)));
    if (pinned && pinned[i]) {
        vx = vy = 0.0;
        ox = lo[2 * i];
        oy = lo[2 * i + 1];
    }
    vel[2 * i] = vx;
    vel[2 * i + 1] = vy;
    lo_out[2 * i] = ox;
    lo_out[2 * i + 1] = oy;
}

// fit_hi_for_new_landmark (ref: som.py:82-101): d2_j = |lo_j - p|^2 (f64);
// the first minimum below eps returns hi_j verbatim, else the inverse-distance
// weighted mean sum_j w_j hi_j / sum_j w_j, w_j = 1 / (d2_j + eps).  One CTA.
__global__ void fit_hi_kernel(const float* __restrict__ hi, const float* __restrict__ lo, int g, int d, double px,
                              double py, double eps, float* __restrict__ out) {
    extern __shared__ double w[];  // g weights
    __shared__ double s_min[32], s_sum[32];
    __shared__ int s_arg[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    double best = INFINITY, wsum = 0.0;
    int arg = 0x7fffffff;
    for (int j = tid; j < g; j += blockDim.x) {
        const double dx = __dsub_rn((double)lo[2 * j], px), dy = __dsub_rn((double)lo[2 * j + 1], py);
        const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
        if (d2 < best) best = d2, arg = j;  // j ascending per thread: first minimum kept
        w[j] = __ddiv_rn(1.0, __dadd_rn(d2, eps));
    }
    __syncthreads();
    for (int j = tid; j < g; j += blockDim.x) wsum = __dadd_rn(wsum, w[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, o);
        const int oa = __shfl_down_sync(0xffffffffu, arg, o);
        if (ob < best || (ob == best && oa < arg)) best = ob, arg = oa;
        wsum = __dadd_rn(wsum, __shfl_down_sync(0xffffffffu, wsum, o));
    }
    if (lane == 0) s_min[warp] = best, s_arg[warp] = arg, s_sum[warp] = wsum;
    __syncthreads();
    if (tid == 0) {
        for (int q = 1; q < nw; ++q) {
            if (s_min[q] < s_min[0] || (s_min[q] == s_min[0] && s_arg[q] < s_arg[0])) s_min[0] = s_min[q], s_arg[0] = s_arg[q];
            s_sum[0] = __dadd_rn(s_sum[0], s_sum[q]);
        }
    }
    __syncthreads();
    const bool hit = s_min[0] < eps;
    const int jb = s_arg[0];
    const double W = s_sum[0];
    for (int c = tid; c < d; c += blockDim.x) {
        if (hit) {
            out[c] = hi[(int64_t)jb * d + c];
            continue;
        }
        double acc = 0.0;
        for (int j = 0; j < g; ++j) acc = fma(w[j], (double)hi[(int64_t)j * d + c], acc);
        out[c] = __double2float_rn(__ddiv_rn(acc, W));
    }
}


__global__ void transform4_kernel(const float4* __restrict__ X, int64_t n4, int d, const int32_t* __restrict__ kind,
                                  const double* __restrict__ pa, const double* __restrict__ pb,
                                  const double* __restrict__ mn, const double* __restrict__ mx,
                                  const double* __restrict__ mean, const double* __restrict__ sd,
                                  float4* __restrict__ out, int32_t* flag) {
    extern __shared__ ColXf cx4[];
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        ColXf t;
        t.kind = kind[c];
        if (t.kind == 1) {
            t.p = mn[c];
            t.q = __dsub_rn(mx[c], mn[c]);
        } else if (t.kind == 2) {
            t.p = mean[c];
            t.q = sd[c];
        } else {
            t.p = pa ? pa[c] : 1.0;
            t.q = pb ? pb[c] : 0.0;
        }
        cx4[c] = t;
    }
    __syncthreads();
    bool bad = false;
    const int d4 = d >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int cstep = (int)(stride % d4);
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int c4 = (int)(e % d4);
    if (cstep == 0) {  // the grid stride is a multiple of the row: this thread's 4 columns never change
        const ColXf t0 = cx4[4 * c4], t1 = cx4[4 * c4 + 1], t2 = cx4[4 * c4 + 2], t3 = cx4[4 * c4 + 3];
        for (; e < n4; e += stride) {
            const float4 v = __ldg(X + e);
            float4 o;
            o.x = xform1(t0, v.x);
            o.y = xform1(t1, v.y);
            o.z = xform1(t2, v.z);
            o.w = xform1(t3, v.w);
            bad |= !finite_f(o.x) | !finite_f(o.y) | !finite_f(o.z) | !finite_f(o.w);
            out[e] = o;
        }
        flag_nonfinite(flag, bad);
        return;
    }
    for (; e < n4; e += stride, c4 = (c4 + cstep >= d4) ? c4 + cstep - d4 : c4 + cstep) {
        const float4 v = __ldg(X + e);
        const int c = 4 * c4;
        float4 o;
        o.x = xform1(cx4[c], v.x);
        o.y = xform1(cx4[c + 1], v.y);
        o.z = xform1(cx4[c + 2], v.z);
        o.w = xform1(cx4[c + 3], v.w);
        bad |= !finite_f(o.x) | !finite_f(o.y) | !finite_f(o.z) | !finite_f(o.w);
        out[e] = o;
    }
    flag_nonfinite(flag, bad);
}
}  // namespace

extern "C" {

int esom_color_channel(const float* X, int64_t n, int32_t d, int32_t color_dim, double lo, double span, uint8_t* out,
                       cudaStream_t stream) {
    if (color_dim < 0 || color_dim >= d)
        return set_err(ESOM_ERR_PARAM, "color_dim=%lld out of range for d=%lld", (long long)color_dim, (long long)d);
    if (n <= 0) return ESOM_OK;
    color_channel_kernel<<<stream_grid(n, 256), 256, 0, stream>>>(X, n, d, color_dim, lo, span, out);
    return cuda_check("color_channel_kernel");
}

size_t esom_frame_points_bytes(int64_t n) { return (size_t)(13 + 9 * n); }

void* esom_mapped_device_ptr(void* host_ptr) {
    void* dptr = nullptr;
    if (cudaHostGetDevicePointer(&dptr, host_ptr, 0) != cudaSuccess) {
        cudaGetLastError();  // not page-locked / not mapped: clear the sticky-free error
        return nullptr;
    }
    return dptr;
}

int esom_frame_points_pack(const float* xy, const uint8_t* colors, int64_t n, uint32_t frame_id, uint8_t* out,
                           cudaStream_t stream) {
    if (n < 0 || 9 + 9 * n > 0xffffffffLL)
        return set_err(ESOM_ERR_PARAM, "frame of %lld points does not fit the u32 length field", (long long)n);
    if ((((uintptr_t)out) & 15) || (((uintptr_t)xy) & 3))
        return set_err(ESOM_ERR_PARAM, "frame buffer must be 16-byte aligned%s", "");
    const int64_t chunks = (13 + 9 * n + 15) / 16;
    frame_points_pack_kernel<<<stream_grid(chunks, 256), 256, 0, stream>>>(xy, colors, n, frame_id, out);
    return cuda_check("frame_points_pack_kernel");
}

int esom_fcs_decode(const void* raw, int64_t count, int32_t big_endian, float* out, int32_t* nonfinite_flag,
                    cudaStream_t stream) {
    if (count < 0) return set_err(ESOM_ERR_PARAM, "negative value count%s", "");
    if ((((uintptr_t)raw) & 15) || (((uintptr_t)out) & 15))
        return set_err(ESOM_ERR_PARAM, "DATA staging buffers must be 16-byte aligned%s", "");
    if (count == 0) return ESOM_OK;
    fcs_decode_kernel<<<stream_grid((count + 3) / 4, 256), 256, 0, stream>>>(reinterpret_cast<const uint32_t*>(raw),
                                                                             count, big_endian, out, nonfinite_flag);
    return cuda_check("fcs_decode_kernel");
}

size_t esom_dim_stats_workspace_bytes(int64_t n, int32_t d) { return (size_t)stat_blocks(n) * 3 * d * 8 + 256; }

int esom_dim_stats(const float* X, int64_t n, int32_t d, double* mn, double* mx, double* mean, double* sd,
                   void* workspace, size_t ws_bytes, cudaStream_t stream) {
    if (n < 1 || d < 1) return set_err(ESOM_ERR_INPUT, "empty dataset%s", "");
    if (ws_bytes < esom_dim_stats_workspace_bytes(n, d)) return set_err(ESOM_ERR_PARAM, "workspace too small%s", "");
    const int nb = stat_blocks(n);
    const int64_t rows = (n + nb - 1) / nb;
    double* part = reinterpret_cast<double*>(workspace);
    const bool v4 = stats_vec4(d) && (((uintptr_t)X) & 15) == 0;
    const size_t sm4 = v4 ? (size_t)3 * (kStatThreads / (d / 4)) * d * 8 : 0;
    if (v4) dim_partial4_kernel<false><<<nb, kStatThreads, sm4, stream>>>(X, n, d, rows, nullptr, part);
    else dim_partial_kernel<false><<<nb, kStatThreads, 0, stream>>>(X, n, d, rows, nullptr, part);
    dim_final_kernel<false><<<d, 32, 0, stream>>>(part, nb, n, d, mn, mx, mean, sd);
    if (v4) dim_partial4_kernel<true><<<nb, kStatThreads, sm4, stream>>>(X, n, d, rows, mean, part);
    else dim_partial_kernel<true><<<nb, kStatThreads, 0, stream>>>(X, n, d, rows, mean, part);
    dim_final_kernel<true><<<d, 32, 0, stream>>>(part, nb, n, d, mn, mx, mean, sd);
    return cuda_check("dim_stats", 4);
}

int esom_apply_transform(const float* X, int64_t n, int32_t d, const int32_t* kind, const double* a, const double* b,
                         const double* mn, const double* mx, const double* mean, const double* sd, float* out,
                         int32_t* nonfinite_flag, cudaStream_t stream) {
    if (n < 0 || d < 1) return set_err(ESOM_ERR_PARAM, "bad shape%s", "");
    if (n == 0) return ESOM_OK;
    const size_t smem = (size_t)d * sizeof(ColXf);
    if (smem > 48 * 1024) return set_err(ESOM_ERR_UNSUPPORTED, "d=%lld too large for the transform kernel", (long long)d);
    if ((d & 3) == 0 && !(((uintptr_t)X) & 15) && !(((uintptr_t)out) & 15)) {
        const int64_t n4 = n * d / 4;
        transform4_kernel<<<stream_grid(n4, 256), 256, smem, stream>>>(reinterpret_cast<const float4*>(X), n4, d, kind,
                                                                       a, b, mn, mx, mean, sd,
                                                                       reinterpret_cast<float4*>(out), nonfinite_flag);
        return cuda_check("transform4_kernel");
    }
    transform_kernel<<<stream_grid(n * d, 256), 256, smem, stream>>>(X, n, d, kind, a, b, mn, mx, mean, sd, out,
                                                                     nonfinite_flag);
    return cuda_check("transform_kernel");
}


int esom_layout_tick(const float* lo, int32_t g, const int32_t* pairs, const float* rest, const int32_t* csr_ptr,
                     const int32_t* csr_edge, const uint8_t* pinned, double stiffness, double repulsion, double eps,
                     double damping, double dt, double* vel_inout, float* lo_out, double* forces_or_null,
                     cudaStream_t stream) {
    if (g < 0) return set_err(ESOM_ERR_PARAM, "negative landmark count%s", "");
    if (!(damping > 0.0 && damping < 1.0)) return set_err(ESOM_ERR_PARAM, "damping must be in (0, 1)%s", "");
    if (!(dt > 0.0)) return set_err(ESOM_ERR_PARAM, "dt must be > 0%s", "");
    if (g == 0) return ESOM_OK;
    const int threads = 256;
    const int blocks = (int)(((int64_t)g * 32 + threads - 1) / threads);
    layout_tick_kernel<<<blocks, threads, 0, stream>>>(lo, g, pairs, rest, csr_ptr, csr_edge, pinned, stiffness,
                                                       repulsion, eps, damping, dt, vel_inout, lo_out, forces_or_null);
    return cuda_check("layout_tick_kernel");
}

int esom_fit_hi(const float* hi, const float* lo, int32_t g, int32_t d, double px, double py, double eps, float* out,
                cudaStream_t stream) {
    if (g < 1) return set_err(ESOM_ERR_INPUT, "empty model%s", "");
    const size_t smem = (size_t)g * 8;
    if (smem > (size_t)max_smem_optin()) return set_err(ESOM_ERR_UNSUPPORTED, "g=%lld too large for fit_hi", (long long)g);
    cudaFuncSetAttribute(fit_hi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fit_hi_kernel<<<1, 1024, smem, stream>>>(hi, lo, g, d, px, py, eps, out);
    return cuda_check("fit_hi_kernel");
}

}  // extern "C"
