// esom_project.cuh -- fast EmbedSOM projection from exact neighbour lists
// (ref: projection.py:38-59 scores, 68-121 _project_rows).
//
// One thread per point.  For every kept pair (u < v, w = s_u s_v > 0) the
// high-dimensional line coordinate comes from the law of cosines on the
// EXACT squared distances the k-NN scan already produced:
//     dnum/hd2 = (x - h_u).(h_v - h_u) / |h_v - h_u|^2 = 1/2 + (sqd_u - sqd_v) * T_uv
// with T_uv = 0.5 / hd2_uv from a per-model pair table (packed upper
// triangle, f32, -1 where the reference skips the pair: hd2 < 1e-12).  No
// landmark rows are gathered per pair.  The table lives in shared memory
// when it fits (g <= ~256), otherwise in L2.  Layout terms and the normal
// equations are evaluated in f64, like the reference's accumulators.
//
// Accuracy: the law of cosines has absolute error ~ u*sqrt(d)*(sqd_u+sqd_v)
// in dnum; points whose kappa = max (sqd_u+sqd_v)*T_uv exceeds kKappaMax
// recompute their k distances in f64 (precise_sqd), and the rare far
// outliers and ill-conditioned systems run the reference's own arithmetic
// (faithful_point).  Checked against the reference to <= 1e-4 x extent.
#pragma once
#include <stdlib.h>

#include "esom_common.cuh"
#include "esom_faithful.cuh"
#include "esom_host.h"
#include "esom_scan_args.h"

namespace esom {

// threads per CTA: 384 for k <= 16 (per-thread rows fit next to a smem pair
// table of g <= 256), fewer for larger k so the per-thread rows still fit
template <int KP>
__host__ __device__ constexpr int proj_threads() { return KP <= 16 ? 384 : (KP <= 32 ? 256 : 128); }

// Exact f64 pair accumulation from x and the landmark rows (outlier path).
static __device__ __noinline__ void pairs_exact_f64(const float* __restrict__ x, int d,
                                                    const float* __restrict__ hi, const float* __restrict__ lo,
                                                    int k, const int* J, const float* S, int stride, double* out5) {
    double a11 = 0.0, a12 = 0.0, a22 = 0.0, c1 = 0.0, c2 = 0.0;
    for (int u = 0; u < k; ++u) {
        const double su = S[u * stride];
        if (su <= 0.0) continue;
        const int ju = J[u * stride];
        const float* hu = hi + (int64_t)ju * d;
        for (int v = u + 1; v < k; ++v) {
            const double w = su * (double)S[v * stride];
            if (!(w > 0.0)) continue;
            const int jv = J[v * stride];
            const float* hv = hi + (int64_t)jv * d;
            double hd2 = 0.0, hd2f = 0.0, dnum = 0.0;
            for (int c = 0; c < d; ++c) {
                const double e = (double)hv[c] - (double)hu[c];
                const float ef = __fsub_rn(hv[c], hu[c]);
                hd2f = __dadd_rn(hd2f, (double)__fmul_rn(ef, ef));
                hd2 = fma(e, e, hd2);
                dnum = fma((double)x[c] - (double)hu[c], e, dnum);
            }
            if (hd2f < kPairEps) continue;
            const float exf = __fsub_rn(lo[2 * jv], lo[2 * ju]);
            const float eyf = __fsub_rn(lo[2 * jv + 1], lo[2 * ju + 1]);
            const float ld2f = __fadd_rn(__fmul_rn(exf, exf), __fmul_rn(eyf, eyf));
            if ((double)ld2f < kPairEps) continue;
            const double ex = exf, ey = eyf, ld2 = (double)ld2f;
            const double g1 = ex / ld2, g2 = ey / ld2;
            const double h = dnum / hd2 + g1 * (double)lo[2 * ju] + g2 * (double)lo[2 * ju + 1];
            const double wg1 = w * g1, wg2 = w * g2, wh = w * h;
            a11 = fma(wg1, g1, a11);
            a12 = fma(wg1, g2, a12);
            a22 = fma(wg2, g2, a22);
            c1 = fma(wh, g1, c1);
            c2 = fma(wh, g2, c2);
        }
    }
    out5[0] = a11;
    out5[1] = a12;
    out5[2] = a22;
    out5[3] = c1;
    out5[4] = c2;
}

// smallest f32 value v with (double)v >= 1e-12: ld2 (f32, as the reference
// computes it) is skipped iff ld2 < kLd2Min  (ref: projection.py:346)
constexpr float kLd2Min = 1.000000104e-12f;  // 0x2b8cbccd

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

constexpr float kCondMax = 100.0f;

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float r;
    asm("ex2.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Squared distances that the law of cosines can trust far from the landmarks.
// dnum/hd2 = 1/2 + (s_u - s_v) T_uv needs s_u - s_v to ~1e-7 hd2, but the
// reference's f32 sums carry ~sqrt(d) eps32 s of rounding: once s T (kappa)
// is large -- points far from a trained SOM's tightly packed landmarks --
// that error dominates.  Recomputing the k distances in f64 (O(kd), rows from
// L1) and keeping them as f32 OFFSETS e_j = fl(s_j - s_0) from the nearest
// makes e_u - e_v = s_u - s_v up to eps32 (|s_u - s_0| + |s_v - s_0|): the
// rounding now scales with the spread of the neighbour distances, not with
// their size, and the f32 pair loop stays valid far out (kKappaMax64 bounds
// (s_{k-1} - s_0) T_max before the exact x-based f64 loop takes over).
constexpr double kKappaMax64 = 1e5;

// Far-point census for the host's visiting-order choice (esom_embed_prepared_ex):
// one warp-aggregated atomic per warp.
__device__ __forceinline__ void count_prec(int32_t* cnt, bool prec) {
    if (!cnt) return;
    const unsigned am = __activemask();
    const unsigned b = __ballot_sync(am, prec);
    if ((threadIdx.x & 31) == __ffs(am) - 1 && b) atomicAdd(cnt, __popc(b));
}



template <int KP, bool SMEM = false>
__device__ __forceinline__ void precise_sqd(const float* __restrict__ x, int d, const double* __restrict__ hi64,
                                            int hs, const int (&jj)[KP], int k, float (&qe)[KP]) {
    // rows (stride hs doubles) in shared memory (plain loads) or the model workspace (read-only path)
    auto row2 = [&](int j, int c) {
        const double2* p = reinterpret_cast<const double2*>(hi64 + (int64_t)j * hs + c);
        return SMEM ? *p : __ldg(p);
    };
    auto row1 = [&](int j, int c) {
        const double* p = hi64 + (int64_t)j * hs + c;
        return SMEM ? *p : __ldg(p);
    };
    // landmark rows come pre-widened (model workspace), so the only f32 -> f64
    // conversions are x's: 2 per dimension pair per chunk of neighbours (the
    // per-element F2F of both operands used to dominate trained-model frames)
    constexpr int QC = KP < 8 ? KP : 8;  // neighbours per pass (bounds the live f64 accumulators)
    double s0 = 0.0;
#pragma unroll
    for (int q0 = 0; q0 < KP; q0 += QC) {
        double acc[QC];
#pragma unroll
        for (int q = 0; q < QC; ++q) acc[q] = 0.0;
        if ((d & 1) == 0) {
            for (int c = 0; c < d; c += 2) {
                const float2 xv = __ldg(reinterpret_cast<const float2*>(x + c));
                const double x0 = (double)xv.x, x1 = (double)xv.y;
#pragma unroll
                for (int q = 0; q < QC; ++q) {
                    if (q0 + q < k) {
                        const double2 hv = row2(jj[q0 + q], c);
                        double t = x0 - hv.x;
                        acc[q] = fma(t, t, acc[q]);
                        t = x1 - hv.y;
                        acc[q] = fma(t, t, acc[q]);
                    }
                }
            }
        } else {
            for (int c = 0; c < d; ++c) {
                const double xc = (double)__ldg(x + c);
#pragma unroll
                for (int q = 0; q < QC; ++q) {
                    if (q0 + q < k) {
                        const double t = xc - row1(jj[q0 + q], c);
                        acc[q] = fma(t, t, acc[q]);
                    }
                }
            }
        }
        if (q0 == 0) s0 = acc[0];
#pragma unroll
        for (int q = 0; q < QC; ++q) qe[q0 + q] = q0 + q < k ? (float)(acc[q] - s0) : 0.0f;
    }
}

// precise_sqd for a compile-time d (d = 32: C2-C4), in the dot-product form
//   s_j - s_0 = (|h_j|^2 - |h_0|^2) - 2 x.(h_j - h_0),  x.h_j = sum_c x_c h_jc
// (one f64 FMA per element, |h_j|^2 precomputed per model; f64 keeps the
// cancellation harmless: ~1e-13 absolute at these magnitudes), with x held in
// registers (its loads all in flight at once) and the dimension loop unrolled
// so the row loads of the next step issue early.
// FULL (frames where most points are far, i.e. trained models): x held in
// registers and every step unrolled -- the most loads in flight, at the price of
// registers the common case needs elsewhere; otherwise x streams one step ahead.
template <int KP, int D, bool SMEM, bool FULL>
__device__ __forceinline__ void precise_sqd_fixed(const float* __restrict__ xg, const double* __restrict__ hi64,
                                                  int hs, const double* __restrict__ hn, const int (&jj)[KP], int k,
                                                  float (&qe)[KP]) {
    constexpr int QC = KP < 4 ? KP : 4;
    float xr[FULL ? D : 4];
    if (FULL) {
#pragma unroll
        for (int c = 0; c < D; c += 4) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(xg + c));
            xr[c] = v.x; xr[c + 1] = v.y; xr[c + 2] = v.z; xr[c + 3] = v.w;
        }
    }
    double s0 = 0.0;
#pragma unroll
    for (int q0 = 0; q0 < KP; q0 += QC) {
        double acc[QC];
#pragma unroll
        for (int q = 0; q < QC; ++q) acc[q] = 0.0;
        float4 xn = FULL ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg(reinterpret_cast<const float4*>(xg));
#pragma unroll (FULL ? D / 4 : 2)
        for (int c = 0; c < D; c += 4) {
            float4 xc;
            if (FULL) {
                xc = make_float4(xr[c % (FULL ? D : 4)], xr[(c + 1) % (FULL ? D : 4)], xr[(c + 2) % (FULL ? D : 4)],
                                 xr[(c + 3) % (FULL ? D : 4)]);
            } else {
                xc = xn;
                if (c + 4 < D) xn = __ldg(reinterpret_cast<const float4*>(xg + c + 4));  // one step ahead
            }
            const double x0 = (double)xc.x, x1 = (double)xc.y, x2 = (double)xc.z, x3 = (double)xc.w;
#pragma unroll
            for (int q = 0; q < QC; ++q) {
                if (q0 + q < k) {
                    const double2* pr = reinterpret_cast<const double2*>(hi64 + (int64_t)jj[q0 + q] * hs + c);
                    const double2 h01 = SMEM ? pr[0] : __ldg(pr);
                    const double2 h23 = SMEM ? pr[1] : __ldg(pr + 1);
                    acc[q] = fma(x0, h01.x, acc[q]);
                    acc[q] = fma(x1, h01.y, acc[q]);
                    acc[q] = fma(x2, h23.x, acc[q]);
                    acc[q] = fma(x3, h23.y, acc[q]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < QC; ++q) {
            const double hq = q0 + q < k ? (SMEM ? hn[jj[q0 + q]] : __ldg(hn + jj[q0 + q])) : 0.0;
            acc[q] = fma(-2.0, acc[q], hq);  // s_j - |x|^2
        }
        if (q0 == 0) s0 = acc[0];
#pragma unroll
        for (int q = 0; q < QC; ++q) qe[q0 + q] = q0 + q < k ? (float)(acc[q] - s0) : 0.0f;
    }
}

// precise_sqd from the exact phase's f32 landmark rows in shared memory (the
// fused kernel; rows in screen order, located through inv = landmark -> row):
// the same dot-product form in f64, each row element widened on the fly.
template <int KP>
__device__ __forceinline__ void precise_sqd_rows32(const float* __restrict__ xg, const float* Ls, int ls,
                                                   const int32_t* inv, const double* __restrict__ hn,
                                                   const int (&jj)[KP], int k, float (&qe)[KP]) {
    constexpr int QC = KP < 4 ? KP : 4;
    double s0 = 0.0;
#pragma unroll
    for (int q0 = 0; q0 < KP; q0 += QC) {
        double acc[QC];
        const float* rw[QC];
#pragma unroll
        for (int q = 0; q < QC; ++q) {
            acc[q] = 0.0;
            rw[q] = Ls + (size_t)inv[q0 + q < k ? jj[q0 + q] : 0] * ls;
        }
        float4 xn = __ldg(reinterpret_cast<const float4*>(xg));
#pragma unroll 2
        for (int c = 0; c < 32; c += 4) {
            const float4 xc = xn;
            if (c + 4 < 32) xn = __ldg(reinterpret_cast<const float4*>(xg + c + 4));
            const double x0 = (double)xc.x, x1 = (double)xc.y, x2 = (double)xc.z, x3 = (double)xc.w;
#pragma unroll
            for (int q = 0; q < QC; ++q) {
                const float4 h = *reinterpret_cast<const float4*>(rw[q] + c);
                acc[q] = fma(x0, (double)h.x, acc[q]);
                acc[q] = fma(x1, (double)h.y, acc[q]);
                acc[q] = fma(x2, (double)h.z, acc[q]);
                acc[q] = fma(x3, (double)h.w, acc[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < QC; ++q) {
            const double hq = q0 + q < k ? __ldg(hn + jj[q0 + q]) : 0.0;
            acc[q] = fma(-2.0, acc[q], hq);  // s_j - |x|^2
        }
        if (q0 == 0) s0 = acc[0];
#pragma unroll
        for (int q = 0; q < QC; ++q) qe[q0 + q] = q0 + q < k ? (float)(acc[q] - s0) : 0.0f;
    }
}

// Ill-conditioned systems (tr^2 > kCondMax det: the solution amplifies every
// rounding) and far outliers: the reference's own scores and projection op
// for op (esom_faithful.cuh) -- bit-faithful given the scores, so even the
// wild solutions of near-singular systems match (fuzz: kappa ~ 5e5).  Rare.
static __device__ __noinline__ void faithful_point(const ProjArgs& a, int64_t i) {
    double sc[64];
    const float* row = a.sqd + i * a.k;
    score_row_dev(a.k, [&](int t) { return __ldg(row + t); }, sc);
    project_row_faithful(a.X + i * a.d, a.hi, a.lo, a.idx + i * a.k, sc, a.d, a.k, a.xy + 2 * i);
}

template <int KP>
__global__ void __launch_bounds__(proj_threads<KP>()) project_fast_kernel(ProjArgs a) {
    constexpr int PT = proj_threads<KP>();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int g = a.g, k = a.k;
    // layout: lo [g] float2 | RB [g] int | J [KP][PT] int | S [KP][PT] f32 | Q, QB [KP][PT] f32 | (T table)
    // 16-byte aligned regions (the T table below is copied with float4 stores;
    // odd g used to misalign it: fuzz test)
    float2* LO = reinterpret_cast<float2*>(smem_raw);
    int* RB = reinterpret_cast<int*>(smem_raw + (((size_t)g * 8 + 15) & ~(size_t)15));
    int* J = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(RB) + (((size_t)g * 4 + 15) & ~(size_t)15));
    float* S = reinterpret_cast<float*>(J + KP * PT);
    float* Q = S + KP * PT;
    const float tmax_model = a.tmax ? __ldg(a.tmax) : 0.0f;
    const float* Ts = a.T;
    if (a.t_smem) {
        float* tsm = Q + KP * PT;
        const int ntri = g * (g - 1) / 2;
        const float4* src = reinterpret_cast<const float4*>(a.T);
        float4* dst = reinterpret_cast<float4*>(tsm);
        for (int e = tid; e < ntri / 4; e += PT) dst[e] = src[e];
        for (int e = (ntri / 4) * 4 + tid; e < ntri; e += PT) tsm[e] = a.T[e];
        Ts = tsm;
    }
    for (int j = tid; j < g; j += PT) {
        LO[j] = make_float2(a.lo[2 * j], a.lo[2 * j + 1]);
        RB[j] = j * (2 * g - j - 1) / 2 - j - 1;  // tri(j, b) = RB[j] + b for b > j
    }
    __syncthreads();

    for (int64_t i = blockIdx.x * (int64_t)PT + tid; i < a.n; i += (int64_t)gridDim.x * PT) {
        const int32_t* irow = a.idx + i * k;
        const float* drow = a.sqd + i * k;
        // scores: the scale-free f32 form of project_reg2_kernel
        float sig = 0.0f, sqk = 0.0f;
        for (int q = 0; q < k; ++q) {
            const float sq = __ldg(drow + q);
            sig += sqrt_approx(sq);
            J[q * PT + tid] = __ldg(irow + q);
            Q[q * PT + tid] = sq;
            sqk = sq;  // rows ascending: the last is the largest
        }
        sig = sig / (float)k;
        bool uniform = sig < (float)kScoreEps;
        // far from the landmarks (kappa bound large): f64 paths below
        const bool prec = 2.0f * sqk * tmax_model > (float)kKappaMax;
        count_prec(a.prec_count, prec);
        if (!uniform) {
            const float inv = 1.0f / (2.0f * sig * sig);
            const float tail = ex2_approx(-1.44269504f * sqk * inv);
            const double dk = (double)__fsqrt_rn(sqk);
            for (int q = 0; q < k; ++q) {
                const float sq = Q[q * PT + tid];
                // far points: the exponent differences from the reference's own d_t^2 = (f64 sqrtf(sq))^2
                const double dq = (double)__fsqrt_rn(sq);
                const float dl = prec ? (float)((dk * dk - dq * dq) * (double)inv) : (sqk - sq) * inv;
                const float poly = dl * fmaf(dl, fmaf(dl, fmaf(dl, fmaf(dl, fmaf(dl, 1.0f / 720.0f, 1.0f / 120.0f),
                                                                       1.0f / 24.0f), 1.0f / 6.0f), 0.5f), 1.0f);
                S[q * PT + tid] = dl < 0.3f ? poly : ex2_approx(1.44269504f * dl) - 1.0f;
                if (q == 0) uniform = ex2_approx(-1.44269504f * sq * inv) - tail < (float)kScoreEps;
            }
        }
        if (uniform)
            for (int q = 0; q < k; ++q) S[q * PT + tid] = q == k - 1 ? 0.0f : 1.0f;

        // far points: Q <- f64 squared distances as f32 offsets from the nearest
        // (precise_sqd; the reference's sq are re-read for the f64 score fallback)
        if (prec) {
            const float* x = a.X + i * a.d;
            double s0 = 0.0;
            for (int q = 0; q < k; ++q) {
                const float* h = a.hi + (int64_t)J[q * PT + tid] * a.d;
                double acc = 0.0;
                for (int c = 0; c < a.d; ++c) {
                    const double t = (double)__ldg(x + c) - (double)__ldg(h + c);
                    acc = fma(t, t, acc);
                }
                if (q == 0) s0 = acc;
                Q[q * PT + tid] = (float)(acc - s0);
            }
        }
        // pairs in f32 about o = lo[idx0] (see project_reg2_kernel), solved in f64
        const float2 o = LO[J[tid]];
        float a11 = 0.0f, a12 = 0.0f, a22 = 0.0f, c1 = 0.0f, c2 = 0.0f;
        float kappa = 0.0f;
        for (int u = 0; u + 1 < k; ++u) {
            const float su = S[u * PT + tid];
            if (!(su > 0.0f)) continue;
            const int ju = J[u * PT + tid];
            const float squ = Q[u * PT + tid];
            const float2 lu = LO[ju];
            const int rbu = RB[ju];
            const float lux = lu.x - o.x, luy = lu.y - o.y;
#pragma unroll 4
            for (int v = u + 1; v < k; ++v) {
                const float sv = S[v * PT + tid];
                const int jv = J[v * PT + tid];
                const float sqv = Q[v * PT + tid];
                const int ti = ju < jv ? rbu + jv : RB[jv] + ju;
                const float tv = Ts[ti];
                const float2 lv = LO[jv];
                // layout terms in f32 exactly as the reference forms them (ref: projection.py:341-348)
                const float ex = __fsub_rn(lv.x, lu.x), ey = __fsub_rn(lv.y, lu.y);
                const float ld2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
                const float w = su * sv;
                const bool keep = (w > 0.0f) & (tv >= 0.0f) & (ld2 >= kLd2Min);
                kappa = keep ? fmaxf(kappa, (prec ? fabsf(squ) + fabsf(sqv) : squ + sqv) * tv) : kappa;
                const float rr = keep ? rcp_approx(ld2) : 0.0f;
                const float g1 = ex * rr, g2 = ey * rr, wr = w * rr;
                const float h = fmaf(squ - sqv, tv, 0.5f) + fmaf(g1, lux, g2 * luy);
                const float wg1 = wr * ex, wg2 = wr * ey;
                a11 = fmaf(wg1, g1, a11);
                a12 = fmaf(wg1, g2, a12);
                a22 = fmaf(wg2, g2, a22);
                c1 = fmaf(wg1, h, c1);
                c2 = fmaf(wg2, h, c2);
            }
        }
        double A11 = a11, A12 = a12, A22 = a22, C1 = c1, C2 = c2;
        const bool illc = a11 * a22 - a12 * a12 < (a11 + a22) * (a11 + a22) * (1.0f / kCondMax);
        const bool far = kappa > (float)(prec ? kKappaMax64 : kKappaMax);
        if (far || illc) {
            faithful_point(a, i);
            continue;
        }
        const double det = A11 * A22 - A12 * A12;
        const double tr = A11 + A22;
        float2 out;
        if (det < kDetRel * tr * tr + kDetAbs) {
            out = o;
        } else {
            out.x = (float)((C1 * A22 - C2 * A12) / det + (double)o.x);
            out.y = (float)((A11 * C2 - A12 * C1) / det + (double)o.y);
        }
        reinterpret_cast<float2*>(a.xy)[i] = out;
    }
}

constexpr int kRegThreads = 512;  // project_reg3_kernel: 16 warps/SM at <= 128 registers

// ---------------------------------------------------------------------------
// k <= 16 (default; the pair triangle in shared memory up to g ~ 330): the
// law-of-cosines projection with the whole per-point state in registers and
// the pair loop fully unrolled (static register indices).
//  * scores in f32 (MUFU sqrt/ex2; ~1e-7 relative, far inside the embedding
//    tolerance), normal equations accumulated in f32 about the nearest
//    landmark's layout position o = lo[idx0] (small magnitudes), solved in f64;
//  * points whose system is ill-conditioned (tr^2 > kCondMax det) or whose
//    law-of-cosines error bound trips (kappa) are recomputed in f64 (rare);
//  * pair-table index from per-slot row bases (no triangle arithmetic per pair),
//    unconditional table reads, vector loads of the neighbour rows.
// ---------------------------------------------------------------------------
constexpr int kReg2Threads = 512;  // 16 warps/SM at <= 128 registers (one CTA: the pair table fills smem)

// shared-memory bytes of project_reg2_kernel: LO, RB | pair triangle | f64 rows
__host__ __device__ inline size_t reg2_tri_offset(int g) { return ((size_t)g * 12 + 4 + 15) & ~(size_t)15; }
__host__ __device__ inline size_t reg2_hi64_offset(int g) {
    return (reg2_tri_offset(g) + (size_t)g * (g - 1) / 2 * 4 + 15) & ~(size_t)15;
}
// row stride (doubles) of the f64 rows in shared memory: an odd number of 16-byte
// units, so the rows of different neighbours start in different bank groups
// (a 256-byte stride put every lane's 128-bit load on the same banks)
__host__ __device__ inline int reg2_hi64_stride(int d) {
    const int u = (d + 1) / 2;  // 16-byte units
    return 2 * (u | 1);
}

// One point of project_reg2_kernel: scores + law-of-cosines projection from the
// point's k neighbour indices jj and exact squared distances sq (slots >= k:
// padding with zero weight).  Shared with the fused embed kernel
// (esom_fused.cuh; STORE_ROW: the rows are in registers only, so the rare
// faithful fallback first writes them to the point workspace).
template <int KP, bool TSMEM, bool HSMEM, bool FARHEAVY, bool STORE_ROW, bool ROWS32 = false>
__device__ __forceinline__ void reg2_point(const ProjArgs& a, int64_t i, const int (&jj)[KP], const float (&sq)[KP],
                                           const float2* LO, const int* RB, const float* T, const double* h64,
                                           const double* hn_s, int hs, float tmax_model,
                                           const float* rows32 = nullptr, int ls32 = 0,
                                           const int32_t* inv32 = nullptr) {
    const int k = a.k;
    int rb[KP];
    float sc[KP], lx[KP], ly[KP];
    f2 L[KP];  // FARHEAVY: the same layout offsets as (x, y) register pairs for the packed pair loop
    float sqmax = 0.0f;
#pragma unroll
    for (int q = 0; q < KP; ++q) sqmax = fmaxf(sqmax, sq[q]);
    const bool prec = 2.0f * sqmax * tmax_model > (float)kKappaMax;  // far: f64 distance paths
    count_prec(a.prec_count, prec);
    // far from the landmarks: the k squared distances again in f64, kept as f32
    // offsets from the nearest (precise_sqd); first, while little else is live
    float qe[KP];
    if (prec) {
        if (ROWS32)  // (d == 32, the fused kernel)
            precise_sqd_rows32<KP>(a.X + i * 32, rows32, ls32, inv32, a.hn64, jj, k, qe);
        else if (a.d == 32)
            precise_sqd_fixed<KP, 32, HSMEM, FARHEAVY>(a.X + i * 32, HSMEM ? h64 : a.hi64, HSMEM ? hs : 32,
                                             HSMEM ? hn_s : a.hn64, jj, k, qe);
        else
            precise_sqd<KP, HSMEM>(a.X + i * a.d, a.d, HSMEM ? h64 : a.hi64, HSMEM ? hs : a.d, jj, k, qe);
    } else {
#pragma unroll
        for (int q = 0; q < KP; ++q) qe[q] = sq[q];
    }
    const float2 o = LO[jj[0]];
    float sig = 0.0f, sqk = 0.0f;
#pragma unroll
    for (int q = 0; q < KP; ++q) {
        const float2 l = LO[jj[q]];
        lx[q] = l.x - o.x;  // layout about the nearest landmark
        ly[q] = l.y - o.y;
        if (FARHEAVY) L[q] = f2_sub(f2_pack(l.x, l.y), f2_pack(o.x, o.y));
        rb[q] = RB[jj[q]];
        const float dq = q < k ? sqrt_approx(sq[q]) : 0.0f;
        sig += dq;
        if (q == k - 1) sqk = sq[q];
    }
    // scores (ref: projection.py:38-59) in f32, as the scale-free weights
    // s_q / tail = expm1((d_k^2 - d_q^2) / 2 sigma^2): the normal equations
    // are homogeneous in w, and the difference form keeps full relative
    // precision where the reference's e_q - tail cancels (far outliers).
    sig = sig / (float)k;
    bool uniform = sig < (float)kScoreEps;
    if (!uniform) {
        const float inv = 1.0f / (2.0f * sig * sig);
        const float tail = ex2_approx(-1.44269504f * sqk * inv);
        float dls[KP];
        if (prec) {  // far points: exponent differences from the reference's own d_t^2 = (f64 sqrtf(sq))^2
            const double dk = (double)__fsqrt_rn(sqk);
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                const double dq = (double)__fsqrt_rn(sq[q]);
                dls[q] = q < k ? (float)((dk * dk - dq * dq) * (double)inv) : 0.0f;
            }
        } else {
#pragma unroll
            for (int q = 0; q < KP; ++q) dls[q] = q < k ? (sqk - sq[q]) * inv : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < KP; ++q) {
            const float dl = dls[q];  // >= 0 (rows ascending); 0 at q = k-1
            const float poly = dl * fmaf(dl, fmaf(dl, fmaf(dl, fmaf(dl, fmaf(dl, 1.0f / 720.0f, 1.0f / 120.0f),
                                                                   1.0f / 24.0f), 1.0f / 6.0f), 0.5f), 1.0f);
            const float e = dl < 0.3f ? poly : ex2_approx(1.44269504f * dl) - 1.0f;
            sc[q] = e;
            if (q == 0)  // the reference's s_0 = e_0 - tail < 1e-9 test (no underflow of tail * e)
                uniform = ex2_approx(-1.44269504f * sq[0] * inv) - tail < (float)kScoreEps;
        }
    }
    if (uniform) {
#pragma unroll
        for (int q = 0; q < KP; ++q) sc[q] = q < k - 1 ? 1.0f : 0.0f;
    }

    float a11 = 0.0f, a12 = 0.0f, a22 = 0.0f, c1 = 0.0f, c2 = 0.0f;
    // all pairs u < v, fully unrolled (static register indices, no ring rotation).
    // Slot KP-1 never pairs: its score is exactly 0 (the reference's tail
    // s_{k-1} = 0 when k == KP, the uniform fallback's trailing 0, or padding).
    if constexpr (FARHEAVY) {
        // far-heavy frames (trained models): the same operations packed as f32x2 (each lane
        // the scalar form's IEEE operation, so bit-identical): fewer issue slots next to the
        // f64 distance work (trained C2 fused kernel -9 %; on untrained frames the scalar
        // loop's register allocation measured 5 % faster, so it stays there)
        f2 A = f2_pack(0.0f, 0.0f), C = f2_pack(0.0f, 0.0f);  // (a11, a22), (c1, c2)
#pragma unroll
        for (int u = 0; u < KP - 2; ++u) {
#pragma unroll
            for (int v = u + 1; v < KP - 1; ++v) {
                const float w = sc[u] * sc[v];
                const int ti = max(jj[u] < jj[v] ? rb[u] + jj[v] : rb[v] + jj[u], 0);
                const float tv = T[ti];
                const f2 e = f2_sub(L[v], L[u]);  // (ex, ey)
                float exx, eyy;
                f2_unpack(f2_mul(e, e), exx, eyy);
                const float ld2 = __fadd_rn(exx, eyy);
                const bool keep = (tv >= 0.0f) & (ld2 >= kLd2Min);
                const float rr = keep ? rcp_approx(ld2) : 0.0f;
                const float wr = w * rr;
                const f2 g = f2_mul(e, f2_pack(rr, rr));   // (g1, g2)
                const f2 wg = f2_mul(e, f2_pack(wr, wr));  // w g
                float g1, g2, wg1, wg2;
                f2_unpack(g, g1, g2);
                f2_unpack(wg, wg1, wg2);
                const float h = fmaf(qe[u] - qe[v], tv, 0.5f) + fmaf(g1, lx[u], g2 * ly[u]);
                A = f2_fma(wg, g, A);
                a12 = fmaf(wg1, g2, a12);
                C = f2_fma(wg, f2_pack(h, h), C);
            }
        }
        f2_unpack(A, a11, a22);
        f2_unpack(C, c1, c2);
    } else {
#pragma unroll
    for (int u = 0; u < KP - 2; ++u) {
#pragma unroll
        for (int v = u + 1; v < KP - 1; ++v) {
            const float w = sc[u] * sc[v];
            const int ti = max(jj[u] < jj[v] ? rb[u] + jj[v] : rb[v] + jj[u], 0);
            const float tv = T[ti];
            const float ex = __fsub_rn(lx[v], lx[u]), ey = __fsub_rn(ly[v], ly[u]);
            const float ld2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
            // skipped pairs (the reference's hd2 / ld2 tests) get g = 0; w = 0 pairs add 0 anyway
            const bool keep = (tv >= 0.0f) & (ld2 >= kLd2Min);
            const float rr = keep ? rcp_approx(ld2) : 0.0f;  // (ld2 may be 0)
            const float wr = w * rr;
            const float g1 = ex * rr, g2 = ey * rr;
            // dnum/hd2 by the law of cosines + g . (lo_u - o)
            const float h = fmaf(qe[u] - qe[v], tv, 0.5f) + fmaf(g1, lx[u], g2 * ly[u]);
            const float wg1 = wr * ex, wg2 = wr * ey;  // w g
            a11 = fmaf(wg1, g1, a11);
            a12 = fmaf(wg1, g2, a12);
            a22 = fmaf(wg2, g2, a22);
            c1 = fmaf(wg1, h, c1);
            c2 = fmaf(wg2, h, c2);
        }
    }
    }
    double A11 = a11, A12 = a12, A22 = a22, C1 = c1, C2 = c2;
    float spread = sqmax;  // prec: the error of qe_u - qe_v scales with the offsets' spread
    if (prec) {
        spread = 0.0f;
#pragma unroll
        for (int q = 0; q < KP; ++q) spread = fmaxf(spread, fabsf(qe[q]));
    }
    // the model-wide max T bounds every kept pair's T: for a point that passed the
    // prec test (2 sqmax T_max <= kKappaMax) this never trips; far points compare
    // against the f64 path's bound
    const float kappa = 2.0f * spread * tmax_model;
    const bool illc = a11 * a22 - a12 * a12 < (a11 + a22) * (a11 + a22) * (1.0f / kCondMax);
    const bool far = kappa > (float)(prec ? kKappaMax64 : kKappaMax);
    if (far || illc) {
        if (STORE_ROW) {  // the fused kernel keeps the rows in registers: hand them over
#pragma unroll
            for (int q = 0; q < KP; ++q)
                if (q < k) {
                    const_cast<int32_t*>(a.idx)[i * k + q] = jj[q];
                    const_cast<float*>(a.sqd)[i * k + q] = sq[q];
                }
        }
        faithful_point(a, i);
        return;
    }
    const double det = A11 * A22 - A12 * A12;
    const double tr = A11 + A22;
    float2 out;
    if (det < kDetRel * tr * tr + kDetAbs) {
        out = o;
    } else {
        out.x = (float)((C1 * A22 - C2 * A12) / det + (double)o.x);
        out.y = (float)((A11 * C2 - A12 * C1) / det + (double)o.y);
    }
    reinterpret_cast<float2*>(a.xy)[i] = out;
}

template <int KP, bool TSMEM, bool HSMEM, bool FARHEAVY>
__global__ void __launch_bounds__(kReg2Threads, 1) project_reg2_kernel(ProjArgs a) {
    constexpr int PT = kReg2Threads;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int g = a.g, k = a.k;
    float2* LO = reinterpret_cast<float2*>(smem_raw);
    int* RB = reinterpret_cast<int*>(LO + g);
    float* tsm = reinterpret_cast<float*>(smem_raw + reg2_tri_offset(g));
    double* h64 = reinterpret_cast<double*>(smem_raw + reg2_hi64_offset(g));
    double* hn_s = h64 + (size_t)g * reg2_hi64_stride(a.d);  // g row norms after the rows
    if (TSMEM) {
        const int ntri = g * (g - 1) / 2;
        for (int e = tid; e < ntri; e += PT) tsm[e] = __ldg(a.T + e);
    }
    const int hs = reg2_hi64_stride(a.d);
    if (HSMEM) {  // f64 landmark rows for the far-point distances (precise_sqd)
        const int nh = g * a.d;
        for (int e = tid; e < nh; e += PT) h64[(e / a.d) * hs + e % a.d] = __ldg(a.hi64 + e);
        for (int j = tid; j < g; j += PT) hn_s[j] = __ldg(a.hn64 + j);
    }
    for (int j = tid; j < g; j += PT) {
        LO[j] = make_float2(a.lo[2 * j], a.lo[2 * j + 1]);
        RB[j] = j * (2 * g - j - 1) / 2 - j - 1;  // tri(j, b) = RB[j] + b for b > j
    }
    __syncthreads();
    const float* T = TSMEM ? tsm : a.T;
    const bool vec = (k == KP) && ((KP & 3) == 0);
    const bool vec8 = vec && (KP & 7) == 0 && rows32(a.idx, k) && rows32(a.sqd, k);
    const float tmax_model = a.tmax ? __ldg(a.tmax) : 0.0f;

    for (int64_t pos = blockIdx.x * (int64_t)PT + tid; pos < a.n; pos += (int64_t)gridDim.x * PT) {
        const int64_t i = a.perm ? (int64_t)__ldg(a.perm + pos) : pos;
        int jj[KP];
        float sq[KP];
        const int32_t* irow = a.idx + i * k;
        const float* drow = a.sqd + i * k;
        if (vec8) {
#pragma unroll
            for (int q = 0; q + 8 <= KP; q += 8) {
                int4 iv, iw;
                float4 dv, dw;
                ldg8(irow + q, iv, iw);
                ldg8(drow + q, dv, dw);
                jj[q] = iv.x; jj[q + 1] = iv.y; jj[q + 2] = iv.z; jj[q + 3] = iv.w;
                jj[q + 4] = iw.x; jj[q + 5] = iw.y; jj[q + 6] = iw.z; jj[q + 7] = iw.w;
                sq[q] = dv.x; sq[q + 1] = dv.y; sq[q + 2] = dv.z; sq[q + 3] = dv.w;
                sq[q + 4] = dw.x; sq[q + 5] = dw.y; sq[q + 6] = dw.z; sq[q + 7] = dw.w;
            }
        } else if (vec) {
#pragma unroll
            for (int q = 0; q < KP; q += 4) {
                const int4 iv = __ldg(reinterpret_cast<const int4*>(irow + q));
                const float4 dv = __ldg(reinterpret_cast<const float4*>(drow + q));
                jj[q] = iv.x; jj[q + 1] = iv.y; jj[q + 2] = iv.z; jj[q + 3] = iv.w;
                sq[q] = dv.x; sq[q + 1] = dv.y; sq[q + 2] = dv.z; sq[q + 3] = dv.w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                jj[q] = q < k ? __ldg(irow + q) : q % g;  // padding slots: valid dummy landmarks, zero weight
                sq[q] = q < k ? __ldg(drow + q) : 0.0f;
            }
        }
        reg2_point<KP, TSMEM, HSMEM, FARHEAVY, false>(a, i, jj, sq, LO, RB, T, h64, hn_s, hs, tmax_model);
    }
}

// ---------------------------------------------------------------------------
// v3 (default for k <= 16, g <= 1024): everything a pair needs that depends
// only on the landmark pair is precomputed per (hi, lo) into a g x g record
// table {T = 0.5/hd2 (or -1 = skip), g = (lo_v - lo_u)/|lo_v - lo_u|^2,
// g . lo_u} (16 MB at g = 1024, L2-resident; points are visited in BMU order
// so a warp's lanes share records).  Per pair: one 16-byte load, the weight,
// h = 1/2 + g.lo_u + (sqd_u - sqd_v) T, five FMAs.  Same fallbacks as v2.
// ---------------------------------------------------------------------------
static __global__ void pair_record_kernel(const float* __restrict__ T, const float* __restrict__ lo, int g,
                                   float4* __restrict__ rec) {
    const int64_t total = (int64_t)g * g;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int u = (int)(e / g), v = (int)(e % g);
        float4 r = make_float4(-1.0f, 0.0f, 0.0f, 0.0f);
        if (u != v) {
            const int a = min(u, v), b = max(u, v);
            const float t = __ldg(T + ((int64_t)a * (2 * g - 1 - a) >> 1) + b - a - 1);
            const float lux = lo[2 * u], luy = lo[2 * u + 1];
            const float ex = __fsub_rn(lo[2 * v], lux), ey = __fsub_rn(lo[2 * v + 1], luy);
            const float ld2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));  // as the reference forms it
            if (t >= 0.0f && ld2 >= kLd2Min) {
                const double g1 = (double)ex / (double)ld2, g2 = (double)ey / (double)ld2;
                r = make_float4(t, (float)g1, (float)g2, (float)(g1 * (double)lux + g2 * (double)luy));
            }
        }
        rec[e] = r;
    }
}

// One point of project_reg3_kernel (pair records {T, g, g.lo_u} in L2); shared
// with the record-table variant of the fused kernel (esom_fused.cuh; STORE_ROW
// and ROWS32 as in reg2_point).
template <int KP, bool STORE_ROW, bool ROWS32 = false>
__device__ __forceinline__ void reg3_point(const ProjArgs& a, int64_t i, const int (&jj)[KP], const float (&sq)[KP],
                                           const float4* __restrict__ rec, float tmax_model,
                                           const float* rows32 = nullptr, int ls32 = 0,
                                           const int32_t* inv32 = nullptr) {
    const int g = a.g, k = a.k;
    int rowb[KP];
    float sc[KP];
    float sig = 0.0f, sqk = 0.0f, sqmax = 0.0f;
#pragma unroll
    for (int q = 0; q < KP; ++q) {
        rowb[q] = jj[q] * g;
        sig += q < k ? sqrt_approx(sq[q]) : 0.0f;
        if (q == k - 1) sqk = sq[q];
        sqmax = fmaxf(sqmax, sq[q]);
    }
    // scores as in v2 (scale-free f32 expm1 form)
    sig = sig / (float)k;
    bool uniform = sig < (float)kScoreEps;
    const bool prec = 2.0f * sqmax * tmax_model > (float)kKappaMax;  // far: f64 distance paths
    count_prec(a.prec_count, prec);
    if (!uniform) {
        const float inv = 1.0f / (2.0f * sig * sig);
        const float tail = ex2_approx(-1.44269504f * sqk * inv);
        float dls[KP];
        if (prec) {  // far points: exponent differences from the reference's own d_t^2 = (f64 sqrtf(sq))^2
            const double dk = (double)__fsqrt_rn(sqk);
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                const double dq = (double)__fsqrt_rn(sq[q]);
                dls[q] = q < k ? (float)((dk * dk - dq * dq) * (double)inv) : 0.0f;
            }
        } else {
#pragma unroll
            for (int q = 0; q < KP; ++q) dls[q] = q < k ? (sqk - sq[q]) * inv : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < KP; ++q) {
            const float dl = dls[q];
            const float poly = dl * fmaf(dl, fmaf(dl, fmaf(dl, fmaf(dl, fmaf(dl, 1.0f / 720.0f, 1.0f / 120.0f),
                                                                   1.0f / 24.0f), 1.0f / 6.0f), 0.5f), 1.0f);
            sc[q] = dl < 0.3f ? poly : ex2_approx(1.44269504f * dl) - 1.0f;
            if (q == 0) uniform = ex2_approx(-1.44269504f * sq[0] * inv) - tail < (float)kScoreEps;
        }
    }
    if (uniform) {
#pragma unroll
        for (int q = 0; q < KP; ++q) sc[q] = q < k - 1 ? 1.0f : 0.0f;
    }

    float qe[KP];
    if (prec) {
        if (ROWS32)  // (d == 32, the fused kernel)
            precise_sqd_rows32<KP>(a.X + i * 32, rows32, ls32, inv32, a.hn64, jj, k, qe);
        else
            precise_sqd<KP>(a.X + i * a.d, a.d, a.hi64, a.d, jj, k, qe);
    } else {
#pragma unroll
        for (int q = 0; q < KP; ++q) qe[q] = sq[q];
    }
    float a11 = 0.0f, a12 = 0.0f, a22 = 0.0f, c1 = 0.0f, c2 = 0.0f;
    // all pairs u < v fully unrolled; slot KP-1 has score 0 (see project_reg2_kernel);
    // skipped pairs' records are (-1, 0, 0, 0): g = 0, so they add nothing
#pragma unroll
    for (int u = 0; u < KP - 2; ++u) {
#pragma unroll
        for (int v = u + 1; v < KP - 1; ++v) {
            const float w = sc[u] * sc[v];
            const float4 rc = __ldg(rec + rowb[u] + jj[v]);
            const float h = fmaf(qe[u] - qe[v], rc.x, 0.5f + rc.w);  // dnum/hd2 + g . lo_u
            const float wg1 = w * rc.y, wg2 = w * rc.z;
            a11 = fmaf(wg1, rc.y, a11);
            a12 = fmaf(wg1, rc.z, a12);
            a22 = fmaf(wg2, rc.z, a22);
            c1 = fmaf(wg1, h, c1);
            c2 = fmaf(wg2, h, c2);
        }
    }
    double A11 = a11, A12 = a12, A22 = a22, C1 = c1, C2 = c2;
    float spread = sqmax;  // prec: the error of qe_u - qe_v scales with the offsets' spread
    if (prec) {
        spread = 0.0f;
#pragma unroll
        for (int q = 0; q < KP; ++q) spread = fmaxf(spread, fabsf(qe[q]));
    }
    const float kappa = 2.0f * spread * tmax_model;  // (see reg2_point)
    const bool illc = a11 * a22 - a12 * a12 < (a11 + a22) * (a11 + a22) * (1.0f / kCondMax);
    const bool far = kappa > (float)(prec ? kKappaMax64 : kKappaMax);
    if (far || illc) {
        if (STORE_ROW) {  // the fused kernel keeps the rows in registers: hand them over
#pragma unroll
            for (int q = 0; q < KP; ++q)
                if (q < k) {
                    const_cast<int32_t*>(a.idx)[i * k + q] = jj[q];
                    const_cast<float*>(a.sqd)[i * k + q] = sq[q];
                }
        }
        faithful_point(a, i);
        return;
    }
    const double det = A11 * A22 - A12 * A12;
    const double tr = A11 + A22;
    float2 out;
    if (det < kDetRel * tr * tr + kDetAbs) {
        out = make_float2(__ldg(a.lo + 2 * jj[0]), __ldg(a.lo + 2 * jj[0] + 1));
    } else {
        out.x = (float)((C1 * A22 - C2 * A12) / det);
        out.y = (float)((A11 * C2 - A12 * C1) / det);
    }
    reinterpret_cast<float2*>(a.xy)[i] = out;
}

template <int KP>
__global__ void __launch_bounds__(kRegThreads, 1) project_reg3_kernel(ProjArgs a) {
    constexpr int PT = kRegThreads;
    const int tid = threadIdx.x;
    const int k = a.k;
    const bool vec = (k == KP) && ((KP & 3) == 0);
    const bool vec8 = vec && (KP & 7) == 0 && rows32(a.idx, k) && rows32(a.sqd, k);
    const float4* __restrict__ rec = a.rec;
    const float tmax_model = a.tmax ? __ldg(a.tmax) : 0.0f;

    for (int64_t pos = blockIdx.x * (int64_t)PT + tid; pos < a.n; pos += (int64_t)gridDim.x * PT) {
        const int64_t i = a.perm ? (int64_t)__ldg(a.perm + pos) : pos;
        int jj[KP];
        float sq[KP];
        const int32_t* irow = a.idx + i * k;
        const float* drow = a.sqd + i * k;
        if (vec8) {
#pragma unroll
            for (int q = 0; q + 8 <= KP; q += 8) {
                int4 iv, iw;
                float4 dv, dw;
                ldg8(irow + q, iv, iw);
                ldg8(drow + q, dv, dw);
                jj[q] = iv.x; jj[q + 1] = iv.y; jj[q + 2] = iv.z; jj[q + 3] = iv.w;
                jj[q + 4] = iw.x; jj[q + 5] = iw.y; jj[q + 6] = iw.z; jj[q + 7] = iw.w;
                sq[q] = dv.x; sq[q + 1] = dv.y; sq[q + 2] = dv.z; sq[q + 3] = dv.w;
                sq[q + 4] = dw.x; sq[q + 5] = dw.y; sq[q + 6] = dw.z; sq[q + 7] = dw.w;
            }
        } else if (vec) {
#pragma unroll
            for (int q = 0; q < KP; q += 4) {
                const int4 iv = __ldg(reinterpret_cast<const int4*>(irow + q));
                const float4 dv = __ldg(reinterpret_cast<const float4*>(drow + q));
                jj[q] = iv.x; jj[q + 1] = iv.y; jj[q + 2] = iv.z; jj[q + 3] = iv.w;
                sq[q] = dv.x; sq[q + 1] = dv.y; sq[q + 2] = dv.z; sq[q + 3] = dv.w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                jj[q] = q < k ? __ldg(irow + q) : 0;  // padding slots: zero weight (diagonal record)
                sq[q] = q < k ? __ldg(drow + q) : 0.0f;
            }
        }
        reg3_point<KP, false>(a, i, jj, sq, rec, tmax_model);
    }
}

template <int KP, bool TSMEM, bool HSMEM>
int launch_project_reg(ProjArgs a, size_t smem, cudaStream_t st) {
    auto kern = a.far_heavy ? project_reg2_kernel<KP, TSMEM, HSMEM, true> : project_reg2_kernel<KP, TSMEM, HSMEM, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kReg2Threads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t nblk = (a.n + kReg2Threads - 1) / kReg2Threads;
    int64_t grid = (int64_t)esom_host::num_sms() * per_sm;
    if (grid > nblk) grid = nblk;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kReg2Threads, smem, st>>>(a);
    return esom_host::cuda_check("project_reg_kernel");
}

template <int KP>
int launch_project_t(ProjArgs a, cudaStream_t st) {
    if constexpr (KP <= 16) {
        if (a.rec) {
            auto kern = project_reg3_kernel<KP>;
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRegThreads, 0);
            if (per_sm < 1) per_sm = 1;
            const int64_t nblk = (a.n + kRegThreads - 1) / kRegThreads;
            int64_t grid = (int64_t)esom_host::num_sms() * per_sm;
            if (grid > nblk) grid = nblk;
            if (grid < 1) grid = 1;
            kern<<<(unsigned)grid, kRegThreads, 0, st>>>(a);
            return esom_host::cuda_check("project_reg3_kernel");
        }
        const size_t cap = (size_t)esom_host::max_smem_optin() - 1024;
        const size_t with_t = reg2_hi64_offset(a.g);
        const size_t with_h = with_t + (size_t)a.g * (reg2_hi64_stride(a.d) + 1) * 8;
        if (with_h <= cap) return launch_project_reg<KP, true, true>(a, with_h, st);
        if (with_t <= cap) return launch_project_reg<KP, true, false>(a, with_t, st);
        return launch_project_reg<KP, false, false>(a, reg2_tri_offset(a.g), st);
    }
    constexpr int kProjThreads = proj_threads<KP>();
    const size_t base = (size_t)a.g * 12 + (size_t)KP * kProjThreads * 12 + 64;
    const size_t tbytes = (size_t)a.g * (a.g - 1) / 2 * 4;
    const size_t cap = (size_t)esom_host::max_smem_optin() - 1024;
    if (base > cap) return esom_host::set_err(ESOM_ERR_UNSUPPORTED, "g too large for the projection kernel%s", "");
    a.t_smem = base + tbytes <= cap ? 1 : 0;
    const size_t smem = base + (a.t_smem ? tbytes : 0);
    auto kern = project_fast_kernel<KP>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kProjThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t nblk = (a.n + kProjThreads - 1) / kProjThreads;
    int64_t grid = (int64_t)esom_host::num_sms() * per_sm;
    if (grid > nblk) grid = nblk;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kProjThreads, smem, st>>>(a);
    return esom_host::cuda_check("project_fast_kernel");
}

}  // namespace esom
