// esom_faithful.cuh -- the reference's scores and projection op for op
// (SURVEY.md Appendix A.2/A.3), shared by the faithful kernels
// (esom_kernels.cu: scores_kernel, project_kernel) and the fast projection
// kernels' fallback for ill-conditioned systems (esom_project.cuh).
#pragma once
#include <stdint.h>

#include "esom_common.cuh"

namespace esom {

// Scores (ref: projection.py:38-59).  numba's float(f32) stays f32, so the
// root is sqrtf, widened; the rest is f64.  `exp` is CUDA's (<= 1 ulp from
// glibc); everything else is correctly rounded like the reference.
template <typename Get>
__device__ __forceinline__ void score_row_dev(int k, Get sqd_at, double* out) {
    double sigma = 0.0;
    for (int t = 0; t < k; ++t) {
        out[t] = (double)__fsqrt_rn(sqd_at(t));
        sigma = __dadd_rn(sigma, out[t]);
    }
    sigma = __ddiv_rn(sigma, (double)k);
    if (sigma < kScoreEps) {
        for (int t = 0; t < k - 1; ++t) out[t] = 1.0;
        out[k - 1] = 0.0;
        return;
    }
    const double denom = __dmul_rn(__dmul_rn(2.0, sigma), sigma);
    const double tail = exp(__ddiv_rn(-__dmul_rn(out[k - 1], out[k - 1]), denom));
    for (int t = 0; t < k; ++t) {
        const double v = __dsub_rn(exp(__ddiv_rn(-__dmul_rn(out[t], out[t]), denom)), tail);
        out[t] = v > 0.0 ? v : 0.0;
    }
    if (out[0] < kScoreEps) {
        for (int t = 0; t < k - 1; ++t) out[t] = 1.0;
        out[k - 1] = 0.0;
    }
}

// ---------------------------------------------------------------------------
// Faithful projection (ref: projection.py:68-121), the mixed f32/f64 typing
// of SURVEY Appendix A.3 with every operation separately rounded.
// ---------------------------------------------------------------------------
// d <= 32: the same operations in the same order, with x - l_u (formed by the
// reference inside the pair loop; it does not depend on v) and l_u held in
// registers once per u and l_v read 8 dimensions per 256-bit load.
// Bit-identical to project_row_faithful.
__device__ __forceinline__ void project_row_faithful32(const float* __restrict__ x, const float* __restrict__ hi,
                                                       const float* __restrict__ lo, const int32_t* __restrict__ nbr,
                                                       const double* __restrict__ sc, int d, int k, float* out) {
    float xr[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) xr[c] = c < d ? __ldg(x + c) : 0.0f;
    double a11 = 0.0, a12 = 0.0, a22 = 0.0, c1 = 0.0, c2 = 0.0;
    for (int u = 0; u < k; ++u) {
        const double su = __ldg(sc + u);
        if (su <= 0.0) continue;
        const int ju = __ldg(nbr + u);
        const float* hu = hi + (int64_t)ju * d;
        float lu[32], xu[32];
#pragma unroll
        for (int c0 = 0; c0 < 32; c0 += 8) {
            float4 p0 = make_float4(0.f, 0.f, 0.f, 0.f), p1 = p0;
            if (c0 < d) ldg8(hu + c0, p0, p1);
            lu[c0] = p0.x; lu[c0 + 1] = p0.y; lu[c0 + 2] = p0.z; lu[c0 + 3] = p0.w;
            lu[c0 + 4] = p1.x; lu[c0 + 5] = p1.y; lu[c0 + 6] = p1.z; lu[c0 + 7] = p1.w;
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) xu[c] = __fsub_rn(xr[c], lu[c]);
        const float lux = __ldg(lo + 2 * ju), luy = __ldg(lo + 2 * ju + 1);
        for (int v = u + 1; v < k; ++v) {
            const double w = __dmul_rn(su, __ldg(sc + v));
            if (w <= 0.0) continue;
            const int jv = __ldg(nbr + v);
            const float* hv = hi + (int64_t)jv * d;
            double hd2 = 0.0, dnum = 0.0;
#pragma unroll
            for (int c0 = 0; c0 < 32; c0 += 8) {
                if (c0 < d) {
                    float4 p0, p1;
                    ldg8(hv + c0, p0, p1);
                    const float lv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float e = __fsub_rn(lv[q], lu[c0 + q]);
                        hd2 = __dadd_rn(hd2, (double)__fmul_rn(e, e));
                        dnum = __dadd_rn(dnum, (double)__fmul_rn(xu[c0 + q], e));
                    }
                }
            }
            if (hd2 < kPairEps) continue;
            const float ex = __fsub_rn(__ldg(lo + 2 * jv), lux);
            const float ey = __fsub_rn(__ldg(lo + 2 * jv + 1), luy);
            const float ld2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
            if ((double)ld2 < kPairEps) continue;
            const float g1 = __fdiv_rn(ex, ld2);
            const float g2 = __fdiv_rn(ey, ld2);
            const double h = __dadd_rn(__dadd_rn(__ddiv_rn(dnum, hd2), (double)__fmul_rn(g1, lux)),
                                       (double)__fmul_rn(g2, luy));
            const double G1 = g1, G2 = g2;
            a11 = __dadd_rn(a11, __dmul_rn(__dmul_rn(w, G1), G1));
            a12 = __dadd_rn(a12, __dmul_rn(__dmul_rn(w, G1), G2));
            a22 = __dadd_rn(a22, __dmul_rn(__dmul_rn(w, G2), G2));
            c1 = __dadd_rn(c1, __dmul_rn(__dmul_rn(w, h), G1));
            c2 = __dadd_rn(c2, __dmul_rn(__dmul_rn(w, h), G2));
        }
    }
    const double det = __dsub_rn(__dmul_rn(a11, a22), __dmul_rn(a12, a12));
    const double tr = __dadd_rn(a11, a22);
    if (det < __dadd_rn(__dmul_rn(__dmul_rn(kDetRel, tr), tr), kDetAbs)) {
        const int nearest = __ldg(nbr);
        out[0] = __ldg(lo + 2 * nearest);
        out[1] = __ldg(lo + 2 * nearest + 1);
    } else {
        out[0] = (float)__ddiv_rn(__dsub_rn(__dmul_rn(c1, a22), __dmul_rn(c2, a12)), det);
        out[1] = (float)__ddiv_rn(__dsub_rn(__dmul_rn(a11, c2), __dmul_rn(a12, c1)), det);
    }
}

// Any d % 8 == 0 with 32-byte rows: the generic loop with x, l_u and l_v read
// 8 dimensions per 256-bit load (same operations, same order).
__device__ __forceinline__ void project_row_faithful_v8(const float* __restrict__ x, const float* __restrict__ hi,
                                                        const float* __restrict__ lo, const int32_t* __restrict__ nbr,
                                                        const double* __restrict__ sc, int d, int k, float* out) {
    double a11 = 0.0, a12 = 0.0, a22 = 0.0, c1 = 0.0, c2 = 0.0;
    for (int u = 0; u < k; ++u) {
        const double su = __ldg(sc + u);
        if (su <= 0.0) continue;
        const int ju = __ldg(nbr + u);
        const float* hu = hi + (int64_t)ju * d;
        const float lux = __ldg(lo + 2 * ju), luy = __ldg(lo + 2 * ju + 1);
        for (int v = u + 1; v < k; ++v) {
            const double w = __dmul_rn(su, __ldg(sc + v));
            if (w <= 0.0) continue;
            const int jv = __ldg(nbr + v);
            const float* hv = hi + (int64_t)jv * d;
            double hd2 = 0.0, dnum = 0.0;
            for (int c0 = 0; c0 < d; c0 += 8) {
                float4 x0, x1, u0, u1, v0, v1;
                ldg8(x + c0, x0, x1);
                ldg8(hu + c0, u0, u1);
                ldg8(hv + c0, v0, v1);
                const float xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
                const float us[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
                const float vs[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float e = __fsub_rn(vs[q], us[q]);
                    hd2 = __dadd_rn(hd2, (double)__fmul_rn(e, e));
                    dnum = __dadd_rn(dnum, (double)__fmul_rn(__fsub_rn(xs[q], us[q]), e));
                }
            }
            if (hd2 < kPairEps) continue;
            const float ex = __fsub_rn(__ldg(lo + 2 * jv), lux);
            const float ey = __fsub_rn(__ldg(lo + 2 * jv + 1), luy);
            const float ld2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
            if ((double)ld2 < kPairEps) continue;
            const float g1 = __fdiv_rn(ex, ld2);
            const float g2 = __fdiv_rn(ey, ld2);
            const double h = __dadd_rn(__dadd_rn(__ddiv_rn(dnum, hd2), (double)__fmul_rn(g1, lux)),
                                       (double)__fmul_rn(g2, luy));
            const double G1 = g1, G2 = g2;
            a11 = __dadd_rn(a11, __dmul_rn(__dmul_rn(w, G1), G1));
            a12 = __dadd_rn(a12, __dmul_rn(__dmul_rn(w, G1), G2));
            a22 = __dadd_rn(a22, __dmul_rn(__dmul_rn(w, G2), G2));
            c1 = __dadd_rn(c1, __dmul_rn(__dmul_rn(w, h), G1));
            c2 = __dadd_rn(c2, __dmul_rn(__dmul_rn(w, h), G2));
        }
    }
    const double det = __dsub_rn(__dmul_rn(a11, a22), __dmul_rn(a12, a12));
    const double tr = __dadd_rn(a11, a22);
    if (det < __dadd_rn(__dmul_rn(__dmul_rn(kDetRel, tr), tr), kDetAbs)) {
        const int nearest = __ldg(nbr);
        out[0] = __ldg(lo + 2 * nearest);
        out[1] = __ldg(lo + 2 * nearest + 1);
    } else {
        out[0] = (float)__ddiv_rn(__dsub_rn(__dmul_rn(c1, a22), __dmul_rn(c2, a12)), det);
        out[1] = (float)__ddiv_rn(__dsub_rn(__dmul_rn(a11, c2), __dmul_rn(a12, c1)), det);
    }
}

static __device__ __noinline__ void project_row_faithful(const float* __restrict__ x, const float* __restrict__ hi,
                                     const float* __restrict__ lo, const int32_t* __restrict__ nbr,
                                     const double* __restrict__ sc, int d, int k, float* out) {
    double a11 = 0.0, a12 = 0.0, a22 = 0.0, c1 = 0.0, c2 = 0.0;
    for (int u = 0; u < k; ++u) {
        const double su = sc[u];
        if (su <= 0.0) continue;
        const int ju = nbr[u];
        const float* hu = hi + (int64_t)ju * d;
        for (int v = u + 1; v < k; ++v) {
            const double w = __dmul_rn(su, sc[v]);
            if (w <= 0.0) continue;
            const int jv = nbr[v];
            const float* hv = hi + (int64_t)jv * d;
            double hd2 = 0.0, dnum = 0.0;
            for (int c = 0; c < d; ++c) {
                const float lu = hu[c];
                const float e = __fsub_rn(hv[c], lu);
                hd2 = __dadd_rn(hd2, (double)__fmul_rn(e, e));
                dnum = __dadd_rn(dnum, (double)__fmul_rn(__fsub_rn(x[c], lu), e));
            }
            if (hd2 < kPairEps) continue;
            const float lux = lo[2 * ju], luy = lo[2 * ju + 1];
            const float ex = __fsub_rn(lo[2 * jv], lux);
            const float ey = __fsub_rn(lo[2 * jv + 1], luy);
            const float ld2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
            if ((double)ld2 < kPairEps) continue;
            const float g1 = __fdiv_rn(ex, ld2);
            const float g2 = __fdiv_rn(ey, ld2);
            const double h = __dadd_rn(__dadd_rn(__ddiv_rn(dnum, hd2), (double)__fmul_rn(g1, lux)),
                                       (double)__fmul_rn(g2, luy));
            const double G1 = g1, G2 = g2;
            a11 = __dadd_rn(a11, __dmul_rn(__dmul_rn(w, G1), G1));
            a12 = __dadd_rn(a12, __dmul_rn(__dmul_rn(w, G1), G2));
            a22 = __dadd_rn(a22, __dmul_rn(__dmul_rn(w, G2), G2));
            c1 = __dadd_rn(c1, __dmul_rn(__dmul_rn(w, h), G1));
            c2 = __dadd_rn(c2, __dmul_rn(__dmul_rn(w, h), G2));
        }
    }
    const double det = __dsub_rn(__dmul_rn(a11, a22), __dmul_rn(a12, a12));
    const double tr = __dadd_rn(a11, a22);
    if (det < __dadd_rn(__dmul_rn(__dmul_rn(kDetRel, tr), tr), kDetAbs)) {
        const int nearest = nbr[0];
        out[0] = lo[2 * nearest];
        out[1] = lo[2 * nearest + 1];
    } else {
        out[0] = (float)__ddiv_rn(__dsub_rn(__dmul_rn(c1, a22), __dmul_rn(c2, a12)), det);
        out[1] = (float)__ddiv_rn(__dsub_rn(__dmul_rn(a11, c2), __dmul_rn(a12, c1)), det);
    }
}



}  // namespace esom
