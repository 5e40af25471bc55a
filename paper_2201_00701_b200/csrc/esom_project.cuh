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
// (far outliers, where that error would matter) are redone with the exact
// x-based f64 pair loop.  Checked against the reference to <= 1e-4 x extent.
#pragma once
#include "esom_common.cuh"
#include "esom_host.h"
#include "esom_scan_args.h"

namespace esom {

// threads per CTA: 256 for k <= 16 (per-thread rows fit next to a smem pair
// table), fewer for larger k so the per-thread rows still fit
template <int KP>
__host__ __device__ constexpr int proj_threads() { return KP <= 16 ? 256 : (KP <= 32 ? 128 : 64); }

__device__ __forceinline__ int64_t tri_index(int a, int b, int g) {
    // a < b; row a holds pairs (a, a+1..g-1)
    return (int64_t)a * (2 * (int64_t)g - a - 1) / 2 + (b - a - 1);
}

// Exact f64 pair accumulation from x and the landmark rows (outlier path).
static __device__ __noinline__ void pairs_exact_f64(const float* __restrict__ x, int d,
                                                    const float* __restrict__ hi, const float* __restrict__ lo,
                                                    int k, const int* J, const double* S, int stride, double* out5) {
    double a11 = 0.0, a12 = 0.0, a22 = 0.0, c1 = 0.0, c2 = 0.0;
    for (int u = 0; u < k; ++u) {
        const double su = S[u * stride];
        if (su <= 0.0) continue;
        const int ju = J[u * stride];
        const float* hu = hi + (int64_t)ju * d;
        for (int v = u + 1; v < k; ++v) {
            const double w = su * S[v * stride];
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
            const double ex = (double)lo[2 * jv] - (double)lo[2 * ju];
            const double ey = (double)lo[2 * jv + 1] - (double)lo[2 * ju + 1];
            const double ld2 = ex * ex + ey * ey;
            if (ld2 < kPairEps) continue;
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

template <int KP>
__global__ void __launch_bounds__(proj_threads<KP>()) project_fast_kernel(ProjArgs a) {
    constexpr int kProjThreads = proj_threads<KP>();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int g = a.g, k = a.k;
    // layout: lo64 [g] double2 | J [KP][T] int | Q [KP][T] double | S [KP][T] double | (T table)
    double2* lo64 = reinterpret_cast<double2*>(smem_raw);
    int* J = reinterpret_cast<int*>(lo64 + g);
    double* Q = reinterpret_cast<double*>(J + KP * kProjThreads);
    double* S = Q + KP * kProjThreads;
    const float* Ts = a.T;
    if (a.t_smem) {
        float* tsm = reinterpret_cast<float*>(S + KP * kProjThreads);
        const int64_t ntri = (int64_t)g * (g - 1) / 2;
        for (int64_t e = tid; e < ntri; e += kProjThreads) tsm[e] = a.T[e];
        Ts = tsm;
    }
    for (int j = tid; j < g; j += kProjThreads)
        lo64[j] = make_double2((double)a.lo[2 * j], (double)a.lo[2 * j + 1]);
    __syncthreads();

    for (int64_t i = blockIdx.x * (int64_t)kProjThreads + tid; i < a.n; i += (int64_t)gridDim.x * kProjThreads) {
        const int32_t* irow = a.idx + i * k;
        const float* drow = a.sqd + i * k;
        // scores (f64; ref: projection.py:38-59)
        double sigma = 0.0, dk = 0.0;
        for (int q = 0; q < k; ++q) {
            const float sq = __ldg(drow + q);
            const double dq = (double)__fsqrt_rn(sq);
            sigma += dq;
            J[q * kProjThreads + tid] = __ldg(irow + q);
            Q[q * kProjThreads + tid] = (double)sq;
            S[q * kProjThreads + tid] = dq;  // distances for now
            dk = dq;
        }
        sigma /= (double)k;
        bool uniform = sigma < kScoreEps;
        if (!uniform) {
            const double inv = -1.0 / (2.0 * sigma * sigma);
            const double tail = exp(dk * dk * inv);
            for (int q = 0; q < k; ++q) {
                const double dq = S[q * kProjThreads + tid];
                const double v = exp(dq * dq * inv) - tail;
                S[q * kProjThreads + tid] = v > 0.0 ? v : 0.0;
                if (q == 0) uniform = v < kScoreEps;
            }
        }
        if (uniform)
            for (int q = 0; q < k; ++q) S[q * kProjThreads + tid] = q == k - 1 ? 0.0 : 1.0;

        double a11 = 0.0, a12 = 0.0, a22 = 0.0, c1 = 0.0, c2 = 0.0;
        double kappa = 0.0;
        for (int u = 0; u + 1 < k; ++u) {
            const double su = S[u * kProjThreads + tid];
            if (!(su > 0.0)) continue;
            const int ju = J[u * kProjThreads + tid];
            const double squ = Q[u * kProjThreads + tid];
            const double2 lu = lo64[ju];
            for (int v = u + 1; v < k; ++v) {
                const double w = su * S[v * kProjThreads + tid];
                if (!(w > 0.0)) continue;
                const int jv = J[v * kProjThreads + tid];
                const float tv = ju < jv ? Ts[tri_index(ju, jv, g)] : Ts[tri_index(jv, ju, g)];
                if (tv < 0.0f) continue;  // hd2 < 1e-12: the reference skips the pair
                const double2 lv = lo64[jv];
                const double ex = lv.x - lu.x, ey = lv.y - lu.y;
                const double ld2 = fma(ex, ex, ey * ey);
                if (ld2 < kPairEps) continue;
                const double t = (double)tv;
                const double sqv = Q[v * kProjThreads + tid];
                kappa = fmax(kappa, (squ + sqv) * t);
                const double r = __drcp_rn(ld2);
                const double g1 = ex * r, g2 = ey * r;
                const double h = fma(squ - sqv, t, 0.5) + fma(g1, lu.x, g2 * lu.y);
                const double wg1 = w * g1, wg2 = w * g2, wh = w * h;
                a11 = fma(wg1, g1, a11);
                a12 = fma(wg1, g2, a12);
                a22 = fma(wg2, g2, a22);
                c1 = fma(wh, g1, c1);
                c2 = fma(wh, g2, c2);
            }
        }
        if (kappa > kKappaMax) {
            double o5[5];
            pairs_exact_f64(a.X + i * a.d, a.d, a.hi, a.lo, k, J + tid, S + tid, kProjThreads, o5);
            a11 = o5[0];
            a12 = o5[1];
            a22 = o5[2];
            c1 = o5[3];
            c2 = o5[4];
        }
        const double det = a11 * a22 - a12 * a12;
        const double tr = a11 + a22;
        float2 out;
        if (det < kDetRel * tr * tr + kDetAbs) {
            const int j0 = J[tid];
            out = make_float2(a.lo[2 * j0], a.lo[2 * j0 + 1]);
        } else {
            out.x = (float)((c1 * a22 - c2 * a12) / det);
            out.y = (float)((a11 * c2 - a12 * c1) / det);
        }
        reinterpret_cast<float2*>(a.xy)[i] = out;
    }
}

template <int KP>
int launch_project_t(ProjArgs a, cudaStream_t st) {
    constexpr int kProjThreads = proj_threads<KP>();
    const size_t base = (size_t)a.g * 16 + (size_t)KP * kProjThreads * (4 + 8 + 8);
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
