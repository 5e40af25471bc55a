// esom_scan.cuh -- the fused scan kernel (distance + top-k [+ scores +
// projection | + BMU statistics]) and its launcher template.  Instantiated
// per (DC, KP, MODE) in inst/*.cu so the library builds in parallel.
#pragma once
#include "esom_common.cuh"
#include "esom_host.h"
#include "esom_knn.cuh"
#include "esom_scan_args.h"

namespace esom {


// ---------------------------------------------------------------------------
// Fused scan kernel.
//
// MODE 0: k-NN only -> idx/sqd rows.
// MODE 1: embed -> scores + fast projection -> xy; optional batch-SOM stats
//         (BMU = idx[0]) and the quantization-error sum.
//
// Fast projection ("law of cosines"): for a kept pair,
//   dnum = (x - h_u).(h_v - h_u) = (sqd_u - sqd_v + hd2) / 2
// so h = dnum/hd2 + g.lo_u = 0.5 + (sqd_u - sqd_v) * T[u,v] + g.lo_u with
// T = 0.5/hd2 from pair_table_kernel.  Its absolute error is bounded by
// ~u*sqrt(d)*(sqd_u + sqd_v)/hd2; points whose kappa = max (sqd_u+sqd_v)/hd2
// exceeds kKappaMax (far outliers) are redone with the exact f64 pair loop.
// ---------------------------------------------------------------------------


template <int DC>
__device__ __forceinline__ bool load_x(const float* __restrict__ X, int64_t i, int64_t n, int d, int c0,
                                       float (&x)[DC]) {
    bool bad = false;
    const float* row = X + i * d;
#pragma unroll
    for (int c = 0; c < DC; ++c) {
        const int cc = c0 + c;
        float v = 0.0f;
        if (i < n && cc < d) {
            v = __ldg(row + cc);
            bad |= !finite_f(v);
        }
        x[c] = v;
    }
    return bad;
}

// Exact (f64, x-based) pair accumulation for one point: used for outliers.
static __device__ __noinline__ void pairs_exact(const float* __restrict__ X, int64_t i, int d, const float* __restrict__ hi,
                            const float* __restrict__ lo, int k, const int* sj, const float* ss, int tid,
                            double& a11, double& a12, double& a22, double& c1, double& c2) {
    a11 = a12 = a22 = c1 = c2 = 0.0;
    const float* x = X + i * d;
    for (int u = 0; u < k; ++u) {
        const float su = ss[u * kThreads + tid];
        if (su <= 0.0f) continue;
        const int ju = sj[u * kThreads + tid];
        const float* hu = hi + (int64_t)ju * d;
        for (int v = u + 1; v < k; ++v) {
            const float sv = ss[v * kThreads + tid];
            const double w = (double)su * (double)sv;
            if (!(w > 0.0)) continue;
            const int jv = sj[v * kThreads + tid];
            const float* hv = hi + (int64_t)jv * d;
            double hd2 = 0.0, hd2f = 0.0, dnum = 0.0;
            for (int c = 0; c < d; ++c) {
                const double hu_c = hu[c];
                const double e = (double)hv[c] - hu_c;
                const float ef = __fsub_rn(hv[c], hu[c]);
                hd2f = __dadd_rn(hd2f, (double)__fmul_rn(ef, ef));
                hd2 = fma(e, e, hd2);
                dnum = fma((double)x[c] - hu_c, e, dnum);
            }
            if (hd2f < kPairEps) continue;
            const float lux = lo[2 * ju], luy = lo[2 * ju + 1];
            const float ex = __fsub_rn(lo[2 * jv], lux);
            const float ey = __fsub_rn(lo[2 * jv + 1], luy);
            const float ld2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
            if ((double)ld2 < kPairEps) continue;
            const double G1 = (double)ex / (double)ld2, G2 = (double)ey / (double)ld2;
            const double h = dnum / hd2 + G1 * (double)lux + G2 * (double)luy;
            const double wg1 = w * G1, wg2 = w * G2, wh = w * h;
            a11 = fma(wg1, G1, a11);
            a12 = fma(wg1, G2, a12);
            a22 = fma(wg2, G2, a22);
            c1 = fma(wh, G1, c1);
            c2 = fma(wh, G2, c2);
        }
    }
}

template <int DC, int KP, int MODE>
__global__ void __launch_bounds__(kThreads) scan_kernel(ScanArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[2];  // TMA completion barriers
    const int tid = threadIdx.x;
    const int tile_floats = a.dp * kTile;
    const uint32_t tile_bytes = (uint32_t)tile_floats * 4u;
    const int nbuf = a.res_tiles ? a.res_tiles : 2;
    float* tiles = reinterpret_cast<float*>(smem_raw);
    float* cbuf = tiles + (size_t)nbuf * tile_floats;              // [32][kThreads] candidates
    // MODE 1 per-thread neighbour rows [KP][kThreads], aliasing cbuf (the
    // candidate rows are dead once the tile loop of a point block is done)
    int* sj = reinterpret_cast<int*>(cbuf);
    float* ssq = reinterpret_cast<float*>(sj + KP * kThreads);
    float* ssc = ssq + KP * kThreads;

    const f2 nz = f2_pack(a.nz, a.nz);
    const bool stream = a.res_tiles == 0;
    uint32_t uses0 = 0, uses1 = 0;

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (!stream) {
        if (tid == 0) {
            mbar_expect_tx(&bars[0], tile_bytes * (uint32_t)a.ntiles);
            for (int t = 0; t < a.ntiles; ++t)
                tma_bulk_g2s(tiles + (size_t)t * tile_floats, a.Lt + (size_t)t * tile_floats, tile_bytes, &bars[0]);
        }
        mbar_wait(&bars[0], 0);
    }

    const int64_t nblk = (a.n + kThreads - 1) / kThreads;
    bool bad = false;
    double qe_local = 0.0;
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int64_t i = blk * kThreads + tid;
        float x[DC];
        if (a.nch == 1) bad |= load_x<DC>(a.X, i, a.n, a.d, 0, x);

        float td[KP];
        int ti[KP];
        topk_init<KP>(td, ti, a.k, a.g);
        const int off = KP - a.k;  // live slots are [off, KP)
        if (stream && tid == 0) {
            // prefetch tiles 0 and 1 of this block's pass
            for (int b = 0; b < 2 && b < a.ntiles; ++b) {
                mbar_expect_tx(&bars[b], tile_bytes);
                tma_bulk_g2s(tiles + (size_t)b * tile_floats, a.Lt + (size_t)b * tile_floats, tile_bytes, &bars[b]);
            }
        }
        for (int t = 0; t < a.ntiles; ++t) {
            const float* tl;
            if (stream) {
                const int b = t & 1;
                uint32_t& u = b ? uses1 : uses0;
                mbar_wait(&bars[b], u & 1u);
                ++u;
                tl = tiles + (size_t)b * tile_floats;
            } else {
                tl = tiles + (size_t)t * tile_floats;
            }
            f2 acc[16];
            for (int ch = 0; ch < a.nch; ++ch) {
                if (a.nch > 1) bad |= load_x<DC>(a.X, i, a.n, a.d, ch * DC, x);
                tile_accumulate<DC>(x, tl + ch * DC * kTile, nz, acc, ch == 0);
            }
            topk_tile<KP>(td, ti, acc, t * kTile, a.k, cbuf, tid);
            if (stream) {
                __syncthreads();  // everyone done with buffer (t & 1)
                if (tid == 0 && t + 2 < a.ntiles) {
                    const int b = t & 1;
                    fence_proxy_async();
                    mbar_expect_tx(&bars[b], tile_bytes);
                    tma_bulk_g2s(tiles + (size_t)b * tile_floats, a.Lt + (size_t)(t + 2) * tile_floats, tile_bytes,
                                 &bars[b]);
                }
            }
        }

        const bool valid = i < a.n;
        if (MODE == 0) {
            if (valid) {
                int32_t* oi = a.out_idx + i * a.k;
                float* od = a.out_sqd + i * a.k;
#pragma unroll
                for (int q = 0; q < KP; ++q) {
                    if (q >= off) {
                        oi[q - off] = ti[q];
                        od[q - off] = td[q];
                    }
                }
            }
            continue;
        }

        // ---------------- MODE 1/2: BMU statistics ----------------
        const int k = a.k;
        float d0 = td[KP - 1];
        int b0 = ti[KP - 1];
#pragma unroll
        for (int q = KP - 1; q >= 0; --q) {
            if (q >= off) {
                d0 = td[q];
                b0 = ti[q];
            }
        }
        if (valid && a.qe_sum) qe_local += (double)d0;
        if (valid && a.bmu) a.bmu[i] = b0;
        if (valid && a.accS) {
            const int b = b0;
            atomicAdd(a.accC + b, 1.0);
            if (a.nch == 1) {
#pragma unroll
                for (int c = 0; c < DC; ++c)
                    if (c < a.d) atomicAdd(a.accS + (int64_t)b * a.d + c, (double)x[c]);
            } else {
                for (int c = 0; c < a.d; ++c) atomicAdd(a.accS + (int64_t)b * a.d + c, (double)a.X[i * a.d + c]);
            }
        }
        if (MODE == 2) continue;
        // ---------------- MODE 1: scores + projection ----------------
        // scores (f64 like the reference; ref: projection.py:38-59), parked in
        // smem with the neighbour rows: [q][kThreads], q = rank 0..k-1
        {
            double sigma = 0.0;
            const double dk = (double)__fsqrt_rn(td[KP - 1]);
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                if (q >= off) {
                    sigma += (double)__fsqrt_rn(td[q]);
                    sj[(q - off) * kThreads + tid] = ti[q];
                    ssq[(q - off) * kThreads + tid] = td[q];
                }
            }
            sigma /= (double)k;
            bool uniform = sigma < kScoreEps;
            if (!uniform) {
                const double inv = -1.0 / (2.0 * sigma * sigma);
                const double tail = exp(dk * dk * inv);
#pragma unroll
                for (int q = 0; q < KP; ++q) {
                    if (q >= off) {
                        const double dq = (double)__fsqrt_rn(td[q]);
                        const double v = exp(dq * dq * inv) - tail;
                        const float sv = v > 0.0 ? (float)v : 0.0f;
                        ssc[(q - off) * kThreads + tid] = sv;
                        if (q == off) uniform = v < kScoreEps;
                    }
                }
            }
            if (uniform) {
                for (int q = 0; q < k; ++q) ssc[q * kThreads + tid] = q == k - 1 ? 0.0f : 1.0f;
            }
        }
        if (!valid) continue;
        double a11 = 0.0, a12 = 0.0, a22 = 0.0, c1 = 0.0, c2 = 0.0;
        float kappa = 0.0f;
        for (int u = 0; u + 1 < k; ++u) {
            const float su = ssc[u * kThreads + tid];
            if (su <= 0.0f) continue;
            const int ju = sj[u * kThreads + tid];
            const float squ = ssq[u * kThreads + tid];
            const float2 lou = __ldg(reinterpret_cast<const float2*>(a.lo) + ju);
            const float* Trow = a.T + (int64_t)ju * a.g;
            for (int v = u + 1; v < k; ++v) {
                const float sv = ssc[v * kThreads + tid];
                const float wf = su * sv;
                if (!(wf > 0.0f)) continue;
                const int jv = sj[v * kThreads + tid];
                const float tv = __ldg(Trow + jv);
                if (tv < 0.0f) continue;  // hd2 < 1e-12: reference skips the pair
                const float2 lov = __ldg(reinterpret_cast<const float2*>(a.lo) + jv);
                const float ex = __fsub_rn(lov.x, lou.x);
                const float ey = __fsub_rn(lov.y, lou.y);
                const float ld2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
                if ((double)ld2 < kPairEps) continue;
                const float sqv = ssq[v * kThreads + tid];
                kappa = fmaxf(kappa, (squ + sqv) * tv);
                const float r = __frcp_rn(ld2);
                const double G1 = (double)(ex * r), G2 = (double)(ey * r);
                const double h = fma((double)(squ - sqv), (double)tv, 0.5) + G1 * (double)lou.x + G2 * (double)lou.y;
                const double w = (double)wf;
                const double wg1 = w * G1, wg2 = w * G2, wh = w * h;
                a11 = fma(wg1, G1, a11);
                a12 = fma(wg1, G2, a12);
                a22 = fma(wg2, G2, a22);
                c1 = fma(wh, G1, c1);
                c2 = fma(wh, G2, c2);
            }
        }
        if (kappa > (float)(2.0 * kKappaMax))  // kappa here is (sqd_u+sqd_v)*0.5/hd2
            pairs_exact(a.X, i, a.d, a.hi, a.lo, k, sj, ssc, tid, a11, a12, a22, c1, c2);
        const double det = a11 * a22 - a12 * a12;
        const double tr = a11 + a22;
        float2 out;
        if (det < kDetRel * tr * tr + kDetAbs) {
            out = __ldg(reinterpret_cast<const float2*>(a.lo) + b0);
        } else {
            out.x = (float)((c1 * a22 - c2 * a12) / det);
            out.y = (float)((a11 * c2 - a12 * c1) / det);
        }
        reinterpret_cast<float2*>(a.xy)[i] = out;
    }
    flag_nonfinite(a.flag, bad);
    if (MODE != 0 && a.qe_sum) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) qe_local += __shfl_xor_sync(0xffffffffu, qe_local, o);
        if ((tid & 31) == 0 && qe_local != 0.0) atomicAdd(a.qe_sum, qe_local);
    }
}


template <int DC, int KP, int MODE>
int launch_scan_t(ScanArgs a, cudaStream_t st) {
    const size_t tile_bytes = (size_t)a.dp * kTile * 4;
    size_t extra = (size_t)kTile * kThreads * 4;
    if (MODE == 1 && (size_t)KP * kThreads * 12 > extra) extra = (size_t)KP * kThreads * 12;
    const size_t cap = (size_t)esom_host::max_smem_optin() - 2048;
    size_t smem;
    if ((size_t)a.ntiles * tile_bytes + extra <= cap && (size_t)a.ntiles * tile_bytes <= esom_host::resident_limit()) {
        a.res_tiles = a.ntiles;
        smem = (size_t)a.ntiles * tile_bytes + extra;
    } else {
        a.res_tiles = 0;
        smem = 2 * tile_bytes + extra;
        if (smem > cap) return esom_host::set_err(ESOM_ERR_UNSUPPORTED, "dimension too large for smem tiles%s", "");
    }
    auto kern = scan_kernel<DC, KP, MODE>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t nblk = (a.n + kThreads - 1) / kThreads;
    int64_t grid = (int64_t)esom_host::num_sms() * per_sm;
    if (grid > nblk) grid = nblk;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kThreads, smem, st>>>(a);
    return esom_host::cuda_check("scan_kernel");
}


}  // namespace esom
