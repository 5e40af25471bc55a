// esom_scan.cuh -- the exact k-NN scan kernel (distance tiles + selection,
// optional batch-SOM statistics) and its launcher template.  Instantiated
// per (DC, KP) in inst/*.cu so the library builds in parallel.
//
//   ref: knn.py:56-62 (_sqdist_f32), 65-92 (_knn_base_kernel),
//        148-184 (_knn_bitonic_kernel; identical output), 201-243 (API)
#pragma once
#include "esom_common.cuh"
#include "esom_host.h"
#include "esom_knn.cuh"
#include "esom_scan_args.h"

namespace esom {

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

// Rare exact fallback for one point whose candidate log overflowed (massive
// exact ties / overflowing distances): the reference's own insertion scan
// (ref: knn.py:65-92) over row-major landmarks, writing rank-ordered rows.
struct SlowNearest {
    int b0;
    float d0;
};

static __device__ __noinline__ SlowNearest knn_point_slow(const float* __restrict__ x, int d, const float* __restrict__ L,
                                                          int g, int k, int32_t* oi, float* od) {
    float bd[64];
    int bi[64];
    int cnt = 0;
    for (int j = 0; j < g; ++j) {
        const float* l = L + (int64_t)j * d;
        float s = 0.0f;
        for (int c = 0; c < d; ++c) {
            const float t = __fsub_rn(x[c], l[c]);
            s = __fadd_rn(s, __fmul_rn(t, t));
        }
        int p;
        if (cnt < k) {
            p = cnt++;
        } else {
            if (s > bd[k - 1] || (s == bd[k - 1] && j > bi[k - 1])) continue;
            p = k - 1;
        }
        while (p > 0 && (s < bd[p - 1] || (s == bd[p - 1] && j < bi[p - 1]))) {
            bd[p] = bd[p - 1];
            bi[p] = bi[p - 1];
            --p;
        }
        bd[p] = s;
        bi[p] = j;
    }
    for (int q = 0; q < k; ++q) {
        if (oi) {
            oi[q] = bi[q];
            od[q] = bd[q];
        }
    }
    return SlowNearest{bi[0], bd[0]};
}

template <int DC, int KP>
__global__ void __launch_bounds__(kThreads) knn_scan_kernel(ScanArgs a) {
    constexpr int LOGCAP = KP + kTile;  // one tile of appends on top of a compacted log
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[2];  // TMA completion barriers
    const int tid = threadIdx.x;
    const int tile_floats = a.dp * kTile;
    const uint32_t tile_bytes = (uint32_t)tile_floats * 4u;
    const int nbuf = a.res_tiles ? a.res_tiles : 2;
    float* tiles = reinterpret_cast<float*>(smem_raw);
    float* logv = tiles + (size_t)nbuf * tile_floats;                                // [LOGCAP][kThreads]
    unsigned short* logj = reinterpret_cast<unsigned short*>(logv + LOGCAP * kThreads);  // [LOGCAP][kThreads], g < 65536

    const f2 nz = f2_pack(a.nz, a.nz);
    const bool stream = a.res_tiles == 0;
    const int k = a.k;
    const int off = KP - k;
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
        const bool valid = i < a.n;
        float x[DC];
        if (a.nch == 1) bad |= load_x<DC>(a.X, i, a.n, a.d, 0, x);

        float vd[KP];
        vlist_init<KP>(vd, k);
        int cnt = 0;
        bool ovf = false;

        if (stream && tid == 0) {
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
            if (!ovf) {
                const float tau = vd[KP - 1];
                const bool open = tau == kInf;
                const int jb = t * kTile;
                const int cnt0 = cnt;
#pragma unroll
                for (int p = 0; p < 16; ++p) {
                    float va, vb;
                    f2_unpack(acc[p], va, vb);
                    const int ja = jb + 2 * p;
                    if (va < tau || (open && ja < a.g)) {
                        logv[cnt * kThreads + tid] = va;
                        logj[cnt * kThreads + tid] = (unsigned short)ja;
                        ++cnt;
                    }
                    if (vb < tau || (open && ja + 1 < a.g)) {
                        logv[cnt * kThreads + tid] = vb;
                        logj[cnt * kThreads + tid] = (unsigned short)(ja + 1);
                        ++cnt;
                    }
                }
                for (int e = cnt0; e < cnt; ++e) {
                    const float v = logv[e * kThreads + tid];
                    if (v < vd[KP - 1]) vlist_insert<KP>(vd, v);
                }
                if (cnt > LOGCAP - kTile) {  // compact: keep what can still make the top k
                    const float tf = vd[KP - 1];
                    int w = 0;
                    for (int e = 0; e < cnt; ++e) {
                        const float v = logv[e * kThreads + tid];
                        if (v <= tf) {
                            logj[w * kThreads + tid] = logj[e * kThreads + tid];
                            logv[w * kThreads + tid] = v;
                            ++w;
                        }
                    }
                    cnt = w;
                    ovf = cnt > LOGCAP - kTile;
                }
            }
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
        if (!valid) continue;

        // ---- final selection: rank the logged candidates by (v, j) ----
        int32_t* oi = a.out_idx ? a.out_idx + i * k : nullptr;
        float* od = a.out_sqd ? a.out_sqd + i * k : nullptr;
        int b0 = 0;
        float d0 = 0.0f;
        int written = 0;
        if (!ovf) {
            const float tf = vd[KP - 1];
            int quota = k - (vlist_count_lt<KP>(vd, tf) - off);  // entries == tf still admitted
            for (int e = 0; e < cnt; ++e) {
                const float v = logv[e * kThreads + tid];
                int r;
                if (v < tf) {
                    r = vlist_count_lt<KP>(vd, v) - off;
                    // exact duplicates below tf: earlier-index copies rank first
                    int le = 0;
#pragma unroll
                    for (int q = 0; q < KP; ++q) le += vd[q] <= v ? 1 : 0;
                    if (le - off - r > 1) {
                        for (int e2 = 0; e2 < e; ++e2) r += logv[e2 * kThreads + tid] == v ? 1 : 0;
                    }
                } else if (v == tf && quota > 0) {
                    r = k - quota;  // ties at the k-th value: lowest indices, in log (= index) order
                    --quota;
                } else {
                    continue;
                }
                const int j = logj[e * kThreads + tid];
                if (oi) {
                    oi[r] = j;
                    od[r] = v;
                }
                if (r == 0) {
                    b0 = j;
                    d0 = v;
                }
                ++written;
            }
        }
        // log overflow (pathological ties) or NaN inputs (flagged as
        // non-finite; rows must still hold valid indices): the reference's
        // own insertion scan for this point
        if (ovf || written != k) {
            const SlowNearest sn = knn_point_slow(a.X + i * a.d, a.d, a.L, a.g, k, oi, od);
            b0 = sn.b0;
            d0 = sn.d0;
        }
        if (a.bmu) a.bmu[i] = b0;
        if (a.qe_sum) qe_local += (double)d0;
        if (a.accS) {
            atomicAdd(a.accC + b0, 1ull);
            if (a.nch == 1) {
#pragma unroll
                for (int c = 0; c < DC; ++c)
                    if (c < a.d) atomicAdd(a.accS + (int64_t)b0 * a.d + c, acc_fx(x[c], a.acc_scale));
            } else {
                for (int c = 0; c < a.d; ++c) atomicAdd(a.accS + (int64_t)b0 * a.d + c, acc_fx(a.X[i * a.d + c], a.acc_scale));
            }
        }
    }
    flag_nonfinite(a.flag, bad);
    if (a.qe_sum) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) qe_local += __shfl_xor_sync(0xffffffffu, qe_local, o);
        if ((tid & 31) == 0 && qe_local != 0.0) atomicAdd(a.qe_sum, qe_local);
    }
}

template <int DC, int KP>
int launch_scan_t(ScanArgs a, cudaStream_t st) {
    constexpr int LOGCAP = KP + kTile;
    const size_t tile_bytes = (size_t)a.dp * kTile * 4;
    const size_t extra = (size_t)LOGCAP * kThreads * 6;
    if (a.g >= 65536) return esom_host::set_err(ESOM_ERR_UNSUPPORTED, "g >= 65536 unsupported by the scan kernel%s", "");
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
    auto kern = knn_scan_kernel<DC, KP>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t nblk = (a.n + kThreads - 1) / kThreads;
    int64_t grid = (int64_t)esom_host::num_sms() * per_sm;
    if (grid > nblk) grid = nblk;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kThreads, smem, st>>>(a);
    return esom_host::cuda_check("knn_scan_kernel");
}

}  // namespace esom
