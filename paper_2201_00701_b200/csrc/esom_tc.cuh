// esom_tc.cuh -- tensor-core screened EXACT k-NN (tcgen05 + TMEM).
//
// The dense part of the distance evaluation, x . l, runs on the 5th-gen
// tensor cores as a split-BF16 GEMM (x = x_hi + x_lo, l = l_hi + l_lo;
// p ~= x_hi.l_hi + x_hi.l_lo + x_lo.l_hi, three kind::f16 MMAs into one f32
// TMEM accumulator).  Each epilogue thread owns one point (TMEM lane = row)
// and forms approximate distances d~_j = |x|^2 + |l_j|^2 - 2 p_j with a
// rigorous per-point error bound eps (see tc_eps).  Every landmark the exact
// top k could contain satisfies d~_j <= tau~ + 2 eps (tau~ = k-th smallest
// d~), so only those candidates get their EXACT distance recomputed with the
// reference's sequential f32 arithmetic (ref: knn.py:56-62), and the exact
// top k is selected among them by (distance, index).  Output is therefore
// bit-identical to knn_base (ref: knn.py:65-92) -- the tensor cores only
// prune.
//
// Layouts: operands are K-major bf16 in the canonical
// no-swizzle UMMA layout [8-row group][16-byte K chunk][8 rows][8 elems]
// (LBO = 128 B between K chunks, SBO = (K/8)*128 B between row groups).
// Landmarks (B, hi and lo), |l_j|^2 and the f32 exact tiles are prepared
// per model and staged once per CTA with 1-D TMA bulk copies.
#pragma once
#include "esom_common.cuh"
#include "esom_host.h"
#include "esom_knn.cuh"
#include "esom_scan.cuh"  // knn_point_slow
#include "esom_scan_args.h"

namespace esom {

constexpr int kTcThreads = 256;  // two 128-point tiles per CTA, one per TMEM column half



__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t desc = 0;
    desc |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    desc |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    desc |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    desc |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
    return desc;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both K-major.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 consecutive f32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]);
}

__device__ __forceinline__ uint16_t bf16_bits(float f) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}
__device__ __forceinline__ float bf16_val(uint16_t b) { return __bfloat162float(__ushort_as_bfloat16(b)); }

// byte offset of element (row, kk) in the canonical K-major no-swizzle layout
__device__ __forceinline__ uint32_t canon_off(int row, int kk, int K) {
    return (uint32_t)((((row >> 3) * (K >> 3) + (kk >> 3)) << 7) + ((row & 7) << 4) + ((kk & 7) << 1));
}

// Rigorous bound on |d~ - d_ref| for one point (d~ from the split-bf16
// product, d_ref the reference's sequential f32 sum):
//  * split residual: |x - x_hi - x_lo| <= 2^-18|x| per component, dropped
//    x_lo*l_lo <= 2^-18|x||l|  ->  <= 4*2^-18 sum|x_c||l_c|
//  * tensor-core f32 accumulation of 3*d16 exact bf16 products: budgeted at
//    3*d16 * 2^-22 sum|x_c||l_c| (2x the sequential-RN bound)
//  * |x|^2, |l|^2 and the final combination: (d + 4) 2^-23 (|x|^2 + |l|^2)
//  * the reference's own rounding: d 2^-24 d_true <= d 2^-23 (|x|^2 + |l|^2)
// with sum|x_c||l_c| <= |x||l| (Cauchy-Schwarz) and a further 2x margin; all
// norms are of the centred vectors x - c, l - c (c = landmark centroid; the
// centring rounding is inside the (d + 4) 2^-23 term's slack).
__device__ __forceinline__ float tc_eps(float xnorm, float xn, float lmax, float lnmax, int d, int d16) {
    const float c1 = 2.0f * (4.0f * 3.8147e-6f + 3.0f * d16 * 2.3842e-7f);
    const float c2 = 2.0f * (2.0f * d + 4.0f) * 1.1921e-7f;
    return 2.0f * (c1 * xnorm * lmax + c2 * (xn + lnmax));
}

template <int KP>
__global__ void __launch_bounds__(kTcThreads, 1) knn_tc_kernel(TcArgs a) {
    constexpr int LOGCAP = KP + kTile;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bar_load, bar_mma, bar_b[2];
    __shared__ uint32_t tmem_base_sh;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int d = a.d, d16 = a.d16, gpad = a.gpad, k = a.k;
    const int off = KP - k;
    const int R = (gpad + 255) >> 8;           // landmark rounds of <= 256 TMEM columns
    const bool streamB = R > 1;                // B streamed round by round (double buffered)
    const bool lt_res = a.Lt != nullptr;       // exact tiles resident in smem (else rows from L2)
    const uint32_t a_bytes = 128u * d16 * 2u;  // one operand tile (hi or lo), bytes
    const uint32_t b_bytes = (uint32_t)(streamB ? 256 : gpad) * d16 * 2u;
    const uint32_t lt_bytes = lt_res ? (uint32_t)(gpad / kTile) * a.dp * kTile * 4u : 0u;
    // ---- shared memory carve-up (all 128-byte aligned) ----
    unsigned char* p = smem_raw;
    unsigned char* Ahi = p;  p += 2 * a_bytes;  // [tile 0 | tile 1]
    unsigned char* Alo = p;  p += 2 * a_bytes;
    unsigned char* Bhi = p;  p += (streamB ? 2 : 1) * b_bytes;
    unsigned char* Blo = p;  p += (streamB ? 2 : 1) * b_bytes;
    float* Lt = reinterpret_cast<float*>(p);  p += lt_bytes;
    float* lns = reinterpret_cast<float*>(p);  p += ((gpad * 4 + 127) / 128) * 128;
    float* xrow = reinterpret_cast<float*>(p);  p += (((size_t)kTcThreads * (d + 1) * 4 + 127) / 128) * 128;
    float* logv = reinterpret_cast<float*>(p);  p += (size_t)(LOGCAP + 1) * kTcThreads * 4;
    unsigned short* logj = reinterpret_cast<unsigned short*>(p);

    if (tid == 0) {
        mbar_init(&bar_load, 1);
        mbar_init(&bar_mma, 1);
        mbar_init(&bar_b[0], 1);
        mbar_init(&bar_b[1], 1);
        fence_mbar_init();
    }
    if (warp == 0) {  // 512 TMEM columns: tile t accumulates in columns [256 t, 256 t + 256)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    const float lmax = __ldg(a.lstats), lnmax = __ldg(a.lstats + 1);
    const int64_t nblk = (a.n + kTcThreads - 1) / kTcThreads;

    // B round v (of the periodic visit sequence: two passes x R rounds per block)
    auto load_round = [&](int64_t v) {
        const int b = (int)(v & 1), r = (int)(v % R);
        const int rows = min(256, gpad - 256 * r);
        const uint32_t bytes = (uint32_t)rows * d16 * 2u;
        const size_t off_el = (size_t)256 * r * d16;
        mbar_expect_tx(&bar_b[b], 2 * bytes);
        tma_bulk_g2s(Bhi + b * b_bytes, a.Bhi + off_el, bytes, &bar_b[b]);
        tma_bulk_g2s(Blo + b * b_bytes, a.Blo + off_el, bytes, &bar_b[b]);
    };
    if (tid == 0) {
        mbar_expect_tx(&bar_load, (streamB ? 0u : 2 * b_bytes) + lt_bytes + (uint32_t)gpad * 4u);
        if (!streamB) {
            tma_bulk_g2s(Bhi, a.Bhi, b_bytes, &bar_load);
            tma_bulk_g2s(Blo, a.Blo, b_bytes, &bar_load);
        }
        if (lt_res) tma_bulk_g2s(Lt, a.Lt, lt_bytes, &bar_load);
        tma_bulk_g2s(lns, a.ln, (uint32_t)gpad * 4u, &bar_load);
        if (streamB && blockIdx.x < nblk) {
            load_round(0);
            load_round(1);
        }
    }
    mbar_wait(&bar_load, 0);

    const int tile = tid >> 7, row = tid & 127;
    const uint32_t sbo = (uint32_t)(d16 >> 3) << 7, lbo = 128;
    const uint32_t lane_col = ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(256 * tile);
    float* myx = xrow + (size_t)tid * (d + 1);
    uint32_t mma_phase = 0, bph0 = 0, bph1 = 0;
    int64_t visit = 0;
    bool bad = false;
    double qe_local = 0.0;

    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int64_t i = blk * kTcThreads + tid;
        const bool valid = i < a.n;
        // ---- stage the point: f32 row (exact recompute) + split bf16 operand ----
        float xn = 0.0f;
        bool xbad = false;
        {
            const float* xr = a.X + i * d;
            unsigned char* ah = Ahi + tile * a_bytes;
            unsigned char* al = Alo + tile * a_bytes;
            for (int c0 = 0; c0 < d16; c0 += 8) {
                uint32_t hw[4], lw[4];
#pragma unroll
                for (int q = 0; q < 8; q += 2) {
                    float v0 = 0.0f, v1 = 0.0f;
                    if (valid && c0 + q < d) v0 = __ldg(xr + c0 + q);
                    if (valid && c0 + q + 1 < d) v1 = __ldg(xr + c0 + q + 1);
                    xbad |= !finite_f(v0) || !finite_f(v1);
                    if (c0 + q < d) myx[c0 + q] = v0;
                    if (c0 + q + 1 < d) myx[c0 + q + 1] = v1;
                    v0 -= __ldg(a.center + c0 + q);  // centred operands (|x - l| is translation invariant)
                    v1 -= __ldg(a.center + c0 + q + 1);
                    xn = fmaf(v0, v0, xn);
                    xn = fmaf(v1, v1, xn);
                    const uint16_t h0 = bf16_bits(v0), h1 = bf16_bits(v1);
                    const uint16_t l0 = bf16_bits(v0 - bf16_val(h0)), l1 = bf16_bits(v1 - bf16_val(h1));
                    hw[q >> 1] = (uint32_t)h0 | ((uint32_t)h1 << 16);
                    lw[q >> 1] = (uint32_t)l0 | ((uint32_t)l1 << 16);
                }
                const uint32_t o = canon_off(row, c0, d16);
                *reinterpret_cast<uint4*>(ah + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                *reinterpret_cast<uint4*>(al + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
        }
        bad |= xbad;
        fence_proxy_async();  // generic smem writes -> visible to the tensor core (async proxy)
        tc_fence_before();
        __syncthreads();

        const float xnorm = sqrtf(xn);
        const float eps2 = 2.0f * tc_eps(xnorm, xn, lmax, lnmax, d, d16);
        float gm[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) gm[q] = kInf;
        float tcut = kInf;
        int cnt = 0;
        // two passes over the R landmark rounds: pass 0 builds the bound, pass 1 logs candidates
        for (int s2 = 0; s2 < 2 * R; ++s2, ++visit) {
            const int r = s2 % R, pass = s2 / R;
            const int nr = min(256, gpad - 256 * r);
            const int bb = streamB ? (int)(visit & 1) : 0;
            if (tid == 0) {
                if (streamB) {
                    mbar_wait(&bar_b[bb], bb ? bph1 : bph0);
                }
                tc_fence_after();
                const uint32_t idesc = umma_idesc_bf16(128, nr);
                const uint32_t bbase_h = smem_u32(Bhi + bb * b_bytes), bbase_l = smem_u32(Blo + bb * b_bytes);
                for (int t = 0; t < 2; ++t) {
                    const uint32_t abase_h = smem_u32(Ahi + t * a_bytes), abase_l = smem_u32(Alo + t * a_bytes);
                    const uint32_t dcol = tmem + (uint32_t)(256 * t);
                    for (int ks = 0; ks < (d16 >> 4); ++ks) {
                        const uint32_t ko = (uint32_t)ks * 256u;  // two 16-byte K chunks per MMA
                        umma_bf16(dcol, umma_desc(abase_h + ko, lbo, sbo), umma_desc(bbase_h + ko, lbo, sbo), idesc,
                                  ks > 0);
                        umma_bf16(dcol, umma_desc(abase_h + ko, lbo, sbo), umma_desc(bbase_l + ko, lbo, sbo), idesc, 1);
                        umma_bf16(dcol, umma_desc(abase_l + ko, lbo, sbo), umma_desc(bbase_h + ko, lbo, sbo), idesc, 1);
                    }
                }
                umma_commit(&bar_mma);
            }
            if (streamB) {
                if (bb) bph1 ^= 1u; else bph0 ^= 1u;
            }
            mbar_wait(&bar_mma, mma_phase);
            mma_phase ^= 1u;
            tc_fence_after();
            if (streamB && tid == 0) {
                // buffer bb is free again: prefetch visit + 2 (next block's rounds included)
                const bool more = s2 + 2 < 2 * R || blk + gridDim.x < nblk;
                if (more) load_round(visit + 2);
            }
            const int cbase = 256 * r;
            if (pass == 0) {
                // minima of the 32 landmark groups j = q (mod 32): the k-th smallest
                // group minimum bounds the k-th smallest d~ (k distinct landmarks)
                for (int c0 = 0; c0 < nr; c0 += 32) {
                    float v[32];
                    tmem_ld32(tmem + lane_col + (uint32_t)c0, v);
#pragma unroll
                    for (int q = 0; q < 32; ++q) gm[q] = fminf(gm[q], v[q] + (xn + lns[cbase + c0 + q]));  // B = -2 l
                }
                if (r == R - 1) {
                    float vd[KP];
                    vlist_init<KP>(vd, k);
#pragma unroll
                    for (int q = 0; q < 32; ++q) vlist_insert<KP>(vd, gm[q]);
                    tcut = vd[KP - 1] + eps2;
                }
            } else {
                // log every landmark that can still be in the top k
                for (int c0 = 0; c0 < nr; c0 += 32) {
                    float v[32];
                    tmem_ld32(tmem + lane_col + (uint32_t)c0, v);
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const float dt = v[q] + (xn + lns[cbase + c0 + q]);  // B = -2 l; +inf on padding rows
                        const bool keep = dt <= tcut;
                        const int slot = min(cnt, LOGCAP);  // slot LOGCAP is a dump row
                        if (keep) {
                            logv[slot * kTcThreads + tid] = dt;
                            logj[slot * kTcThreads + tid] = (unsigned short)(cbase + c0 + q);
                        }
                        cnt += keep ? 1 : 0;
                    }
                }
            }
            tc_fence_before();
            __syncthreads();  // TMEM columns are rewritten by the next visit's MMA
        }
        const bool ovf = cnt > LOGCAP;
        // refine: the exact k-th smallest d~ among the logged candidates
        float vd[KP];
        vlist_init<KP>(vd, k);
        if (!ovf)
            for (int e = 0; e < cnt; ++e) {
                const float dv = logv[e * kTcThreads + tid];
                if (dv < vd[KP - 1]) vlist_insert<KP>(vd, dv);
            }
        // ---- exact phase: reference f32 distances of the surviving candidates ----
        if (!valid) continue;
        int32_t* oi = a.out_idx ? a.out_idx + i * k : nullptr;
        float* od = a.out_sqd ? a.out_sqd + i * k : nullptr;
        int b0 = 0;
        float d0 = 0.0f;
        int written = 0;
        if (!ovf && !xbad) {
            const float tf = vd[KP - 1] + eps2;
            int m = 0;  // compact the survivors of the refined threshold (index order kept)
            for (int e = 0; e < cnt; ++e) {
                const float dv = logv[e * kTcThreads + tid];
                if (dv <= tf) {
                    logj[m * kTcThreads + tid] = logj[e * kTcThreads + tid];
                    ++m;
                }
            }
            // exact f32 distances (four independent sequential chains in flight),
            // inserted in index order into a (dist, idx) register list
            float td[KP];
            int ti[KP];
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                td[q] = q >= off ? kInf : -kInf;
                ti[q] = a.g;
            }
            for (int e = 0; e < m; e += 4) {
                const float* lt[4];
                int jq[4];
                int stride;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    jq[u] = logj[min(e + u, m - 1) * kTcThreads + tid];
                    lt[u] = lt_res ? Lt + (size_t)(jq[u] >> 5) * a.dp * kTile + (jq[u] & 31) : a.L + (size_t)jq[u] * d;
                }
                stride = lt_res ? kTile : 1;
                float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                for (int c = 0; c < d; ++c) {
                    const float xc = myx[c];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float t = __fsub_rn(xc, lt[u][c * stride]);
                        s4[u] = __fadd_rn(s4[u], __fmul_rn(t, t));
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (e + u < m && s4[u] < td[KP - 1]) topk_insert<KP>(td, ti, s4[u], jq[u]);
            }
            if (a.stats) atomicAdd(a.stats, m);
            written = 0;
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                if (q >= off) {
                    written += ti[q] < a.g ? 1 : 0;
                    if (oi) {
                        oi[q - off] = ti[q];
                        od[q - off] = td[q];
                    }
                    if (q == off) {
                        b0 = ti[q];
                        d0 = td[q];
                    }
                }
            }
        }
        if (written != k) {
            // log overflow, non-finite input or a candidate set short of k:
            // the reference's insertion scan for this point
            const SlowNearest sn = knn_point_slow(a.X + i * d, d, a.L, a.g, k, oi, od);
            b0 = sn.b0;
            d0 = sn.d0;
        }
        if (a.bmu) a.bmu[i] = b0;
        if (a.qe_sum) qe_local += (double)d0;
        if (a.accS) {
            atomicAdd(a.accC + b0, 1ull);
            for (int c = 0; c < d; ++c) atomicAdd(a.accS + (int64_t)b0 * d + c, acc_fx(myx[c], a.acc_scale));
        }
    }
    flag_nonfinite(a.flag, bad);
    if (a.qe_sum) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) qe_local += __shfl_xor_sync(0xffffffffu, qe_local, o);
        if ((tid & 31) == 0 && qe_local != 0.0) atomicAdd(a.qe_sum, qe_local);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int KP>
size_t tc_smem_bytes(const TcArgs& a) {
    constexpr int LOGCAP = KP + kTile;
    const bool streamB = a.gpad > 256;
    size_t b = 4 * (size_t)128 * a.d16 * 2;                          // A hi/lo, two tiles
    b += 2 * (size_t)(streamB ? 2 * 256 : a.gpad) * a.d16 * 2;       // B hi/lo (two round buffers when streamed)
    if (a.Lt) b += (size_t)(a.gpad / kTile) * a.dp * kTile * 4;      // exact tiles (resident)
    b += ((size_t)a.gpad * 4 + 127) / 128 * 128;                     // |l|^2
    b += (((size_t)kTcThreads * (a.d + 1) * 4 + 127) / 128) * 128;   // f32 rows
    b += (size_t)(LOGCAP + 1) * kTcThreads * 6;                      // candidate log (+ dump row)
    return b + 1024;
}

template <int KP>
int launch_tc_t(TcArgs a, cudaStream_t st) {
    const size_t smem = tc_smem_bytes<KP>(a);
    if (smem > (size_t)esom_host::max_smem_optin())
        return esom_host::set_err(ESOM_ERR_UNSUPPORTED, "tensor-core screen: shape exceeds shared memory%s", "");
    auto kern = knn_tc_kernel<KP>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t nblk = (a.n + kTcThreads - 1) / kTcThreads;
    int64_t grid = esom_host::num_sms();
    if (grid > nblk) grid = nblk;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kTcThreads, smem, st>>>(a);
    return esom_host::cuda_check("knn_tc_kernel");
}

}  // namespace esom
