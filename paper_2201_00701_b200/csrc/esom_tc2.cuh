// esom_tc2.cuh -- pipelined tensor-core screened EXACT k-NN (d <= 32).
//
// Same contract as esom_tc.cuh (bit-identical to knn_base, ref:
// knn.py:65-92; the tensor cores only prune), re-organised for throughput:
//
//  * W warpgroups per CTA ("WG", 4 warps = the 128 TMEM lanes = one 128-point
//    tile each) run independent tile loops; the CTA's 512 TMEM columns form
//    S = 2 accumulator slots of 256 columns that the tiles take in turn
//    (tile t uses slot t mod S and waits for tile t - S to release it).  A WG
//    releases its slot as soon as its screen has read TMEM, so the MMA of the
//    next tile overlaps the exact phase of this one.
//  * The accumulator is initialised with |l_j|^2 (tcgen05.st) and the
//    landmark operand is B = -2 l (split bf16), so the tensor cores deliver
//    D~_j = |l_j|^2 - 2 x.l_j = |x - l_j|^2 - |x|^2 directly: the screen is one
//    TMEM read + one min per value (pass A) and one compare per value (pass B).
//  * Pass A: minima of the 32 landmark groups j = q (mod 32); the k-th
//    smallest group minimum tau bounds the k-th smallest D~ (k distinct
//    landmarks).  Pass B logs every column with D~_j <= tau + 2E in index
//    order (E = per-point bound on |D~_j - (d_ref_j - |x|^2)|, see tc2_eps).
//    Every member of the exact top k satisfies that, so the exact phase --
//    reference f32 distances of the logged landmarks (ref: knn.py:56-62,
//    packed f32x2 sub/square, sequential scalar adds), inserted in index
//    order by (distance, index) -- reproduces knn_base bit for bit.
//  * Landmarks (B operand, |l|^2, padded f32 rows) are staged once per CTA by
//    1-D TMA bulk copies; rows come from L2 when they do not fit in smem.
#pragma once
#include <stdlib.h>

#include <utility>

#include "esom_tc.cuh"

namespace esom {


constexpr int kTc2Slots = 2;     // TMEM accumulator slots of 256 columns
constexpr int kTc2SlotCols = 256;

__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
        "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
        "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
        "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// m | (1 << Q) when v <= t (FSETP + predicated LOP3 with an immediate)
template <int Q>
__device__ __forceinline__ uint32_t or_if_le(uint32_t m, float v, float t) {
    uint32_t r;
    asm("{\n\t.reg .pred p;\n\tsetp.le.f32 p, %1, %2;\n\tmov.b32 %0, %3;\n\t@p or.b32 %0, %3, %4;\n\t}"
        : "=r"(r) : "f"(v), "f"(t), "r"(m), "n"(1u << Q));
    return r;
}
template <int... Q>
__device__ __forceinline__ uint32_t le_mask32(const uint32_t (&v)[32], float t, std::integer_sequence<int, Q...>) {
    uint32_t m = 0;
    ((m = or_if_le<Q>(m, __uint_as_float(v[Q]), t)), ...);
    return m;
}

__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// Rigorous bound E on |D~_j - (d_ref_j - |x|^2)| for one point:
//   split residual of x.l (x_lo l_lo dropped, bf16 residuals): 4 2^-18 S, x2 for B = -2l
//   tensor-core f32 accumulation of 3 d16 products onto |l|^2: 3 d16 2^-23 (N + 2S)
//   |l|^2 rounded to f32: 2^-24 N
//   the reference's own rounding of d_ref: (d + 2) 2^-23 (|x| + |l|)^2
//   centring (x' = fl(x - c), l' = fl(l - c), c = landmark mean; |x - l| is
//   translation invariant): 2^-23 (|x'| + |l'|)^2
// with all norms of the centred vectors, S = |x'| max|l'| >= sum_c |x'_c l'_c|
// (Cauchy-Schwarz), N = max |l'|^2, and a further 2x margin.
__device__ __forceinline__ float tc2_eps(float xnorm, float lmax, float lnmax, int d, int d16) {
    const float S = xnorm * lmax;
    const float r = xnorm + lmax;
    const float e = 8.0f * 3.8147e-6f * S + 3.0f * d16 * 1.1921e-7f * (lnmax + 2.0f * S) + 5.97e-8f * lnmax +
                    (d + 3.0f) * 1.1921e-7f * r * r;
    return 2.0f * e;
}

// Batcher odd-even merge sort of 16 register values (63 comparators, generated).
#define ESOM_CE(a, b)                          \
    {                                          \
        const float lo_ = fminf(v[a], v[b]);   \
        v[b] = fmaxf(v[a], v[b]);              \
        v[a] = lo_;                            \
    }
__device__ __forceinline__ void sort16(float (&v)[16]) {
    ESOM_CE(0, 1);
    ESOM_CE(2, 3);
    ESOM_CE(4, 5);
    ESOM_CE(6, 7);
    ESOM_CE(8, 9);
    ESOM_CE(10, 11);
    ESOM_CE(12, 13);
    ESOM_CE(14, 15);
    ESOM_CE(0, 2);
    ESOM_CE(1, 3);
    ESOM_CE(4, 6);
    ESOM_CE(5, 7);
    ESOM_CE(8, 10);
    ESOM_CE(9, 11);
    ESOM_CE(12, 14);
    ESOM_CE(13, 15);
    ESOM_CE(1, 2);
    ESOM_CE(5, 6);
    ESOM_CE(9, 10);
    ESOM_CE(13, 14);
    ESOM_CE(0, 4);
    ESOM_CE(1, 5);
    ESOM_CE(2, 6);
    ESOM_CE(3, 7);
    ESOM_CE(8, 12);
    ESOM_CE(9, 13);
    ESOM_CE(10, 14);
    ESOM_CE(11, 15);
    ESOM_CE(2, 4);
    ESOM_CE(3, 5);
    ESOM_CE(10, 12);
    ESOM_CE(11, 13);
    ESOM_CE(1, 2);
    ESOM_CE(3, 4);
    ESOM_CE(5, 6);
    ESOM_CE(9, 10);
    ESOM_CE(11, 12);
    ESOM_CE(13, 14);
    ESOM_CE(0, 8);
    ESOM_CE(1, 9);
    ESOM_CE(2, 10);
    ESOM_CE(3, 11);
    ESOM_CE(4, 12);
    ESOM_CE(5, 13);
    ESOM_CE(6, 14);
    ESOM_CE(7, 15);
    ESOM_CE(4, 8);
    ESOM_CE(5, 9);
    ESOM_CE(6, 10);
    ESOM_CE(7, 11);
    ESOM_CE(2, 4);
    ESOM_CE(3, 5);
    ESOM_CE(6, 8);
    ESOM_CE(7, 9);
    ESOM_CE(10, 12);
    ESOM_CE(11, 13);
    ESOM_CE(1, 2);
    ESOM_CE(3, 4);
    ESOM_CE(5, 6);
    ESOM_CE(7, 8);
    ESOM_CE(9, 10);
    ESOM_CE(11, 12);
    ESOM_CE(13, 14);
}
#undef ESOM_CE

// k-th smallest of the 32 group minima (an upper bound of the k-th smallest D~).
// k == 16: sort both halves (Batcher, 63 comparators each), then the 16th
// smallest of two sorted 16-lists = min over splits i of max(A[i-1], B[15-i]).
template <int KP>
__device__ __forceinline__ float kth_of_32(const float (&gm)[32], int k) {
    if (KP == 16 && k == 16) {
        float A[16], B[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            A[q] = gm[q];
            B[q] = gm[16 + q];
        }
        sort16(A);
        sort16(B);
        float t = fminf(A[15], B[15]);
#pragma unroll
        for (int i = 1; i < 16; ++i) t = fminf(t, fmaxf(A[i - 1], B[15 - i]));
        return t;
    }
    float vd[KP];
    vlist_init<KP>(vd, k);
#pragma unroll
    for (int q = 0; q < 32; ++q) vlist_insert<KP>(vd, gm[q]);
    return vd[KP - 1];
}

template <int KP, int W>
__host__ __device__ constexpr int tc2_slot_bars() { return (W + kTc2Slots - 1) / kTc2Slots + 1; }

template <int KP, int W, bool RS, bool SPLIT>
__global__ void __launch_bounds__(128 * W, 1) knn_tc2_kernel(Tc2Args a) {
    constexpr int S = kTc2Slots;
    constexpr int M = tc2_slot_bars<KP, W>();  // release barriers per slot (no parity aliasing, see acquire)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bar_load, bar_mma[W], bar_slot[S][M];
    __shared__ uint32_t tmem_base_sh;
    __shared__ __align__(16) float cen[32];  // landmark centroid (zero-padded to 32 dims)

    const int tid = threadIdx.x;
    const int w = tid >> 7;        // warpgroup
    const bool x32 = rows32(a.X, a.d);
    const int wt = tid & 127;      // TMEM lane / row of the tile
    const int d = a.d, d16 = a.d16, gpad = a.gpad, k = a.k;
    const int off = KP - k;
    const int R = (gpad + kTc2SlotCols - 1) / kTc2SlotCols;  // landmark rounds per pass
    const int nwords = gpad >> 5;                             // candidate bitmap words per point
    const uint32_t a_bytes = 128u * d16 * 2u;
    const uint32_t b_bytes = (uint32_t)gpad * d16 * 2u;
    const uint32_t r_bytes = RS ? (uint32_t)gpad * a.ls * 4u : 0u;
    unsigned char* p = smem_raw;
    unsigned char* Bhi = p;  p += b_bytes;
    unsigned char* Blo = p;  p += b_bytes;
    float* lns = reinterpret_cast<float*>(p);  p += ((gpad * 4 + 127) / 128) * 128;
    float* Ls = reinterpret_cast<float*>(p);  p += ((r_bytes + 127) / 128) * 128;
    unsigned char* Ahi = p + (size_t)w * 2 * a_bytes;
    unsigned char* Alo = Ahi + a_bytes;
    p += (size_t)W * 2 * a_bytes;
    // fused mode: candidate bitmaps and locality-sort keys in smem; SPLIT mode: bitmaps to global
    uint32_t* bmap0 = reinterpret_cast<uint32_t*>(p) + (size_t)w * nwords * 128;  // [word][128]
    uint32_t* bmap = bmap0 + wt;
    if (!SPLIT) p += (size_t)W * nwords * 128 * 4;
    uint32_t* pkey = reinterpret_cast<uint32_t*>(p) + (size_t)w * 4 * 128;  // per WG: key | cnt | nzw | bad

    if (tid == 0) {
        mbar_init(&bar_load, 1);
        for (int q = 0; q < W; ++q) mbar_init(&bar_mma[q], 1);
        for (int q = 0; q < S; ++q)
            for (int u = 0; u < M; ++u) mbar_init(&bar_slot[q][u], 128);
        fence_mbar_init();
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    if (tid == 0) {
        mbar_expect_tx(&bar_load, 2 * b_bytes + (uint32_t)gpad * 4u + r_bytes + 128u);
        tma_bulk_g2s(cen, a.center, 128u, &bar_load);
        tma_bulk_g2s(Bhi, a.Bhi, b_bytes, &bar_load);
        tma_bulk_g2s(Blo, a.Blo, b_bytes, &bar_load);
        tma_bulk_g2s(lns, a.ln, (uint32_t)gpad * 4u, &bar_load);
        if (RS) tma_bulk_g2s(Ls, a.Lrow, r_bytes, &bar_load);
    }
    mbar_wait(&bar_load, 0);

    const float lmax = __ldg(a.lstats), lnmax = __ldg(a.lstats + 1);
    const int64_t ntiles = (a.n + 127) / 128;
    const uint32_t sbo = (uint32_t)(d16 >> 3) << 7, lbo = 128;
    const uint32_t lane_off = (uint32_t)(32 * ((tid >> 5) & 3)) << 16;
    const float* Lr = RS ? Ls : a.Lrow;
    const int ls = a.ls;
    uint32_t mma_phase = 0;
    bool bad = false;
    double qe_local = 0.0;
    int stat_local = 0, slow_local = 0;
    const f2 nz = f2_pack(-0.0f, -0.0f);

    for (int64_t t = w;; t += W) {
        const int64_t tile = blockIdx.x + t * (int64_t)gridDim.x;
        if (tile >= ntiles) break;
        int64_t i = tile * 128 + wt;
        bool valid = i < a.n;
        // ---- stage the centred point as the split-bf16 A operand ----
        float xn = 0.0f;
        bool xbad = false;
        {
            const float* xr = a.X + i * d;
            for (int c0 = 0; c0 < d16; c0 += 8) {
                float v[8];
                if (valid && (d & 3) == 0 && c0 + 8 <= d) {
                    float4 u0, u1;
                    if (x32) {
                        ldg8(xr + c0, u0, u1);
                    } else {
                        u0 = __ldg(reinterpret_cast<const float4*>(xr + c0));
                        u1 = __ldg(reinterpret_cast<const float4*>(xr + c0 + 4));
                    }
                    v[0] = u0.x; v[1] = u0.y; v[2] = u0.z; v[3] = u0.w;
                    v[4] = u1.x; v[5] = u1.y; v[6] = u1.z; v[7] = u1.w;
                } else {
#pragma unroll
                    for (int q = 0; q < 8; ++q) v[q] = (valid && c0 + q < d) ? __ldg(xr + c0 + q) : 0.0f;
                }
                uint32_t hw[4], lw[4];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    xbad |= !finite_f(v[q]);
                    v[q] = v[q] - cen[c0 + q];  // centred operand (padding dims: 0 - 0)
                }
#pragma unroll
                for (int q = 0; q < 8; q += 2) {
                    xn = fmaf(v[q], v[q], xn);
                    xn = fmaf(v[q + 1], v[q + 1], xn);
                    const uint16_t h0 = bf16_bits(v[q]), h1 = bf16_bits(v[q + 1]);
                    const uint16_t l0 = bf16_bits(v[q] - bf16_val(h0)), l1 = bf16_bits(v[q + 1] - bf16_val(h1));
                    hw[q >> 1] = (uint32_t)h0 | ((uint32_t)h1 << 16);
                    lw[q >> 1] = (uint32_t)l0 | ((uint32_t)l1 << 16);
                }
                const uint32_t o = canon_off(wt, c0, d16);
                *reinterpret_cast<uint4*>(Ahi + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                *reinterpret_cast<uint4*>(Alo + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
        }
        bad |= xbad;
        fence_proxy_async();  // generic smem writes -> async proxy (tensor core)
        const float xnorm = sqrtf(xn);
        const float E2 = 2.0f * tc2_eps(xnorm, lmax, lnmax, d, d16);

        // ---- acquire the TMEM slot: tile t takes slot t%S after use u-1 = t/S - 1
        // was released.  Releases of a slot happen in use order, and this WG's
        // previous tile (t - W) already saw use (t-W)/S - 1 released, so the
        // barrier of use u-1 (one of M per slot) is at most one phase behind:
        // its parity cannot alias (M >= W/S + 1).
        const int slot = (int)(t % S);
        const int64_t use = t / S;
        if (use > 0) mbar_wait(&bar_slot[slot][(use - 1) % M], (uint32_t)(((use - 1) / M) & 1));
        tc_fence_after();
        const uint32_t scol = tmem + (uint32_t)(kTc2SlotCols * slot);

        // one landmark round: |l|^2 into the slot, MMA onto it, wait (all WG threads)
        auto run_round = [&](int r) {
            const int c0r = kTc2SlotCols * r;
            const int nr = min(kTc2SlotCols, gpad - c0r);
            for (int c0 = 0; c0 < nr; c0 += 32) {
                float nv[32];
                const float4* s4 = reinterpret_cast<const float4*>(lns + c0r + c0);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 u = s4[q];
                    nv[4 * q] = u.x; nv[4 * q + 1] = u.y; nv[4 * q + 2] = u.z; nv[4 * q + 3] = u.w;
                }
                tmem_st32(scol + lane_off + (uint32_t)c0, nv);
            }
            tmem_wait_st();
            tc_fence_before();
            named_bar(1 + w, 128);
            if (wt == 0) {
                tc_fence_after();
                const uint32_t idesc = umma_idesc_bf16(128, nr);
                const uint32_t ah = smem_u32(Ahi), al = smem_u32(Alo);
                const uint32_t boff = (uint32_t)(c0r >> 3) * sbo;
                const uint32_t bh = smem_u32(Bhi) + boff, bl = smem_u32(Blo) + boff;
                for (int ks = 0; ks < (d16 >> 4); ++ks) {
                    const uint32_t ko = (uint32_t)ks * 256u;
                    umma_bf16(scol, umma_desc(ah + ko, lbo, sbo), umma_desc(bh + ko, lbo, sbo), idesc, 1);
                    umma_bf16(scol, umma_desc(ah + ko, lbo, sbo), umma_desc(bl + ko, lbo, sbo), idesc, 1);
                    umma_bf16(scol, umma_desc(al + ko, lbo, sbo), umma_desc(bh + ko, lbo, sbo), idesc, 1);
                }
                umma_commit(&bar_mma[w]);
            }
            mbar_wait(&bar_mma[w], mma_phase);
            mma_phase ^= 1u;
            tc_fence_after();
            return nr;
        };

        // ---- pass A: minima of the 32 landmark groups j = q (mod 32) ----
        float gm[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) gm[q] = kInf;
        for (int r = 0; r < R; ++r) {
            const int nr = run_round(r);
            int c0 = 0;
            for (; c0 + 64 <= nr; c0 += 64) {
                uint32_t v0[32], v1[32];
                tmem_ld32_async(scol + lane_off + (uint32_t)c0, v0);
                tmem_ld32_async(scol + lane_off + (uint32_t)(c0 + 32), v1);
                tmem_wait_ld();
#pragma unroll
                for (int q = 0; q < 32; ++q) gm[q] = fmin3(gm[q], __uint_as_float(v0[q]), __uint_as_float(v1[q]));
            }
            if (c0 < nr) {
                uint32_t v0[32];
                tmem_ld32_async(scol + lane_off + (uint32_t)c0, v0);
                tmem_wait_ld();
#pragma unroll
                for (int q = 0; q < 32; ++q) gm[q] = fminf(gm[q], __uint_as_float(v0[q]));
            }
        }
        const float tau = kth_of_32<KP>(gm, k);
        const float tcut = tau + E2 + 9.6e-7f * fabsf(tau);
        // ---- pass B: candidate bitmap (bit q of word c/32 <=> D~_c <= tcut) and
        // the mask of non-empty words (gpad <= 1024: one 32-bit word) ----
        int cnt = 0;
        uint32_t nzw = 0;
        int first = -1;  // a candidate (split mode: locality sort key)
        // the last round of pass A is still in the slot: pass B starts with it (no
        // MMA recompute), then redoes rounds 0 .. R-2
        for (int rr = 0; rr < R; ++rr) {
            const int r = rr == 0 ? R - 1 : rr - 1;
            const int nr = rr > 0 ? run_round(r) : min(kTc2SlotCols, gpad - kTc2SlotCols * r);
            const int wb = (kTc2SlotCols * r) >> 5;
            for (int c0 = 0; c0 < nr; c0 += 32) {
                uint32_t v0[32];
                tmem_ld32_async(scol + lane_off + (uint32_t)c0, v0);
                tmem_wait_ld();
                const uint32_t m = le_mask32(v0, tcut, std::make_integer_sequence<int, 32>{});
                const int wd = wb + (c0 >> 5);
                if (SPLIT) {
                    if (valid) a.cbits[(size_t)i * nwords + wd] = m;
                    // locality key: the first candidate met (lowest one of the first round
                    // visited that has any) -- any candidate groups a cluster's points
                    if (first < 0 && m) first = 32 * wd + __ffs(m) - 1;
                } else {
                    bmap[(size_t)wd * 128] = m;
                }
                nzw |= (m != 0u) ? (1u << wd) : 0u;
                cnt += __popc(m);
            }
        }
        // ---- release the slot: the next tile's MMA may overwrite it ----
        tc_fence_before();
        mbar_arrive(&bar_slot[slot][use % M]);
        if (SPLIT) {  // the exact phase runs in knn_exact_bits_kernel
            if (valid) {
                a.cinfo[i] = make_int2(xbad ? -1 : cnt, (int)nzw);
                if (a.ckey) a.ckey[i] = first < 0 ? 0 : first;
            }
            stat_local += valid ? cnt : 0;
            continue;
        }

        const uint32_t* bx;  // bitmap column of the point this thread re-evaluates
        // ---- locality: the WG's threads take the tile's points in order of their
        // lowest candidate (points of one cluster share candidate rows, so a warp's
        // row loads hit the same smem banks / L1 lines); bitonic sort of 128 keys
        {
            const int w0 = __ffs(nzw) - 1;
            const uint32_t m0 = w0 >= 0 ? bmap[(size_t)w0 * 128] : 0u;
            const uint32_t j0 = (valid && m0) ? (uint32_t)(32 * w0 + __ffs(m0) - 1) : 0xFFFFFFu;
            pkey[wt] = (j0 << 7) | (uint32_t)wt;
            pkey[128 + wt] = (uint32_t)cnt;
            pkey[256 + wt] = nzw;
            pkey[384 + wt] = (valid ? 1u : 0u) | (xbad ? 2u : 0u);
            named_bar(1 + w, 128);
            for (int size = 2; size <= 128; size <<= 1) {
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    const int pt = wt ^ stride;
                    if (pt > wt) {
                        const uint32_t ka = pkey[wt], kb = pkey[pt];
                        if ((ka > kb) == ((wt & size) == 0)) {
                            pkey[wt] = kb;
                            pkey[pt] = ka;
                        }
                    }
                    named_bar(1 + w, 128);
                }
            }
            const int pp = (int)(pkey[wt] & 127u);
            stat_local += cnt;
            cnt = (int)pkey[128 + pp];
            nzw = pkey[256 + pp];
            const uint32_t fl = pkey[384 + pp];
            named_bar(1 + w, 128);  // pkey is rewritten by this WG's next tile
            i = tile * 128 + pp;
            valid = (fl & 1u) != 0;
            xbad = (fl & 2u) != 0;
            bx = bmap0 + pp;
        }

        // ---- exact phase: reference f32 distances of the candidates, index order ----
        if (!valid) continue;
        int32_t* oi = a.out_idx ? a.out_idx + i * k : nullptr;
        float* od = a.out_sqd ? a.out_sqd + i * k : nullptr;
        int b0 = 0;
        float d0 = 0.0f;
        int written = 0;
        if (!xbad) {
            float x[32];
            const float* xr = a.X + i * d;
            if (x32) {
#pragma unroll
                for (int c = 0; c < 32; c += 8) {
                    float4 u = make_float4(0.f, 0.f, 0.f, 0.f), u2 = u;
                    if (c < d) ldg8(xr + c, u, u2);
                    x[c] = u.x; x[c + 1] = u.y; x[c + 2] = u.z; x[c + 3] = u.w;
                    x[c + 4] = u2.x; x[c + 5] = u2.y; x[c + 6] = u2.z; x[c + 7] = u2.w;
                }
            } else if ((d & 3) == 0) {
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (c < d) u = __ldg(reinterpret_cast<const float4*>(xr + c));
                    x[c] = u.x; x[c + 1] = u.y; x[c + 2] = u.z; x[c + 3] = u.w;
                }
            } else {
#pragma unroll
                for (int c = 0; c < 32; ++c) x[c] = c < d ? __ldg(xr + c) : 0.0f;
            }
            float td[KP];
            int ti[KP];
#pragma unroll
            for (int q = 0; q < KP; ++q) {
                td[q] = q >= off ? kInf : -kInf;
                ti[q] = a.g;
            }
            const int d4 = (d16 + 3) >> 2;  // float4 steps (rows zero-padded to ls >= d16)
            int wi = 0;
            uint32_t m = 0;
            for (int e = 0; e < cnt; e += 4) {
                int jq[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {  // next set bit in index order (branch-free word advance)
                    if (m == 0u) {
                        wi = __ffs(nzw) - 1;  // nzw == 0 only past the last candidate (jq unused)
                        nzw &= nzw - 1u;
                        m = bx[(size_t)(wi < 0 ? 0 : wi) * 128];
                    }
                    jq[u] = max(32 * wi + (__ffs(m) - 1), 0);  // past the last candidate: any valid row
                    m &= m - 1u;
                }
                const float4* lr[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) lr[u] = reinterpret_cast<const float4*>(Lr + (size_t)jq[u] * ls);
                float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                for (int c4 = 0; c4 < 8; ++c4) {
                    if (c4 < d4) {
                        const f2 x01 = f2_pack(x[4 * c4], x[4 * c4 + 1]);
                        const f2 x23 = f2_pack(x[4 * c4 + 2], x[4 * c4 + 3]);
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const float4 l4 = RS ? lr[u][c4] : __ldg(lr[u] + c4);
                            const f2 q01 = f2_sq(f2_sub(x01, f2_pack(l4.x, l4.y)), nz);
                            const f2 q23 = f2_sq(f2_sub(x23, f2_pack(l4.z, l4.w)), nz);
                            float a0, a1, a2, a3;
                            f2_unpack(q01, a0, a1);
                            f2_unpack(q23, a2, a3);
                            s4[u] = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s4[u], a0), a1), a2), a3);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int jo = a.rowmap ? __ldg(a.rowmap + jq[u]) : jq[u];  // screen row -> landmark
                    if (e + u < cnt && key_lt(s4[u], jo, td[KP - 1], ti[KP - 1])) topk_insert_lex<KP>(td, ti, s4[u], jo);
                }
            }
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
            // non-finite input or overflowing distances: the reference's insertion scan
            const SlowNearest sn = knn_point_slow(a.X + i * d, d, a.L, a.g, k, oi, od);
            b0 = sn.b0;
            d0 = sn.d0;
            ++slow_local;
        }
        if (a.bmu) a.bmu[i] = b0;
        if (a.qe_sum) qe_local += (double)d0;
        if (a.accS) {
            atomicAdd(a.accC + b0, 1ull);
            for (int c = 0; c < d; ++c) atomicAdd(a.accS + (int64_t)b0 * d + c, acc_fx(__ldg(a.X + i * d + c), a.acc_scale));
        }
    }
    flag_nonfinite(a.flag, bad);
    if (a.stats && stat_local) atomicAdd(a.stats, stat_local);
    if (a.stats && slow_local) atomicAdd(a.stats + 1, slow_local);
    if (a.qe_sum) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) qe_local += __shfl_xor_sync(0xffffffffu, qe_local, o);
        if ((tid & 31) == 0 && qe_local != 0.0) atomicAdd(a.qe_sum, qe_local);
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int W>
size_t tc2_smem_bytes(const Tc2Args& a, bool rows_smem, bool split = false) {
    size_t b = 2 * (size_t)a.gpad * a.d16 * 2;                             // B hi/lo
    b += ((size_t)a.gpad * 4 + 127) / 128 * 128;                           // |l|^2
    if (rows_smem && !split) b += ((size_t)a.gpad * a.ls * 4 + 127) / 128 * 128;  // f32 rows
    b += (size_t)W * 2 * 128 * a.d16 * 2;                                  // A hi/lo per WG
    if (!split) {
        b += (size_t)W * (a.gpad / 32) * 128 * 4;                          // candidate bitmaps
        b += (size_t)W * 4 * 128 * 4;                                      // locality sort keys
    }
    return b + 256;
}

template <int KP, int W>
int launch_tc2_t(Tc2Args a, cudaStream_t st) {
    const size_t cap = (size_t)esom_host::max_smem_optin();
    const bool split = a.cbits != nullptr;
    const bool rs = !split && tc2_smem_bytes<W>(a, true) <= cap;
    const size_t smem = tc2_smem_bytes<W>(a, rs, split);
    if (smem > cap) return esom_host::set_err(ESOM_ERR_UNSUPPORTED, "tc2: shape exceeds shared memory%s", "");
    auto kern = split ? knn_tc2_kernel<KP, W, false, true>
                      : (rs ? knn_tc2_kernel<KP, W, true, false> : knn_tc2_kernel<KP, W, false, false>);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t ntiles = (a.n + 127) / 128;
    int64_t grid = esom_host::num_sms();
    const int64_t need = (ntiles + W - 1) / W;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, 128 * W, smem, st>>>(a);
    return esom_host::cuda_check("knn_tc2_kernel");
}

// ---------------------------------------------------------------------------
// Exact phase of the split screen (g > 256, esom_tc2.cuh SPLIT mode): thread =
// point, landmark rows (gpad x ls f32, up to 147 KB at g = 1024) staged once per
// CTA by TMA, candidate bitmaps from the screen; same arithmetic and ordered
// insertion as the fused kernel.  Splitting frees the screen's shared memory
// (B stays resident, more warpgroups) and gives the exact phase the rows.
// ---------------------------------------------------------------------------
constexpr int kExactBitsThreads = 512;

// One point of the exact phase: the reference-exact top k of the point's
// candidates (bitmap in bsm, screen rows in Ls, row map rmap), in (distance,
// landmark index) order.  rj / rd hold the k results in slots [KP - k, KP);
// written = k unless the point needs the reference scan (non-finite input or
// overflowing distances).  Shared by knn_exact_bits_kernel and the fused
// embed kernel (esom_fused.cuh).
struct ExactPoint {
    int b0;
    float d0;
    int written;
};

// LIST: the candidates are first unpacked into a per-thread index list in shared
// memory (lst: [e][BS] u16, up to kExactListCap entries) while the point's x row is
// in flight, so the distance loop reads its next landmark with one independent
// load instead of the bitmap word -> ffs -> row-address chain (points with more
// candidates walk the bitmap as before).
constexpr int kExactListCap = 32;

template <int KP, int BS = kExactBitsThreads, bool LIST = false>  // BS: thread stride of bsm / lst
__device__ __forceinline__ ExactPoint exact_bits_point(const Tc2Args& a, int64_t i, int cnt, uint32_t nzw,
                                                       const float* __restrict__ Ls, const uint32_t* bsm,
                                                       const int32_t* rmap, int (&rj)[KP], float (&rd)[KP],
                                                       uint16_t* lst = nullptr) {
    const int d = a.d, d16 = a.d16, k = a.k, ls = a.ls;
    const int off = KP - k;
    const f2 nz2 = f2_pack(-0.0f, -0.0f);
    const int d4 = (d16 + 3) >> 2;
    const bool full = d4 == 8;
    const bool x32 = rows32(a.X, d);
        int b0 = 0;
        float d0 = 0.0f;
        int written = 0;
        if (cnt >= 0) {
            float x[32];
            const float* xr = a.X + i * d;
            if (x32) {
#pragma unroll
                for (int c = 0; c < 32; c += 8) {
                    float4 u = make_float4(0.f, 0.f, 0.f, 0.f), u2 = u;
                    if (c < d) ldg8(xr + c, u, u2);
                    x[c] = u.x; x[c + 1] = u.y; x[c + 2] = u.z; x[c + 3] = u.w;
                    x[c + 4] = u2.x; x[c + 5] = u2.y; x[c + 6] = u2.z; x[c + 7] = u2.w;
                }
            } else if ((d & 3) == 0) {
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (c < d) u = __ldg(reinterpret_cast<const float4*>(xr + c));
                    x[c] = u.x; x[c + 1] = u.y; x[c + 2] = u.z; x[c + 3] = u.w;
                }
            } else {
#pragma unroll
                for (int c = 0; c < 32; ++c) x[c] = c < d ? __ldg(xr + c) : 0.0f;
            }
            const uint32_t nzw0 = nzw;
            const bool listed = LIST && cnt <= kExactListCap;
            if (listed) {  // unpack the bitmap (index order) while x is loading
                int e = 0;
                uint32_t nz = nzw;
                while (nz) {
                    const int w = __ffs(nz) - 1;
                    nz &= nz - 1u;
                    uint32_t m = bsm[w * BS];
                    while (m) {
                        lst[e * BS] = (uint16_t)(32 * w + __ffs(m) - 1);
                        ++e;
                        m &= m - 1u;
                    }
                }
            }
            int cur_e = 0;  // list cursor
            // exact distances of the next 4 candidates of the bitmap (index order)
            auto next4 = [&](int& wi, uint32_t& m, uint32_t& nz, int* jq, float* s4) {
                if (LIST && listed) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int e = cur_e + u;
                        jq[u] = e < cnt ? (int)lst[e * BS] : 0;  // past the last candidate: any valid row
                    }
                    cur_e += 4;
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (m == 0u) {
                            wi = __ffs(nz) - 1;
                            nz &= nz - 1u;
                            m = bsm[(wi < 0 ? 0 : wi) * BS];
                        }
                        jq[u] = max(32 * wi + (__ffs(m) - 1), 0);  // past the last candidate: any valid row
                        m &= m - 1u;
                    }
                }
                const float4* lr[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) lr[u] = reinterpret_cast<const float4*>(Ls + (size_t)jq[u] * ls);
#pragma unroll
                for (int u = 0; u < 4; ++u) s4[u] = 0.0f;
                if (full) {
                    // d16 == 32: no per-chunk guard, so the row loads of the next
                    // chunk are issued while the current one is summed (one-chunk
                    // register prefetch hides the shared-memory latency)
                    float4 cur[4], nxt[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) cur[u] = lr[u][0];
#pragma unroll
                    for (int c4 = 0; c4 < 8; ++c4) {
                        if (c4 < 7) {
#pragma unroll
                            for (int u = 0; u < 4; ++u) nxt[u] = lr[u][c4 + 1];
                        }
                        const f2 x01 = f2_pack(x[4 * c4], x[4 * c4 + 1]);
                        const f2 x23 = f2_pack(x[4 * c4 + 2], x[4 * c4 + 3]);
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const float4 l4 = cur[u];
                            const f2 q01 = f2_sq(f2_sub(x01, f2_pack(l4.x, l4.y)), nz2);
                            const f2 q23 = f2_sq(f2_sub(x23, f2_pack(l4.z, l4.w)), nz2);
                            float a0, a1, a2, a3;
                            f2_unpack(q01, a0, a1);
                            f2_unpack(q23, a2, a3);
                            s4[u] = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s4[u], a0), a1), a2), a3);
                        }
                        if (c4 < 7) {
#pragma unroll
                            for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
                        }
                    }
                    return;
                }
#pragma unroll
                for (int c4 = 0; c4 < 8; ++c4) {
                    if (c4 < d4) {
                        const f2 x01 = f2_pack(x[4 * c4], x[4 * c4 + 1]);
                        const f2 x23 = f2_pack(x[4 * c4 + 2], x[4 * c4 + 3]);
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const float4 l4 = lr[u][c4];
                            const f2 q01 = f2_sq(f2_sub(x01, f2_pack(l4.x, l4.y)), nz2);
                            const f2 q23 = f2_sq(f2_sub(x23, f2_pack(l4.z, l4.w)), nz2);
                            float a0, a1, a2, a3;
                            f2_unpack(q01, a0, a1);
                            f2_unpack(q23, a2, a3);
                            s4[u] = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s4[u], a0), a1), a2), a3);
                        }
                    }
                }
            };
            bool done = false;
            if (KP == 16 && k == 16) {
                // batches of 8: sort, half-clean + bitonic-merge into the sorted 16-list
                float L[16], dmin = kInf;
                int LJ[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    L[q] = kInf;
                    LJ[q] = a.g;
                }
                int wi = 0;
                uint32_t m = 0, nz = nzw0;
                cur_e = 0;
                for (int e = 0; e < cnt; e += 8) {
                    float bv[8];
                    int bj[8];
                    next4(wi, m, nz, bj, bv);
                    if (e + 4 < cnt) {
                        next4(wi, m, nz, bj + 4, bv + 4);
                    } else {
#pragma unroll
                        for (int u = 4; u < 8; ++u) bv[u] = kInf;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (e + u >= cnt) bv[u] = kInf;
                    sort8_vj(bv, bj);
                    merge16_8(L, LJ, bv, bj, dmin);
                }
                bool amb = !(L[15] < kInf) || dmin == L[15];
#pragma unroll
                for (int q = 0; q < 15; ++q) amb |= L[q] == L[q + 1];
                if (!amb) {  // distinct distances: value order is the (d, j) order
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        rj[q] = rmap[LJ[q]];
                        rd[q] = L[q];
                    }
                    b0 = rmap[LJ[0]];
                    d0 = L[0];
                    written = k;
                    done = true;
                }
            }
            if (!done) {  // k < KP, or equal distances: index-ordered insertion
                float td[KP];
                int ti[KP];
#pragma unroll
                for (int q = 0; q < KP; ++q) {
                    td[q] = q >= off ? kInf : -kInf;
                    ti[q] = a.g;
                }
                int wi = 0;
                uint32_t m = 0, nz = nzw0;
                cur_e = 0;
                for (int e = 0; e < cnt; e += 4) {
                    int jq[4];
                    float s4[4];
                    next4(wi, m, nz, jq, s4);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int jo = rmap[jq[u]];  // screen row -> landmark index
                        if (e + u < cnt && key_lt(s4[u], jo, td[KP - 1], ti[KP - 1]))
                            topk_insert_lex<KP>(td, ti, s4[u], jo);
                    }
                }
#pragma unroll
                for (int q = 0; q < KP; ++q) {
                    rj[q] = ti[q];
                    rd[q] = td[q];
                    if (q >= off) {
                        written += ti[q] < a.g ? 1 : 0;
                        if (q == off) {
                            b0 = ti[q];
                            d0 = td[q];
                        }
                    }
                }
            }
        }
    return ExactPoint{b0, d0, written};
}

template <int KP, bool LIST>
__global__ void __launch_bounds__(kExactBitsThreads, 1) knn_exact_bits_kernel(Tc2Args a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bar_load;
    const int tid = threadIdx.x;
    const int d = a.d, k = a.k, ls = a.ls;
    const int off = KP - k;
    const int nwords = a.gpad >> 5;
    float* Ls = reinterpret_cast<float*>(smem_raw);
    const uint32_t r_bytes = (uint32_t)a.gpad * ls * 4u;
    // per-thread copy of the point's candidate bitmap ([word][thread]): the extraction
    // then waits on shared, not global, memory
    uint32_t* bsm = reinterpret_cast<uint32_t*>(smem_raw + ((r_bytes + 127) / 128) * 128) + tid;
    // screen row -> landmark index (after the bitmaps)
    int32_t* rmap = reinterpret_cast<int32_t*>(bsm - tid + (size_t)nwords * kExactBitsThreads);
    uint16_t* lst = reinterpret_cast<uint16_t*>(rmap + a.gpad) + tid;  // LIST: [e][thread] candidate indices
    for (int j = tid; j < a.gpad; j += kExactBitsThreads) rmap[j] = a.rowmap ? __ldg(a.rowmap + j) : j;
    if (tid == 0) {
        mbar_init(&bar_load, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(&bar_load, r_bytes);
        tma_bulk_g2s(Ls, a.Lrow, r_bytes, &bar_load);
    }
    mbar_wait(&bar_load, 0);
    double qe_local = 0.0;
    int slow_local = 0;
    for (int64_t pos = blockIdx.x * (int64_t)kExactBitsThreads + tid; pos < a.n;
         pos += (int64_t)gridDim.x * kExactBitsThreads) {
        // points grouped by lowest candidate: a warp's lanes share landmark rows (smem broadcasts)
        const int64_t i = a.perm ? (int64_t)__ldg(a.perm + pos) : pos;
        const int2 info = a.cinfo[i];
        const int cnt = info.x;
        uint32_t nzw = (uint32_t)info.y;
        {
            const uint32_t* bg = a.cbits + (size_t)i * nwords;
            if ((nwords & 3) == 0) {
                for (int w4 = 0; w4 < nwords; w4 += 4) {
                    const uint4 u = __ldg(reinterpret_cast<const uint4*>(bg + w4));
                    bsm[(w4 + 0) * kExactBitsThreads] = u.x;
                    bsm[(w4 + 1) * kExactBitsThreads] = u.y;
                    bsm[(w4 + 2) * kExactBitsThreads] = u.z;
                    bsm[(w4 + 3) * kExactBitsThreads] = u.w;
                }
            } else {
                for (int w1 = 0; w1 < nwords; ++w1) bsm[w1 * kExactBitsThreads] = __ldg(bg + w1);
            }
        }
        int rj[KP];
        float rd[KP];
        ExactPoint ep = exact_bits_point<KP, kExactBitsThreads, LIST>(a, i, cnt, nzw, Ls, bsm, rmap, rj, rd, lst);
        int32_t* oi = a.out_idx ? a.out_idx + i * k : nullptr;
        float* od = a.out_sqd ? a.out_sqd + i * k : nullptr;
        int b0 = ep.b0;
        float d0 = ep.d0;
        const int written = ep.written;
        if (written == k && oi) {
#pragma unroll
            for (int q = 0; q < KP; ++q)
                if (q >= off) {
                    oi[q - off] = rj[q];
                    od[q - off] = rd[q];
                }
        }
        if (written != k) {
            const SlowNearest sn = knn_point_slow(a.X + i * d, d, a.L, a.g, k, oi, od);
            b0 = sn.b0;
            d0 = sn.d0;
            ++slow_local;
        }
        if (a.bmu) a.bmu[i] = b0;
        if (a.qe_sum) qe_local += (double)d0;
        if (a.accS) {
            atomicAdd(a.accC + b0, 1ull);
            for (int c = 0; c < d; ++c) atomicAdd(a.accS + (int64_t)b0 * d + c, acc_fx(__ldg(a.X + i * d + c), a.acc_scale));
        }
    }
    if (a.stats && slow_local) atomicAdd(a.stats + 1, slow_local);
    if (a.qe_sum) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) qe_local += __shfl_xor_sync(0xffffffffu, qe_local, o);
        if ((tid & 31) == 0 && qe_local != 0.0) atomicAdd(a.qe_sum, qe_local);
    }
}

template <int KP>
int launch_exact_bits_t(Tc2Args a, cudaStream_t st) {
    const size_t smem = ((size_t)a.gpad * a.ls * 4 + 127) / 128 * 128 + (size_t)(a.gpad / 32) * kExactBitsThreads * 4 +
                        (size_t)a.gpad * 4;  // + the row map
    if (smem > (size_t)esom_host::max_smem_optin())
        return esom_host::set_err(ESOM_ERR_UNSUPPORTED, "exact rows exceed shared memory%s", "");
    const size_t smem_list = smem + (size_t)kExactListCap * kExactBitsThreads * 2;
    const bool list = smem_list <= (size_t)esom_host::max_smem_optin();
    auto kern = list ? knn_exact_bits_kernel<KP, true> : knn_exact_bits_kernel<KP, false>;
    const size_t sm = list ? smem_list : smem;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int64_t grid = (a.n + kExactBitsThreads - 1) / kExactBitsThreads;
    if (grid > esom_host::num_sms()) grid = esom_host::num_sms();
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kExactBitsThreads, sm, st>>>(a);
    return esom_host::cuda_check("knn_exact_bits_kernel");
}

}  // namespace esom
