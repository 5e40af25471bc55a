// esom_tc3.cuh -- tensor-core GEMM screen for high-dimensional EXACT k-NN
// (d > 32, e.g. C5: 2^20 x 512, 4096 landmarks, k = 32; tensor
// bound).  Same exactness contract as esom_tc.cuh / esom_tc2.cuh: the tensor
// cores only prune, the output equals knn_base (ref: knn.py:65-92) bit for bit.
//
// Pipeline (three kernels per <= kT3Chunk points, all on the caller's stream):
//  1. t3_split_points: x' = x - c (c = landmark centroid) as split bf16
//     (hi, lo) in canonical K-major tiles [128-point tile][32-wide K chunk],
//     |x'| per point.  Landmarks were split the same way per model (B = -2 l',
//     tiles [256-landmark round][K chunk]).
//  2. knn_gemm_kernel: a persistent, warp-specialised tcgen05 GEMM.  A CTA owns
//     256 points (two M = 128 tiles sharing every B chunk); one producer warp
//     streams A/B chunks with 1-D TMA bulk copies through a 2-stage smem ring,
//     one MMA warp issues 3 x kind::f16 MMAs per 16-wide K step per tile
//     (x_hi l_hi + x_hi l_lo + x_lo l_hi) into TMEM (2 x 256 columns), and
//     8 epilogue warps (thread = point = TMEM lane) read the accumulators in
//     ONE pass over the landmark rounds: every landmark with D~_j <= cut is
//     logged in smem (<= 64 per thread); when a lane's log could overflow, the
//     warp's lanes with more than k entries compact it (cut -> the k-th smallest
//     logged D~ + 2E, E: per-point error bound, t3_eps; the cut only falls, and
//     the k-th smallest logged D~ bounds the k-th smallest overall).  The final
//     log (<= kT3CMax candidates, index order) and the approximate nearest
//     landmark (for a locality sort) go to the exact kernel.
//  3. knn_exact_group_kernel (d % 8 == 0; else knn_exact_warp_kernel, one warp
//     per point): points in approximate-BMU order, a warp per 4 points; lanes
//     re-evaluate the union of their candidates with the reference's sequential
//     f32 sum (ref: knn.py:56-62), each point ranks its own candidates by
//     (distance, index) and writes the k-NN row.
// A point whose log overflows or whose candidate list exceeds kT3CMax is
// flagged and re-done by the reference insertion scan (knn_point_slow).
#pragma once
#include "esom_tc2.cuh"

namespace esom {

constexpr int kT3Kc = 32;            // K elements per pipeline stage
constexpr int kT3Rows = 256;         // landmarks per round (MMA N)
constexpr int kT3Stages = 2;
constexpr int kT3Epi = 256;          // epilogue threads: two 128-point tiles
constexpr int kT3Threads = kT3Epi + 64;
constexpr int kT3CMax = 64;          // candidates handed to the exact kernel per point
constexpr int kT3LogCap = 64;        // per-thread candidate log in smem
constexpr uint32_t kT3AChunk = 128u * kT3Kc * 2u;   // one A tile chunk (hi or lo), bytes
constexpr uint32_t kT3BChunk = 256u * kT3Kc * 2u;   // one B round chunk (hi or lo), bytes
// MMA N = 128: a 256-landmark round is issued as two half-rounds into
// alternating TMEM buffers (2 x [2 tiles x 128 columns]), so the MMAs of
// half-round h + 1 run while the epilogue reads half-round h (one buffer
// serialised MMA and epilogue: tensor pipe ~54 % active).
constexpr int kT3N = 128;
constexpr uint32_t kT3BHalf = kT3BChunk / 2;          // rows [128 h, 128 h + 128) of a round chunk
constexpr uint32_t kT3Stage = 4u * kT3AChunk + 2u * kT3BHalf;

// Rigorous-by-model bound E on |D~_j - (d_ref_j - |x'|^2)|:
//  split residual 8 2^-18 S; tensor-core accumulation budgeted at 4 2^-23 (N + 2S)
//  per MMA instruction (3 dk/16 of them); |l'|^2 rounding and the epilogue add
//  2^-23 (N + |D|); the reference's own sequential rounding (d + 3) 2^-24 d_true
//  with d_true <= |x'|^2 + tau + 4 + E0; all x2.
__device__ __forceinline__ float t3_eps(float xnorm, float lmax, float lnmax, int d, int dk, float tau) {
    const float S = xnorm * lmax;
    const float nm = 3.0f * (float)(dk >> 4);
    const float e0 = 8.0f * 3.8147e-6f * S + 4.0f * nm * 1.1921e-7f * (lnmax + 2.0f * S) +
                     1.1921e-7f * (2.0f * lnmax + xnorm * xnorm + fabsf(tau));
    const float dtrue = fmaxf(xnorm * xnorm + tau, 0.0f) + 4.0f * e0 + 1.0f;
    return 2.0f * (e0 + (d + 3.0f) * 5.9605e-8f * dtrue);
}


template <int KP>
struct T3Compacted {
    int m;
    float tcut;
};

// One-pass compaction: the k smallest logged D~ persist in shared memory
// (vds, KP slots strided by kT3Epi) across compactions -- an entry a compaction
// drops lies above the cut, so it is never among them -- and only the entries
// logged since the last compaction, [ins, cnt), are inserted.  Then the cut
// falls to the k-th smallest + 2E and the log keeps the entries at or below it.
template <int KP>
__device__ __noinline__ T3Compacted<KP> t3_compact_keep(float* logv, unsigned short* logj, float* vds, int cnt, int ins,
                                                        float xnorm, float lmax, float lnmax, int d, int dk,
                                                        float tcut) {
    float vd[KP];
#pragma unroll
    for (int q = 0; q < KP; ++q) vd[q] = vds[q * kT3Epi];
    for (int e = ins; e < cnt; ++e) {
        const float v = logv[e * kT3Epi];
        if (v < vd[KP - 1]) vlist_insert<KP>(vd, v);
    }
#pragma unroll
    for (int q = 0; q < KP; ++q) vds[q * kT3Epi] = vd[q];
    const float tau = vd[KP - 1];
    const float nt = tau + 2.0f * t3_eps(xnorm, lmax, lnmax, d, dk, tau) + 9.6e-7f * fabsf(tau);
    T3Compacted<KP> r;
    r.tcut = nt < tcut ? nt : tcut;
    int m = 0;
    for (int e = 0; e < cnt; ++e) {
        const float v = logv[e * kT3Epi];
        if (v <= r.tcut) {
            logv[m * kT3Epi] = v;
            logj[m * kT3Epi] = logj[e * kT3Epi];
            ++m;
        }
    }
    r.m = m;
    return r;
}

template <int KP>
__global__ void __launch_bounds__(kT3Threads, 1) knn_gemm_kernel(Tc3Args a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kT3Stages], empty[kT3Stages], tmem_full[2], tmem_empty[2];
    __shared__ uint32_t tmem_base_sh;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int nkc = a.dk / kT3Kc;                 // K chunks
    const int R = a.gpad / kT3N;                  // landmark half-rounds (MMA N = 128)
    const int64_t nsup = (a.n + 255) / 256;       // 256-point super tiles
    unsigned char* stage = smem_raw;
    float* logv = reinterpret_cast<float*>(smem_raw + kT3Stages * kT3Stage);
    unsigned short* logj = reinterpret_cast<unsigned short*>(logv + kT3LogCap * kT3Epi);
    float* vdsm = reinterpret_cast<float*>(logj + kT3LogCap * kT3Epi);  // [KP][kT3Epi]: the k smallest logged

    if (tid == 0) {
        for (int s = 0; s < kT3Stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tmem_full[b], 1);
            mbar_init(&tmem_empty[b], kT3Epi);
        }
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    if (warp == kT3Epi / 32) {
        // ---------------- producer: TMA bulk copies of A / B chunks ----------------
        if ((tid & 31) == 0) {
            uint32_t q = 0;
            for (int64_t st = blockIdx.x; st < nsup; st += gridDim.x)
                for (int r = 0; r < R; ++r)
                    for (int kc = 0; kc < nkc; ++kc, ++q) {
                        const int s = (int)(q % kT3Stages);
                        mbar_wait(&empty[s], ((q / kT3Stages) & 1u) ^ 1u);
                        unsigned char* sb = stage + (size_t)s * kT3Stage;
                        mbar_expect_tx(&full[s], kT3Stage);
                        for (int t = 0; t < 2; ++t) {
                            const size_t ao = ((size_t)(2 * st + t) * nkc + kc) * (kT3AChunk / 2);
                            tma_bulk_g2s(sb + (2 * t) * kT3AChunk, a.Ahi + ao, kT3AChunk, &full[s]);
                            tma_bulk_g2s(sb + (2 * t + 1) * kT3AChunk, a.Alo + ao, kT3AChunk, &full[s]);
                        }
                        const size_t bo = ((size_t)(r >> 1) * nkc + kc) * (kT3BChunk / 2) +
                                          (size_t)(r & 1) * (kT3BHalf / 2);  // bf16 elements
                        tma_bulk_g2s(sb + 4 * kT3AChunk, a.Bhi + bo, kT3BHalf, &full[s]);
                        tma_bulk_g2s(sb + 4 * kT3AChunk + kT3BHalf, a.Blo + bo, kT3BHalf, &full[s]);
                    }
        }
    } else if (warp == kT3Epi / 32 + 1) {
        // ---------------- MMA issuer ----------------
        if ((tid & 31) == 0) {
            uint32_t q = 0, rr = 0;
            const uint32_t idesc = umma_idesc_bf16(128, kT3N);
            const uint32_t sboA = (kT3Kc / 8) * 128, sboB = (kT3Kc / 8) * 128, lbo = 128;
            for (int64_t st = blockIdx.x; st < nsup; st += gridDim.x)
                for (int r = 0; r < R; ++r, ++rr) {
                    const uint32_t buf = rr & 1u;
                    mbar_wait(&tmem_empty[buf], ((rr >> 1) & 1u) ^ 1u);  // epilogue read this buffer's last use
                    tc_fence_after();
                    for (int kc = 0; kc < nkc; ++kc, ++q) {
                        const int s = (int)(q % kT3Stages);
                        mbar_wait(&full[s], (q / kT3Stages) & 1u);
                        tc_fence_after();
                        const uint32_t sb = smem_u32(stage + (size_t)s * kT3Stage);
                        const uint32_t bh = sb + 4 * kT3AChunk, bl = bh + kT3BHalf;
                        for (int ks = 0; ks < kT3Kc / 16; ++ks) {
                            const uint32_t ko = (uint32_t)ks * 256u;
                            for (int t = 0; t < 2; ++t) {
                                const uint32_t ah = sb + (2 * t) * kT3AChunk, al = ah + kT3AChunk;
                                const uint32_t dcol = tmem + buf * 256u + (uint32_t)(kT3N * t);
                                const uint32_t acc0 = (kc | ks) ? 1u : 0u;
                                umma_bf16(dcol, umma_desc(ah + ko, lbo, sboA), umma_desc(bh + ko, lbo, sboB), idesc,
                                          acc0);
                                umma_bf16(dcol, umma_desc(ah + ko, lbo, sboA), umma_desc(bl + ko, lbo, sboB), idesc,
                                          1);
                                umma_bf16(dcol, umma_desc(al + ko, lbo, sboA), umma_desc(bh + ko, lbo, sboB), idesc,
                                          1);
                            }
                        }
                        umma_commit(&empty[s]);  // stage reusable once these MMAs retire
                    }
                    umma_commit(&tmem_full[buf]);
                }
        }
    } else {
        // ---------------- epilogue: thread = point = TMEM lane ----------------
        const int t = tid >> 7;              // tile within the super tile
        const int lane_row = tid & 127;
        const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
        const uint32_t tcol0 = tmem + lane_off + (uint32_t)(kT3N * t);
        const float lmax = __ldg(a.lstats), lnmax = __ldg(a.lstats + 1);
        float* lv = logv + tid;
        unsigned short* lj = logj + tid;
        float* vs = vdsm + tid;
        const int k = a.k;
        uint32_t rr = 0;
        int stat_local = 0, ovf_local = 0;
        for (int64_t st = blockIdx.x; st < nsup; st += gridDim.x) {
            const int64_t i = st * 256 + t * 128 + lane_row;
            const bool valid = i < a.n;
            const float xnorm = valid ? __ldg(a.xnorm + i) : 0.0f;
            int cnt = 0;
            bool ovf = false;
            // ---- one pass: log under a running cut (t3_compact_keep: the k-th smallest
            // logged D~ + 2E).  Whenever a lane's log could overflow with the next 32
            // columns, every lane holding more than k entries compacts: one warp-wide
            // event instead of one per lane (divergent per-lane compactions made an
            // earlier one-pass mode slower than two passes). ----
            float tcut = kInf;
            int ins = 0;  // log entries [ins, cnt) are not among the kept k smallest yet
#pragma unroll
            for (int q = 0; q < KP; ++q) vs[q * kT3Epi] = q >= KP - k ? kInf : -kInf;  // (vlist_init)
            for (int r = 0; r < R; ++r, ++rr) {
                const uint32_t buf = rr & 1u, tcol = tcol0 + buf * 256u;
                mbar_wait(&tmem_full[buf], (rr >> 1) & 1u);
                tc_fence_after();
                const float* lnr = a.ln + (size_t)r * kT3N;
#pragma unroll 1
                for (int c0 = 0; c0 < kT3N; c0 += 32) {
                    uint32_t v0[32];
                    tmem_ld32_async(tcol + (uint32_t)c0, v0);
                    tmem_wait_ld();
                    float vv[32];
                    int need = 0;
#pragma unroll
                    for (int q = 0; q < 32; q += 8) {  // |l'|^2 of 8 columns per 256-bit load (uniform address)
                        float4 l0, l1;
                        ldg8(lnr + c0 + q, l0, l1);
                        const float lq[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            vv[q + u] = __uint_as_float(v0[q + u]) + lq[u];
                            need += vv[q + u] <= tcut ? 1 : 0;
                        }
                    }
                    const bool ev = __any_sync(0xffffffffu, cnt + need > kT3LogCap);
                    if (ev && cnt > k) {
                        const T3Compacted<KP> cr =
                            t3_compact_keep<KP>(lv, lj, vs, cnt, ins, xnorm, lmax, lnmax, a.d, a.dk, tcut);
                        cnt = ins = cr.m;
                        tcut = cr.tcut;
                    }
                    if (a.stats && ev && (tid & 31) == 0) atomicAdd(a.stats + 5, 1);  // warp compaction events
                    const uint16_t j0 = (uint16_t)(r * kT3N + c0);
                    if (__all_sync(0xffffffffu, cnt + need <= kT3LogCap)) {  // (the common case) no overflow: predicated appends
#pragma unroll
                        for (int q = 0; q < 32; ++q) {
                            const bool lg = vv[q] <= tcut;
                            if (lg) {
                                lv[cnt * kT3Epi] = vv[q];
                                lj[cnt * kT3Epi] = (uint16_t)(j0 + q);
                            }
                            cnt += lg ? 1 : 0;
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < 32; ++q) {
                            const float v = vv[q];
                            if (v <= tcut) {
                                if (cnt == kT3LogCap) {
                                    if (a.stats) atomicAdd(a.stats + 6, 1);  // per-lane (divergent) compactions
                                    const T3Compacted<KP> cr =
                                        t3_compact_keep<KP>(lv, lj, vs, cnt, ins, xnorm, lmax, lnmax, a.d, a.dk, tcut);
                                    cnt = ins = cr.m;
                                    tcut = cr.tcut;
                                    ovf |= cnt == kT3LogCap;
                                }
                                if (cnt < kT3LogCap && v <= tcut) {
                                    lv[cnt * kT3Epi] = v;
                                    lj[cnt * kT3Epi] = (unsigned short)(r * kT3N + c0 + q);
                                    ++cnt;
                                }
                            }
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(&tmem_empty[buf]);
            }
            if (!valid) continue;
            // ---- refine and hand the candidates to the exact kernel ----
            if (!ovf && cnt > k) {
                const T3Compacted<KP> cr =
                    t3_compact_keep<KP>(lv, lj, vs, cnt, ins, xnorm, lmax, lnmax, a.d, a.dk, tcut);
                cnt = cr.m;
            }
            int best = 0;
            float bv = kInf;
            unsigned short* outc = a.cand + (size_t)i * kT3CMax;
            const bool fits = !ovf && cnt <= kT3CMax;
            for (int e = 0; e < cnt; ++e) {
                const float v = lv[e * kT3Epi];
                const unsigned short j = lj[e * kT3Epi];
                if (v < bv) {
                    bv = v;
                    best = j;
                }
                if (fits) outc[e] = j;
            }
            a.ccount[i] = fits ? cnt : -1;  // -1: exact kernel runs the reference scan for this point
            a.bmu_approx[i] = best;
            stat_local += cnt;
            ovf_local += fits ? 0 : 1;
        }
        if (a.stats) {
            if (stat_local) atomicAdd(a.stats, stat_local);
            if (ovf_local) atomicAdd(a.stats + 1, ovf_local);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int KP>
int launch_gemm_t(Tc3Args a, cudaStream_t st) {
    const size_t smem = (size_t)kT3Stages * kT3Stage + (size_t)kT3LogCap * kT3Epi * 6 + (size_t)KP * kT3Epi * 4 + 128;
    if (smem > (size_t)esom_host::max_smem_optin())
        return esom_host::set_err(ESOM_ERR_UNSUPPORTED, "gemm screen: shared memory%s", "");
    auto kern = knn_gemm_kernel<KP>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t nsup = (a.n + 255) / 256;
    int64_t grid = esom_host::num_sms();
    if (grid > nsup) grid = nsup;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kT3Threads, smem, st>>>(a);
    return esom_host::cuda_check("knn_gemm_kernel");
}

// ---------------------------------------------------------------------------
// Operand preparation: one warp per row; lane l handles the 8-wide K groups
// l, l + 32, ... (coalesced 32-byte reads).  Canonical no-swizzle K-major
// layout per (row block, 32-wide K chunk): [8-row group][8-elem K group][8 rows][8 elems].
// ---------------------------------------------------------------------------
__device__ __forceinline__ size_t t3_canon(int64_t row, int c, int rows_blk, int nkc) {
    const int64_t blk = row / rows_blk;
    const int r = (int)(row % rows_blk), kc = c / kT3Kc, cc = c % kT3Kc;
    return ((size_t)blk * nkc + kc) * ((size_t)rows_blk * kT3Kc) +
           (size_t)(((r >> 3) * (kT3Kc / 8) + (cc >> 3)) * 64 + (r & 7) * 8);
}

// scale = 1 for points (x - c), -2 for landmarks (B = -2 (l - c)); nrm: |v'| (points) or |l'|^2 (landmarks)
__global__ void t3_split_kernel(const float* __restrict__ X, int64_t n, int64_t npad, int d, int dk,
                                const float* __restrict__ cen, float scale, int rows_blk, uint16_t* __restrict__ Hi,
                                uint16_t* __restrict__ Lo, float* __restrict__ nrm, int nrm_sq, float* __restrict__ lstats,
                                int32_t* flag) {
    const int lane = threadIdx.x & 31;
    const int64_t wpb = blockDim.x >> 5;
    const int nkc = dk / kT3Kc;
    bool bad = false;
    for (int64_t row = blockIdx.x * wpb + (threadIdx.x >> 5); row < npad; row += (int64_t)gridDim.x * wpb) {
        const bool valid = row < n;
        double s = 0.0;
        for (int c0 = lane * 8; c0 < dk; c0 += 256) {
            float v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int c = c0 + q;
                float x = 0.0f;
                if (valid && c < d) {
                    x = X[row * d + c];
                    bad |= !finite_f(x);
                    x = x - cen[c];
                }
                s += (double)x * (double)x;
                v[q] = scale * x;
            }
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int q = 0; q < 8; q += 2) {
                const uint16_t h0 = bf16_bits(v[q]), h1 = bf16_bits(v[q + 1]);
                const uint16_t l0 = bf16_bits(v[q] - bf16_val(h0)), l1 = bf16_bits(v[q + 1] - bf16_val(h1));
                hw[q >> 1] = (uint32_t)h0 | ((uint32_t)h1 << 16);
                lw[q >> 1] = (uint32_t)l0 | ((uint32_t)l1 << 16);
            }
            const size_t o = t3_canon(row, c0, rows_blk, nkc);
            *reinterpret_cast<uint4*>(Hi + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(Lo + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0 && nrm) {
            if (nrm_sq) {  // landmark norms |l'|^2 (+inf on padding rows) and the bound's maxima
                nrm[row] = valid ? (float)s : __int_as_float(0x7f800000);
                if (valid && lstats) {
                    atomicMax(reinterpret_cast<int*>(lstats), __float_as_int((float)(sqrt(s) * (1.0 + 1e-6))));
                    atomicMax(reinterpret_cast<int*>(lstats + 1), __float_as_int((float)(s * (1.0 + 1e-6))));
                }
            } else if (valid) {
                nrm[row] = (float)(sqrt(s) * (1.0 + 1e-6));  // |x'| rounded up
            }
        }
    }
    if (flag) flag_nonfinite(flag, bad);
}

// ---------------------------------------------------------------------------
// Exact re-evaluation: one warp per point (approximate-BMU order), lane e owns
// candidates e and e + 32; (distance, index) ranks by warp shuffles.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool t3_less(float va, int ja, float vb, int jb) { return va < vb || (va == vb && ja < jb); }

constexpr int kT3ExactWarps = 32;  // one 1024-thread CTA per SM: its warps walk consecutive (BMU-sorted)
                                   // points, so their candidate rows are shared in L1

template <int KP>
__global__ void __launch_bounds__(kT3ExactWarps * 32) knn_exact_warp_kernel(T3ExactArgs a) {
    extern __shared__ __align__(16) float xs_all[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    float* xs = xs_all + (size_t)wib * a.dpad;
    const int d = a.d, k = a.k;
    const f2 nz = f2_pack(-0.0f, -0.0f);
    double qe_local = 0.0;
    const bool vec = (d & 7) == 0;
    // contiguous range of the visiting order per CTA
    const int64_t per = (a.n + gridDim.x - 1) / gridDim.x;
    const int64_t p0 = (int64_t)blockIdx.x * per, p1 = p0 + per < a.n ? p0 + per : a.n;
    for (int64_t pos = p0 + wib; pos < p1; pos += kT3ExactWarps) {
        const int64_t i = a.perm ? (int64_t)__ldg(a.perm + pos) : pos;
        const float* xr = a.X + i * d;
        const int cnt = __ldg(a.ccount + i);
        int32_t* oi = a.out_idx ? a.out_idx + i * k : nullptr;
        float* od = a.out_sqd ? a.out_sqd + i * k : nullptr;
        int b0 = 0;
        float d0 = 0.0f;
        if (cnt < k || cnt > kT3CMax) {
            if (lane == 0) {
                const SlowNearest sn = knn_point_slow(xr, d, a.L, a.g, k, oi, od);
                b0 = sn.b0;
                d0 = sn.d0;
            }
            b0 = __shfl_sync(0xffffffffu, b0, 0);
            d0 = __shfl_sync(0xffffffffu, d0, 0);
        } else {
            for (int c = lane * 4; c < d; c += 128) {
                if ((d & 3) == 0) {
                    *reinterpret_cast<float4*>(xs + c) = __ldg(reinterpret_cast<const float4*>(xr + c));
                } else {
                    for (int q = 0; q < 4 && c + q < d; ++q) xs[c + q] = __ldg(xr + c + q);
                }
            }
            __syncwarp();
            const unsigned short* cr = a.cand + (size_t)i * kT3CMax;
            const bool h0 = lane < cnt, h1 = lane + 32 < cnt;
            const int j0 = h0 ? (int)cr[lane] : 0, j1 = h1 ? (int)cr[lane + 32] : 0;
            float s0 = 0.0f, s1 = 0.0f;
            const float* l0 = a.L + (size_t)j0 * d;
            const float* l1 = a.L + (size_t)j1 * d;
            if (vec) {
                // 8 dims (one full 32-byte sector of the candidate row) per step
                auto acc8 = [&](float s, const float* lr, int c, const float4& xa, const float4& xb) {
                    const float4 la = __ldg(reinterpret_cast<const float4*>(lr + c));
                    const float4 lb = __ldg(reinterpret_cast<const float4*>(lr + c + 4));
                    float q0, q1, q2, q3, q4, q5, q6, q7;
                    f2_unpack(f2_sq(f2_sub(f2_pack(xa.x, xa.y), f2_pack(la.x, la.y)), nz), q0, q1);
                    f2_unpack(f2_sq(f2_sub(f2_pack(xa.z, xa.w), f2_pack(la.z, la.w)), nz), q2, q3);
                    f2_unpack(f2_sq(f2_sub(f2_pack(xb.x, xb.y), f2_pack(lb.x, lb.y)), nz), q4, q5);
                    f2_unpack(f2_sq(f2_sub(f2_pack(xb.z, xb.w), f2_pack(lb.z, lb.w)), nz), q6, q7);
                    s = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s, q0), q1), q2), q3);
                    return __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s, q4), q5), q6), q7);
                };
                for (int c = 0; c < d; c += 8) {
                    const float4 xa = *reinterpret_cast<const float4*>(xs + c);
                    const float4 xb = *reinterpret_cast<const float4*>(xs + c + 4);
                    s0 = acc8(s0, l0, c, xa, xb);
                    if (h1) s1 = acc8(s1, l1, c, xa, xb);
                }
            } else {
                for (int c = 0; c < d; ++c) {
                    const float t0 = __fsub_rn(xs[c], __ldg(l0 + c));
                    s0 = __fadd_rn(s0, __fmul_rn(t0, t0));
                    if (h1) {
                        const float t1 = __fsub_rn(xs[c], __ldg(l1 + c));
                        s1 = __fadd_rn(s1, __fmul_rn(t1, t1));
                    }
                }
            }
            const float v0 = h0 ? s0 : kInf, v1 = h1 ? s1 : kInf;
            const int k0 = h0 ? j0 : 0x7fffffff, k1 = h1 ? j1 : 0x7fffffff;
            int r0 = 0, r1 = 0;
            const int nsrc = cnt < 32 ? cnt : 32;
            for (int sl = 0; sl < nsrc; ++sl) {
                const float wv0 = __shfl_sync(0xffffffffu, v0, sl), wv1 = __shfl_sync(0xffffffffu, v1, sl);
                const int wj0 = __shfl_sync(0xffffffffu, k0, sl), wj1 = __shfl_sync(0xffffffffu, k1, sl);
                r0 += (t3_less(wv0, wj0, v0, k0) ? 1 : 0) + (t3_less(wv1, wj1, v0, k0) ? 1 : 0);
                r1 += (t3_less(wv0, wj0, v1, k1) ? 1 : 0) + (t3_less(wv1, wj1, v1, k1) ? 1 : 0);
            }
            if (h0 && r0 < k && oi) {
                oi[r0] = j0;
                od[r0] = v0;
            }
            if (h1 && r1 < k && oi) {
                oi[r1] = j1;
                od[r1] = v1;
            }
            const unsigned m0 = __ballot_sync(0xffffffffu, h0 && r0 == 0), m1 = __ballot_sync(0xffffffffu, h1 && r1 == 0);
            const int src = m0 ? __ffs(m0) - 1 : __ffs(m1) - 1;
            const float sv = m0 ? v0 : v1;
            const int sj = m0 ? j0 : j1;
            d0 = __shfl_sync(0xffffffffu, sv, src);
            b0 = __shfl_sync(0xffffffffu, sj, src);
        }
        if (lane == 0) {
            if (a.bmu) a.bmu[i] = b0;
            if (a.qe_sum) qe_local += (double)d0;
            if (a.accC) atomicAdd(a.accC + b0, 1ull);
        }
        if (a.accS)
            for (int c = lane; c < d; c += 32) atomicAdd(a.accS + (int64_t)b0 * d + c, acc_fx(__ldg(xr + c), a.acc_scale));
        __syncwarp();
    }
    if (a.qe_sum && lane == 0 && qe_local != 0.0) atomicAdd(a.qe_sum, qe_local);
}

// ---------------------------------------------------------------------------
// Grouped exact re-evaluation (d % 8 == 0): a warp takes 4 consecutive points
// of the approximate-BMU order, forms the union U of their candidate lists
// (<= kT3UMax landmarks; points of one Voronoi cell share most candidates) and
// lane e evaluates landmark U_e against all 4 points (each candidate row is
// read once per group, 4 sequential f32 chains per landmark).  U contains
// every point's true top k, so the top k of U by (distance, index) is exact.
//
// The lanes' row reads are the bound (every lane a different row: one L1
// wavefront per lane per load), so each lane fetches its 32-byte row sector
// with ONE 256-bit load (ld.global.nc.v8.f32 -> LDG.E.ENL2.256) instead of two
// 128-bit loads: 14.6 -> 11.5 ms per 2^20 points at C5.  (A CTA-shared
// cp.async ring of the tile's union rows in shared memory removed the L1
// bound but was slower, 15.7 ms: per-tile barriers at 8-16 warps per SM and
// 3.8-way bank conflicts on the lane-divergent rows.)
// ---------------------------------------------------------------------------
constexpr int kT3GP = 4;       // points per warp group
constexpr int kT3UMax = 96;    // union capacity (three landmark slots per lane)
constexpr int kT3GWarps = 8;   // warps per CTA (two CTAs per SM at d = 512)

__device__ __forceinline__ float acc8f(float s, const float4& la, const float4& lb, const float4& xa, const float4& xb,
                                       f2 nz) {
    float q0, q1, q2, q3, q4, q5, q6, q7;
    f2_unpack(f2_sq(f2_sub(f2_pack(xa.x, xa.y), f2_pack(la.x, la.y)), nz), q0, q1);
    f2_unpack(f2_sq(f2_sub(f2_pack(xa.z, xa.w), f2_pack(la.z, la.w)), nz), q2, q3);
    f2_unpack(f2_sq(f2_sub(f2_pack(xb.x, xb.y), f2_pack(lb.x, lb.y)), nz), q4, q5);
    f2_unpack(f2_sq(f2_sub(f2_pack(xb.z, xb.w), f2_pack(lb.z, lb.w)), nz), q6, q7);
    s = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s, q0), q1), q2), q3);
    return __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s, q4), q5), q6), q7);
}

__host__ __device__ constexpr int t3_group_stride(int dpad, int g) {  // floats per warp, 16-B aligned
    return (kT3GP * dpad + 2 * ((g + 31) / 32) + kT3UMax + 3) / 4 * 4;  // x rows | bitmap | word prefix | list
}

// Set bits of bm[0, gw) -> ascending landmark list out[0, min(U, cap)); returns U.
// pre (nullable): exclusive prefix popcount per word (the list position of the word's first bit).
__device__ __forceinline__ int t3_bits_to_list(const uint32_t* bm, int gw, int* out, int cap, int* pre, int lane) {
    int U = 0;
    for (int w0 = 0; w0 < gw; w0 += 32) {
        const uint32_t m = w0 + lane < gw ? bm[w0 + lane] : 0u;
        const int c = __popc(m);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        int pos = U + incl - c;
        if (pre && w0 + lane < gw) pre[w0 + lane] = pos;
        uint32_t mm = m;
        while (mm) {
            const int b = __ffs(mm) - 1;
            mm &= mm - 1u;
            if (pos < cap) out[pos] = ((w0 + lane) << 5) + b;
            ++pos;
        }
        U += __shfl_sync(0xffffffffu, incl, 31);
    }
    return U;
}

// Per point of subset sm: rank its OWN candidates (its list contains its true top
// k, so the top k of the list is exact; ref: knn.py:84-90) by (distance, index)
// and write the k-NN row and the statistics.  The evaluated distances sit in
// union slots (lane u & 31, slot u >> 5); a candidate's union position u comes
// from the subset's union bitmap bm and its per-word prefix pre.  Lane e takes
// the point's candidates e and e + 32, so the rank loop runs over cnt (~k + 10)
// sources instead of the union (~3k).
// xs (nullable): the points' rows in shared memory (dpad apart), else read from X.
__device__ __forceinline__ void t3_rank_write(const T3ExactArgs& a, int lane, unsigned sm, int64_t ip, int cp,
                                              const uint32_t* bm, const int* pre, const float (&acc)[3][kT3GP],
                                              const float* xs, int dpad, double& qe_local) {
    const int d = a.d, k = a.k;
#pragma unroll
    for (int p = 0; p < kT3GP; ++p) {
        if (!((sm >> p) & 1u)) continue;
        const int64_t i = __shfl_sync(0xffffffffu, ip, p);
        const int c = __shfl_sync(0xffffffffu, cp, p);
        const unsigned short* cr = a.cand + (size_t)i * kT3CMax;
        float cv[2];
        int ck[2], rk[2] = {0, 0};
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int e = 32 * q + lane;
            const bool has = e < c;
            const int j = has ? (int)cr[e] : 0;
            const int u = has ? pre[j >> 5] + __popc(bm[j >> 5] & ((1u << (j & 31)) - 1u)) : 0;
            const float a0 = __shfl_sync(0xffffffffu, acc[0][p], u & 31);
            const float a1 = __shfl_sync(0xffffffffu, acc[1][p], u & 31);
            const float a2 = __shfl_sync(0xffffffffu, acc[2][p], u & 31);
            cv[q] = has ? (u < 32 ? a0 : (u < 64 ? a1 : a2)) : kInf;
            ck[q] = has ? j : 0x7fffffff;
        }
        const int n0 = c < 32 ? c : 32;
        for (int src = 0; src < n0; ++src) {
            const float wv = __shfl_sync(0xffffffffu, cv[0], src);
            const int wj = __shfl_sync(0xffffffffu, ck[0], src);
            rk[0] += t3_less(wv, wj, cv[0], ck[0]) ? 1 : 0;
            rk[1] += t3_less(wv, wj, cv[1], ck[1]) ? 1 : 0;
        }
        for (int src = 0; src < c - 32; ++src) {
            const float wv = __shfl_sync(0xffffffffu, cv[1], src);
            const int wj = __shfl_sync(0xffffffffu, ck[1], src);
            rk[0] += t3_less(wv, wj, cv[0], ck[0]) ? 1 : 0;
            rk[1] += t3_less(wv, wj, cv[1], ck[1]) ? 1 : 0;
        }
        int32_t* oi = a.out_idx ? a.out_idx + i * k : nullptr;
        float* od = a.out_sqd ? a.out_sqd + i * k : nullptr;
        if (oi) {
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (32 * q + lane < c && rk[q] < k) {
                    oi[rk[q]] = ck[q];
                    od[rk[q]] = cv[q];
                }
        }
        const unsigned m0 = __ballot_sync(0xffffffffu, lane < c && rk[0] == 0);
        const unsigned m1 = __ballot_sync(0xffffffffu, 32 + lane < c && rk[1] == 0);
        const int src0 = m0 ? __ffs(m0) - 1 : __ffs(m1) - 1;
        const float d0 = __shfl_sync(0xffffffffu, m0 ? cv[0] : cv[1], src0);
        const int b0 = __shfl_sync(0xffffffffu, m0 ? ck[0] : ck[1], src0);
        if (lane == 0) {
            if (a.bmu) a.bmu[i] = b0;
            if (a.qe_sum) qe_local += (double)d0;
            if (a.accC) atomicAdd(a.accC + b0, 1ull);
        }
        if (a.accS) {
            const float* xr = a.X + i * d;
            for (int cc = lane; cc < d; cc += 32)
                atomicAdd(a.accS + (int64_t)b0 * d + cc, acc_fx(xs ? xs[p * dpad + cc] : __ldg(xr + cc), a.acc_scale));
        }
    }
}

// Points of the group the screen could not bound (log overflow / too few
// candidates): the reference insertion scan.
__device__ __forceinline__ void t3_slow_points(const T3ExactArgs& a, int lane, int64_t gpos, int64_t p1, unsigned nmask,
                                               int64_t ip, double& qe_local) {
    const int d = a.d, k = a.k;
    for (int p = 0; p < kT3GP; ++p) {
        if (gpos + p >= p1) break;
        if ((nmask >> p) & 1u) continue;
        const int64_t i = __shfl_sync(0xffffffffu, ip, p);
        int32_t* oi = a.out_idx ? a.out_idx + i * k : nullptr;
        float* od = a.out_sqd ? a.out_sqd + i * k : nullptr;
        const float* xr = a.X + i * d;
        int b0 = 0;
        if (lane == 0) {
            const SlowNearest sn = knn_point_slow(xr, d, a.L, a.g, k, oi, od);
            b0 = sn.b0;
            if (a.bmu) a.bmu[i] = b0;
            if (a.qe_sum) qe_local += (double)sn.d0;
            if (a.accC) atomicAdd(a.accC + b0, 1ull);
        }
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (a.accS)
            for (int c = lane; c < d; c += 32) atomicAdd(a.accS + (int64_t)b0 * d + c, acc_fx(__ldg(xr + c), a.acc_scale));
    }
}

// One warp group from L2: stage the normal points' rows in xs, then per subset
// (all points, else halves, else single points) union -> evaluate -> rank.
template <bool V8>
__device__ __forceinline__ void t3_group_l2(const T3ExactArgs& a, int lane, float* xs, uint32_t* bm, int* pre,
                                            int* ul, int64_t ip, int cp, unsigned nmask, double& qe_local) {
    const int d = a.d, dpad = a.dpad;
    const int gw = (a.g + 31) >> 5;
    const f2 nz = f2_pack(-0.0f, -0.0f);
    for (int p = 0; p < kT3GP; ++p) {
        if (!((nmask >> p) & 1u)) continue;
        const int64_t i = __shfl_sync(0xffffffffu, ip, p);
        const float* xr = a.X + i * d;
        for (int c = lane * 4; c < d; c += 128)
            *reinterpret_cast<float4*>(xs + p * dpad + c) = __ldg(reinterpret_cast<const float4*>(xr + c));
    }
    // (a single point's list has <= kT3CMax <= kT3UMax landmarks, so the split always terminates)
    unsigned todo[8];
    int ntodo = 0;
    if (nmask) todo[ntodo++] = nmask;
    while (ntodo > 0) {
        const unsigned sm = todo[--ntodo];
        __syncwarp();
        for (int w = lane; w < gw; w += 32) bm[w] = 0u;
        __syncwarp();
        for (int p = 0; p < kT3GP; ++p) {
            if (!((sm >> p) & 1u)) continue;
            const int64_t i = __shfl_sync(0xffffffffu, ip, p);
            const int c = __shfl_sync(0xffffffffu, cp, p);
            const unsigned short* cr = a.cand + (size_t)i * kT3CMax;
            for (int e = lane; e < c; e += 32) {
                const int j = cr[e];
                atomicOr(bm + (j >> 5), 1u << (j & 31));
            }
        }
        __syncwarp();
        const int U = t3_bits_to_list(bm, gw, ul, kT3UMax, pre, lane);
        if (a.stats && lane == 0) {
            atomicAdd(a.stats + 2, U);
            atomicAdd(a.stats + (U > kT3UMax ? 4 : 3), 1);
        }
        if (U > kT3UMax) {  // split the subset in two halves
            unsigned lo = 0u, rest = sm;
            const int half = __popc(sm) / 2;
            for (int q = 0; q < half; ++q) {
                const unsigned bit = rest & (0u - rest);
                lo |= bit;
                rest ^= bit;
            }
            todo[ntodo++] = rest;
            todo[ntodo++] = lo;
            continue;
        }
        __syncwarp();
        int jj[3];
        bool hv[3];
        const float* lr[3];
#pragma unroll
        for (int sl = 0; sl < 3; ++sl) {
            hv[sl] = 32 * sl + lane < U;
            jj[sl] = hv[sl] ? ul[32 * sl + lane] : 0;
            lr[sl] = a.L + (size_t)jj[sl] * d;
        }
        float acc[3][kT3GP];
#pragma unroll
        for (int sl = 0; sl < 3; ++sl)
#pragma unroll
            for (int p = 0; p < kT3GP; ++p) acc[sl][p] = 0.0f;
        const bool two = U > 32, three = U > 64;  // warp-uniform slot counts
        // landmark rows stream from L2: the next 8-dim chunk is loaded while the
        // current one is accumulated (one-chunk register prefetch)
        float4 la[3], lb[3];
#pragma unroll
        for (int sl = 0; sl < 3; ++sl) {
            la[sl] = lb[sl] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (sl == 0 || (sl == 1 && two) || (sl == 2 && three)) {
                if (V8) {
                    ldg8(lr[sl], la[sl], lb[sl]);
                } else {
                    la[sl] = __ldg(reinterpret_cast<const float4*>(lr[sl]));
                    lb[sl] = __ldg(reinterpret_cast<const float4*>(lr[sl] + 4));
                }
            }
        }
        for (int c = 0; c < d; c += 8) {
            float4 na[3], nb[3];
#pragma unroll
            for (int sl = 0; sl < 3; ++sl) {
                na[sl] = la[sl];
                nb[sl] = lb[sl];
                if (c + 8 < d && (sl == 0 || (sl == 1 && two) || (sl == 2 && three))) {
                    if (V8) {
                        ldg8(lr[sl] + c + 8, na[sl], nb[sl]);
                    } else {
                        na[sl] = __ldg(reinterpret_cast<const float4*>(lr[sl] + c + 8));
                        nb[sl] = __ldg(reinterpret_cast<const float4*>(lr[sl] + c + 12));
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < kT3GP; ++p) {
                if (!((sm >> p) & 1u)) continue;
                const float4 xa = *reinterpret_cast<const float4*>(xs + p * dpad + c);
                const float4 xb = *reinterpret_cast<const float4*>(xs + p * dpad + c + 4);
                acc[0][p] = acc8f(acc[0][p], la[0], lb[0], xa, xb, nz);
                if (two) acc[1][p] = acc8f(acc[1][p], la[1], lb[1], xa, xb, nz);
                if (three) acc[2][p] = acc8f(acc[2][p], la[2], lb[2], xa, xb, nz);
            }
#pragma unroll
            for (int sl = 0; sl < 3; ++sl) {
                la[sl] = na[sl];
                lb[sl] = nb[sl];
            }
        }
        __syncwarp();
        t3_rank_write(a, lane, sm, ip, cp, bm, pre, acc, xs, dpad, qe_local);
    }
}

template <int KP, bool V8>
__global__ void __launch_bounds__(kT3GWarps * 32, 2) knn_exact_group_kernel(T3ExactArgs a) {
    extern __shared__ __align__(16) float sm_all[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int k = a.k, dpad = a.dpad;
    const int gw = (a.g + 31) >> 5;  // bitmap words
    float* xs = sm_all + (size_t)wib * t3_group_stride(dpad, a.g);
    uint32_t* bm = reinterpret_cast<uint32_t*>(xs + kT3GP * dpad);
    int* pre = reinterpret_cast<int*>(bm + gw);
    int* ul = pre + gw;
    double qe_local = 0.0;
    const int64_t per = ((a.n + gridDim.x - 1) / gridDim.x + kT3GP - 1) / kT3GP * kT3GP;
    const int64_t p0 = (int64_t)blockIdx.x * per, p1 = p0 + per < a.n ? p0 + per : a.n;
    for (int64_t gpos = p0 + (int64_t)wib * kT3GP; gpos < p1; gpos += (int64_t)kT3GWarps * kT3GP) {
        int64_t ip = 0;
        int cp = -1;
        if (lane < kT3GP && gpos + lane < p1) {
            ip = a.perm ? (int64_t)__ldg(a.perm + gpos + lane) : gpos + lane;
            cp = __ldg(a.ccount + ip);
        }
        const unsigned nmask = __ballot_sync(0xffffffffu, lane < kT3GP && cp >= k && cp <= kT3CMax);
        t3_group_l2<V8>(a, lane, xs, bm, pre, ul, ip, cp, nmask, qe_local);
        t3_slow_points(a, lane, gpos, p1, nmask, ip, qe_local);
        __syncwarp();
    }
    if (a.qe_sum && lane == 0 && qe_local != 0.0) atomicAdd(a.qe_sum, qe_local);
}

template <int KP>
int launch_exact_warp_t(T3ExactArgs a, cudaStream_t st) {
    if ((a.d & 7) == 0) {  // (the per-point kernel below measured 22 vs 15 ms at C5)
        const size_t per_warp = (size_t)t3_group_stride(a.dpad, a.g) * 4;
        const size_t smem = (size_t)kT3GWarps * per_warp;
        if (smem <= (size_t)esom_host::max_smem_optin()) {
            const bool v8 = (reinterpret_cast<uintptr_t>(a.L) & 31) == 0;  // 256-bit loads need 32-B rows
            auto kern = v8 ? knn_exact_group_kernel<KP, true> : knn_exact_group_kernel<KP, false>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kT3GWarps * 32, smem);
            if (per_sm < 1) per_sm = 1;
            int64_t grid = (a.n + kT3GWarps * kT3GP - 1) / (kT3GWarps * kT3GP);
            const int64_t cap = (int64_t)esom_host::num_sms() * per_sm;
            if (grid > cap) grid = cap;
            if (grid < 1) grid = 1;
            kern<<<(unsigned)grid, kT3GWarps * 32, smem, st>>>(a);
            return esom_host::cuda_check("knn_exact_group_kernel");
        }
    }
    const size_t smem = (size_t)kT3ExactWarps * a.dpad * 4;
    auto kern = knn_exact_warp_kernel<KP>;
    if (smem > (size_t)esom_host::max_smem_optin())
        return esom_host::set_err(ESOM_ERR_UNSUPPORTED, "exact re-evaluation: d too large%s", "");
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int64_t grid = (a.n + kT3ExactWarps - 1) / kT3ExactWarps;
    const int64_t cap = (int64_t)esom_host::num_sms();
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kT3ExactWarps * 32, smem, st>>>(a);
    return esom_host::cuda_check("knn_exact_warp_kernel");
}

}  // namespace esom
