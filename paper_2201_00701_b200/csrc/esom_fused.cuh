// esom_fused.cuh -- the exact k-NN phase and the projection in ONE kernel
// (embed, d <= 32, k = 16, g <= ~330: the landmark rows, the candidate bitmaps
// and the pair triangle all fit one SM's shared memory).
//
// Per point: the exact re-evaluation of the tensor-core screen's candidates
// (exact_bits_point, esom_tc2.cuh: the reference's sequential f32 distances,
// (distance, index) order) leaves the 16 neighbours and their exact squared
// distances in registers, and the projection (reg2_point, esom_project.cuh:
// scores + law-of-cosines normal equations) consumes them there -- the
// neighbour rows (128 B per point written and read back through HBM by the
// two-kernel path) never leave the SM, and one launch (and one prologue of
// the pair table) disappears per chunk.  The nearest landmark goes to column
// 0 of the point workspace's index rows for the batch-SOM statistics; the
// rare reference-scan and faithful-projection fallbacks stage their rows
// there too.
#pragma once
#include "esom_project.cuh"
#include "esom_tc2.cuh"

namespace esom {

constexpr int kFusedThreads = kExactBitsThreads;  // 512: one CTA per SM, 128 registers (384 threads at 168 registers: slower)

__host__ __device__ inline size_t fused_rows_bytes(int gpad, int ls) { return ((size_t)gpad * ls * 4 + 127) / 128 * 128; }
__host__ __device__ inline size_t fused_proj_offset(int gpad, int ls) {
    // rows | bitmaps [word][thread] | row map | inverse row map | (aligned) projection tables (reg2 layout)
    return (fused_rows_bytes(gpad, ls) + (size_t)(gpad / 32) * kFusedThreads * 4 + (size_t)gpad * 8 + 127) / 128 * 128;
}
inline size_t fused_smem_bytes(int gpad, int ls, int g) { return fused_proj_offset(gpad, ls) + reg2_hi64_offset(g); }
inline size_t fused_list_bytes() { return (size_t)kExactListCap * kFusedThreads * 2; }

template <int KP, bool LIST, bool FH>
__global__ void __launch_bounds__(kFusedThreads, 1) embed_fused_kernel(Tc2Args a, ProjArgs q) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bar_load;
    const int tid = threadIdx.x;
    const int d = a.d, k = a.k, g = a.g;
    const int nwords = a.gpad >> 5;
    float* Ls = reinterpret_cast<float*>(smem_raw);
    const uint32_t r_bytes = (uint32_t)a.gpad * a.ls * 4u;
    uint32_t* bsm = reinterpret_cast<uint32_t*>(smem_raw + fused_rows_bytes(a.gpad, a.ls)) + tid;
    int32_t* rmap = reinterpret_cast<int32_t*>(bsm - tid + (size_t)nwords * kFusedThreads);
    int32_t* inv = rmap + a.gpad;  // landmark -> screen row (the far-point distances read the rows)
    unsigned char* pj = smem_raw + fused_proj_offset(a.gpad, a.ls);
    float2* LO = reinterpret_cast<float2*>(pj);
    int* RB = reinterpret_cast<int*>(LO + g);
    float* tsm = reinterpret_cast<float*>(pj + reg2_tri_offset(g));
    uint16_t* lst = reinterpret_cast<uint16_t*>(pj + reg2_hi64_offset(g)) + tid;  // LIST: candidate indices
    for (int j = tid; j < a.gpad; j += kFusedThreads) {
        const int r = a.rowmap ? __ldg(a.rowmap + j) : j;
        rmap[j] = r;
        if (r < a.gpad) inv[r] = j;
    }
    const int ntri = g * (g - 1) / 2;
    for (int e = tid; e < ntri; e += kFusedThreads) tsm[e] = __ldg(q.T + e);
    for (int j = tid; j < g; j += kFusedThreads) {
        LO[j] = make_float2(q.lo[2 * j], q.lo[2 * j + 1]);
        RB[j] = j * (2 * g - j - 1) / 2 - j - 1;  // tri(j, b) = RB[j] + b for b > j
    }
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
    const float tmax_model = q.tmax ? __ldg(q.tmax) : 0.0f;
    double qe_local = 0.0;
    int slow_local = 0;
    for (int64_t pos = blockIdx.x * (int64_t)kFusedThreads + tid; pos < a.n;
         pos += (int64_t)gridDim.x * kFusedThreads) {
        // points grouped by lowest candidate (the exact phase's locality order)
        const int64_t i = a.perm ? (int64_t)__ldg(a.perm + pos) : pos;
        const int2 info = a.cinfo[i];
        const int cnt = info.x;
        {
            const uint32_t* bgw = a.cbits + (size_t)i * nwords;
            if ((nwords & 3) == 0) {
                for (int w4 = 0; w4 < nwords; w4 += 4) {
                    const uint4 u = __ldg(reinterpret_cast<const uint4*>(bgw + w4));
                    bsm[(w4 + 0) * kFusedThreads] = u.x;
                    bsm[(w4 + 1) * kFusedThreads] = u.y;
                    bsm[(w4 + 2) * kFusedThreads] = u.z;
                    bsm[(w4 + 3) * kFusedThreads] = u.w;
                }
            } else {
                for (int w1 = 0; w1 < nwords; ++w1) bsm[w1 * kFusedThreads] = __ldg(bgw + w1);
            }
        }
        int rj[KP];
        float rd[KP];
        const ExactPoint ep =
            exact_bits_point<KP, kFusedThreads, LIST>(a, i, cnt, (uint32_t)info.y, Ls, bsm, rmap, rj, rd, lst);
        int32_t* wi = const_cast<int32_t*>(q.idx) + i * k;  // point workspace rows (chunk-relative)
        float* wd = const_cast<float*>(q.sqd) + i * k;
        int b0 = ep.b0;
        float d0 = ep.d0;
        if (ep.written != k) {
            // non-finite input or overflowing distances: the reference's insertion scan
            const SlowNearest sn = knn_point_slow(a.X + i * d, d, a.L, g, k, wi, wd);
            b0 = sn.b0;
            d0 = sn.d0;
            ++slow_local;
#pragma unroll
            for (int t = 0; t < KP; ++t) {
                rj[t] = wi[t];
                rd[t] = wd[t];
            }
        }
        if (q.store_bmu) wi[0] = b0;  // the nearest landmark: batch-SOM statistics read column 0
        if (a.bmu) a.bmu[i] = b0;
        if (a.qe_sum) qe_local += (double)d0;
        reg2_point<KP, true, false, FH, true, true>(q, i, rj, rd, LO, RB, tsm, nullptr, nullptr, 0, tmax_model, Ls,
                                                    a.ls, inv);
    }
    if (a.stats && slow_local) atomicAdd(a.stats + 1, slow_local);
    if (a.qe_sum) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) qe_local += __shfl_xor_sync(0xffffffffu, qe_local, o);
        if ((tid & 31) == 0 && qe_local != 0.0) atomicAdd(a.qe_sum, qe_local);
    }
}

// ESOM_ERR_UNSUPPORTED when the shape does not qualify (the caller runs the two kernels)
inline int launch_embed_fused(Tc2Args a, ProjArgs q, cudaStream_t st) {
    if (a.k != 16 || a.d != 32 || !a.cbits || q.k != 16) return ESOM_ERR_UNSUPPORTED;
    size_t smem = fused_smem_bytes(a.gpad, a.ls, a.g);
    const size_t cap = (size_t)esom_host::max_smem_optin() - 1024;
    if (smem > cap) return ESOM_ERR_UNSUPPORTED;
    const bool list = smem + fused_list_bytes() <= cap;
    if (list) smem += fused_list_bytes();
    const bool fh = q.far_heavy != 0;  // far-heavy (trained) frames: the packed pair loop
    auto kern = list ? (fh ? embed_fused_kernel<16, true, true> : embed_fused_kernel<16, true, false>)
                     : (fh ? embed_fused_kernel<16, false, true> : embed_fused_kernel<16, false, false>);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int64_t grid = (a.n + kFusedThreads - 1) / kFusedThreads;
    if (grid > esom_host::num_sms()) grid = esom_host::num_sms();
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kFusedThreads, smem, st>>>(a, q);
    return esom_host::cuda_check("embed_fused_kernel");
}

}  // namespace esom
