// esom_knn.cuh -- fused exact f32 distance scan + register top-k selection.
//
// One thread owns one point (ref: knn.py:65-92 `_knn_base_kernel` walks the
// landmarks of one point in ascending j).  Landmarks sit in shared memory as
// transposed 32-landmark tiles Lt[tile][c][32] (staged by 1-D TMA bulk copies
// from a packed, zero/inf-padded copy), so one LDS.128 broadcast feeds two
// packed f32x2 lanes for two landmarks; the point's coordinates stay in
// registers.  Per tile each thread produces 32 exact squared distances.
//
// Selection keeps a sorted (dist, idx) list of KP >= k entries in registers.
// Because j only grows, a new candidate precedes an equal-distance entry
// never (lexicographic key (s, j), ref: knn.py:79,85,96-97), so insertion
// uses strict '<'.  Candidates that beat the current k-th key are parked in
// a per-thread shared-memory slot row and inserted in a divergent loop whose
// trip count is the warp's max candidate count (not the tile size).
#pragma once
#include "esom_common.cuh"

namespace esom {

// Compute 32 exact squared distances of x (DC dims, zero padded) against a
// tile slab Lt[c][32] for dims [c0, c0+DC).  acc holds 16 packed pairs.
template <int DC>
__device__ __forceinline__ void tile_accumulate(const float (&x)[DC], const float* __restrict__ slab,
                                                f2 nz, f2 (&acc)[16], bool first) {
#pragma unroll
    for (int c = 0; c < DC; ++c) {
        const float4* row = reinterpret_cast<const float4*>(slab + c * kTile);
        const f2 xx = f2_pack(x[c], x[c]);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 l4 = row[q];
            f2 t0 = f2_sub(f2_pack(l4.x, l4.y), xx);
            f2 t1 = f2_sub(f2_pack(l4.z, l4.w), xx);
            f2 s0 = f2_sq(t0, nz);
            f2 s1 = f2_sq(t1, nz);
            if (first && c == 0) {
                acc[2 * q] = s0;          // 0 + t^2 == t^2 exactly
                acc[2 * q + 1] = s1;
            } else {
                acc[2 * q] = f2_add(acc[2 * q], s0);
                acc[2 * q + 1] = f2_add(acc[2 * q + 1], s1);
            }
        }
    }
}

// Insert (v, j) into the sorted register list; j exceeds every held index.
template <int KP>
__device__ __forceinline__ void topk_insert(float (&td)[KP], int (&ti)[KP], float v, int j) {
#pragma unroll
    for (int q = KP - 1; q > 0; --q) {
        const bool gp = td[q - 1] > v;
        const bool gc = td[q] > v;
        td[q] = gp ? td[q - 1] : (gc ? v : td[q]);
        ti[q] = gp ? ti[q - 1] : (gc ? j : ti[q]);
    }
    if (td[0] > v) {
        td[0] = v;
        ti[0] = j;
    }
}

// Exact lexicographic insertion, only needed when v == +inf (an overflowed
// distance competing with the (+inf, g) sentinels of still-empty slots).
template <int KP>
__device__ __forceinline__ void topk_insert_lex(float (&td)[KP], int (&ti)[KP], float v, int j) {
#pragma unroll
    for (int q = KP - 1; q > 0; --q) {
        const bool gp = td[q - 1] > v || (td[q - 1] == v && ti[q - 1] > j);
        const bool gc = td[q] > v || (td[q] == v && ti[q] > j);
        td[q] = gp ? td[q - 1] : (gc ? v : td[q]);
        ti[q] = gp ? ti[q - 1] : (gc ? j : ti[q]);
    }
    if (td[0] > v || (td[0] == v && ti[0] > j)) {
        td[0] = v;
        ti[0] = j;
    }
}

// The live list occupies slots [KP-k, KP); slots below hold -inf and never
// move, so the k-th key is always td[KP-1] (a static register).
template <int KP>
__device__ __forceinline__ void topk_init(float (&td)[KP], int (&ti)[KP], int k, int sentinel) {
#pragma unroll
    for (int q = 0; q < KP; ++q) {
        td[q] = q >= KP - k ? __int_as_float(0x7f800000) : __int_as_float(0xff800000);
        ti[q] = sentinel;
    }
}

template <int KP>
__device__ __forceinline__ float topk_tau(const float (&td)[KP], int) {
    return td[KP - 1];
}

// Merge one tile's 32 distances into the top-k list.
template <int KP>
__device__ __forceinline__ void topk_tile(float (&td)[KP], int (&ti)[KP], const f2 (&acc)[16], int jbase,
                                          int k, float* __restrict__ cbuf, int tid) {
    float tau = topk_tau<KP>(td, k);
    const bool open = tau == __int_as_float(0x7f800000);  // k-th slot still empty
    uint32_t m = 0;
#pragma unroll
    for (int p = 0; p < 16; ++p) {
        float a, b;
        f2_unpack(acc[p], a, b);
        if (a < tau || (open && a == tau)) {
            m |= 1u << (2 * p);
            cbuf[(2 * p) * kThreads + tid] = a;
        }
        if (b < tau || (open && b == tau)) {
            m |= 1u << (2 * p + 1);
            cbuf[(2 * p + 1) * kThreads + tid] = b;
        }
    }
    while (m) {
        const int t = __ffs(m) - 1;
        m &= m - 1;
        const float v = cbuf[t * kThreads + tid];
        if (v < tau) {
            topk_insert<KP>(td, ti, v, jbase + t);
            tau = topk_tau<KP>(td, k);
        } else if (v == tau && tau == __int_as_float(0x7f800000) && jbase + t < 0x7fffffff) {
            topk_insert_lex<KP>(td, ti, v, jbase + t);
            tau = topk_tau<KP>(td, k);
        }
    }
}

}  // namespace esom
