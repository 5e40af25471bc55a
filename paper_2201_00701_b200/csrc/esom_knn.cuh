// esom_knn.cuh -- exact f32 distance tiles and the register/shared-memory
// top-k selection of the k-NN scan kernel.
//
// One thread owns one point (ref: knn.py:65-92 `_knn_base_kernel` walks the
// landmarks of one point in ascending j).  Landmarks sit in shared memory as
// transposed 32-landmark tiles Lt[tile][c][32] (staged by 1-D TMA bulk copies
// from a packed, zero/inf-padded copy), so one LDS.128 broadcast feeds two
// packed f32x2 lanes for two landmarks; the point's coordinates stay in
// registers.  Per tile each thread produces 32 exact squared distances.
//
// Selection (exact, equal to the reference's lexicographic (dist, index)
// order, ref: knn.py:79,85,96-97):
//  * a VALUES-ONLY sorted list vd[KP] in registers (min/max insertion, two
//    FMNMX per slot, no index bookkeeping) gives the running k-th distance tau;
//  * every landmark that beats tau when scanned is appended, in index order,
//    to a per-thread candidate log in shared memory (value, index);
//  * at the end the final set is {log entries with v < tau_f} plus the
//    lowest-index entries with v == tau_f, ranked by (v, j).
// A landmark that is not logged had v >= tau at scan time, and tau only
// decreases, so it cannot be in the top k (ties go to lower indices, which
// were scanned earlier) -- the selection is exact, ties included.
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
                acc[2 * q] = s0;  // 0 + t^2 == t^2 exactly
                acc[2 * q + 1] = s1;
            } else {
                acc[2 * q] = f2_add(acc[2 * q], s0);
                acc[2 * q + 1] = f2_add(acc[2 * q + 1], s1);
            }
        }
    }
}

constexpr float kInf = __builtin_huge_valf();

// Live slots of the values list are [KP-k, KP); slots below hold -inf and
// never move, so the k-th smallest value is always vd[KP-1].
template <int KP>
__device__ __forceinline__ void vlist_init(float (&vd)[KP], int k) {
#pragma unroll
    for (int q = 0; q < KP; ++q) vd[q] = q >= KP - k ? kInf : -kInf;
}

template <int KP>
__device__ __forceinline__ void vlist_insert(float (&vd)[KP], float v) {
#pragma unroll
    for (int q = KP - 1; q > 0; --q) vd[q] = fmaxf(vd[q - 1], fminf(vd[q], v));
    vd[0] = fminf(vd[0], v);
}

// Insert (v, j) into a sorted (dist, idx) register list whose held indices
// are all smaller than j (strict '<' then realises the (dist, idx) order).
// Slots below KP-k hold -inf and never move.
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

// (distance, index) lexicographic insertion: the (d, j) order of knn_base
// whatever order the candidates are visited in (the tensor-core screens visit
// them in screen-row order, a permutation of the landmark indices)
__device__ __forceinline__ bool key_lt(float va, int ja, float vb, int jb) {
    return va < vb || (va == vb && ja < jb);
}
template <int KP>
__device__ __forceinline__ void topk_insert_lex(float (&td)[KP], int (&ti)[KP], float v, int j) {
#pragma unroll
    for (int q = KP - 1; q > 0; --q) {
        const bool gp = key_lt(v, j, td[q - 1], ti[q - 1]);
        const bool gc = key_lt(v, j, td[q], ti[q]);
        td[q] = gp ? td[q - 1] : (gc ? v : td[q]);
        ti[q] = gp ? ti[q - 1] : (gc ? j : ti[q]);
    }
    if (key_lt(v, j, td[0], ti[0])) {
        td[0] = v;
        ti[0] = j;
    }
}

// number of values (live or -inf padding) strictly below v
template <int KP>
__device__ __forceinline__ int vlist_count_lt(const float (&vd)[KP], float v) {
    int c = 0;
#pragma unroll
    for (int q = 0; q < KP; ++q) c += vd[q] < v ? 1 : 0;
    return c;
}

// ---- batched top-16 (exact phase): sort 8 new candidates, merge into the
// sorted 16-list by a bitonic half-cleaner + bitonic merge.  Compares values
// only; equal values are detected afterwards (adjacent equal list entries, or
// a discarded value equal to the last kept one) and the caller falls back to
// the index-ordered insertion, so the result is the (distance, index) order.
__device__ __forceinline__ void ce_vj(float& va, int& ja, float& vb, int& jb) {
    const bool sw = va > vb;
    const float lo = fminf(va, vb), hi = fmaxf(va, vb);
    const int jl = sw ? jb : ja, jh = sw ? ja : jb;
    va = lo;
    vb = hi;
    ja = jl;
    jb = jh;
}

// Batcher odd-even merge sort of 8 (19 comparators, generated)
__device__ __forceinline__ void sort8_vj(float (&v)[8], int (&j)[8]) {
    ce_vj(v[0], j[0], v[1], j[1]);
    ce_vj(v[2], j[2], v[3], j[3]);
    ce_vj(v[4], j[4], v[5], j[5]);
    ce_vj(v[6], j[6], v[7], j[7]);
    ce_vj(v[0], j[0], v[2], j[2]);
    ce_vj(v[1], j[1], v[3], j[3]);
    ce_vj(v[4], j[4], v[6], j[6]);
    ce_vj(v[5], j[5], v[7], j[7]);
    ce_vj(v[1], j[1], v[2], j[2]);
    ce_vj(v[5], j[5], v[6], j[6]);
    ce_vj(v[0], j[0], v[4], j[4]);
    ce_vj(v[1], j[1], v[5], j[5]);
    ce_vj(v[2], j[2], v[6], j[6]);
    ce_vj(v[3], j[3], v[7], j[7]);
    ce_vj(v[2], j[2], v[4], j[4]);
    ce_vj(v[3], j[3], v[5], j[5]);
    ce_vj(v[1], j[1], v[2], j[2]);
    ce_vj(v[3], j[3], v[4], j[4]);
    ce_vj(v[5], j[5], v[6], j[6]);
}

// L (ascending, 16) <- the 16 smallest of L and B (8, ascending); dmin tracks the
// smallest discarded value
__device__ __forceinline__ void merge16_8(float (&L)[16], int (&LJ)[16], const float (&B)[8], const int (&BJ)[8],
                                          float& dmin) {
#pragma unroll
    for (int i = 8; i < 16; ++i) {  // half-cleaner against the reversed, +inf-padded B
        const float y = B[15 - i];
        const bool take = y < L[i];
        dmin = fminf(dmin, fmaxf(L[i], y));
        LJ[i] = take ? BJ[15 - i] : LJ[i];
        L[i] = fminf(L[i], y);
    }
#pragma unroll
    for (int st = 8; st > 0; st >>= 1)  // bitonic merge (ascending)
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if ((i & st) == 0) ce_vj(L[i], LJ[i], L[i + st], LJ[i + st]);
}

}  // namespace esom
