// esom_common.cuh -- shared device helpers for the sm_100a EmbedSOM kernels.
//
// Exactness note: the reference's distance kernel
// (ref: knn.py:56-62) rounds every sub, mul and add separately in f32.  We
// use either the __f*_rn intrinsics (never contracted) or packed f32x2 PTX
// where the square is issued as fma(t, t, NZ) with NZ a *runtime* -0.0f so
// ptxas cannot fold the following add into an FFMA2 (it does contract
// mul.rn.f32x2 + add.rn.f32x2; verified with cuobjdump).  fma(t,t,-0) is the
// correctly rounded t*t for every t, including t = 0 (+0 + -0 = +0).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cuda_bf16.h>

#define ESOM_OK 0
#define ESOM_ERR_PARAM 1
#define ESOM_ERR_INPUT 2
#define ESOM_ERR_CUDA 3
#define ESOM_ERR_UNSUPPORTED 4

namespace esom {

constexpr int kTile = 32;          // landmarks per smem tile (one per accumulator slot)
constexpr int kThreads = 128;      // points per CTA iteration (one per thread)

typedef unsigned long long f2;     // two packed f32 lanes (lo = first, hi = second)

// Batch-SOM statistics are exact int64 fixed point (units of 2^-fx, two's
// complement in unsigned atomics): integer addition is associative, so S and C
// are independent of the accumulation order, of atomic scheduling and of how
// the points are split across ranks -- training is bit-identical at any GPU
// count (SURVEY §7 hard part 6).  x -> round(x 2^fx) is exact f64 arithmetic
// (a power-of-two scale) followed by one deterministic rounding.
typedef unsigned long long acc_t;
__device__ __forceinline__ acc_t acc_fx(float x, double scale) {
    // scale = 2^fx (0 <= fx <= 40) and |x| 2^fx < 2^61: x * 2^fx is exact in f32
    // as in f64, so rounding the f32 product gives the same integer as rounding
    // (double)x * scale -- one F2I instead of F2F + DMUL + F2I
    return (acc_t)__float2ll_rn(x * (float)scale);
}

__device__ __forceinline__ f2 f2_pack(float a, float b) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2_unpack(f2 v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2 f2_sub(f2 a, f2 b) {
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// t*t correctly rounded, kept a separate rounding from the following add.
__device__ __forceinline__ f2 f2_sq(f2 t, f2 nz) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(t), "l"(nz));
    return r;
}
__device__ __forceinline__ f2 f2_add(f2 a, f2 b) {
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2_mul(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2_fma(f2 a, f2 b, f2 c) {  // a*b + c, one rounding per lane
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// 32 bytes per lane in ONE 256-bit load (ld.global.nc.v8 -> LDG.E.ENL2.256):
// when every lane of a warp reads its own row, each load costs one L1 wavefront
// per lane, so halving the load count halves the L1 work.  p: 32-byte aligned.
__device__ __forceinline__ void ldg8(const float* p, float4& a, float4& b) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                 : "l"(p));
}
__device__ __forceinline__ void ldg8(const int32_t* p, int4& a, int4& b) {
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                 : "l"(p));
}
__device__ __forceinline__ bool rows32(const void* base, int row_floats) {  // every row 32-byte aligned
    return ((reinterpret_cast<uintptr_t>(base) | (uintptr_t)(row_floats * 4)) & 31) == 0;
}

__device__ __forceinline__ bool finite_f(float v) { return fabsf(v) <= 3.402823466e38f; }

// mbarrier + 1-D TMA bulk copy (cp.async.bulk) helpers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// Global -> shared bulk copy completing on an mbarrier (size multiple of 16 B,
// both addresses 16-B aligned).  SASS: UBLKCP.S.G.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

constexpr double kScoreEps = 1e-9;   // ref: projection.py:25
constexpr double kPairEps = 1e-12;   // ref: projection.py:26
constexpr double kDetRel = 1e-9;     // ref: projection.py:27
constexpr double kDetAbs = 1e-30;    // ref: projection.py:28
constexpr double kKappaMax = 256.0;  // law-of-cosines guard (see scan_kernel)

__device__ __forceinline__ void flag_nonfinite(int32_t* flag, bool bad) {
    if (__any_sync(0xffffffffu, bad) && flag) {
        if ((threadIdx.x & 31) == 0) atomicOr(flag, 1);
    }
}

}  // namespace esom
