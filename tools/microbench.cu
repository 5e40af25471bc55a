// Pipe-throughput microbenchmarks on the B200 (evidence for DESIGN.md):
// scalar FADD/FMUL chains vs packed f32x2 FADD2/FFMA2, F2F.F64.F32,
// DADD/DFMA, and broadcast LDS.128.  Each kernel runs independent chains
// per thread so issue throughput (not latency) binds.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
#define ITERS 4096
__global__ void k_scalar(float* out, float a, float b) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __fadd_rn(__fmul_rn(x[i], a), b);
    }
    float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_packed(float* out, float a, float b) {
    u64 x[8], A, B;
    asm("mov.b64 %0, {%1,%1};" : "=l"(A) : "f"(a));
    asm("mov.b64 %0, {%1,%1};" : "=l"(B) : "f"(b));
    for (int i = 0; i < 8; ++i) { float v = threadIdx.x * 0.001f + i; asm("mov.b64 %0, {%1,%1};" : "=l"(x[i]) : "f"(v)); }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            u64 t;
            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(t) : "l"(x[i]), "l"(A), "l"(B));
            asm("add.rn.f32x2 %0, %1, %2;" : "=l"(x[i]) : "l"(t), "l"(B));
        }
    }
    float s = 0; for (int i = 0; i < 8; ++i) { float p, q; asm("mov.b64 {%0,%1}, %2;" : "=f"(p), "=f"(q) : "l"(x[i])); s += p + q; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(float* out, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
__global__ void k_f2f(float* out, float a) {
    float x[8]; double acc[8];
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 0.001f + i; acc[i] = 0; }
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { acc[i] = (double)x[i]; x[i] = (float)acc[i] + a; }
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += acc[i] + x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
__global__ void k_lds(float* out, int n) {
    __shared__ float4 sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { float4 v = sm[(it * 8 + i) & 1023]; acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}
template <typename F>
float timeit(F f) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); cudaDeviceSynchronize();
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out; cudaMalloc(&out, sms * 8 * 256 * 4);
    dim3 grid(sms * 8), blk(256);
    double threads = (double)sms * 8 * 256;
    float t;
    t = timeit([&] { k_scalar<<<grid, blk>>>(out, 1.0001f, 0.5f); });
    printf("{\"op\": \"FMUL+FADD scalar\", \"ms\": %.3f, \"Gop_per_s\": %.1f}\n", t, threads * ITERS * 8 * 2 / t / 1e6);
    t = timeit([&] { k_packed<<<grid, blk>>>(out, 1.0001f, 0.5f); });
    printf("{\"op\": \"FFMA2+FADD2 packed (lane-ops)\", \"ms\": %.3f, \"Gop_per_s\": %.1f}\n", t, threads * ITERS * 8 * 4 / t / 1e6);
    t = timeit([&] { k_dfma<<<grid, blk>>>(out, 1.0000001, 0.5); });
    printf("{\"op\": \"DFMA\", \"ms\": %.3f, \"Gop_per_s\": %.1f}\n", t, threads * ITERS * 8 / t / 1e6);
    t = timeit([&] { k_f2f<<<grid, blk>>>(out, 0.5f); });
    printf("{\"op\": \"F2F.F64.F32+F2F.F32.F64+FADD (per pair)\", \"ms\": %.3f, \"Gpair_per_s\": %.1f}\n", t, threads * ITERS / 4 * 8 / t / 1e6);
    t = timeit([&] { k_lds<<<grid, blk>>>(out, 0); });
    printf("{\"op\": \"LDS.128 broadcast\", \"ms\": %.3f, \"Ginstr_per_s\": %.1f}\n", t, threads / 32 * ITERS * 8 / t / 1e6);
    printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
    return 0;
}
