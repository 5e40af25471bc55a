// esom_scan_args.h -- launch arguments of the k-NN scan and projection kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace esom {

struct ScanArgs {
    const float* X;          // n×d points (row-major)
    int64_t n;
    int d, dp, nch;          // dims, padded dims, x chunks (dp = nch * DC)
    const float* Lt;         // packed landmark tiles [tile][dp][32]
    const float* L;          // row-major landmarks g×d (rare exact slow path)
    int g, ntiles, k;
    int res_tiles;           // tiles resident in smem (== ntiles) or 0 = streamed
    int32_t* out_idx;        // n×k (nullable: statistics only)
    float* out_sqd;          // n×k
    int32_t* bmu;            // n   (nullable)
    unsigned long long* accS;  // g×d batch-SOM sums, int64 fixed point x 2^fx (nullable)
    unsigned long long* accC;  // g   counts (int64, nullable)
    double acc_scale;          // 2^fx
    double* qe_sum;          // sum of nearest squared distances (nullable)
    int32_t* flag;           // non-finite input flag
    float nz;                // -0.0f, opaque to ptxas
};

struct ProjArgs {
    const int32_t* idx;      // n×k neighbour rows (ascending)
    const float* sqd;        // n×k exact squared distances
    int64_t n;
    int k, g;
    const float* lo;         // g×2 layout
    const float* T;          // packed upper-triangular 0.5/hd2 (f32), -1 = pair skipped
    int t_smem;              // stage T in shared memory
    float* xy;               // n×2 out
    const float* X;          // outlier exact path
    const float* hi;
    const double* hi64;      // hi widened to f64 (model workspace): far-point distances
    const double* hn64;      // |h_j|^2 in f64 (model workspace)
    int d;
    const int32_t* perm;     // optional visiting order (nullable)
    const float4* rec;       // g x g pair records {T, g1, g2, g.lo_u} (project_reg3_kernel; nullable)
    const float* tmax;       // device scalar: max kept T of the model (f64-distance decision)
    int32_t* prec_count;     // += points that took the f64 far-point path (nullable)
    int far_heavy;           // the caller expects most points far (nearest-landmark order): far-path codegen
    int store_bmu;           // fused kernel: write the nearest landmark to idx[i * k] (batch-SOM statistics)
};

// tensor-core screened k-NN (esom_tc.cuh)
struct TcArgs {
    const float* X;          // n×d points
    int64_t n;
    int d, d16, dp;          // dims, dims padded to 16 (MMA K), dims of the exact tiles
    int g, gpad, k;          // landmarks, landmarks padded to 32
    const uint16_t* Bhi;     // gpad × d16 bf16, canonical K-major layout
    const uint16_t* Blo;
    const float* ln;         // gpad |l_j|^2 (f32; +inf for padding rows)
    const float* Lt;         // exact tiles [tile][dp][32]
    const float* L;          // row-major landmarks (slow path)
    const float* lstats;     // [0] = max_j |l'_j|, [1] = max_j |l'_j|^2 (device, centred)
    const float* center;     // landmark centroid c (padded to d16); operands are x - c, l - c
    int32_t* out_idx;
    float* out_sqd;
    int32_t* bmu;
    unsigned long long* accS;
    unsigned long long* accC;
    double acc_scale;
    double* qe_sum;
    int32_t* flag;
    int32_t* stats;          // [0] += candidates examined exactly (diagnostic, nullable)
};

// pipelined tensor-core screened k-NN (esom_tc2.cuh)
struct Tc2Args {
    const float* X;          // n×d points
    int64_t n;
    int d, d16, g, gpad, k;  // d16 = MMA K (16 or 32), gpad = g padded to 32
    const uint16_t* Bhi;     // gpad×d16 bf16 of -2 l (hi part), canonical K-major
    const uint16_t* Blo;     // lo part
    const float* ln;         // gpad |l_j|^2 (f32, +inf on padding rows)
    const float* Lrow;       // gpad×ls f32 rows, zero-padded dims (global), in screen-row order
    const int32_t* rowmap;   // screen row -> landmark index (gpad; nullable = identity)
    int ls;                  // Lrow stride (floats, multiple of 4, ls/4 odd)
    const float* L;          // row-major g×d (slow path)
    const float* lstats;     // [0] max|l'_j|, [1] max|l'_j|^2 (centred)
    const float* center;     // 32 f32: landmark centroid c (zero-padded), operands are x - c, l - c
    int32_t* out_idx;
    float* out_sqd;
    int32_t* bmu;
    unsigned long long* accS;
    unsigned long long* accC;
    double acc_scale;
    double* qe_sum;
    int32_t* flag;
    int32_t* stats;          // [0] += logged candidates, [1] += slow-path points (diagnostic, nullable)
    uint32_t* cbits;         // split mode (g > 256): n x gpad/32 candidate bitmaps (nullable = fused)
    int2* cinfo;             // split mode: n x {candidates (-1: non-finite input), non-empty word mask}
    int32_t* ckey;           // split mode: n x lowest candidate (locality sort key)
    const int32_t* perm;     // split mode, exact kernel: visiting order (nullable)
};

// tensor-core GEMM screen for d > 32 (esom_tc3.cuh)
struct Tc3Args {
    const uint16_t* Ahi;     // points x - c, split bf16, [128-row tile][32-wide K chunk] canonical
    const uint16_t* Alo;
    const float* xnorm;      // n: |x - c| (rounded up)
    int64_t n;
    int d, dk, gpad, k;      // dk = d padded to 32, gpad = g padded to 256
    const uint16_t* Bhi;     // -2 (l - c) split bf16, [256-row round][K chunk] canonical
    const uint16_t* Blo;
    const float* ln;         // gpad: |l - c|^2 (+inf padding)
    const float* lstats;     // [0] max|l - c|, [1] max|l - c|^2
    uint16_t* cand;          // n x 64 candidate landmark indices (index order)
    int32_t* ccount;         // n: candidates, -1 = reference scan needed
    int32_t* bmu_approx;     // n: landmark of the smallest screened distance
    int32_t* stats;          // [0] += candidates, [1] += overflowed points (nullable)
};

struct T3ExactArgs {
    const float* X;          // n x d points
    int64_t n;
    int d, dpad, g, k;       // dpad: d rounded up to 4 (smem row of one warp)
    const float* L;          // g x d landmarks (row-major)
    const uint16_t* cand;
    const int32_t* ccount;
    const int32_t* perm;     // visiting order (approximate-BMU sorted; nullable)
    int32_t* out_idx;        // n x k (nullable: statistics only)
    float* out_sqd;
    int32_t* bmu;
    double* qe_sum;
    unsigned long long* accS;
    unsigned long long* accC;
    double acc_scale;
    int32_t* stats;          // diagnostic: [2] += union sizes, [3] += groups evaluated, [4] += splits
};

template <int KP>
int launch_gemm_t(Tc3Args a, cudaStream_t st);        // esom_tc3.cuh, instantiated in inst/tc3.cu
template <int KP>
int launch_exact_warp_t(T3ExactArgs a, cudaStream_t st);
// operand split of esom_tc3.cuh (rows x - c or -2 (l - c), canonical bf16 tiles, norms)
int t3_split(const float* X, int64_t n, int64_t npad, int d, int dk, const float* cen, float scale, int rows_blk,
             uint16_t* Hi, uint16_t* Lo, float* nrm, int nrm_sq, float* lstats, int32_t* flag, cudaStream_t st);

template <int KP>
int launch_tc_t(TcArgs a, cudaStream_t st);  // esom_tc.cuh, instantiated in inst/tc.cu

template <int KP, int W>
int launch_tc2_t(Tc2Args a, cudaStream_t st);  // esom_tc2.cuh, instantiated in inst/tc2.cu
template <int KP>
int launch_exact_bits_t(Tc2Args a, cudaStream_t st);

template <int DC, int KP>
int launch_scan_t(ScanArgs a, cudaStream_t st);   // esom_scan.cuh, instantiated in inst/*.cu

template <int KP>
int launch_project_t(ProjArgs a, cudaStream_t st);
// exact k-NN + projection in one kernel (esom_fused.cuh; k = 16, d <= 32, small g);
// ESOM_ERR_UNSUPPORTED when the shape does not qualify
int launch_embed_fused_c(Tc2Args a, ProjArgs q, cudaStream_t st);
// g x g pair records of project_reg3_kernel from the pair triangle T and the layout lo
int launch_pair_records(const float* T, const float* lo, int g, float4* rec, cudaStream_t st);  // esom_project.cuh, instantiated in inst/*.cu

}  // namespace esom
