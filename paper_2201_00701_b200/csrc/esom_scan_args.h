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
    double* accS;            // g×d batch-SOM sums (nullable)
    double* accC;            // g   counts as f64 (nullable)
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
    int d;
};

template <int DC, int KP>
int launch_scan_t(ScanArgs a, cudaStream_t st);   // esom_scan.cuh, instantiated in inst/*.cu

template <int KP>
int launch_project_t(ProjArgs a, cudaStream_t st);  // esom_project.cuh, instantiated in inst/*.cu

}  // namespace esom
