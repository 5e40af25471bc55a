// esom_scan_args.h -- launch arguments of the fused scan kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace esom {

struct ScanArgs {
    const float* X;
    int64_t n;
    int d, dp, nch;          // dims, padded dims, x chunks (dp = nch * DC)
    const float* Lt;         // packed tiles
    int g, ntiles, k;
    int res_tiles;           // tiles resident in smem (== ntiles) or 0 = stream
    int32_t* out_idx;
    float* out_sqd;
    const float* hi;         // row-major hi (outlier path)
    const float* lo;         // g×2
    const float* T;          // pair table
    float* xy;
    int32_t* bmu;
    double* accS;
    double* accC;            // counts as f64 (all-reduce friendly)
    double* qe_sum;
    int32_t* flag;
    float nz;                // -0.0f, opaque to ptxas
};

template <int DC, int KP, int MODE>
int launch_scan_t(ScanArgs a, cudaStream_t st);  // esom_scan.cuh, instantiated in inst/*.cu

}  // namespace esom
