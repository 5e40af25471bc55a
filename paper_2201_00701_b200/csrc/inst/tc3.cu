// generated: explicit instantiations of the tensor-core GEMM screen (d > 32)
#include "../esom_tc3.cuh"
namespace esom {
template int launch_gemm_t<4>(Tc3Args, cudaStream_t);
template int launch_gemm_t<8>(Tc3Args, cudaStream_t);
template int launch_gemm_t<16>(Tc3Args, cudaStream_t);
template int launch_gemm_t<32>(Tc3Args, cudaStream_t);
template int launch_exact_warp_t<32>(T3ExactArgs, cudaStream_t);

int t3_split(const float* X, int64_t n, int64_t npad, int d, int dk, const float* cen, float scale, int rows_blk,
             uint16_t* Hi, uint16_t* Lo, float* nrm, int nrm_sq, float* lstats, int32_t* flag, cudaStream_t st) {
    if (npad <= 0) return ESOM_OK;
    int64_t blocks = (npad + 7) / 8;  // 8 warps (rows) per 256-thread block
    const int64_t cap = (int64_t)esom_host::num_sms() * 16;
    if (blocks > cap) blocks = cap;
    t3_split_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, n, npad, d, dk, cen, scale, rows_blk, Hi, Lo, nrm, nrm_sq,
                                                     lstats, flag);
    return esom_host::cuda_check("t3_split_kernel");
}
}
