// generated: explicit instantiations of the projection kernel
#include "../esom_project.cuh"
namespace esom {
template int launch_project_t<4>(ProjArgs, cudaStream_t);
template int launch_project_t<8>(ProjArgs, cudaStream_t);
template int launch_project_t<16>(ProjArgs, cudaStream_t);
template int launch_project_t<32>(ProjArgs, cudaStream_t);
template int launch_project_t<64>(ProjArgs, cudaStream_t);

int launch_pair_records(const float* T, const float* lo, int g, float4* rec, cudaStream_t st) {
    const int64_t total = (int64_t)g * g;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)esom_host::num_sms() * 16;
    if (blocks > cap) blocks = cap;
    pair_record_kernel<<<(unsigned)blocks, 256, 0, st>>>(T, lo, g, rec);
    return esom_host::cuda_check("pair_record_kernel");
}
}
