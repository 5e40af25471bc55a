// generated: explicit instantiations of the projection kernel
#include "../esom_project.cuh"
namespace esom {
template int launch_project_t<4>(ProjArgs, cudaStream_t);
template int launch_project_t<8>(ProjArgs, cudaStream_t);
template int launch_project_t<16>(ProjArgs, cudaStream_t);
template int launch_project_t<32>(ProjArgs, cudaStream_t);
template int launch_project_t<64>(ProjArgs, cudaStream_t);
}
