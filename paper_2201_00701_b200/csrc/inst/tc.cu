// generated: explicit instantiations of the tensor-core screened k-NN kernel
#include "../esom_tc.cuh"
namespace esom {
template int launch_tc_t<4>(TcArgs, cudaStream_t);
template int launch_tc_t<8>(TcArgs, cudaStream_t);
template int launch_tc_t<16>(TcArgs, cudaStream_t);
}
