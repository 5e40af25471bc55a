// generated: explicit instantiations of the pipelined tensor-core screened k-NN kernel
#include "../esom_tc2.cuh"
namespace esom {
#define ESOM_TC2(KP) \
    template int launch_exact_bits_t<KP>(Tc2Args, cudaStream_t); \
    template int launch_tc2_t<KP, 2>(Tc2Args, cudaStream_t); \
    template int launch_tc2_t<KP, 3>(Tc2Args, cudaStream_t); \
    template int launch_tc2_t<KP, 4>(Tc2Args, cudaStream_t);
ESOM_TC2(4)
ESOM_TC2(8)
ESOM_TC2(16)
#undef ESOM_TC2
}
