// the fused exact k-NN + projection embed kernel (esom_fused.cuh)
#include "../esom_fused.cuh"
namespace esom {
int launch_embed_fused_c(Tc2Args a, ProjArgs q, cudaStream_t st) { return launch_embed_fused(a, q, st); }
}
