// generated: explicit instantiations of the k-NN scan kernel
#include "../esom_scan.cuh"
namespace esom {
template int launch_scan_t<16, 4>(ScanArgs, cudaStream_t);
template int launch_scan_t<16, 8>(ScanArgs, cudaStream_t);
template int launch_scan_t<16, 16>(ScanArgs, cudaStream_t);
template int launch_scan_t<16, 32>(ScanArgs, cudaStream_t);
template int launch_scan_t<16, 64>(ScanArgs, cudaStream_t);
}
