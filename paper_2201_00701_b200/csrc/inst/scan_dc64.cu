// generated: explicit instantiations of the k-NN scan kernel
#include "../esom_scan.cuh"
namespace esom {
template int launch_scan_t<64, 4>(ScanArgs, cudaStream_t);
template int launch_scan_t<64, 8>(ScanArgs, cudaStream_t);
template int launch_scan_t<64, 16>(ScanArgs, cudaStream_t);
template int launch_scan_t<64, 32>(ScanArgs, cudaStream_t);
template int launch_scan_t<64, 64>(ScanArgs, cudaStream_t);
}
