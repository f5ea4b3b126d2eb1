// bp_scatter.cu: the Back-Projection kernels with the NEXT-4 scatter epilogue (every finished
// tile stored, or reduced, into the images of all ranks over NVLink: P2P stores / red, or
// multimem.st / multimem.red to the NVSwitch multicast address; under a chirp split the last
// chunk of each tile publishes it).  Same kernel template as bp_kernel.cu (bp_kernel.cuh).
#include "bp_kernel.cuh"

namespace sar {

cudaError_t launch_bp_scatter(const BpArgs& a, bool bistatic, bool doppler, bool near, cudaStream_t s) {
  return launch_shapes<true>(a, bistatic, doppler, near, s);
}

}  // namespace sar

#ifdef SAR_DEBUG_CHECKS
extern "C" int sar_debug_violations_scatter(unsigned long long* out4, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out4, sar::g_violations, sizeof(sar::g_violations));
  if (reset) {
    const unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(sar::g_violations, z, sizeof(z));
  }
  return (int)e;
}
#endif
