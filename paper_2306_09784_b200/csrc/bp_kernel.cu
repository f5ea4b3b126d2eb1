// bp_kernel.cu: the plain Back-Projection kernels (image store / accumulate / chirp-split
// reductions) and the launch entry; the kernel template is in bp_kernel.cuh, the NEXT-4
// scatter family in bp_scatter.cu.
#include "bp_kernel.cuh"

namespace sar {

// Supported CTA shapes (consumer warps x pixels per thread); tile = 32 x (NCW * PB).
bool bp_shape_supported(int ncw, int pb) {
  return (ncw == 8 && pb == 4) || (ncw == 4 && pb == 8) || (ncw == 4 && pb == 4) || (ncw == 8 && pb == 8);
}

size_t bp_smem_bytes(int W, int CB, int n_rx, int S, bool bistatic) {
  return make_layout(W, CB, n_rx, S, bistatic).total;
}

cudaError_t launch_bp(const BpArgs& a, bool bistatic, bool doppler, bool near, cudaStream_t s) {
  // the scatter family only for split scatters (its publish epilogue); unsplit scatters take
  // the plain family, whose generic epilogue stores to peers (and whose schedule is faster)
  if (a.n_peer > 0 && a.ws && a.tile_count) return launch_bp_scatter(a, bistatic, doppler, near, s);
  return launch_shapes<false>(a, bistatic, doppler, near, s);
}

}  // namespace sar

#ifdef SAR_BP_TRACE
extern "C" int sar_debug_trace(void* dst, void* dst_wid) {
  cudaMemcpyFromSymbol(dst, sar::g_trace, sizeof(sar::g_trace));
  return (int)cudaMemcpyFromSymbol(dst_wid, sar::g_trace_wid, sizeof(sar::g_trace_wid));
}
#endif

#ifdef SAR_DEBUG_CHECKS
extern "C" int sar_debug_violations_plain(unsigned long long* out4, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out4, sar::g_violations, sizeof(sar::g_violations));
  if (reset) {
    const unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(sar::g_violations, z, sizeof(z));
  }
  return (int)e;
}
extern "C" int sar_debug_modes_plain(unsigned long long* out8, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out8, sar::g_modes, sizeof(sar::g_modes));
  if (reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(sar::g_modes, z, sizeof(z));
  }
  return (int)e;
}
#endif
