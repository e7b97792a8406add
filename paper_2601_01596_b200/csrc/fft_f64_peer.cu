// FP64 instantiations of the slab passes whose outputs are scattered into the other ranks'
// receive buffers (fused all-to-all, kernels.cuh PeerScatter): a separate translation unit so
// they compile in parallel with the other FP64 passes.
#include "fft_dispatch.cuh"

namespace ffcz_gpu {

template void launch_col<double, HookScatter>(long long, int, const double2*, double2*, long long,
                                              long long, long long, int, Twiddles<double>&,
                                              const int*, HookScatter, cudaStream_t);
template void launch_col<double, HookFClipScatter<double>>(long long, int, const double2*,
                                                           double2*, long long, long long,
                                                           long long, int, Twiddles<double>&,
                                                           const int*, HookFClipScatter<double>,
                                                           cudaStream_t);

}  // namespace ffcz_gpu
