// FP64 instantiations of the batched-frame loop passes (tiled per-frame hooks, kernels.cuh).
#include "fft_dispatch.cuh"

namespace ffcz_gpu {

template void launch_col<double, HookFReduceB>(long long, int, const double2*, double2*, long long,
                                               long long, long long, int, Twiddles<double>&,
                                               const int*, HookFReduceB, cudaStream_t);
template void launch_col<double, HookFClipB<double>>(long long, int, const double2*, double2*,
                                                     long long, long long, long long, int,
                                                     Twiddles<double>&, const int*,
                                                     HookFClipB<double>, cudaStream_t);
template void launch_row_c2r_hook<double, HookSClipB<double>>(long long, const double2*, long long,
                                                              double*, long long, long long, double,
                                                              Twiddles<double>&, const int*,
                                                              HookSClipB<double>, cudaStream_t);
template void launch_row_r2c_hook<double, HookSkipB<true>>(long long, const double*, long long,
                                                           double2*, long long, long long,
                                                           Twiddles<double>&, const int*,
                                                           HookSkipB<true>, cudaStream_t);

} // namespace ffcz_gpu
