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

namespace ffcz_gpu {

// batched-frame gate (engine.cu gate_frames): per-frame masks and bounds
template void launch_col<double, HookFRebuildB>(long long, int, const double2*, double2*, long long,
                                                long long, long long, int, Twiddles<double>&,
                                                const int*, HookFRebuildB, cudaStream_t);
template void launch_col<double, HookMaskB<false>>(long long, int, const double2*, double2*,
                                                   long long, long long, long long, int,
                                                   Twiddles<double>&, const int*,
                                                   HookMaskB<false>, cudaStream_t);
template void launch_col<double, HookMarkViolB>(long long, int, const double2*, double2*, long long,
                                                long long, long long, int, Twiddles<double>&,
                                                const int*, HookMarkViolB, cudaStream_t);
template void launch_col<double, HookVerifyFB>(long long, int, const double2*, double2*, long long,
                                               long long, long long, int, Twiddles<double>&,
                                               const int*, HookVerifyFB, cudaStream_t);
template void launch_row_r2c_hook<double, HookMaskB<true>>(long long, const double*, long long,
                                                           double2*, long long, long long,
                                                           Twiddles<double>&, const int*,
                                                           HookMaskB<true>, cudaStream_t);
#define FFCZ_FR_C2R(H)                                                                        \
    template void launch_row_c2r_hook<double, H>(long long, const double2*, long long, double*, \
                                                 long long, long long, double, Twiddles<double>&, \
                                                 const int*, H, cudaStream_t);
FFCZ_FR_C2R(HookRepairVerifySB<float>)
FFCZ_FR_C2R(HookRepairVerifySB<double>)
FFCZ_FR_C2R(HookVerifySB<float>)
FFCZ_FR_C2R(HookVerifySB<double>)
#undef FFCZ_FR_C2R

} // namespace ffcz_gpu
