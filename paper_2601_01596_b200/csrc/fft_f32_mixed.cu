// FP32 instantiations of the mixed policy's FP32 phase (check / clip column passes, C2R with the
// s-cube clip); the accumulators S and F stay FP64 (the hooks compute in FP64).
#include "fft_dispatch.cuh"

namespace ffcz_gpu {

template void launch_col<float, HookFReduce>(long long, int, const float2*, float2*, long long,
                                             long long, long long, int, Twiddles<float>&,
                                             const int*, HookFReduce, cudaStream_t);
template void launch_col<float, HookFClip<float>>(long long, int, const float2*, float2*,
                                                  long long, long long, long long, int,
                                                  Twiddles<float>&, const int*, HookFClip<float>,
                                                  cudaStream_t);
template void launch_row_c2r_hook<float, HookSClip<float>>(long long, const float2*, long long,
                                                           float*, long long, long long, float,
                                                           Twiddles<float>&, const int*,
                                                           HookSClip<float>, cudaStream_t);

} // namespace ffcz_gpu
