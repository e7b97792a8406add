// FP32 instantiations of the FFT engine (engine tests, per-pass roofline bench, mixed policy).
#include "fft_dispatch.cuh"

namespace ffcz_gpu {

template struct FftPlan<float>;
template void launch_col<float, HookNone>(long long, int, const float2*, float2*, long long,
                                          long long, long long, int, Twiddles<float>&, const int*,
                                          HookNone, cudaStream_t);
template void launch_row_r2c<float>(long long, const float*, long long, float2*, long long,
                                    long long, Twiddles<float>&, const int*, cudaStream_t);
template void launch_row_c2r<float>(long long, const float2*, long long, float*, long long,
                                    long long, float, Twiddles<float>&, const int*, cudaStream_t);

} // namespace ffcz_gpu
