// FP64 instantiation of the loop's round-trip column pass (check + clip between the forward and
// the inverse transform of the completing axis): its own translation unit so it compiles in
// parallel with the other pass templates.
#include "fft_dispatch.cuh"

namespace ffcz_gpu {
template void launch_col_rt<double, HookRT>(long long, const double2*, double2*, long long,
                                            long long, long long, int, Twiddles<double>&,
                                            const int*, HookRT, cudaStream_t);
template void launch_col_frebuild<double>(long long, const double2*, const double2*, double2*,
                                          const unsigned char*, long long, long long, long long,
                                          int, Twiddles<double>&, cudaStream_t);
} // namespace ffcz_gpu
