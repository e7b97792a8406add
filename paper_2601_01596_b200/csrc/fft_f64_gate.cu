// FP64 instantiations of the gate-side passes (escape-repair rounds, verify, F rebuild): a
// separate translation unit so the FP64 pass templates compile in parallel.
#include "fft_dispatch.cuh"

namespace ffcz_gpu {

// FP64 gate: fused escape-repair rounds and verify
#define FFCZ_ROW_C2R_HOOK(H)                                                                  \
    template void launch_row_c2r_hook<double, H>(long long, const double2*, long long, double*, \
                                                 long long, long long, double, Twiddles<double>&, \
                                                 const int*, H, cudaStream_t);
FFCZ_ROW_C2R_HOOK(HookSClip<double>)
FFCZ_ROW_C2R_HOOK(HookVerifyS<float>)
FFCZ_ROW_C2R_HOOK(HookVerifyS<double>)
FFCZ_ROW_C2R_HOOK(HookRepairVerifyS<float>)
FFCZ_ROW_C2R_HOOK(HookRepairVerifyS<double>)
#undef FFCZ_ROW_C2R_HOOK
template void launch_col<double, HookMarkViol>(long long, int, const double2*, double2*, long long,
                                               long long, long long, int, Twiddles<double>&,
                                               const int*, HookMarkViol, cudaStream_t);
template void launch_col<double, HookFRebuild>(long long, int, const double2*, double2*, long long,
                                               long long, long long, int, Twiddles<double>&,
                                               const int*, HookFRebuild, cudaStream_t);
template void launch_col<double, HookVerifyF>(long long, int, const double2*, double2*, long long,
                                              long long, long long, int, Twiddles<double>&,
                                              const int*, HookVerifyF, cudaStream_t);

// gate rounds with FFCZ_GATE_ROW_FUSED=1: C2R -> repair -> R2C in one row pass
template void launch_row_fused<double, HookRepairVerifyS<float>>(
    long long, double2*, long long, long long, long long, double, Twiddles<double>&, const int*,
    HookRepairVerifyS<float>, cudaStream_t, double2*);
template void launch_row_fused<double, HookRepairVerifyS<double>>(
    long long, double2*, long long, long long, long long, double, Twiddles<double>&, const int*,
    HookRepairVerifyS<double>, cudaStream_t, double2*);
} // namespace ffcz_gpu
