/*
 * Minimal FFTW3-API provider for building the CPU reference (oracle/_ref).
 *
 * TEST INFRASTRUCTURE ONLY.  The reference (`/root/reference/proj/core/src/transform.cpp:3,20-41`)
 * calls exactly fftw_plan_dft / fftw_execute / fftw_destroy_plan with
 * FFTW_ESTIMATE|FFTW_PRESERVE_INPUT on complex<double> buffers.  FFTW itself is
 * not installed in this image, so this header + fftw_shim.cpp
 * provide those three entry points with FFTW's documented semantics:
 * unnormalised transforms, sign -1 forward / +1 backward, row-major extents,
 * out-of-place, input preserved.
 */
#pragma once

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct ffcz_shim_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_PRESERVE_INPUT (1U << 4)

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign,
                        unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif
