// FFTW3-API provider backed by Intel MKL's DFTI (the copy statically linked into PyTorch's
// libtorch_cpu.so, which exports the DFTI C entry points).  TEST INFRASTRUCTURE ONLY.
//
// Same three entry points and semantics as fftw_shim.cpp (the reference calls exactly these,
// /root/reference/proj/core/src/transform.cpp:20-41): an N-d complex<double> DFT, unnormalised,
// sign -1 forward / +1 backward, row-major extents, out-of-place, input preserved.  This is the
// "MKL-backed shim" of BASELINE.md §3 / SURVEY.md §8c option (i): an FFTW-class CPU FFT, so the
// reference arm of bench.py and the large golden runs time the reference's algorithm rather
// than the dependency-free radix-2 stand-in (~17x slower at 64^3).
//
// FFCZ_SHIM_THREADS=<k> (default 1) sets MKL's thread count for the transforms (the reference
// itself is single-threaded; k > 1 is the "FFT-threaded" CPU figure).

#include "fftw3.h"

#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <vector>

extern "C" {
// mkl_dfti.h (LP64 MKL_LONG = long); enum values from the public MKL headers.
typedef struct DFTI_DESCRIPTOR* DFTI_DESCRIPTOR_HANDLE;
long DftiCreateDescriptor_d_1d(DFTI_DESCRIPTOR_HANDLE*, int domain, long length);
long DftiCreateDescriptor_d_md(DFTI_DESCRIPTOR_HANDLE*, int domain, long dim, long* lengths);
long DftiSetValue(DFTI_DESCRIPTOR_HANDLE, int param, ...);
long DftiCommitDescriptor(DFTI_DESCRIPTOR_HANDLE);
long DftiComputeForward(DFTI_DESCRIPTOR_HANDLE, void*, ...);
long DftiComputeBackward(DFTI_DESCRIPTOR_HANDLE, void*, ...);
long DftiFreeDescriptor(DFTI_DESCRIPTOR_HANDLE*);
char* DftiErrorMessage(long);
void omp_set_num_threads(int);  // libgomp (torch's MKL threads through OpenMP)
}

namespace {
constexpr int DFTI_PLACEMENT = 11;
constexpr int DFTI_THREAD_LIMIT = 27;
constexpr int DFTI_COMPLEX = 32;
constexpr int DFTI_NOT_INPLACE = 44;

int shim_threads() {
    const char* s = std::getenv("FFCZ_SHIM_THREADS");
    int k = s ? std::atoi(s) : 1;
    return k < 1 ? 1 : k;
}

void check(long st, const char* what) {
    if (st != 0) throw std::runtime_error(std::string("MKL DFTI ") + what + ": " + DftiErrorMessage(st));
}
}  // namespace

struct ffcz_shim_plan_s {
    DFTI_DESCRIPTOR_HANDLE h = nullptr;
    fftw_complex* in = nullptr;
    fftw_complex* out = nullptr;
    int sign = -1;
    int threads = 1;
};

extern "C" fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out,
                                   int sign, unsigned /*flags*/) {
    auto* p = new ffcz_shim_plan_s;
    p->in = in;
    p->out = out;
    p->sign = sign;
    p->threads = shim_threads();
    if (rank == 1) {
        check(DftiCreateDescriptor_d_1d(&p->h, DFTI_COMPLEX, long(n[0])), "create");
    } else {
        std::vector<long> len(n, n + rank);
        check(DftiCreateDescriptor_d_md(&p->h, DFTI_COMPLEX, long(rank), len.data()), "create");
    }
    check(DftiSetValue(p->h, DFTI_PLACEMENT, DFTI_NOT_INPLACE), "placement");
    check(DftiSetValue(p->h, DFTI_THREAD_LIMIT, p->threads), "threads");
    omp_set_num_threads(p->threads);
    check(DftiCommitDescriptor(p->h), "commit");
    return p;
}

extern "C" void fftw_execute(const fftw_plan p) {
    // MKL's out-of-place transforms leave the input intact (FFTW_PRESERVE_INPUT)
    if (p->sign < 0)
        check(DftiComputeForward(p->h, p->in, p->out), "forward");
    else
        check(DftiComputeBackward(p->h, p->in, p->out), "backward");
}

extern "C" void fftw_destroy_plan(fftw_plan p) {
    if (p) {
        DftiFreeDescriptor(&p->h);
        delete p;
    }
}
