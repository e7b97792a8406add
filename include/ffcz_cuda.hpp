// ffcz_cuda.hpp — header-only C++ shim that keeps the reference's host API and types and runs
// the correction step on the B200 engine through the C-ABI (ffcz_cuda.h).
//
// A caller of the reference (/root/reference/proj/core/include/ffcz/*.hpp) switches by calling
// ffcz::cuda::correct / alternating_projection / forward_dft / inverse_dft instead of the ffcz::
// functions of the same names (or by forwarding those bodies here): the
// arguments, the returned structs and the exception classes are the reference's own.
//   ffcz::correct                 proj/core/include/ffcz/pipeline.hpp:22-24
//   ffcz::alternating_projection  proj/core/include/ffcz/projection.hpp:65-70
//   ffcz::forward_dft/inverse_dft proj/core/include/ffcz/transform.hpp:7-17
#pragma once

#include <complex>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "ffcz/archive.hpp"
#include "ffcz/bounds.hpp"
#include "ffcz/errors.hpp"
#include "ffcz/field.hpp"
#include "ffcz/metrics.hpp"
#include "ffcz/pipeline.hpp"
#include "ffcz/projection.hpp"
#include "ffcz_cuda.h"

namespace ffcz::cuda {

// Maps C-ABI status codes back onto the reference's exception taxonomy (errors.hpp:9-48).
inline void check(int status) {
    if (status == FFCZ_OK) return;
    const std::string msg = ffcz_cuda_last_error();
    switch (status) {
        case FFCZ_VALIDATION_ERROR: throw ffcz::validation_error(msg);
        case FFCZ_SYMMETRY_ERROR: throw ffcz::symmetry_error(msg);
        case FFCZ_FORMAT_ERROR: throw ffcz::format_error(msg);
        case FFCZ_IO_ERROR: throw ffcz::io_error(msg);
        case FFCZ_UNDEFINED_METRIC: throw ffcz::undefined_metric_error(msg);
        default: throw ffcz::error("ffcz_cuda: " + msg);
    }
}

// One engine context per device, created on first use (the reference is reentrant; the
// context serialises calls internally).
inline ffcz_cuda_ctx* context(int device = 0) {
    static std::mutex mu;
    static std::vector<std::unique_ptr<ffcz_cuda_ctx, void (*)(ffcz_cuda_ctx*)>> ctxs;
    std::lock_guard<std::mutex> lk(mu);
    while (static_cast<int>(ctxs.size()) <= device)
        ctxs.emplace_back(nullptr, &ffcz_cuda_destroy);
    if (!ctxs[device]) {
        ffcz_cuda_ctx* c = nullptr;
        check(ffcz_cuda_create(&c, device, nullptr));
        ctxs[device].reset(c);
    }
    return ctxs[device].get();
}

inline ffcz_field_desc describe(const Dims& dims, Precision p) {
    ffcz_field_desc d{};
    d.ndim = static_cast<int32_t>(dims.size());
    for (std::size_t a = 0; a < dims.size() && a < 3; ++a) d.dims[a] = dims[a];
    d.dtype = FFCZ_F64;  // ScalarField holds doubles (field.hpp:32-38)
    d.precision = p == Precision::f32 ? FFCZ_PRECISION_F32 : FFCZ_PRECISION_F64;
    return d;
}

inline ffcz_bounds_desc describe(const DualBounds& b) {
    ffcz_bounds_desc d{};
    d.spatial_per_point = b.spatial.per_point;
    d.spatial_global = b.spatial.global;
    d.spatial_values = b.spatial.per_point ? b.spatial.values.data() : nullptr;
    d.freq_per_component = b.frequency.per_component;
    d.freq_global = b.frequency.global;
    d.freq_re = b.frequency.per_component ? b.frequency.re.data() : nullptr;
    d.freq_im = b.frequency.per_component ? b.frequency.im.data() : nullptr;
    return d;
}

// ffcz::correct on the GPU: same arguments, same CorrectionResult (archive bytes in the .ffcz
// format, the projection report, escape count, the FP64 verification against the original
// bounds).
inline CorrectionResult correct(const ScalarField& original, const ScalarField& decompressed,
                                const DualBounds& bounds_original, int m = 16,
                                std::size_t max_iters = 1000, int device = 0) {
    bounds_original.validate_for(original.dims);
    if (original.dims != decompressed.dims || original.precision != decompressed.precision)
        throw validation_error("compute_error: dims/precision mismatch");
    const ffcz_field_desc fd = describe(original.dims, original.precision);
    const ffcz_bounds_desc bd = describe(bounds_original);
    ffcz_cuda_options opt;
    ffcz_cuda_default_options(&opt);
    opt.flags = FFCZ_WANT_ARCHIVE | FFCZ_BOUNDS_VALIDATED;  // built by DualBounds' factories
    ffcz_cuda_result r{};
    const int st = ffcz_cuda_correct(context(device), &fd, original.values.data(),
                                     decompressed.values.data(), &bd, m, max_iters, &opt, &r);
    struct Guard {
        ffcz_cuda_result* r;
        ~Guard() { ffcz_cuda_result_free(r); }
    } guard{&r};
    check(st);
    CorrectionResult out;
    out.archive_bytes.assign(r.archive, r.archive + r.archive_len);
    out.report.iterations = r.report.iterations;
    out.report.active_spatial = r.report.active_spatial;
    out.report.active_frequency = r.report.active_frequency;
    out.report.converged = r.report.converged != 0;
    out.report.residual_f = r.report.residual_f;
    out.report.residual_s = r.report.residual_s;
    out.report.wall_time_s = r.report.wall_time_s;
    out.escape_count = r.escape_count;
    out.verification.ok = r.verify_ok != 0;
    out.verification.max_spatial_excess = r.verify_max_spatial_excess;
    out.verification.max_freq_excess = r.verify_max_freq_excess;
    return out;
}

// ffcz::alternating_projection on the GPU (bounds are the WORKING bounds, as in the reference).
inline ProjectionOutcome alternating_projection(const ScalarField& epsilon0,
                                                const DualBounds& bounds_working,
                                                std::size_t max_iters,
                                                double precondition_slack = 0x1p-20,
                                                int device = 0) {
    bounds_working.validate_for(epsilon0.dims);
    const ffcz_field_desc fd = describe(epsilon0.dims, epsilon0.precision);
    const ffcz_bounds_desc bd = describe(bounds_working);
    const std::size_t n = epsilon0.size();
    ProjectionOutcome out;
    out.edits.spatial.assign(n, 0.0);
    out.edits.frequency.assign(n, {0.0, 0.0});
    out.final_epsilon = ScalarField{epsilon0.dims, std::vector<double>(n), epsilon0.precision};
    ffcz_cuda_report rep{};
    ffcz_cuda_options opt;
    ffcz_cuda_default_options(&opt);
    opt.flags = FFCZ_BOUNDS_VALIDATED;  // built by DualBounds' factories (and shrink_bounds)
    check(ffcz_cuda_alternating_projection(
        context(device), &fd, epsilon0.values.data(), &bd, max_iters, precondition_slack, &opt,
        out.edits.spatial.data(), reinterpret_cast<double*>(out.edits.frequency.data()),
        out.final_epsilon.values.data(), &rep));
    out.report.iterations = rep.iterations;
    out.report.active_spatial = rep.active_spatial;
    out.report.active_frequency = rep.active_frequency;
    out.report.converged = rep.converged != 0;
    out.report.residual_f = rep.residual_f;
    out.report.residual_s = rep.residual_s;
    out.report.wall_time_s = rep.wall_time_s;
    return out;
}

// ffcz::forward_dft on the GPU (FP64, unnormalised, full spectrum).
inline ComplexSpectrum forward_dft(const ScalarField& field, int device = 0) {
    validate_dims(field.dims);
    const ffcz_field_desc fd = describe(field.dims, Precision::f64);
    ComplexSpectrum s{field.dims, std::vector<std::complex<double>>(field.size())};
    check(ffcz_cuda_forward_dft(context(device), &fd, field.values.data(),
                                reinterpret_cast<double*>(s.values.data())));
    return s;
}

// ffcz::inverse_dft on the GPU (1/N, imaginary-residue gate -> symmetry_error).
inline ScalarField inverse_dft(const ComplexSpectrum& spectrum,
                               Precision out_precision = Precision::f64, int device = 0) {
    validate_dims(spectrum.dims);
    const ffcz_field_desc fd = describe(spectrum.dims, Precision::f64);
    ScalarField f{spectrum.dims, std::vector<double>(spectrum.size()), out_precision};
    check(ffcz_cuda_inverse_dft(context(device), &fd,
                                reinterpret_cast<const double*>(spectrum.values.data()),
                                out_precision == Precision::f32 ? FFCZ_PRECISION_F32
                                                                : FFCZ_PRECISION_F64,
                                f.values.data()));
    return f;
}

// ffcz::spectrum_bound_to_freq_bounds(ffcz::forward_dft(original), rho) (metrics.cpp:107-128) on
// the GPU.  Takes the ORIGINAL field (the device transforms it), as the CLI's --rho path does
// (proj/tools/ffcz.cpp:97-102).
inline FrequencyBounds spectrum_bound_to_freq_bounds(const ScalarField& original, double rho,
                                                     int device = 0) {
    validate_dims(original.dims);
    const ffcz_field_desc fd = describe(original.dims, Precision::f64);
    std::vector<double> d(original.size());
    check(ffcz_cuda_spectrum_bound(context(device), &fd, original.values.data(), 0, rho,
                                   d.data()));
    std::vector<double> im = d;
    return DualBounds::frequency_per_component(original.dims, std::move(d), std::move(im));
}

// ffcz::power_spectrum (metrics.cpp:11-62) on the GPU.
inline PowerSpectrum power_spectrum(const ScalarField& field, int device = 0) {
    validate_dims(field.dims);
    const ffcz_field_desc fd = describe(field.dims, Precision::f64);
    uint64_t nb = 0;
    check(ffcz_cuda_power_spectrum(context(device), &fd, field.values.data(), 0, 0, nullptr,
                                   nullptr, &nb, nullptr, nullptr));
    PowerSpectrum ps;
    ps.power.assign(nb, 0.0);
    std::vector<uint64_t> counts(nb, 0);
    int fb = 0;
    check(ffcz_cuda_power_spectrum(context(device), &fd, field.values.data(), 0, nb,
                                   ps.power.data(), counts.data(), &nb, &ps.mean, &fb));
    ps.mean_fallback = fb != 0;
    ps.k_bins.resize(nb);
    ps.counts.resize(nb);
    for (uint64_t b = 0; b < nb; ++b) {
        ps.k_bins[b] = b;
        ps.counts[b] = static_cast<std::size_t>(counts[b]);
    }
    return ps;
}

// The `ffcz metrics` quantities (proj/tools/ffcz.cpp:246-256) in one device pass set:
// psnr(original, reconstructed), ssnr(FFT(original), FFT(reconstructed)), max over
// rfe(FFT(reconstructed - original), FFT(original)), max |reconstructed - original|.
struct Metrics {
    double psnr_db, ssnr_db, max_rfe, max_spatial;
};
inline Metrics metrics(const ScalarField& original, const ScalarField& reconstructed,
                       int device = 0) {
    if (original.dims != reconstructed.dims) throw validation_error("metrics: dims mismatch");
    validate_dims(original.dims);
    const ffcz_field_desc fd = describe(original.dims, Precision::f64);
    ffcz_cuda_metrics_out m{};
    check(ffcz_cuda_metrics(context(device), &fd, original.values.data(),
                            reconstructed.values.data(), 0, &m));
    return Metrics{m.psnr_db, m.ssnr_db, m.max_rfe, m.max_spatial};
}

} // namespace ffcz::cuda
