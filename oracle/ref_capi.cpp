// C entry points over the UNMODIFIED CPU reference (compiled from /root/reference/proj/core/src
// by oracle/Makefile into oracle/_ref/libffcz_ref.so).  TEST INFRASTRUCTURE ONLY: used by
// tests/ (golden-vector generation, oracle pinning) and by bench.py's reference / cpu_baseline
// leg.  Nothing in the product path links or loads this.
//
// Each function wraps one reference API and maps its exception taxonomy
// (/root/reference/proj/core/include/ffcz/errors.hpp:9-48) onto integer status codes:
//   0 ok, 1 validation_error, 2 symmetry_error, 3 format_error, 4 io_error, 5 other ffcz::error,
//   6 std::exception.

#include <chrono>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ffcz/archive.hpp"
#include "ffcz/editset.hpp"
#include "ffcz/metrics.hpp"
#include "ffcz/pipeline.hpp"
#include "ffcz/projection.hpp"
#include "ffcz/synth.hpp"
#include "ffcz/transform.hpp"

using namespace ffcz;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const validation_error& e) {
        g_err = e.what();
        return 1;
    } catch (const symmetry_error& e) {
        g_err = e.what();
        return 2;
    } catch (const format_error& e) {
        g_err = e.what();
        return 3;
    } catch (const io_error& e) {
        g_err = e.what();
        return 4;
    } catch (const ffcz::error& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 6;
    }
}

Dims make_dims(int ndim, const std::uint64_t* dims) {
    Dims d(ndim);
    for (int a = 0; a < ndim; ++a) d[a] = dims[a];
    return d;
}

ScalarField make_field(int ndim, const std::uint64_t* dims, const double* v, int precision) {
    Dims d = make_dims(ndim, dims);
    std::size_t n = total_samples(d);
    return ScalarField::create(d, std::vector<double>(v, v + n),
                               precision ? Precision::f64 : Precision::f32);
}

// Bounds exactly as the reference's DualBounds factories build them.
DualBounds make_bounds(int ndim, const std::uint64_t* dims, int spatial_per_point, double e_global,
                       const double* e_values, int freq_per_component, double d_global,
                       const double* d_re, const double* d_im) {
    Dims d = make_dims(ndim, dims);
    std::size_t n = total_samples(d);
    DualBounds b;
    b.spatial = spatial_per_point ? DualBounds::spatial_per_point(std::vector<double>(e_values, e_values + n))
                                  : DualBounds::spatial_global(e_global);
    b.frequency = freq_per_component
                      ? DualBounds::frequency_per_component(d, std::vector<double>(d_re, d_re + n),
                                                            std::vector<double>(d_im, d_im + n))
                      : DualBounds::frequency_global(d_global);
    return b;
}

template <typename T>
T* dup_vec(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(v.size() * sizeof(T) + 8));
    if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
    return p;
}

} // namespace

extern "C" {

struct ref_report {
    std::uint64_t iterations, active_spatial, active_frequency;
    std::int32_t converged;
    double residual_f, residual_s, wall_time_s;
};

struct ref_correct_out {
    ref_report report;
    std::uint64_t escape_count;
    std::int32_t verify_ok;
    double verify_max_spatial_excess, verify_max_freq_excess;
    std::uint8_t* archive;        // malloc'd; free with ffcz_ref_free
    std::uint64_t archive_len;
    double correct_wall_s;        // wall time of the whole ffcz::correct() call
};

const char* ffcz_ref_last_error() { return g_err.c_str(); }
void ffcz_ref_free(void* p) { std::free(p); }

static void fill_report(ref_report& o, const ProjectionReport& r) {
    o.iterations = r.iterations;
    o.active_spatial = r.active_spatial;
    o.active_frequency = r.active_frequency;
    o.converged = r.converged;
    o.residual_f = r.residual_f;
    o.residual_s = r.residual_s;
    o.wall_time_s = r.wall_time_s;
}

// ffcz::correct (proj/core/include/ffcz/pipeline.hpp:22-24)
int ffcz_ref_correct(int ndim, const std::uint64_t* dims, int precision, const double* original,
                     const double* decompressed, int spatial_per_point, double e_global,
                     const double* e_values, int freq_per_component, double d_global,
                     const double* d_re, const double* d_im, int m, std::uint64_t max_iters,
                     ref_correct_out* out) {
    return guarded([&] {
        ScalarField orig = make_field(ndim, dims, original, precision);
        ScalarField dec = make_field(ndim, dims, decompressed, precision);
        DualBounds b = make_bounds(ndim, dims, spatial_per_point, e_global, e_values,
                                   freq_per_component, d_global, d_re, d_im);
        auto t0 = std::chrono::steady_clock::now();
        CorrectionResult r = correct(orig, dec, b, m, max_iters);
        out->correct_wall_s =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        fill_report(out->report, r.report);
        out->escape_count = r.escape_count;
        out->verify_ok = r.verification.ok;
        out->verify_max_spatial_excess = r.verification.max_spatial_excess;
        out->verify_max_freq_excess = r.verification.max_freq_excess;
        out->archive_len = r.archive_bytes.size();
        out->archive = static_cast<std::uint8_t*>(std::malloc(r.archive_bytes.size() + 1));
        std::memcpy(out->archive, r.archive_bytes.data(), r.archive_bytes.size());
    });
}

// ffcz::alternating_projection (proj/core/include/ffcz/projection.hpp:65-70).
// Outputs dense S (N), F (N complex, interleaved re/im, FULL spectrum), final epsilon (N).
int ffcz_ref_alternating_projection(int ndim, const std::uint64_t* dims, int precision,
                                    const double* eps0, int spatial_per_point, double e_global,
                                    const double* e_values, int freq_per_component, double d_global,
                                    const double* d_re, const double* d_im, std::uint64_t max_iters,
                                    double slack, double* s_out, double* f_out, double* eps_out,
                                    ref_report* rep) {
    return guarded([&] {
        ScalarField e0 = make_field(ndim, dims, eps0, precision);
        DualBounds b = make_bounds(ndim, dims, spatial_per_point, e_global, e_values,
                                   freq_per_component, d_global, d_re, d_im);
        ProjectionOutcome o = alternating_projection(e0, b, max_iters, slack);
        std::size_t n = e0.size();
        std::memcpy(s_out, o.edits.spatial.data(), n * sizeof(double));
        std::memcpy(f_out, o.edits.frequency.data(), n * 2 * sizeof(double));
        std::memcpy(eps_out, o.final_epsilon.values.data(), n * sizeof(double));
        fill_report(*rep, o.report);
    });
}

// forward_dft (proj/core/src/transform.cpp:45-50): full complex spectrum, interleaved.
int ffcz_ref_forward_dft(int ndim, const std::uint64_t* dims, const double* x, double* out) {
    return guarded([&] {
        ScalarField f = make_field(ndim, dims, x, 1);
        ComplexSpectrum s = forward_dft(f);
        std::memcpy(out, s.values.data(), s.size() * 2 * sizeof(double));
    });
}

// inverse_dft (proj/core/src/transform.cpp:64-80), with its imaginary-residue gate.
int ffcz_ref_inverse_dft(int ndim, const std::uint64_t* dims, const double* spec, int precision,
                         double* out) {
    return guarded([&] {
        Dims d = make_dims(ndim, dims);
        std::size_t n = total_samples(d);
        std::vector<std::complex<double>> v(n);
        std::memcpy(v.data(), spec, n * 2 * sizeof(double));
        ScalarField f = inverse_dft(ComplexSpectrum::create(d, std::move(v)),
                                    precision ? Precision::f64 : Precision::f32);
        std::memcpy(out, f.values.data(), n * sizeof(double));
    });
}

// brute_force_dft (proj/core/src/transform.cpp:82-103)
int ffcz_ref_brute_force_dft(int ndim, const std::uint64_t* dims, const double* x, double* out) {
    return guarded([&] {
        ScalarField f = make_field(ndim, dims, x, 1);
        ComplexSpectrum s = brute_force_dft(f);
        std::memcpy(out, s.values.data(), s.size() * 2 * sizeof(double));
    });
}

// read_archive + apply_edits (proj/core/src/archive.cpp:137-273): corrected field.
int ffcz_ref_apply_archive(const std::uint8_t* bytes, std::uint64_t len, int ndim,
                           const std::uint64_t* dims, int precision, const double* decompressed,
                           double* corrected_out) {
    return guarded([&] {
        DecodedArchive a = read_archive(std::vector<std::uint8_t>(bytes, bytes + len));
        ScalarField dec = make_field(ndim, dims, decompressed, precision);
        ScalarField c = apply_edits(dec, a);
        std::memcpy(corrected_out, c.values.data(), c.size() * sizeof(double));
    });
}

// verify_bounds (proj/core/src/archive.cpp:275-297)
int ffcz_ref_verify_bounds(int ndim, const std::uint64_t* dims, int precision,
                           const double* original, const double* corrected, int spatial_per_point,
                           double e_global, const double* e_values, int freq_per_component,
                           double d_global, const double* d_re, const double* d_im,
                           double* max_s, double* max_f, int* ok) {
    return guarded([&] {
        ScalarField o = make_field(ndim, dims, original, precision);
        ScalarField c = make_field(ndim, dims, corrected, precision);
        DualBounds b = make_bounds(ndim, dims, spatial_per_point, e_global, e_values,
                                   freq_per_component, d_global, d_re, d_im);
        VerifyResult v = verify_bounds(o, c, b);
        *max_s = v.max_spatial_excess;
        *max_f = v.max_freq_excess;
        *ok = v.ok;
    });
}

// synth_field (proj/core/src/synth.cpp:53-88); kind: 0 white,1 power-law,2 exponential,3 impulse,4 constant
int ffcz_ref_synth_field(int kind, int ndim, const std::uint64_t* dims, std::uint64_t seed,
                         double param, double* out) {
    return guarded([&] {
        ScalarField f = synth_field(static_cast<SynthKind>(kind), make_dims(ndim, dims), seed, param);
        std::memcpy(out, f.values.data(), f.size() * sizeof(double));
    });
}

// spectrum_bound_to_freq_bounds (proj/core/src/metrics.cpp:107-128) on forward_dft(original).
int ffcz_ref_rho_bounds(int ndim, const std::uint64_t* dims, const double* original, double rho,
                        double* delta_out) {
    return guarded([&] {
        ScalarField f = make_field(ndim, dims, original, 1);
        FrequencyBounds fb = spectrum_bound_to_freq_bounds(forward_dft(f), rho);
        std::memcpy(delta_out, fb.re.data(), fb.re.size() * sizeof(double));
    });
}

// read_archive (proj/core/src/archive.cpp:137-225) -> the edit set as the archive carries it:
// flag bytes (LSB-first), int32 codes (re-quantised from the dequantised values with the
// reference's own quantize_edits, editset.cpp:86-119 — exact, value = code * step), escapes.
// Buffers malloc'd; free each with ffcz_ref_free.  Used to pin flags / codes of large goldens
// by digest (tests/golden/make_golden.py) without a Python Huffman decoder.
struct ref_archive_edits {
    std::uint8_t* spatial_flags;   std::uint64_t spatial_flag_bytes;
    std::uint8_t* frequency_flags; std::uint64_t frequency_flag_bytes;
    std::int32_t* spatial_codes;   std::uint64_t n_spatial;
    std::int32_t* frequency_codes; std::uint64_t n_frequency;   // 2 lanes per entry
    std::uint64_t* escape_index;   std::int32_t* escape_freq;   std::uint64_t n_escapes;
    std::int32_t converged;
};

int ffcz_ref_archive_edits(const std::uint8_t* bytes, std::uint64_t len, ref_archive_edits* out) {
    return guarded([&] {
        DecodedArchive a = read_archive(std::vector<std::uint8_t>(bytes, bytes + len));
        out->spatial_flags = dup_vec(a.edits.spatial_flags.bytes());
        out->spatial_flag_bytes = a.edits.spatial_flags.bytes().size();
        out->frequency_flags = dup_vec(a.edits.frequency_flags.bytes());
        out->frequency_flag_bytes = a.edits.frequency_flags.bytes().size();
        auto si = flagged_indices(a.edits.spatial_flags);
        auto fi = flagged_indices(a.edits.frequency_flags);
        out->spatial_codes = dup_vec(quantize_edits(a.edits.spatial_values, si, a.params));
        out->n_spatial = si.size();
        out->frequency_codes = dup_vec(quantize_edits(a.dims, a.edits.frequency_values, fi, a.params));
        out->n_frequency = fi.size();
        std::vector<std::uint64_t> ei;
        std::vector<std::int32_t> ef;
        for (const auto& e : a.escapes) {
            ei.push_back(e.index);
            ef.push_back(e.frequency ? 1 : 0);
        }
        out->escape_index = dup_vec(ei);
        out->escape_freq = dup_vec(ef);
        out->n_escapes = ei.size();
        out->converged = a.converged;
    });
}

} // extern "C"
