// Drop-in parity through the C++ shim (include/ffcz_cuda.hpp): the SAME reference types go to
// the unmodified reference (ffcz::correct, CPU) and to ffcz::cuda::correct (B200), and the
// reference's own read_archive / apply_edits / verify_bounds decode the GPU archive.
// Built by `make -C oracle shim_parity` where /root/reference exists; run by
// tests/test_gpu_shim.py on the GPU box.  Prints one JSON line per case; exit status = failures.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "ffcz/archive.hpp"
#include "ffcz/baseline.hpp"
#include "ffcz/metrics.hpp"
#include "ffcz/pipeline.hpp"
#include "ffcz/projection.hpp"
#include "ffcz/transform.hpp"
#include "ffcz_cuda.hpp"

using namespace ffcz;

namespace {

ScalarField noise(const Dims& dims, std::uint64_t seed, Precision p) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    std::vector<double> v(total_samples(dims));
    for (double& x : v) {
        x = dist(rng);
        if (p == Precision::f32) x = static_cast<float>(x);
    }
    return ScalarField::create(dims, std::move(v), p);
}

double range_of(const ScalarField& f) {
    double lo = f.values[0], hi = f.values[0];
    for (double v : f.values) {
        lo = std::min(lo, v);
        hi = std::max(hi, v);
    }
    return hi - lo;
}

double peak_of(const ComplexSpectrum& s) {
    double m = 0;
    for (auto& v : s.values) m = std::max(m, std::abs(v));
    return m;
}

int failures = 0;

void run_case(const std::string& name, const ScalarField& orig, const ScalarField& dec,
              const DualBounds& b, int m) {
    CorrectionResult ref = correct(orig, dec, b, m);
    CorrectionResult gpu = ffcz::cuda::correct(orig, dec, b, m);
    // the reference decoder accepts the GPU archive and its guarantee holds
    DecodedArchive a = read_archive(gpu.archive_bytes);
    ScalarField corrected = apply_edits(dec, a);
    VerifyResult v = verify_bounds(orig, corrected, b);
    const bool same_control = ref.report.iterations == gpu.report.iterations &&
                              ref.report.converged == gpu.report.converged &&
                              ref.report.active_spatial == gpu.report.active_spatial &&
                              ref.report.active_frequency == gpu.report.active_frequency;
    const bool identical = ref.archive_bytes == gpu.archive_bytes;
    const bool ok = same_control && (!ref.report.converged || (v.ok && gpu.verification.ok));
    if (!ok) ++failures;
    std::printf(
        "{\"case\": \"%s\", \"ok\": %s, \"iterations\": [%zu, %zu], \"active_s\": [%zu, %zu], "
        "\"active_f\": [%zu, %zu], \"escapes\": [%zu, %zu], \"archive_identical\": %s, "
        "\"archive_len\": [%zu, %zu], \"ref_decoder_verify_ok\": %s, \"gpu_verify_ok\": %s}\n",
        name.c_str(), ok ? "true" : "false", ref.report.iterations, gpu.report.iterations,
        ref.report.active_spatial, gpu.report.active_spatial, ref.report.active_frequency,
        gpu.report.active_frequency, ref.escape_count, gpu.escape_count,
        identical ? "true" : "false", ref.archive_bytes.size(), gpu.archive_bytes.size(),
        v.ok ? "true" : "false", gpu.verification.ok ? "true" : "false");
}

} // namespace

int main() {
    const std::vector<Dims> pool = {{64}, {1000}, {32, 32}, {64, 48}, {16, 16, 16}, {32, 32, 32},
                                    {64, 64, 64}, {128, 128}};
    const double pct[3] = {1e-1, 1e-2, 1e-3};
    for (int c = 0; c < 24; ++c) {
        const Dims& dims = pool[c % pool.size()];
        Precision p = (c / 8) % 2 ? Precision::f64 : Precision::f32;
        ScalarField original = noise(dims, 9000 + c, p);
        const double E = 0.1 / 100.0 * range_of(original);
        const double D = pct[c % 3] / 100.0 * peak_of(forward_dft(original));
        CompressResult base = uniform_quantize_compress(original, E);
        run_case("accept_like_" + std::to_string(c), original, base.decompressed,
                 DualBounds::global(E, D), c % 5 == 4 ? 8 : 16);
    }
    // transform + projection seams
    {
        ScalarField f = noise({16, 12, 10}, 5, Precision::f64);
        ComplexSpectrum a = forward_dft(f), g = ffcz::cuda::forward_dft(f);
        double dev = 0;
        for (std::size_t k = 0; k < a.size(); ++k) dev = std::max(dev, std::abs(a.values[k] - g.values[k]));
        const bool ok = dev <= 1e-12 * peak_of(a);
        if (!ok) ++failures;
        std::printf("{\"case\": \"forward_dft\", \"ok\": %s, \"max_dev_rel\": %.3e}\n",
                    ok ? "true" : "false", dev / peak_of(a));
        ScalarField eps0 = ScalarField::create({2}, {1.0, 1.0});
        ProjectionOutcome o = ffcz::cuda::alternating_projection(eps0, DualBounds::global(1.0, 1.0), 100);
        const bool ok2 = o.report.converged && o.report.iterations == 1 &&
                         std::abs(o.final_epsilon.values[0] - 0.5) < 1e-12 &&
                         std::abs(o.edits.frequency[0].real() + 1.0) < 1e-12;
        if (!ok2) ++failures;
        std::printf("{\"case\": \"hand_trace\", \"ok\": %s}\n", ok2 ? "true" : "false");
        bool threw = false;
        try {
            ffcz::cuda::inverse_dft(ComplexSpectrum{{2}, {{1.0, 0.0}, {0.0, 1.0}}});
        } catch (const symmetry_error&) {
            threw = true;
        }
        if (!threw) ++failures;
        std::printf("{\"case\": \"symmetry_error\", \"ok\": %s}\n", threw ? "true" : "false");
        bool vthrew = false;
        try {
            ScalarField o2 = ScalarField::create({2}, {0.0, 0.0});
            ScalarField d2 = ScalarField::create({2}, {0.0, 3.0});
            ffcz::cuda::correct(o2, d2, DualBounds::global(1.0, 1.0));
        } catch (const validation_error& e) {
            vthrew = std::string(e.what()).find("index 1") != std::string::npos;
        }
        if (!vthrew) ++failures;
        std::printf("{\"case\": \"validation_error\", \"ok\": %s}\n", vthrew ? "true" : "false");
    }
    {
        // device metrics through the shim against the reference's own metrics.cpp
        ScalarField o = noise({24, 20, 18}, 91, Precision::f64);
        for (double& v : o.values) v += 2.0;
        ScalarField r = o;
        std::mt19937_64 rng(92);
        std::uniform_real_distribution<double> u(-1e-3, 1e-3);
        for (double& v : r.values) v += u(rng);
        const ComplexSpectrum X = forward_dft(o), Y = forward_dft(r);
        FrequencyBounds fr = spectrum_bound_to_freq_bounds(X, 1e-3);
        FrequencyBounds fg = ffcz::cuda::spectrum_bound_to_freq_bounds(o, 1e-3);
        double dmax = 0, bmax = 0;
        for (std::size_t k = 0; k < fr.re.size(); ++k) {
            dmax = std::max(dmax, std::abs(fr.re[k] - fg.re[k]));
            bmax = std::max(bmax, fr.re[k]);
        }
        PowerSpectrum pr = power_spectrum(o), pg = ffcz::cuda::power_spectrum(o);
        double pmax = 0, perr = 0;
        for (std::size_t b = 0; b < pr.power.size(); ++b) pmax = std::max(pmax, pr.power[b]);
        bool counts_equal = pr.counts == pg.counts && pr.mean_fallback == pg.mean_fallback;
        for (std::size_t b = 0; b < pr.power.size() && b < pg.power.size(); ++b)
            perr = std::max(perr, std::abs(pr.power[b] - pg.power[b]));
        ffcz::cuda::Metrics mg = ffcz::cuda::metrics(o, r);
        const double p_ref = psnr(o, r), s_ref = ssnr(X, Y);
        ScalarField eps = compute_error(o, r);
        double rfe_ref = 0;
        for (double v : rfe(forward_dft(eps), X)) rfe_ref = std::max(rfe_ref, v);
        const bool ok = dmax <= 1e-12 * bmax && counts_equal && perr <= 1e-12 * pmax &&
                        std::abs(mg.psnr_db - p_ref) <= 1e-10 * std::abs(p_ref) &&
                        std::abs(mg.ssnr_db - s_ref) <= 1e-9 * std::abs(s_ref) &&
                        std::abs(mg.max_rfe - rfe_ref) <= 1e-9 * rfe_ref;
        if (!ok) ++failures;
        std::printf("{\"case\": \"metrics\", \"ok\": %s, \"delta_maxdiff_rel\": %.3g, "
                    "\"counts_equal\": %s, \"power_maxdiff_rel\": %.3g, \"psnr\": [%.12g, %.12g], "
                    "\"ssnr\": [%.12g, %.12g], \"max_rfe\": [%.12g, %.12g]}\n",
                    ok ? "true" : "false", dmax / bmax, counts_equal ? "true" : "false",
                    perr / pmax, p_ref, mg.psnr_db, s_ref, mg.ssnr_db, rfe_ref, mg.max_rfe);
        bool uthrew = false;
        try {
            ffcz::cuda::metrics(ScalarField::create({2}, {3.0, 3.0}),
                                ScalarField::create({2}, {3.0, 3.5}));
        } catch (const undefined_metric_error&) {
            uthrew = true;
        }
        if (!uthrew) ++failures;
        std::printf("{\"case\": \"undefined_metric_error\", \"ok\": %s}\n",
                    uthrew ? "true" : "false");
    }
    std::printf("{\"failures\": %d}\n", failures);
    return failures;
}
