/*
 * ffcz_cuda.h — C-ABI of the B200-native FFCz correction step (libffcz_cuda.so).
 *
 * The reference (/root/reference/proj) has no plugin/FFI layer; its seam is the C++ library
 * call `ffcz::correct(original, decompressed, bounds_original, m, max_iters)`
 * (proj/core/include/ffcz/pipeline.hpp:22-24), with a secondary seam
 * `ffcz::alternating_projection(eps0, bounds_working, max_iters, slack)`
 * (proj/core/include/ffcz/projection.hpp:65-70) and the transform helpers
 * `forward_dft` / `inverse_dft` (proj/core/include/ffcz/transform.hpp:7-17).
 * Every entry point below replaces one of those; the C++ shim in include/ffcz_cuda.hpp maps the
 * reference's own types (ScalarField, DualBounds, CorrectionResult, ...) onto these plain-pointer
 * signatures so callers of the reference are unchanged.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Field buffers are row-major, last index fastest, exactly as
 *    ffcz::ScalarField::values.  Complex buffers are interleaved (re, im) doubles, exactly as
 *    std::vector<std::complex<double>>.
 *  - Inputs are caller-owned.  With FFCZ_INPUTS_ON_DEVICE they are device pointers on the
 *    context's device, otherwise host pointers (copied in inside the call).
 *  - Results are library-owned host buffers released by ffcz_cuda_result_free().
 *  - Status codes mirror the reference's exception classes (errors.hpp:9-48); the message of the
 *    last failure on the calling thread is ffcz_cuda_last_error().
 *  - One CUDA stream per context; a context is internally locked (calls on one context
 *    serialise; distinct contexts run concurrently), matching the reference's reentrancy
 *    (SURVEY.md §8b "Threading").
 */
#ifndef FFCZ_CUDA_H
#define FFCZ_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFCZ_CUDA_ABI_VERSION 1

typedef enum ffcz_cuda_status {
    FFCZ_OK = 0,
    FFCZ_VALIDATION_ERROR = 1, /* ffcz::validation_error: shapes, precondition, quantizer range */
    FFCZ_SYMMETRY_ERROR = 2,   /* ffcz::symmetry_error: inverse of a non-Hermitian spectrum      */
    FFCZ_FORMAT_ERROR = 3,     /* ffcz::format_error: archive encode/decode                      */
    FFCZ_IO_ERROR = 4,         /* ffcz::io_error                                                 */
    FFCZ_CUDA_ERROR = 5,       /* CUDA runtime / launch failure (no reference counterpart)      */
    FFCZ_UNSUPPORTED = 6,      /* shape/size the device engine does not implement yet           */
    FFCZ_OUT_OF_MEMORY = 7,
    FFCZ_UNDEFINED_METRIC = 8  /* ffcz::undefined_metric_error (metrics.cpp: psnr/ssnr/rfe)      */
} ffcz_cuda_status;

/* Sample type of the buffers passed in (the reference always holds doubles; f32 device buffers
 * are accepted so an f32 dataset need not be widened on the host). */
typedef enum ffcz_cuda_dtype { FFCZ_F32 = 0, FFCZ_F64 = 1 } ffcz_cuda_dtype;

/* ffcz::Precision (field.hpp:12): the on-disk width tag carried into the archive. */
typedef enum ffcz_cuda_precision { FFCZ_PRECISION_F32 = 0, FFCZ_PRECISION_F64 = 1 } ffcz_cuda_precision;

typedef struct ffcz_field_desc {
    int32_t ndim;       /* 1..3 (validate_dims, field.cpp:8-18) */
    uint64_t dims[3];   /* row-major extents, dims[ndim-1] fastest */
    int32_t dtype;      /* ffcz_cuda_dtype of original/decompressed/eps0 buffers */
    int32_t precision;  /* ffcz_cuda_precision tag (ScalarField::precision) */
} ffcz_field_desc;

/* ffcz::DualBounds (bounds.hpp:11-47).  Per-point / per-component arrays cover all N samples /
 * the FULL N-entry spectrum, as in the reference; they live where the inputs live. */
typedef struct ffcz_bounds_desc {
    int32_t spatial_per_point;
    double spatial_global;
    const double* spatial_values;  /* N, when spatial_per_point */
    int32_t freq_per_component;
    double freq_global;
    const double* freq_re;         /* N, when freq_per_component */
    const double* freq_im;         /* N, when freq_per_component */
} ffcz_bounds_desc;

/* Arithmetic policy of the projection loop.
 *  FFCZ_POLICY_FP64: every pass in FP64 with the reference control flow (K3a/K3b split):
 *                    iterations, flags and values follow the reference to FFT round-off.
 *  FFCZ_POLICY_MIXED: FP32 fused passes while excess/peak > tau_switch, then FP64 with the
 *                    reference control flow: iterations within +-1 of the
 *                    reference, both bounds still hold exactly (FP64 gate).  Fused shapes only
 *                    (others run FP64); batched frames run it per frame on the lanes.
 *  The FP64 gate (escape repair + verify) always runs in FP64. */
typedef enum ffcz_cuda_policy { FFCZ_POLICY_FP64 = 0, FFCZ_POLICY_MIXED = 1 } ffcz_cuda_policy;

/* option flags */
#define FFCZ_INPUTS_ON_DEVICE (1u << 0) /* original/decompressed/bounds are device pointers      */
#define FFCZ_WANT_ARCHIVE (1u << 1)     /* serialise the .ffcz archive (see zlib_level)        */
#define FFCZ_WANT_EDITS (1u << 2)       /* copy flags, int32 codes and escapes to the host      */
#define FFCZ_WANT_CORRECTED (1u << 3)   /* copy the FP64 corrected field to the host            */
#define FFCZ_FORCE_UNFUSED (1u << 4)    /* use the per-op (unfused) loop even for 2^k shapes    */
#define FFCZ_DEVICE_ENCODE (1u << 5)    /* archive: zigzag + canonical Huffman on the device (same
                                           payload bytes as huffman.cpp); zlib_level 0 = stored  */
#define FFCZ_BOUNDS_VALIDATED (1u << 6) /* the caller guarantees DualBounds' invariants (every
                                           per-point / per-component entry > 0 and finite, Re/Im
                                           lanes Hermitian-consistent: bounds.cpp:10-59), e.g.
                                           the C++ shim, whose ffcz::DualBounds was built by the
                                           reference's factories; otherwise they are checked
                                           (FFCZ_VALIDATION_ERROR with the reference's message) */
#define FFCZ_REPAIR_REFERENCE_ORDER (1u << 7) /* escape repair in the reference's order: check
                                           eps_tilde = eps0 + S_dq + IFFT(F_dq) each round
                                           (pipeline.cpp:134-160), then a separate verify_bounds
                                           transform; default: repair the decoder's own view
                                            */
#define FFCZ_F_ACCUMULATE (1u << 8)     /* accumulate F += displacement in every f-clip
                                           (projection.cpp:117-119); default: mark the clipped
                                           components and rebuild F once at the gate */

/* zlib_level value: the archive is assembled from device-encoded streams (deflate.cu): Huffman
 * payloads byte-identical to huffman.cpp, each stream framed as outer_compress does
 * (streams.cpp:21-32: u64 raw size + a zlib stream) with fixed-Huffman / stored deflate blocks
 * written on the GPU, header CRC-32C over the bound arrays on the GPU when they are resident
 * there.  The reference's read_archive (archive.cpp:137-225, zlib uncompress) decodes it to the
 * same edits; only the outer stage's bytes differ from zlib-9's. */
#define FFCZ_OUTER_DEVICE (-1)

typedef struct ffcz_cuda_options {
    uint32_t flags;
    int32_t policy;          /* ffcz_cuda_policy */
    double tau_switch;       /* MIXED: switch to FP64 when max_excess/peak <= tau (default 1e-4) */
    int32_t zlib_level;      /* archive outer stage: FFCZ_OUTER_DEVICE (default) = every stream
                                encoded on the device; 0..9 = host zlib at that level after the
                                Huffman stage (host, or device with FFCZ_DEVICE_ENCODE); 9 =
                                the reference's bytes (streams.cpp:21-32, Z_BEST_COMPRESSION) */
} ffcz_cuda_options;

/* ffcz::ProjectionReport (projection.hpp:17-25) */
typedef struct ffcz_cuda_report {
    uint64_t iterations;
    uint64_t active_spatial;
    uint64_t active_frequency; /* counted over the FULL spectrum, as the reference */
    int32_t converged;
    double residual_f;
    double residual_s;
    double wall_time_s;        /* device time of the loop (CUDA events) */
} ffcz_cuda_report;

/* ffcz::EscapeEntry (editset.hpp:34-39) */
typedef struct ffcz_cuda_escape {
    int32_t frequency;
    uint64_t index;
    double re;
    double im;
} ffcz_cuda_escape;

/* ffcz::CorrectionResult (pipeline.hpp:11-16) + the device-side products. */
typedef struct ffcz_cuda_result {
    ffcz_cuda_report report;
    uint64_t iterations_fp32;      /* passes run by the FP32 phase (MIXED) */
    uint64_t iterations_fp64;      /* passes run by the FP64 phase */
    uint64_t escape_rounds;        /* escape-repair rounds run (pipeline.cpp:114-163) */
    uint64_t escape_count;
    int32_t verify_ok;             /* ffcz::VerifyResult against the ORIGINAL bounds, FP64 */
    double verify_max_spatial_excess;
    double verify_max_freq_excess;
    /* edit set (FFCZ_WANT_EDITS): LSB-first flag bytes, int32 codes in flag order
     * (frequency codes interleaved Re, Im), escapes ordered as the reference's std::map */
    uint64_t n_spatial, n_frequency;
    uint8_t* spatial_flags;   uint64_t spatial_flag_bytes;
    uint8_t* frequency_flags; uint64_t frequency_flag_bytes;
    int32_t* spatial_codes;   int32_t* frequency_codes;
    ffcz_cuda_escape* escapes;
    double* corrected;        /* FFCZ_WANT_CORRECTED: N doubles, decompressed + decoded edits */
    uint8_t* archive;         /* FFCZ_WANT_ARCHIVE: .ffcz bytes (proj/docs/FORMAT.md) */
    uint64_t archive_len;
    /* timing (CUDA events on the context stream), milliseconds */
    double t_feasible_ms;     /* inputs resident -> verified edits + corrected field resident */
    double t_loop_ms;         /* alternating projection only */
    double t_gate_ms;         /* compaction, quantisation, escape repair, FP64 verify */
    double t_h2d_ms, t_d2h_ms, t_archive_ms;
    uint64_t kernel_launches; /* kernels this call launched (incl. early-exit speculative ones) */
} ffcz_cuda_result;

typedef struct ffcz_cuda_ctx ffcz_cuda_ctx;

/* Context on one device; `stream` is a cudaStream_t to run on (NULL = a private stream). */
int ffcz_cuda_create(ffcz_cuda_ctx** out, int device, void* stream);
void ffcz_cuda_destroy(ffcz_cuda_ctx* ctx);
const char* ffcz_cuda_last_error(void);
int ffcz_cuda_abi_version(void);
void ffcz_cuda_default_options(ffcz_cuda_options* opt);

/* Replaces ffcz::correct (pipeline.cpp:26-178). */
int ffcz_cuda_correct(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const void* original,
                      const void* decompressed, const ffcz_bounds_desc* bounds_original, int m,
                      uint64_t max_iters, const ffcz_cuda_options* opt, ffcz_cuda_result* out);
void ffcz_cuda_result_free(ffcz_cuda_result* r);

/* Batched frames (BASELINE config 3: many independent 2-D frames): nframes independent
 * ffcz::correct() calls (pipeline.cpp:26-178) on frames of shape `frame` stored back to back in
 * `original` / `decompressed` (host or device per opt->flags); bounds[i] / out[i] are frame i's
 * DualBounds and CorrectionResult (free each with ffcz_cuda_result_free).  `lanes` host threads
 * (<= 0: 8) each drive a sub-context with its own stream; the context stream is ordered before
 * and after the batch.  Results are identical to one ffcz_cuda_correct() per frame. */
int ffcz_cuda_correct_batch(ffcz_cuda_ctx* ctx, const ffcz_field_desc* frame, uint64_t nframes,
                            const void* original, const void* decompressed,
                            const ffcz_bounds_desc* bounds, int m, uint64_t max_iters,
                            const ffcz_cuda_options* opt, int lanes, ffcz_cuda_result* out);

/* Slab-decomposed correction of one volume across ranks (BASELINE configs 4/5).
 * The orchestration (transposes = all-to-alls, all-reduced loop decisions, cross-rank escape
 * repair) is paper_2601_01596_b200/slab.py over torch.distributed; this entry point runs one
 * per-rank device step of it on device buffers, on the context stream.  Buffers: real slabs
 * d0 x d1 x n2 FP64 (inputs: `in_dtype`), half spectra d0 x d1 x P complex FP64 with
 * P = round_up(n2/2+1, 16) (ffcz_cuda_slab_pitch), bitmaps uint32 LSB-first.  Bounds are global
 * (e, delta) or per point / per component (e_arr, d_re, d_im); `fscale` scales them to the
 * working bounds (1 - 2^-m) where an op takes working bounds.  Ops that reduce synchronise the stream
 * and return their scalars in out[0..3] -- except in the device-resident loop: FWD_LOCAL,
 * COL0_CHECK, COL0_CLIP_INV and INV_SCLIP take the loop's int32 done flag in p9 (they return at
 * once when it is set) and COL0_CHECK with p1 != NULL writes (peak, excess) to the device doubles
 * p1 instead of returning them, so the orchestrator all-reduces and decides (FFCZ_SLAB_DECIDE)
 * without a host sync per iteration. */
typedef enum ffcz_cuda_slab_opcode {
    FFCZ_SLAB_EPS0 = 0,           /* p0 orig, p1 dec, p2 eps -> out: first bad index (E(1+2^-20)),
                                     first bad index (working E * (1+slack), slack = delta), -1 none */
    FFCZ_SLAB_FWD_LOCAL = 1,      /* p0 real x -> p1 half: R2C rows + forward FFT along axis 1 */
    FFCZ_SLAB_COL0_CHECK = 2,     /* p0 half in place: forward axis 0 + check_convergence
                                     (projection.cpp:29-52) vs delta*fscale -> out: peak, excess */
    FFCZ_SLAB_COL0_CLIP_INV = 3,  /* p0 half in place: project_onto_fcube (F p1 dense on `first`,
                                     clip map p2 |= moved) + inverse axis 0 */
    FFCZ_SLAB_COL0_PLAIN = 4,     /* p0 src -> p1 dst along axis 0, direction `dir` */
    FFCZ_SLAB_COL0_REBUILD = 5,   /* p0 half (FFT(eps0+S) after axis 1) -> F p3 = map p2 ?
                                     delta p1 - forward axis 0 : 0 */
    FFCZ_SLAB_COL0_MARK = 6,      /* p0 half in place: forward axis 0; violation bitmap p1 over
                                     storage offsets vs delta (pipeline.cpp:140-147) -> out: any */
    FFCZ_SLAB_COL0_VERIFY = 7,    /* p0 half: forward axis 0, max(|.|-delta) > 0 -> out: excess */
    FFCZ_SLAB_INV_SCLIP = 8,      /* p0 half (clobbered): inverse axis 1, C2R x 1/n_total,
                                     project_onto_scube vs e*fscale -> p1 eps, S p2 */
    FFCZ_SLAB_INV_REPAIR_VERIFY = 9, /* p0 half (clobbered) -> p1 eps_tilde; p2 orig, p3 dec,
                                     p4 spat_cur (repaired in place), p5 final eps, p6 escape
                                     bitmap, p7 corrected, p8 eps_v -> out: dirty, spatial excess;
                                     p8 NULL: decoder-view repair (p1 receives the decoder view
                                     and the repair checks it) */
    FFCZ_SLAB_INV_VERIFY = 10,    /* p0 half -> p1 eps_v; p2 orig, p3 dec, p4 spat_cur,
                                     p5 corrected -> out: spatial excess */
    FFCZ_SLAB_RESIDUAL_S = 11,    /* p0 eps -> out: max(|eps| - e*fscale, 0) */
    FFCZ_SLAB_EPS0_PLUS_S = 12,   /* p0 orig, p1 dec, p2 S -> p3 (dec - orig) + S */
    FFCZ_SLAB_GATE = 13,          /* p0 S, p1 F (natural half) -> p2 spat_cur, p3 freq_cur,
                                     p4 keep_s, p5 esc_s, p6 keep_f, p7 esc_f bitmaps, p8 codes_s,
                                     p9 codes_f (editset.cpp:43-133, pipeline.cpp:57-106)
                                     -> out: active_s, active_f, kept_s, kept_f */
    FFCZ_SLAB_DECIDE = 14,        /* device-resident loop: p0 all-reduced (peak, excess) doubles,
                                     p1 state (passes, residual_f) doubles, p9 int32 (done,
                                     converged); max_iters in n_total (projection.cpp:106-116) */
    /* fused all-to-all (slab.py peer path, world >= 2): the pass stores its outputs straight into
     * the receive buffers of the ranks that own them in the other layout; p8 = device array of the
     * `world` receive buffers (IPC-mapped, ffcz_cuda_ipc_*), this rank's own at [rank].  The
     * orchestrator orders the ranks (a device-side barrier) after each such op. */
    FFCZ_SLAB_FWD_LOCAL_PEER = 15, /* p0 real x -> p1 half A (c0, n1, P) work buffer: R2C rows,
                                     forward axis 1 scattered into the B (n0, c1, P) buffers p8 */
    FFCZ_SLAB_COL0_CLIP_INV_PEER = 16 /* p0 B half (read only): COL0_CLIP_INV (F p1, map p2)
                                     with the inverse axis-0 outputs scattered into the A
                                     (c0, n1, P) buffers p8 */
} ffcz_cuda_slab_opcode;

/* ffcz_cuda_slab_op.pad flag: a one-rank slab (B layout == natural layout); the COL0 ops
 * transform axis 1 and FWD_LOCAL / INV_* transform axis 0 (the single-volume engine's order) */
#define FFCZ_SLAB_SWAP_AXES 1

typedef struct ffcz_cuda_slab_op {
    int32_t op;          /* ffcz_cuda_slab_opcode */
    int32_t dir;         /* COL0_PLAIN: -1 forward, +1 inverse */
    int32_t first;       /* CLIP passes: the first clip pass (dense F / S write) */
    int32_t in_dtype;    /* ffcz_cuda_dtype of orig / dec */
    int32_t m;           /* GATE: quantiser m */
    int32_t pad;         /* flags: FFCZ_SLAB_SWAP_AXES */
    uint64_t d0, d1, n2; /* local geometry of the buffer(s) the op works on */
    uint64_t n_total;    /* global sample count (C2R normalisation) */
    double e, delta, fscale, slack;
    void* p[10];
    /* per-point E over the op's natural slab (NULL: global e) and per-component Delta lanes in
     * the pitched half layout of the op's spectrum buffer (NULL: global delta; d_im NULL: the Re
     * lane serves both, rho mode); bounds.hpp:11-47 across ranks */
    const double* e_arr;
    const double* d_re;
    const double* d_im;
    int32_t rank, world; /* *_PEER ops: this rank and the slab world size */
} ffcz_cuda_slab_op;
int ffcz_cuda_slab(ffcz_cuda_ctx* ctx, const ffcz_cuda_slab_op* op, double out[4]);
uint64_t ffcz_cuda_slab_pitch(uint64_t n2);
/* Kernels this context has launched so far (every correct / slab op; bench.py's gpu_launches). */
uint64_t ffcz_cuda_launch_count(ffcz_cuda_ctx* ctx);

/* CUDA IPC of the slab receive buffers (the *_PEER ops): handle of the allocation holding `ptr`
 * plus ptr's byte offset in it; open maps another process's handle (its base address), close
 * unmaps it.  No reference counterpart: the reference runs one volume per process. */
int ffcz_cuda_ipc_handle(ffcz_cuda_ctx* ctx, const void* ptr, unsigned char handle[64],
                         uint64_t* offset);
int ffcz_cuda_ipc_open(ffcz_cuda_ctx* ctx, const unsigned char handle[64], void** base);
int ffcz_cuda_ipc_close(ffcz_cuda_ctx* ctx, void* base);

/* Replaces ffcz::alternating_projection (projection.cpp:81-142).  eps0 is a field of
 * field->dtype; bounds are the WORKING bounds.  Outputs (host, caller-allocated, may be NULL):
 * spatial_edits N doubles, frequency_edits 2N doubles (FULL spectrum, interleaved),
 * final_epsilon N doubles. */
int ffcz_cuda_alternating_projection(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field,
                                     const void* eps0, const ffcz_bounds_desc* bounds_working,
                                     uint64_t max_iters, double precondition_slack,
                                     const ffcz_cuda_options* opt, double* spatial_edits,
                                     double* frequency_edits, double* final_epsilon,
                                     ffcz_cuda_report* report);

/* ---- device metrics (proj/core/src/metrics.cpp) ----------------------
 * Field buffers are host pointers, or device pointers with on_device = 1 (then delta_out is a
 * device pointer too).  dtype per field->dtype; everything is computed in FP64. */

/* Replaces ffcz::spectrum_bound_to_freq_bounds(ffcz::forward_dft(original), rho)
 * (metrics.cpp:107-128, called at proj/tools/ffcz.cpp:97-102): writes the FULL-spectrum
 * per-component Delta (N doubles; the Re and Im lanes of the reference's DualBounds are equal).
 * rho < 0 or non-finite -> FFCZ_VALIDATION_ERROR. */
int ffcz_cuda_spectrum_bound(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const void* original,
                             int on_device, double rho, double* delta_out);

/* The quantities `ffcz metrics` reports (proj/tools/ffcz.cpp:246-256): psnr(original,
 * reconstructed), ssnr(FFT(original), FFT(reconstructed)), max over rfe(FFT(reconstructed -
 * original), FFT(original)) and max |reconstructed - original|.  psnr / ssnr are +inf for
 * identical inputs; the reference's undefined_metric_error cases (constant original with
 * nonzero error, zero-energy or all-zero original spectrum) -> FFCZ_UNDEFINED_METRIC. */
typedef struct ffcz_cuda_metrics_out {
    double psnr_db;
    double ssnr_db;
    double max_rfe;
    double max_spatial;
} ffcz_cuda_metrics_out;
int ffcz_cuda_metrics(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const void* original,
                      const void* reconstructed, int on_device, ffcz_cuda_metrics_out* out);

/* Replaces ffcz::power_spectrum (metrics.cpp:11-62): shell-binned power of the normalised
 * fluctuation spectrum.  *nbins_out = round(|centred Nyquist corner|) + 1; power == NULL is a
 * size query; capacity < nbins -> FFCZ_VALIDATION_ERROR.  power[b] = sum |X_k|^2, counts[b] =
 * number of full-spectrum cells in shell b; mean / mean_fallback as PowerSpectrum. */
int ffcz_cuda_power_spectrum(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const void* x,
                             int on_device, uint64_t capacity, double* power, uint64_t* counts,
                             uint64_t* nbins_out, double* mean_out, int* mean_fallback_out);

/* Replaces ffcz::forward_dft (transform.cpp:45-50): FP64, unnormalised; out = FULL spectrum,
 * 2N doubles interleaved.  Host pointers. */
int ffcz_cuda_forward_dft(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const double* x,
                          double* spectrum_out);

/* Replaces ffcz::inverse_dft (transform.cpp:64-80): 1/N-normalised inverse of a FULL spectrum
 * (2N doubles) with the reference's imaginary-residue gate (FFCZ_SYMMETRY_ERROR).  out_precision
 * selects the tolerance (1e-6 f32 / 1e-10 f64 of max|Re|). */
int ffcz_cuda_inverse_dft(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const double* spectrum,
                          int out_precision, double* x_out);

/* Half-spectrum (R2C) transform in FP32 or FP64 on device pointers; out has
 * prod(dims[:-1]) rows of (dims[-1]/2+1) complex, row-major.  Used by the engine tests and
 * the per-pass roofline bench. dtype selects float/double for both buffers. */
int ffcz_cuda_r2c_device(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const void* x_dev,
                         void* half_dev);
int ffcz_cuda_c2r_device(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const void* half_dev,
                         void* x_dev);

/* Per-kernel-class device timing (CUDA events around every launch of the engine's passes),
 * used by bench.py for the roofline of the dominant kernel.  bytes = ALGORITHMIC bytes
 * (each element read once + written once).  Launches shorter than 20% of the
 * longest launch of the same class and size are speculative loop launches that returned at the
 * convergence gate; they are counted in `gated` and excluded from launches / total_ms / bytes. */
typedef struct ffcz_cuda_kernel_stat {
    char name[40];
    uint64_t launches;
    uint64_t gated;
    double total_ms;
    double bytes;
} ffcz_cuda_kernel_stat;
int ffcz_cuda_profile_enable(ffcz_cuda_ctx* ctx, int enable); /* 1: clear + start, 0: stop */
int ffcz_cuda_profile_read(ffcz_cuda_ctx* ctx, ffcz_cuda_kernel_stat* out, int max, int* n);

/* Per-pass micro-benchmark: each pass kind on a synthetic field of this geometry and dtype,
 * `reps` launches each (tools/passbench.py, profiles/). */
int ffcz_cuda_bench_passes(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, int reps,
                           ffcz_cuda_kernel_stat* out, int max, int* n);

/* Replaces ffcz::apply_edits(decompressed, ffcz::read_archive(bytes)) (archive.cpp:137-273):
 * corrected = decompressed + spatial edits + Re(IFFT(frequency edits)) in FP64.  The host parses
 * the container (header, CRC-32C, zlib stages: FFCZ_FORMAT_ERROR on a corrupt archive); the
 * Huffman index streams are decoded, dequantised and scattered on the device.  `field` gives the
 * decompressed field's dims (must match the archive) and dtype; with FFCZ_INPUTS_ON_DEVICE in
 * `flags`, decompressed and corrected (N doubles) are device pointers, else host. */
int ffcz_cuda_apply_archive(ffcz_cuda_ctx* ctx, const uint8_t* archive, uint64_t len,
                            const ffcz_field_desc* field, const void* decompressed, uint32_t flags,
                            double* corrected);

/* Device Huffman encoder on host codes (test hook): writes the huffman::encode payload
 * (huffman.cpp:156-251) of zigzag(codes[0..n)) into out (capacity cap); *len = its length. */
int ffcz_cuda_huffman_encode(ffcz_cuda_ctx* ctx, const int32_t* codes, uint64_t n, uint8_t* out,
                             uint64_t cap, uint64_t* len);

/* The device outer stage (deflate.cu) on n host bytes: writes outer_compress's framing
 * (streams.cpp:21-32: u64 raw size + a zlib stream of fixed-Huffman / stored blocks made on the
 * GPU) into out (capacity cap); *len = its length (out may be NULL to query it). */
int ffcz_cuda_outer_compress(ffcz_cuda_ctx* ctx, const uint8_t* data, uint64_t n, uint8_t* out,
                             uint64_t cap, uint64_t* len);

/* CRC-32C (archive.cpp:61-71) of n bytes computed on the device (crc32c_raw_device + the host
 * combine algebra); data is a device pointer when on_device, else host (copied in first). */
int ffcz_cuda_crc32c_device(ffcz_cuda_ctx* ctx, const uint8_t* data, uint64_t n, int on_device,
                            uint32_t* crc);

/* CRC-32C (archive.cpp:61-71), exported for the format tests. */
uint32_t ffcz_cuda_crc32c(const uint8_t* data, size_t len);

#ifdef __cplusplus
}
#endif

#endif /* FFCZ_CUDA_H */
