/*
 * seriesaug_b200.h -- C ABI of the B200 backend for the seriesaug batched
 * augmentation pipeline (reference: /root/reference/pkg/src/seriesaug).
 *
 * Drop-in boundary.  The reference is a pure-Python package; its plugin API
 * (Augmenter / SpectralAugmenter / Pipeline) stays in Python
 * (package paper_2601_03159_b200) and binds these entry points with ctypes.
 * Each entry point names the reference interface it replaces.
 *
 * Conventions
 *   - Plain C types only; no torch / CUDA types in signatures (streams are
 *     passed as void* holding a cudaStream_t, NULL = legacy default stream).
 *   - Every function is no-throw and returns an int status (SA_OK == 0, <0 on
 *     error); sa_last_error() returns a thread-local message for the last
 *     failure on the calling thread.
 *   - Device pointers (d_*) are owned by the caller.  Host pointers (h_*) are
 *     owned by the caller; the library stages them through its own pinned
 *     buffers unless they are already page-locked.
 *   - Batches are C-contiguous row-major float64 (n_series x length), exactly
 *     the reference's Batch.values layout (reference core.py:85-106).
 *   - Randomness is a pure function of (master_seed, stage index, GLOBAL
 *     series index) (reference core.py:48-82); series_offset is the global
 *     index of row 0, so disjoint row ranges on different GPUs reproduce the
 *     single-device result bit for bit.
 *   - Parameter validation is the Python layer's job (reference core.py:201-212,
 *     pipeline.py:116-131) and happens before any call here; the library only
 *     re-checks what it needs for memory safety.
 */
#ifndef SERIESAUG_B200_H
#define SERIESAUG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SA_ABI_VERSION 1

/* ---- status codes --------------------------------------------------------
 * The Python shim maps SA_ERR_NONFINITE to InvalidInputError (reference
 * core.py:104-105), SA_ERR_WARP_MONOTONE to RuntimeError (reference
 * warp.py:44-45), SA_ERR_INVALID_ARG to InvalidConfigError, everything else to
 * RuntimeError. */
#define SA_OK                   0
#define SA_ERR_INVALID_ARG     -1
#define SA_ERR_NONFINITE       -2
#define SA_ERR_WARP_MONOTONE   -3
#define SA_ERR_CUDA            -4
#define SA_ERR_UNSUPPORTED     -5
#define SA_ERR_NO_DEVICE       -6

/* ---- stage operation codes ----------------------------------------------
 * One per augmenter kind (reference AUGMENTER_REGISTRY, core.py:37,196-199).
 * Parameter slots: f[] doubles, i[] int64s; see each line. */
#define SA_OP_JITTER           1   /* basic.py:30    f0 sigma                           */
#define SA_OP_SCALE            2   /* basic.py:47    f0 sigma_factor                    */
#define SA_OP_ROTATE           3   /* basic.py:63                                       */
#define SA_OP_PERMUTE          4   /* basic.py:74    i0 n_segments                      */
#define SA_OP_CROP             5   /* basic.py:107   i0 size                            */
#define SA_OP_REVERSE          6   /* basic.py:138                                      */
#define SA_OP_RESIZE           7   /* basic.py:149   i0 target_len                      */
#define SA_OP_QUANTIZE         8   /* basic.py:180   i0 n_levels                        */
#define SA_OP_DRIFT            9   /* basic.py:210   f0 max_drift, i0 n_points          */
#define SA_OP_NOISE_UNIFORM   10   /* basic.py:352   f0 half_width                      */
#define SA_OP_NOISE_GAUSSIAN  11   /* basic.py:356   f0 sigma                           */
#define SA_OP_NOISE_SPIKE     12   /* basic.py:360   i0 count, f0 magnitude             */
#define SA_OP_NOISE_SLOPE     13   /* basic.py:371   f0 max_offset                      */
#define SA_OP_REPEAT          14   /* basic.py:378   i0 r                               */
#define SA_OP_APP             15   /* freqaugment.py:79  f0 sigma_amp, f1 sigma_phase   */
#define SA_OP_FREQ_MASK       16   /* freqaugment.py:132 i0 width                       */
#define SA_OP_TIME_WARP       17   /* warp.py:54     i0 n_knots, f0 intensity           */
#define SA_OP_WINDOW_WARP     18   /* warp.py:79     i0 window_size, i1 n_knots, f0 intensity */
/* BASELINE.json operators with no reference implementation (SURVEY.md §8(a)
 * M2-M6); defined by this package in the reference's plugin style. */
#define SA_OP_DROPOUT         19   /* f0 rate, f1 fill                                  */
#define SA_OP_POOL            20   /* i0 size, i1 reducer (0 mean, 1 max, 2 min)        */
#define SA_OP_CONVOLVE        21   /* aux[aux_off .. aux_off+aux_len) = taps            */
#define SA_OP_SPEED_WARP      22   /* i0 n_speed_change, i1 interp (0 linear, 1 cubic), f0 max_speed_ratio */
#define SA_OP_SINUSOID        23   /* f0 amplitude, i0 min_bin                          */
#define SA_OP_MAX             24

#define SA_MAX_STAGES         64

/* One pipeline stage: the reference's {kind, probability, params} record
 * (pipeline.py:48-57) lowered to a fixed-size descriptor. */
typedef struct sa_stage {
    int32_t op;           /* SA_OP_* */
    int32_t index;        /* stage position j = augmenter_index (core.py:242-257) */
    double  probability;  /* per-series gate: fires iff random() < probability   */
    double  f[6];
    int64_t i[6];
    int32_t aux_off;      /* offset into the aux double array (Convolve taps)    */
    int32_t aux_len;
} sa_stage;

/* ---- library --------------------------------------------------------- */
int         sa_abi_version(void);
const char* sa_last_error(void);
/* Select and initialise a CUDA device (idempotent).  */
int         sa_init(int32_t device);
/* Number of kernel launches this library issued on the calling process. */
int64_t     sa_launch_count(void);

/* ---- seeding (reference core.py:71-82 derive_stream) -------------------
 * Writes the 128-bit Philox key of stream (master_seed, stage, series). */
int sa_derive_key(uint64_t master_seed, uint64_t augmenter_index, uint64_t series_index,
                  uint64_t* key_lo, uint64_t* key_hi);

/* ---- the hot path: a whole chain, fused, device-resident ---------------
 * Replaces Pipeline.run (reference pipeline.py:129-157) and, with n_stages
 * == 1, Augmenter.augment_batch (core.py:239-259).  Runs every stage of every
 * series in one pass over HBM (per-sample order, which the reference
 * guarantees is bitwise identical to standard order, pipeline.py:1-12).
 * len_out must equal the projected length (pipeline.py:116-127); a Repeat
 * stage multiplies the row count by its r (basic.py:400-409), so d_out must
 * hold n * r rows.
 * Asynchronous on `stream`; *d_flags (caller-owned device uint32) receives
 * the OR of SA_FLAG_* bits.  */
#define SA_FLAG_NONFINITE      1u
#define SA_FLAG_WARP_MONOTONE  2u
int sa_pipeline_launch(const sa_stage* stages, int32_t n_stages,
                       const double* aux, int32_t n_aux,
                       uint64_t master_seed, int64_t series_offset,
                       const double* d_in, int64_t n, int64_t len_in,
                       double* d_out, int64_t len_out,
                       uint32_t* d_flags, void* stream);

/* Same, then synchronises `stream` and converts the flags into a status
 * (SA_ERR_NONFINITE / SA_ERR_WARP_MONOTONE). */
int sa_pipeline_run(const sa_stage* stages, int32_t n_stages,
                    const double* aux, int32_t n_aux,
                    uint64_t master_seed, int64_t series_offset,
                    const double* d_in, int64_t n, int64_t len_in,
                    double* d_out, int64_t len_out, void* stream);

/* Host-buffer entry (what a reference-side binding calls with Batch.values):
 * chunked H2D -> fused kernel -> D2H with copies overlapped across streams on
 * the current device.  h_in / h_out may be pageable or page-locked.
 * Synchronous; returns the status. */
int sa_pipeline_run_host(const sa_stage* stages, int32_t n_stages,
                         const double* aux, int32_t n_aux,
                         uint64_t master_seed, int64_t series_offset,
                         const double* h_in, int64_t n, int64_t len_in,
                         double* h_out, int64_t len_out);

/* ---- spectral transforms (reference freqtransform.py:101-116) ----------
 * Half-spectrum layout of SpectrumBatch (freqtransform.py:47-88): separate
 * re / im arrays of shape (n, len/2 + 1); im of the DC bin (and of the Nyquist
 * bin for even len) are pinned to 0.0.  Asynchronous on `stream`. */
int sa_fft_forward(const double* d_in, int64_t n, int64_t len,
                   double* d_re, double* d_im, void* stream);
int sa_fft_inverse(const double* d_re, const double* d_im, int64_t n, int64_t len,
                   double* d_out, void* stream);

/* Orthonormal DCT-II / DCT-III along each row (reference freqtransform.py:
 * 91-98: scipy.fft.dct / idct, type 2, norm="ortho"), any length.
 * Asynchronous on `stream`; d_in / d_out are (n, len) float64. */
int sa_dct_forward(const double* d_in, int64_t n, int64_t len, double* d_out, void* stream);
int sa_dct_inverse(const double* d_in, int64_t n, int64_t len, double* d_out, void* stream);

/* ---- DTW quality scoring (reference dtw.py:40-106) ----------------------
 * Row-wise DTW distance of n_pairs (a, b) series pairs, |a_i - b_j| local
 * cost, steps (1,1), (1,0), (0,1); bitwise the reference's accumulated cost.
 * Replaces the per-pair loop of mean_similarity (dtw.py:97-106). Async. */
int sa_dtw_batch(const double* d_a, const double* d_b, int64_t n_pairs, int64_t len_a, int64_t len_b,
                 double* d_dist, void* stream);
/* One pair with its optimal path, ties broken like dtw.py:64-82 (diagonal,
 * then advancing a, then advancing b).  d_acc: len_a * len_b workspace;
 * d_path: 2 * (len_a + len_b) int32 receiving (i, j) pairs from (0, 0).
 * Replaces dtw_distance (dtw.py:40-85). Async. */
int sa_dtw_path(const double* d_a, int64_t len_a, const double* d_b, int64_t len_b, double* d_acc,
                int32_t* d_path, int32_t* d_path_len, double* d_dist, void* stream);

/* ---- host-buffer transforms (freqtransform.py / dtw.py on numpy arrays) --
 * The reference API's arrays live in ordinary host memory.  These run the
 * device entry points above through the host-staging runtime (chunks of rows,
 * parallel copies into page-locked staging overlapped with H2D, kernel and
 * D2H; page-locked buffers are used in place).  Synchronous. */
int sa_fft_forward_host(const double* h_in, int64_t n, int64_t len, double* h_re, double* h_im);
int sa_fft_inverse_host(const double* h_re, const double* h_im, int64_t n, int64_t len, double* h_out);
int sa_dct_forward_host(const double* h_in, int64_t n, int64_t len, double* h_out);
int sa_dct_inverse_host(const double* h_in, int64_t n, int64_t len, double* h_out);
int sa_dtw_batch_host(const double* h_a, const double* h_b, int64_t n_pairs, int64_t len_a, int64_t len_b,
                      double* h_dist);

/* ---- text codec (dataset files, reference datafiles.py) ----------------
 * repr(float(v)) of each value into a 32-byte slot of d_out (length in
 * d_len), bit-exact with CPython's shortest round-trip repr. Async. */
int sa_repr_values(const double* d_values, int64_t n, char* d_out, int32_t* d_len, void* stream);
/* float(field) for the UTF-8 fields d_text[d_offsets[i] .. d_offsets[i+1]),
 * bit-exact with CPython's float(str) (Unicode digits and spaces, '_'
 * separators, inf/nan, correct rounding); d_ok[i] = 0 where float() would
 * raise ValueError. d_scratch: a buffer as large as the text, used only for
 * non-ASCII fields (may be NULL for ASCII text; non-ASCII fields then fail).
 * Async. */
int sa_parse_values(const char* d_text, const int64_t* d_offsets, int64_t n, double* d_out, int32_t* d_ok,
                    char* d_scratch, void* stream);

/* ---- dataset files (reference datafiles.py:70-143) --------------------
 * parse_dataset on device-resident UTF-8 text:
 *   sa_dataset_open   line split (str.splitlines), strip, format detection
 *                     ('@' on the first non-blank line), TS header/label
 *                     split (rsplit ':'), field counts and the reference's
 *                     structural errors in line order.  Synchronizes.  On
 *                     info->status == SA_DS_OK the batch is n_series x length.
 *   sa_dataset_values float() of every field into d_values (row-major
 *                     n_series x length); may report SA_DS_NOT_A_NUMBER or
 *                     SA_DS_NONFINITE.  Synchronizes.
 *   sa_dataset_labels / sa_dataset_headers  the TS labels (stripped) / header
 *                     lines, each followed by '\n', label_bytes / header_bytes
 *                     in total.  Async.
 *   sa_dataset_close  frees the handle's tables (stream ordered).
 * Errors report the first failing line (1-based, as the reference) and for
 * SA_DS_NOT_A_NUMBER the field's byte range [err_begin, err_end) in the text;
 * for SA_DS_BAD_UTF8 err_begin is the first invalid byte. */
#define SA_FORMAT_AUTO (-1)
#define SA_FORMAT_CSV 0
#define SA_FORMAT_TS 1
#define SA_DS_OK 0
#define SA_DS_EMPTY 1             /* "dataset file is empty" */
#define SA_DS_HEADER_AFTER_DATA 2 /* "line N: header after first data row" */
#define SA_DS_MISSING_LABEL 3     /* "line N: missing ':label' separator" */
#define SA_DS_NOT_A_NUMBER 4      /* "line N: not a number: '...'" */
#define SA_DS_RAGGED 5            /* "line N: F fields, but line M has W" */
#define SA_DS_NO_DATA 6           /* "dataset file has headers but no data rows" */
#define SA_DS_NONFINITE 7         /* Batch: "batch contains non-finite values" */
#define SA_DS_BAD_UTF8 8          /* the file is not UTF-8 (UnicodeDecodeError) */

typedef struct sa_dataset sa_dataset;
typedef struct sa_dataset_info {
    int32_t format; /* SA_FORMAT_CSV / SA_FORMAT_TS, detected or forced */
    int32_t status; /* SA_DS_* */
    int64_t n_lines;
    int64_t n_series;
    int64_t length;
    int64_t header_bytes;
    int64_t label_bytes;
    int64_t err_line;
    int64_t err_ref_line;
    int64_t err_fields;
    int64_t err_ref_fields;
    int64_t err_begin;
    int64_t err_end;
} sa_dataset_info;

int sa_dataset_open(const char* d_text, int64_t n_bytes, int32_t format, int32_t validate_utf8, sa_dataset** out,
                    sa_dataset_info* info, void* stream);
int sa_dataset_values(sa_dataset* ds, double* d_values, sa_dataset_info* info);
int sa_dataset_labels(sa_dataset* ds, char* d_out);
int sa_dataset_headers(sa_dataset* ds, char* d_out);
int sa_dataset_close(sa_dataset* ds);

/* format_dataset rows (datafiles.py:127-138): row r of the n x len batch is
 * ",".join(repr(v)) [+ ":" + label r] + "\n".  Labels (TS only, may be NULL
 * for empty labels) are bytes d_labels[d_label_off[r] .. d_label_off[r+1]).
 * sa_dataset_format_size writes each row's absolute offset (base = bytes
 * before the first row, e.g. the header lines) into d_row_off[n] and the
 * file size into *total (synchronizes); sa_dataset_format_write writes the
 * rows into d_out (async). */
int sa_dataset_format_size(const double* d_values, int64_t n, int64_t len, int32_t format,
                           const int64_t* d_label_off, int64_t base, int64_t* d_row_off, int64_t* total,
                           void* stream);
int sa_dataset_format_write(const double* d_values, int64_t n, int64_t len, int32_t format, const char* d_labels,
                            const int64_t* d_label_off, const int64_t* d_row_off, char* d_out, void* stream);

/* SpectralAugmenter.augment_spectrum (reference freqaugment.py:49-76): one
 * spectral stage applied directly to a half spectrum. Synchronous. */
int sa_augment_spectrum(const sa_stage* stage, uint64_t master_seed, int64_t series_offset,
                        const double* d_re, const double* d_im, int64_t n, int64_t len,
                        double* d_re_out, double* d_im_out, void* stream);

/* ---- page-locked host memory helpers (for zero-staging host batches) ---- */
/* memcpy between host buffers on the host-staging runtime's copy threads
 * (what the *_host entry points use to fill their page-locked staging). */
int sa_host_copy(void* dst, const void* src, int64_t bytes);
int sa_host_alloc(void** ptr, int64_t bytes);
int sa_host_free(void* ptr);
/* Batch validation on the host cores: *all_finite = 1 iff none of the n
 * doubles at p is NaN or +-Inf.  Replaces the reference Batch's
 * np.isfinite(values).all() (core.py:103-104) for large host batches; the
 * result is the same predicate, evaluated on the exponent bits. */
int sa_host_all_finite(const double* p, int64_t n, int32_t* all_finite);

#ifdef __cplusplus
}
#endif
#endif /* SERIESAUG_B200_H */
