/*
 * wavepipe_b200.h - C ABI of the B200 (sm_100a) filtering engine.
 *
 * The shared library libwpb200.so replaces the reference's kernel seam, the
 * `_kernels()` module swap in pkg/src/wavepipe/engine.py:74-75, and the chain
 * loop behind the pipe operator (chain.py:66-71). Plain pointers and sizes
 * only; no torch types. All sample buffers are DEVICE memory, planar
 * [channels][ld] float32, row stride `ld` >= frames (in elements).
 *
 * Error convention: every entry point returns WP_OK (0) or a negative
 * WP_E* code and records a message retrievable with wp_last_error()
 * (thread-local). Kernels never fail silently; validation of filter
 * semantics (bound, rate match, stability) stays in the host layer as in the
 * reference (engine.py:126-130, design.py:74-78).
 *
 * Threading / streams: execute calls are asynchronous on the given stream,
 * never allocate and never synchronize. Plan creation allocates device memory
 * for coefficient tables and synchronously uploads them (cuFFT-style plan).
 */
#ifndef WAVEPIPE_B200_H
#define WAVEPIPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *wp_stream_t; /* == cudaStream_t; NULL = legacy default stream */

enum {
    WP_OK = 0,
    WP_EINVAL = -1,    /* bad argument (shape, count, pointer, alignment) */
    WP_ECUDA = -2,     /* CUDA runtime error (launch, memcpy, ...) */
    WP_ENOMEM = -3,    /* workspace too small / allocation failed */
    WP_EARCH = -4,     /* device is not sm_100 (binary carries sm_100a only) */
    WP_EUNSUP = -5,    /* configuration not supported by this build */
};

/* Stage kinds of a chain, applied left to right like Chain.apply
 * (chain.py:66-71). */
enum {
    WP_STAGE_IIR = 1,       /* coef = n sections x {b0,b1,b2,a1,a2}, cascade gain already folded
                               into section 0 (engine.py:133-139) */
    WP_STAGE_FIR = 2,       /* coef = n taps, causal same-length convolution (engine.py:159-178) */
    WP_STAGE_GAIN = 3,      /* y = value * x (fp32 multiply) */
    WP_STAGE_NORMALIZE = 4, /* y = x * (value / max|x|) over the whole buffer; value = target peak */
};

/* Per-stage flags. */
enum {
    WP_FIR_AUTO = 0,        /* direct for short taps, FFT overlap-save for long (measured crossover) */
    WP_FIR_DIRECT = 1,      /* force direct convolution   (strategy="direct", engine.py:170-175) */
    WP_FIR_FFT = 2,         /* force FFT convolution      (strategy="fft",    engine.py:176-177) */
    WP_IIR_PREC_AUTO = 0,   /* fp64 state for a block if any section has pole radius > 0.98 */
    WP_IIR_PREC_F32 = 16,   /* force fp32 recurrence/scan */
    WP_IIR_PREC_F64 = 32,   /* force fp64 recurrence/scan */
};

typedef struct wp_stage {
    int32_t kind;        /* WP_STAGE_* */
    int32_t n;           /* sections (IIR) or taps (FIR); 0 otherwise */
    const double *coef;  /* HOST pointer, read during wp_plan_create only */
    double value;        /* gain factor (GAIN) or target peak (NORMALIZE) */
    int32_t flags;       /* WP_FIR_* / WP_IIR_PREC_* */
    int32_t reserved;
} wp_stage;

typedef struct wp_plan wp_plan; /* opaque */

/* Build a plan for a whole chain: stages are grouped into fused passes
 * (pre-gain -> IIR cascade -> FIR -> post-gains per pass, one HBM round trip
 * each); scan tables are computed in float64 on the host and uploaded to the
 * current device. Replaces the per-stage loop of Chain.apply (chain.py:66-71). */
int wp_plan_create(const wp_stage *stages, int32_t n_stages, wp_plan **out_plan);
int wp_plan_destroy(wp_plan *plan);

/* Device workspace (bytes) an execute call needs for a [channels x frames]
 * signal: look-back records of the scan, ping-pong buffer between passes. */
int wp_plan_workspace_bytes(const wp_plan *plan, int64_t channels, int64_t frames, size_t *bytes);

/* Run the chain: y = chain(x). x and y must not overlap. */
int wp_plan_execute(const wp_plan *plan, const float *x, float *y, int64_t channels, int64_t frames,
                    int64_t ld_x, int64_t ld_y, void *workspace, size_t workspace_bytes,
                    wp_stream_t stream);

/* Host buffers in, host buffers out (the e2e path; Wave.numpy32 over a pinned
 * source): channel blocks (single channels, or pairs when a pass runs the FFT
 * path; `blocks` <= 0 = 16, or 32 from 4 GiB; at most 32) are uploaded, executed and downloaded on
 * three internal streams so both PCIe directions and the kernels overlap.
 * dx, dy: distinct device buffers of [channels x frames] floats (row stride =
 * frames); workspace: wp_plan_workspace_bytes of the largest block (the whole
 * call's size always suffices). Asynchronous: `stream` waits for the last
 * download, so synchronise it before reading hy. Pinned host buffers give the
 * overlap; pageable ones still work. Every block runs the kernels the whole
 * call's shape selects, so hy is bit-identical to one wp_plan_execute over all
 * channels. Not for chains with Normalize (the peak
 * spans all blocks): WP_EUNSUP. Replaces the reference's host-side
 * Chain.apply loop (chain.py:66-71) over numpy buffers for an FFI caller. */
int wp_plan_execute_host(const wp_plan *plan, const float *hx, float *hy, int64_t channels, int64_t frames,
                         int64_t ld_hx, int64_t ld_hy, float *dx, float *dy, void *workspace,
                         size_t workspace_bytes, int32_t blocks, wp_stream_t stream);

/* Number of fused passes and of kernel launches per execute call. */
int wp_plan_num_passes(const wp_plan *plan);
int wp_plan_launches(const wp_plan *plan);
/* Human-readable description of pass i (kernel kind, sections, taps, precision). */
const char *wp_plan_describe(const wp_plan *plan, int32_t pass);
/* The same for one call shape: IIR-only passes run the fused scan kernel for
 * small calls and the single-pass tensor-core chain (chain_lb) for large ones. */
int wp_plan_launches_for(const wp_plan *plan, int64_t channels, int64_t frames);
const char *wp_plan_describe_for(const wp_plan *plan, int32_t pass, int64_t channels, int64_t frames);

/* ---- seam-level one-shot entry points (mirror _kernels_jit functions) ----
 * Each looks up (or builds) a plan for its single stage in a small
 * process-wide cache (64 entries, LRU; shared ownership, so a plan evicted
 * while another thread executes it stays alive until that call returns) and
 * executes it. The *_workspace queries return the workspace bytes one call of
 * that shape needs (it grows with channels x frames for IIR passes: published
 * tile states, ~1 B per 128 samples per state). */

/* iir_cascade_{serial,parallel}(sos, x) (_kernels_jit.py:35-48) */
int wp_iir_cascade(const double *sos, int32_t n_sections, const float *x, float *y, int64_t channels,
                   int64_t frames, int64_t ld_x, int64_t ld_y, int32_t flags, void *workspace,
                   size_t workspace_bytes, wp_stream_t stream);
int wp_iir_cascade_workspace(const double *sos, int32_t n_sections, int64_t channels, int64_t frames, int32_t flags,
                             size_t *bytes);
/* fir_direct_{serial,parallel}(taps, x) (_kernels_jit.py:65-78) and
 * engine._fir_fft (engine.py:206-223) selected by flags */
int wp_fir(const double *taps, int32_t n_taps, const float *x, float *y, int64_t channels, int64_t frames,
           int64_t ld_x, int64_t ld_y, int32_t flags, void *workspace, size_t workspace_bytes,
           wp_stream_t stream);
int wp_fir_workspace(const double *taps, int32_t n_taps, int64_t channels, int64_t frames, int32_t flags,
                     size_t *bytes);

/* ---- signal sources and reductions ---- */

/* white_noise(duration, channels, fs, seed) (wave.py:141-168): splitmix64 +
 * Box-Muller in float64 on the device, channel-major, rounded to float32. */
int wp_white_noise(float *y, int64_t channels, int64_t frames, int64_t ld_y, uint64_t seed,
                   wp_stream_t stream);
/* out[0] = max |x| (float32) */
int wp_peak_abs(const float *x, int64_t channels, int64_t frames, int64_t ld_x, float *out_device,
                wp_stream_t stream);

/* ---- WAV payload codec (wavio.py:49-200), device side ----
 * The RIFF header is parsed/written by the host; these convert the data
 * chunk. payload: DEVICE pointer to the little-endian interleaved frames
 * (channels x frames samples); y / x: planar float32 [channels][ld].
 * Decode is exact (pcm16 / 2^15, pcm24 / 2^23, float32 bit copy); encode
 * clamps to [-1, 1] and quantizes round-half-away-from-zero like
 * wavio.save_wav, counting |x| > 1 samples into *clipped_device (uint64,
 * zeroed by the call; may be NULL for float32). */
enum { WP_ENC_PCM16 = 16, WP_ENC_PCM24 = 24, WP_ENC_F32 = 32 };
int wp_wav_decode(const void *payload, int32_t encoding, float *y, int64_t channels, int64_t frames, int64_t ld_y,
                  wp_stream_t stream);
int wp_wav_encode(const float *x, int64_t channels, int64_t frames, int64_t ld_x, int32_t encoding, void *payload,
                  uint64_t *clipped_device, wp_stream_t stream);

/* ---- diagnostics ---- */
const char *wp_last_error(void);
int wp_abi_version(void);
/* 0 if the current device can run this binary (sm_100), WP_EARCH otherwise */
int wp_check_device(void);
/* Diagnostics: when set, tensor-core chain launches record per-tile stage
 * timestamps (%globaltimer, ns) into this device buffer ([tiles][12]) if it
 * holds enough entries; NULL disables. Not for production use. */
int wp_set_trace(uint64_t *device_buffer, size_t entries);
/* Total kernel launches issued by this process through the library. */
uint64_t wp_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* WAVEPIPE_B200_H */
