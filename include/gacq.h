/*
 * gacq.h -- C ABI of the B200-native GPS L1 C/A acquisition engine (libgacq.so).
 *
 * Drop-in boundary for the reference's acquisition hot path
 * (gnssperf, /root/reference/pkg/src/gnssperf):
 *
 *   gacq_create        replaces the per-(prn, fs, n, precision) conjugate code-spectrum
 *                      cache (acquisition.py:84-105) and the per-bin carrier replicas
 *                      (acquisition.py:139 -> gnss_signal.py:49-72 -> kernels.py:106-114,
 *                      175-185): all tables are built once per plan and kept in HBM.
 *   gacq_run           replaces acquire_all / acquire_channel (acquisition.py:112-208)
 *                      over a batch of snapshots: the hot loop acquisition.py:138-149
 *                      (wipe-off, FFT, x conj(code FFT), IFFT, |.|^2 noncoherent sum)
 *                      and the argmax / exclusion-floor reduction acquisition.py:151-159.
 *                      The host finishes acquisition.py:160-170 (metric = peak/floor in
 *                      double, detection, AcqResult) exactly as the reference does.
 *   gacq_ca_code       replaces generate_ca_code (cacode.py:41-58).
 *
 * Plain C types only: pointers, sizes, POD structs. All functions return 0 on success
 * or a negative GACQ_ERR_* code; gacq_last_error() returns the calling thread's message.
 * A context is bound to one CUDA device; calls on one context are serialized internally,
 * distinct contexts (one per device) may be driven concurrently from different threads.
 */
#ifndef GACQ_H
#define GACQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GACQ_ABI_VERSION 2

#define GACQ_OK 0
#define GACQ_ERR_INVALID (-1)     /* -> InvalidInputError (errors.py:8-9)            */
#define GACQ_ERR_UNSUPPORTED (-2) /* configuration outside the GPU path's support     */
#define GACQ_ERR_CUDA (-3)        /* device / driver failure -> ResourceError          */
#define GACQ_ERR_RESOURCE (-4)    /* allocation failure     -> ResourceError (24-25)   */

/* gacq_params.plan_flags */
#define GACQ_PLAN_GENERIC 1u    /* take the generic power-of-two path even at a chip-aligned
                                   rate (parity tests of that path)                   */

/* gacq_run flags */
#define GACQ_SNAPS_ON_DEVICE 1u /* `snaps` is a device pointer (HBM-resident batch)   */
#define GACQ_ROWS_ON_DEVICE 2u  /* `rows` is a device pointer (no D2H)                */
#define GACQ_ROWS_PER_BIN 4u    /* write [n_snap][n_prn][n_bins] rows, no bin merge   */
#define GACQ_PROFILE 8u         /* time each kernel with CUDA events (gacq_stats)     */

typedef struct gacq_ctx gacq_ctx;

typedef struct gacq_params {
    double sample_rate_hz;            /* IqBuffer.sample_rate_hz (buffers.py:46-66)       */
    int32_t coherent_ms;              /* AcqConfig.coherent_ms      (acquisition.py:49)   */
    int32_t noncoherent_rounds;       /* AcqConfig.noncoherent_rounds (acquisition.py:50) */
    int32_t n_bins;                   /* len(AcqConfig.doppler_bins_hz())                 */
    const double* doppler_bins_hz;    /* the float64 grid itself (acquisition.py:68-70)  */
    int32_t exclusion_radius_samples; /* resolved radius (acquisition.py:155), > 0        */
    int32_t n_prn;                    /* channels searched per snapshot, 1..32            */
    const int32_t* prns;              /* PRN numbers 1..32, distinct                      */
    int32_t device;                   /* CUDA ordinal                                     */
    int32_t plan_flags;               /* GACQ_PLAN_* (0 = default)                        */
    int64_t scratch_bytes;            /* spectrum scratch budget, 0 = default: min(8 GiB,  */
                                      /* free device memory / 4); allocated on demand      */
} gacq_params;

/* One reduced search row: the winning (bin, lag) of a (snapshot, prn) -- or of a
 * (snapshot, prn, bin) with GACQ_ROWS_PER_BIN -- with its float32 power and the float32
 * exclusion floor of that row (acquisition.py:151-159). 16 bytes. */
typedef struct gacq_row {
    int32_t bin;
    int32_t lag;
    float peak;
    float floor;
} gacq_row;

typedef struct gacq_info {
    int32_t samples_per_period; /* P  = round(fs*1023/1.023e6) (acquisition.py:108-109) */
    int32_t n_coh;              /* samples per coherent block  (acquisition.py:116)     */
    int32_t chip_oversample;    /* D  = P / 1023 samples per chip                       */
    int32_t fft_len;            /* transform length on the device: 1023 (path 2) or M (path 4) */
    int32_t n_bins;
    int32_t n_prn;
    int32_t rounds;
    int32_t path;               /* 2 = 1023-point prime-factor path (chip-aligned rates),
                                   4 = generic power-of-two path (any other rate)         */
    int32_t corr_ctas;          /* persistent K2 grid (resident CTAs on the device)      */
} gacq_info;

typedef struct gacq_stats {
    int64_t calls;
    int64_t launches;           /* kernels launched by gacq_run since the last reset    */
    int64_t cells;              /* (snapshot, prn, bin) cells searched                 */
    int64_t h2d_bytes;
    int64_t d2h_bytes;
    double fwd_ms;              /* summed kernel times (GACQ_PROFILE runs only)         */
    double corr_ms;
    double reduce_ms;
    int64_t fwd_launches;
    int64_t corr_launches;
    int64_t reduce_launches;
    double run_ms;              /* device timeline of whole gacq_run calls, first H2D (or
                                   first kernel) to last D2H (GACQ_PROFILE runs only)     */
} gacq_stats;

int gacq_version(void);
const char* gacq_last_error(void);

/* Build a search plan on `device`: validates the configuration, builds the carrier
 * table [n_bins][n_coh] (bit-identical to the reference NCO), the conjugate code spectra
 * and twiddles, and allocates device scratch. */
int gacq_create(gacq_ctx** out, const gacq_params* params);
int gacq_info_get(const gacq_ctx* ctx, gacq_info* out);
void gacq_destroy(gacq_ctx* ctx);

/* Order the context's next device work after everything queued so far on `stream` (a
 * cudaStream_t of the same device; (void*)1 = the legacy default stream, (void*)2 = the
 * per-thread default stream): the __cuda_array_interface__ v3 "stream" contract for device
 * inputs written by another library. */
int gacq_wait_stream(gacq_ctx* ctx, void* stream);

/* Search n_snap snapshots. Snapshot i starts at complex sample i*stride_samples of
 * `snaps` (interleaved float32 I/Q, complex64) and must hold >= rounds*n_coh samples;
 * only the first rounds*n_coh are read (acquisition.py:134-137). `rows` receives
 * n_snap*n_prn records (or n_snap*n_prn*n_bins with GACQ_ROWS_PER_BIN), ordered like the
 * plan's PRN list. Blocks until results are in `rows`. A snapshot holding a NaN or an
 * infinity fails the call with GACQ_ERR_INVALID (the reference's IqBuffer refuses them,
 * buffers.py:62-63); the rows of the other snapshots are still written. */
int gacq_run(gacq_ctx* ctx, const void* snaps, int64_t n_snap, int64_t stride_samples,
             uint32_t flags, gacq_row* rows);

/* Sample formats of gacq_run_quantized: interleaved I/Q integers as in the reference's IF
 * file payload (iffile.py:3-16, 38-43). */
#define GACQ_FMT_INT8 0
#define GACQ_FMT_INT16 1

/* Same search over integer I/Q (the IF-file payload, read_if_file, iffile.py:74-99): each
 * component becomes float32(float64(q) * (scale / limit)), limit = 127 (int8) or 32767
 * (int16) -- bit-identical to read_if_file -- on the device, so only 2 or 4 bytes per sample
 * cross PCIe. `iq` holds n_snap snapshots of 2*stride_samples integers each (host, or device
 * with GACQ_SNAPS_ON_DEVICE). */
int gacq_run_quantized(gacq_ctx* ctx, const void* iq, int32_t sample_format, double scale, int64_t n_snap,
                       int64_t stride_samples, uint32_t flags, gacq_row* rows);

/* Debug/parity hook: the float32 noncoherent power map [n_prn][n_bins][P] of ONE host
 * snapshot (the reference's power_map, acquisition.py:131-149). */
int gacq_power_map(gacq_ctx* ctx, const void* snap_host, float* out_host);

/* Parity hook: the plan's carrier table [n_bins][n_coh] complex64, built on the device
 * and bit-identical to carrier_replica(NcoState(), f, fs, n_coh)
 * (gnss_signal.py:49-72 -> kernels.py:106-114) for every bin f. */
int gacq_carrier_table(gacq_ctx* ctx, void* out_host);

/* ---- On-device synthetic snapshots ------------------------
 * Replaces the benchmark-input side of synthesize_signal / add_awgn (gnss_signal.py:136-186)
 * for large batches: out[s][k] (complex64, device memory, n_snap x n_samples) = the sum, in
 * order, of sats[s][j].amplitude * code * carrier for the n_sat satellites of snapshot s --
 * the same fixed-point NCO words and complex64 rounding as the reference, so with
 * noise_sigma = 0 it is bit-identical to summing synthesize_signal(...) * float32(amp) -- plus
 * complex AWGN of std noise_sigma per component from a counter-based Philox stream (the
 * reference's PCG64 stream is not reproduced: performance inputs only, never parity). */
typedef struct gacq_sat {
    int32_t prn;                 /* 1..32 (SignalSpec.prn)                     */
    int32_t reserved;
    double doppler_hz;           /* SignalSpec.doppler_hz                      */
    double code_phase_samples;   /* SignalSpec.code_phase_samples, [0, P)      */
    double carrier_phase_cycles; /* SignalSpec.carrier_phase_cycles            */
    float amplitude;             /* float32 scale applied to the clean signal  */
    float reserved2;
} gacq_sat;

int gacq_synth(int32_t device, double sample_rate_hz, int64_t n_snap, int64_t n_samples, int32_t n_sat,
               const gacq_sat* sats_host, double noise_sigma, uint64_t seed, void* out_device);

int gacq_stats_get(const gacq_ctx* ctx, gacq_stats* out);
int gacq_stats_reset(gacq_ctx* ctx);

/* ---- Tracking correlators ------------------------------------
 * Replaces epl_correlate (tracking.py:126-165) for a batch of channels: carrier wipe-off
 * with the 48-bit NCO (kernels.py:106-114, fp64 cos/sin rounded to complex64, bit-exact
 * complex64 product) and the three E/P/L dot products against floor-indexed code replicas
 * of the 42-bit code NCO (kernels.py:116-128). The fixed-point starts and steps are given
 * per channel exactly as the reference computes them (kernels.py:56-70), so the replicas
 * are bit-identical; the dot products are complex64 running sums taken left to right,
 * exactly as the reference accumulates them (kernels.py:93-95): the sums are bit-identical. */
typedef struct gacq_epl_chan {
    int64_t block_offset;  /* complex samples from `blocks` to this channel's first sample */
    uint64_t carrier_p0;   /* carrier_phase_to_fixed(state.carrier_phase_cycles)           */
    uint64_t carrier_step; /* carrier_step_to_fixed(state.doppler_hz, fs)                  */
    uint64_t code_p0[3];   /* code_phase_to_fixed((phase + {+d/2, 0, -d/2}) % 1023)        */
    uint64_t code_step;    /* code_step_to_fixed(state.code_rate_hz, fs)                   */
    int32_t prn;           /* 1..32                                                         */
    int32_t reserved;
} gacq_epl_chan;

typedef struct gacq_trk gacq_trk;
int gacq_trk_create(gacq_trk** out, int32_t device);
void gacq_trk_destroy(gacq_trk* trk);
/* gacq_wait_stream for the tracker's device work. */
int gacq_trk_wait_stream(gacq_trk* trk, void* stream);
/* out[c*6 + 0..5] = (ie, qe, ip, qp, il, ql) of channel c over n_samples samples.
 * `blocks` holds total_samples complex64 samples (host, or device with
 * GACQ_SNAPS_ON_DEVICE); every channel's block must lie inside it. */
int gacq_trk_epl(gacq_trk* trk, const void* blocks, int64_t total_samples, int32_t n_samples,
                 const gacq_epl_chan* chans, int64_t n_chan, uint32_t flags, float* out);

/* Host-side loop closure of a struct-of-arrays channel batch (tracking.py:168-275 for every
 * channel, float64, the reference's operation order, bit-identical; no GPU needed). `sums`
 * holds the gacq_trk_epl outputs [n][6]; the batch arrays are updated in place to the next
 * epoch's state; out[c*3 + 0..2] = (dll_error_chips, pll_error_cycles, lock_metric).
 * A channel whose six correlators are all zero fails with GACQ_ERR_INVALID and its index in
 * *bad_channel (DegenerateInputError, tracking.py:173-175, 181-182). */
typedef struct gacq_trk_batch {
    int64_t n;
    const int32_t* prn;
    double* code_phase_chips;
    double* carrier_phase_cycles;
    double* doppler_hz;
    double* code_rate_hz;
    double* dll_acc;
    double* dll_prev;
    double* pll_acc;
    double* pll_prev;
    double* lock_nbd;
    double* lock_nbp;
    int64_t* epoch;
    const double* sample_rate_hz;
} gacq_trk_batch;

typedef struct gacq_trk_config {
    double integration_ms;
    double pll_bandwidth_hz;
    double dll_bandwidth_hz;
    double correlator_spacing_chips;
} gacq_trk_config;

int gacq_trk_close(const float* sums, const gacq_trk_batch* batch, const gacq_trk_config* cfg, double* out,
                   int64_t* bad_channel);

/* The gacq_epl_chan records of a batch (kernels.py:56-70 NCO words; offsets[c] = first sample
 * of channel c), for the next gacq_trk_epl. */
int gacq_trk_chans(const gacq_trk_batch* batch, const gacq_trk_config* cfg, const int64_t* offsets,
                   gacq_epl_chan* chans);

/* One tracking epoch of a whole batch in one call: gacq_trk_chans + gacq_trk_epl + gacq_trk_close
 * (tracking.py:126-275 for every channel), pipelined over channel slices so that one slice's
 * correlator kernel runs while the host computes the next slices' NCO words and closes the
 * previous ones. The block length is round(sample_rate_hz[i] * integration_ms / 1000), which
 * must be the same for every channel (GACQ_ERR_INVALID otherwise). Results
 * are those of the three calls: sums[c*6 + 0..5] the correlators, out[c*3 + 0..2] as
 * gacq_trk_close, the batch advanced in place. On a degenerate channel (*bad_channel = its
 * index, GACQ_ERR_INVALID) the batch may already be partly advanced: pass a copy (the Python
 * track_step does). Replaces the per-epoch loop of tracking.py:226-275 over channels. */
int gacq_trk_step(gacq_trk* trk, const void* blocks, int64_t total_samples, const int64_t* offsets,
                  gacq_trk_batch* batch, const gacq_trk_config* cfg, uint32_t flags, float* sums, double* out,
                  int64_t* bad_channel);

/* Measured FP32 peak of `device` in TFLOP/s (packed FFMA2 chains, the codelets' instruction
 * form): the denominator bench.py reports beside the nominal 148 x 128 x 2 x clock. */
int gacq_fp32_probe(int32_t device, double* tflops);

/* Page-locked host buffers for overlapped H2D (cudaHostAlloc / cudaFreeHost). */
int gacq_host_alloc(int64_t bytes, void** out);
int gacq_host_free(void* ptr);

/* C/A chips (+1/-1) of PRN 1..32 into out[1023] (cacode.py:41-58). */
int gacq_ca_code(int32_t prn, int8_t* out);

#ifdef __cplusplus
}
#endif

#endif /* GACQ_H */
