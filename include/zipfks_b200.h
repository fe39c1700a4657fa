/*
 * zipfks_b200 — C ABI of the B200 (sm_100a) Monte Carlo engine for KS cutoff tables of the
 * discrete power law (Zipf).  Plain pointers and sizes only; no torch types.
 *
 * The reference (zipfks 1.0.0, /root/reference/pkg) is a Python package with no FFI of its
 * own.  These entry points replace the bodies of its Python functions at the batch seam
 * (SURVEY.md §8b); the Python shim paper_1305_6738_b200 binds them with ctypes.  Each
 * declaration cites the reference interface it replaces.
 *
 * Conventions
 *   - Return 0 on success.  ZKS_EINVAL: argument validation (the shim raises ValueError);
 *     ZKS_ECUDA: CUDA failure (RuntimeError).  zks_last_error() gives the thread's message.
 *   - "_dev" pointers are device memory owned by the caller; "_host" pointers host memory.
 *   - Work is enqueued on the engine's stream (zks_engine_set_stream); calls that return host
 *     results synchronise that stream.
 */
#ifndef ZIPFKS_B200_H
#define ZIPFKS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZKS_OK 0
#define ZKS_EINVAL 1
#define ZKS_ECUDA 2

#define ZKS_STATUS_OK 0         /* first stream succeeded                                */
#define ZKS_STATUS_RETRIED 1    /* NoRootError on the first stream, retry at idx + 2^32 ok */
#define ZKS_STATUS_FAILED 2     /* both streams failed (SimulationError in the shim)      */

#define ZKS_RNG_NUMPY 0      /* replicate streams bit-exact with numpy's Philox4x64-10 (default) */
#define ZKS_RNG_PHILOX4X32 1 /* opt-in fast streams: Philox4x32-10, tier-3 (Monte Carlo) parity only */

#define ZKS_MLE_TABLE 0   /* model moments from the device fit tables (default)           */
#define ZKS_MLE_DIRECT 1  /* model moments by direct summation, as the reference forms them */

typedef struct zks_engine zks_engine;
typedef struct zks_table zks_table;

/* One (cell, repetition) slice of replicate indices [first, first + count).
 * Mirrors SimulationConfig (montecarlo.py:50-72) plus the repetition / index range that
 * run_repetition (montecarlo.py:174-191) and _pool_span (montecarlo.py:151-159) iterate. */
typedef struct {
  int32_t support_k;   /* Support.k; 0 = unbounded (draws from 1..65535, distribution.py:26) */
  int32_t reserved;
  double gamma;        /* generating exponent                                             */
  int64_t n;           /* sample size per replicate                                       */
  uint64_t base_seed;  /* stream key (base_seed, repetition, index), distribution.py:182-184 */
  uint64_t repetition;
  uint64_t first;      /* first replicate index                                            */
  uint64_t count;      /* number of replicates                                             */
} zks_cell;

/* ABI version (bumped on any signature change). */
int zks_version(void);

/* Thread-local message for the last non-zero return. */
const char* zks_last_error(void);

/* Create an engine on `device`.  `logs_host[k] = ln k` for k = 0..logs_len-1 (entry 0 = 0),
 * built by the shim with numpy exactly as series.natural_logs (series.py:31-44);
 * logs_len must be >= 65537. */
int zks_engine_create(int device, const double* logs_host, int64_t logs_len, zks_engine** out);
void zks_engine_destroy(zks_engine* engine);

/* Enqueue subsequent work on `stream` (a cudaStream_t; NULL = the legacy default stream).
 * A new engine starts on its own non-blocking stream. */
int zks_engine_set_stream(zks_engine* engine, void* stream);
int zks_engine_sync(zks_engine* engine);

/* Number of CUDA kernels this engine has enqueued since it was created (every launch of every
 * entry point).  Diagnostics: bench.py reports the timed-region delta as gpu_launches. */
int zks_engine_launches(zks_engine* engine, unsigned long long* out);

/* Per-kernel device time: with timing on, every launch is bracketed by CUDA events on the
 * engine stream; zks_engine_kernel_times synchronises the stream, writes the summed milliseconds
 * and launch counts per kind (arrays of ZKS_KERNEL_KINDS) since the last call, and resets. */
enum {
  ZKS_KERNEL_ROW = 0,    /* row_draw_kernel: a row's streams drawn + sorted once, counted per cell */
  ZKS_KERNEL_DRAW = 1,   /* draw_stats_kernel: samples -> head counts, tail values, log-sums */
  ZKS_KERNEL_FIT = 2,    /* fit_ks_kernel: exponent fits + KS of pre-drawn rows */
  ZKS_KERNEL_RETRY = 3,  /* retry_kernel: second attempts */
  ZKS_KERNEL_BATCH = 4,  /* lane_row_kernel: n < 128, one replicate per lane, all cells of a row */
  ZKS_KERNEL_SINGLE = 5, /* replicate_kernel: n > 1024 or direct-sum MLE, one warp per replicate */
  ZKS_KERNEL_SELECT = 6, /* radix selection of order statistics */
  ZKS_KERNEL_OTHER = 7,  /* tables, user-sample fits, series, draws */
  ZKS_KERNEL_KINDS = 8
};
int zks_engine_set_timing(zks_engine* engine, int on);
int zks_engine_kernel_times(zks_engine* engine, double* ms_out, unsigned long long* launches_out);

/* Upload a host-built sampling CDF (ZipfModel._sampling_cdf, distribution.py:99-105):
 * cdf_host[k-1] = P(X <= k) for k = 1..len, len = K or 65535, and build its guide table.
 * Replaces the per-process lru_cache'd table build of _generating_model (montecarlo.py:82-86). */
int zks_table_create(zks_engine* engine, const double* cdf_host, int64_t len, zks_table** out);
void zks_table_destroy(zks_table* table);

/* Replicates [first, first+count) of one cell and repetition: per replicate the KS statistic
 * against the refitted model, the refitted exponent and a status byte.  Replaces
 * run_replicate (montecarlo.py:98-116) looped by run_repetition / _pool_span
 * (montecarlo.py:151-191).  Outputs are indexed by (index - first).  For status
 * ZKS_STATUS_FAILED, ks is NaN and gamma_hat holds the mean log of the retry sample
 * (the "mean log of data" in the NoRootError message, estimate.py:102-105).  Asynchronous. */
int zks_run_replicates(zks_engine* engine, const zks_table* table, const zks_cell* cell, double* ks_dev,
                       double* gamma_hat_dev, uint8_t* status_dev);

/* Sweep rows: the cells of build_table share base_seed (montecarlo.py:276-277), so cells with
 * the same n and repetition consume identical uniform streams.  One call runs replicates
 * [first, first+count) of ncells (<= 32) such cells -- cells[j] must differ only in gamma, with
 * tables[j] its sampling table and ks_dev[j] / gamma_hat_dev[j] / status_dev[j] its outputs as
 * in zks_run_replicates.  In table-MLE mode for n <= 16384 each replicate's stream is drawn
 * ONCE for all the cells (n >= 128: its 53-bit keys bucketed on chip, every cell's counts from
 * where its cdf cuts fall among them; n < 128: the words' top 32 bits kept per lane and
 * classified against each cell's cuts); other sizes run cell by cell.  Results equal
 * zks_run_replicates per cell bit for bit (single cells of these sizes take the same kernels).  Replaces build_table's per-cell
 * run_simulation loop (montecarlo.py:263-314, 194-212) for one row.  Asynchronous. */
int zks_run_cells(zks_engine* engine, int32_t ncells, const zks_table* const* tables, const zks_cell* cells,
                  double* const* ks_dev, double* const* gamma_hat_dev, uint8_t* const* status_dev);

/* Order statistics at zero-based `ranks_host[i]` of `count` non-negative doubles, written to
 * out_host[i].  Replaces the np.sort + index of order_quantiles (montecarlo.py:119-136); the
 * Decimal rank rule stays in the shim.  nranks <= 16.  Synchronous. */
int zks_select_ranks(zks_engine* engine, const double* values_dev, int64_t count, const int64_t* ranks_host,
                     int32_t nranks, double* out_host);

/* Batched selection, asynchronous: for each a < narrays (<= 24), the order statistics of the
 * counts[a] values at device values_dev[a] at ranks ranks_host[a * nranks + i] land in device
 * out_dev[a][i], i < nranks (<= 16).  Optionally (status_dev non-NULL, entry non-NULL) the
 * maximum of the counts[a] status bytes at status_dev[a] lands in *worst_dev[a].  One launch
 * for all arrays (the cells of a sweep row). */
int zks_select_ranks_batch(zks_engine* engine, const double* const* values_dev, const int64_t* counts,
                           int32_t narrays, const int64_t* ranks_host, int32_t nranks, double* const* out_dev,
                           const uint8_t* const* status_dev, uint8_t* const* worst_dev);

/* The batched selection in steps, for arrays sharded over GPUs: each GPU passes its shards
 * values_dev[a] (counts[a] keys) of the full arrays (global_counts[a] keys; ranks refer to
 * those).  zks_select_dist_begin resets the state; then for pass = 0..7:
 * zks_select_dist_count ADDS this GPU's digit counts to hist_dev (uint32, [narrays * nranks][256],
 * zeroed by the caller), the caller sums hist_dev over the GPUs (e.g. an NCCL all-reduce), and
 * zks_select_dist_pick chooses the digits from the sum; zks_select_dist_end writes out_dev[a][i]
 * (identical on every GPU) and this GPU's worst status.  Key work is proportional to the shard.
 * Asynchronous; one selection at a time per engine. */
int zks_select_dist_begin(zks_engine* engine, const double* const* values_dev, const int64_t* counts,
                          const int64_t* global_counts, int32_t narrays, const int64_t* ranks_host, int32_t nranks,
                          double* const* out_dev, const uint8_t* const* status_dev, uint8_t* const* worst_dev);
int zks_select_dist_count(zks_engine* engine, int32_t pass, uint32_t* hist_dev);
int zks_select_dist_pick(zks_engine* engine, int32_t pass, const uint32_t* hist_dev);
int zks_select_dist_end(zks_engine* engine);

/* Same selection, asynchronous: the selected values land in out_dev[0..nranks) (device). */
int zks_select_ranks_async(zks_engine* engine, const double* values_dev, int64_t count, const int64_t* ranks_host,
                           int32_t nranks, double* out_dev);

/* normalization(gamma, support) (distribution.py:71-85): the finite power sum over 1..K
 * (support_k > 0) or the zeta series with its Euler-Maclaurin tail (support_k == 0,
 * series.py:126-138).  Synchronous. */
int zks_normaliser(zks_engine* engine, double gamma, int32_t support_k, double* out_host);

/* First `count` values of RandomStream.for_replicate(seed, rep, idx).uniforms(count)
 * (distribution.py:182-187), bit-exact.  Asynchronous. */
int zks_stream_uniforms(zks_engine* engine, uint64_t seed, uint64_t repetition, uint64_t index, int64_t count,
                        double* out_dev);

/* The same stream for an explicit Philox4x64 key (k0, k1) = SeedSequence(key).generate_state(2,
 * uint64): RandomStream(key) for keys other than [seed, repetition, index] (distribution.py:
 * 173-180 accepts any SeedSequence entropy; the host derives the key, the device the uniforms).
 * Asynchronous. */
/* Replicate streams of later calls: ZKS_RNG_NUMPY = RandomStream.for_replicate (distribution.py:
 * 173-187) bit for bit; ZKS_RNG_PHILOX4X32 = an opt-in faster generator keyed by the same
 * SeedSequence key: different samples, the same distributions, so cutoffs
 * agree with the default only within Monte Carlo error.  User-facing RandomStream uniforms are
 * always numpy's. */
int zks_engine_set_rng(zks_engine* engine, int rng);

/* Memory budget (bytes) of one chunk of pre-drawn rows on the two-kernel path (0, the default: 40 %
 * of the free device memory, at most 48 GiB): a cell whose rows exceed it runs chunk by chunk.
 * Results do not depend on it. */
int zks_engine_set_chunk_bytes(zks_engine* engine, uint64_t bytes);

int zks_stream_uniforms_key(zks_engine* engine, uint64_t k0, uint64_t k1, int64_t count, double* out_dev);

/* Inverse-transform draws for given uniforms: searchsorted(cdf, u, 'left') + 1 clamped to the
 * table length (sample, distribution.py:190-201).  Asynchronous. */
int zks_draw(zks_engine* engine, const zks_table* table, const double* u_dev, int64_t count, int64_t* out_dev);

/* ---- user samples (fit --bespoke, batched dataset fitting) --------------------- */

#define ZKS_FIT_EXPONENT 1  /* estimate the exponent (mle_gamma)                            */
#define ZKS_FIT_KS 2        /* score the KS statistic (against the fit, or gamma_in)         */

#define ZKS_SAMPLE_OK 0
#define ZKS_SAMPLE_NOROOT 2   /* NoRootError (estimate.py:101-105)                         */
#define ZKS_SAMPLE_OUTSIDE 3  /* an observation outside the support (or >= 2^32)           */
#define ZKS_SAMPLE_EMPTY 4

/* MleSettings (estimate.py:24-47). */
typedef struct {
  double initial_guess;
  double absolute_tolerance;
  int32_t max_iterations;
  int32_t reserved;
  double bracket_lo, bracket_hi;
} zks_mle_settings;

/* For each sample i = values_dev[offsets_dev[i] .. offsets_dev[i+1]) (positive int64): its
 * log_mean (estimate.py:59-73), with ZKS_FIT_EXPONENT its mle_gamma (estimate.py:115-146;
 * settings NULL = DEFAULT_SETTINGS), with ZKS_FIT_KS its ks_statistic and argmax_k
 * (gof.py:49-105) against the fitted exponent or, without ZKS_FIT_EXPONENT, against
 * gamma_in_dev[i] with normaliser norm_in_dev[i] (NULL: summed on the device).  Replaces the
 * per-sample calls of cli._cmd_fit (cli.py:197-262).  Asynchronous. */
int zks_fit_samples(zks_engine* engine, int32_t support_k, const int64_t* values_dev, const int64_t* offsets_dev,
                    int64_t nsamples, int32_t mode, const zks_mle_settings* settings, const double* gamma_in_dev,
                    const double* norm_in_dev, double* log_mean_dev, double* gamma_dev, double* ks_dev,
                    int64_t* argmax_dev, uint8_t* status_dev);

/* Reference series at gamma_dev[i]: out_dev[4i..4i+4) = (s0, s1, s2, normaliser) with
 * s_p = sum k^-g (ln k)^p over 1..K (finite_log_moments, series.py:68-73) or the zeta series
 * with its Euler-Maclaurin tail and m-doubling rule (zeta_log_moments, series.py:102-123),
 * normaliser = normalization (distribution.py:71-85).  NaN where the series diverges. */
int zks_series_eval(zks_engine* engine, int32_t support_k, const double* gamma_dev, int64_t count, double* out_dev);

/* tail_mass (series.py:141-160): out_dev[i] = sum_{k >= start_dev[i]} k^-gamma by Euler-Maclaurin
 * through the third-derivative term; every start must exceed 64 (checked by the shim).
 * Asynchronous. */
int zks_tail_mass(zks_engine* engine, double gamma, const double* start_dev, int64_t count, double* out_dev);

/* The exponent for given mean-log targets: Newton/bisection as mle_gamma, or with bisect_only
 * the bisection of _bisect (estimate.py:94-112) on [bracket_lo, bracket_hi].  status 2 =
 * NoRootError.  Asynchronous. */
int zks_solve_exponents(zks_engine* engine, int32_t support_k, const double* target_dev, int64_t count,
                        const zks_mle_settings* settings, int32_t bisect_only, double* gamma_dev, uint8_t* status_dev);

/* ---- diagnostics (bench.py roofline, parity tests; not part of the reference interface) --- */

/* How the replicate kernel evaluates the model functions of the exponent fit
 * (estimate.py:76-83): ZKS_MLE_TABLE (default) or ZKS_MLE_DIRECT. */
int zks_engine_set_mle_mode(zks_engine* engine, int mode);

/* Evaluate the fit table of support_k (0 = unbounded) at x_dev[0..count): model mean of ln X,
 * E[(ln X)^2] and the normaliser (zeta_value for the unbounded support).  Asynchronous. */
int zks_fit_eval(zks_engine* engine, int32_t support_k, const double* x_dev, int64_t count, double* mu_dev,
                 double* m2_dev, double* norm_dev);

/* Accumulate the replicate kernels' work counters into counters_dev[0..13) (u64, caller
 * zeroes): attempts, Philox draws, moment evaluations, moment terms, normaliser terms, KS
 * dense terms, KS endpoints, KS tiles, draws read from staged words, Philox draws made by
 * the staging kernel, staged replicates redrawn from Philox, rows written by the draw kernel
 * (n >= 128), tail values in those rows.  NULL switches counting off. */
int zks_engine_set_counters(zks_engine* engine, unsigned long long* counters_dev);

/* On-device pipe peaks measured by micro-kernels: out_host[0] = FP64 DFMA FLOP/s,
 * out_host[1] = FP64 exp() evaluations/s, out_host[2] = 64x64->128-bit multiplies/s
 * (the Philox4x64 core).  Synchronous. */
int zks_probe_peaks(zks_engine* engine, double* out_host);

#ifdef __cplusplus
}
#endif

#endif /* ZIPFKS_B200_H */
