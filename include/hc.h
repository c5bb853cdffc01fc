/*
 * hc.h — C-ABI of the B200-native Hash Chain (HC) exact string matcher.
 *
 * Method: Palmer, Faro, Scafiti, "Efficient Online String Matching through
 * Linked Weak Factors", arXiv 2310.15711.  P:n = line n of PAPER.md,
 * S:n = line n of SPEC.md (interfaces and contracts only).
 *
 * Problem: find all occurrences of a pattern x of length m in a text y
 * of length n.  hc_prepare() is the paper's Preprocessing(x, m, q, alpha)
 * (Fig. 3); hc_search() is the searching phase of HC(x, m, y, n,
 * q, alpha) (Fig. 5) run on one B200 (sm_100a).
 *
 * Result semantics: exactly { s in [0, n-m] : y[s..s+m-1] == x }, ascending,
 * overlaps included, no duplicates.  HC is an exact
 * matcher: the filter only rejects windows that cannot hold x
 * and every survivor is verified byte by byte, so the set does not
 * depend on q or alpha.  Positions are reported at the window start e-m+1
 * (reading R1).
 *
 * Conventions
 *   - All functions are extern "C" and thread-safe.  A handle is immutable
 *     after hc_prepare(): concurrent hc_search() calls on one handle (on any
 *     streams, from any host threads) are safe.
 *   - Errors: functions returning int / int64_t return a negative hc_status on
 *     failure; hc_prepare() returns NULL.  The code of the last failure on the
 *     calling host thread is available from hc_last_error().
 *   - Bytes are raw unsigned 0..255; no alphabet mapping.
 *   - The word width of F is w = 32 (reading R2).
 */
#ifndef HC_H_
#define HC_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h> /* cudaStream_t */

#ifdef __cplusplus
extern "C" {
#endif

typedef enum hc_status {
    HC_OK = 0,
    HC_EINVAL = -1,    /* NULL x with m > 0, m == 0, q < 1, NULL handle, NULL y with n > 0 */
    HC_ETOOSHORT = -2, /* q > m */
    HC_EALPHA = -3,    /* alpha outside [1, 15]: F = 2^alpha 32-bit words must fit in shared memory */
    HC_ENOMEM = -4,    /* host or device allocation failed */
    HC_ECUDA = -5,     /* a CUDA runtime call failed (see hc_strerror / stderr) */
    HC_ETOOLONG = -6,  /* n > HC_MAX_TEXT or m > HC_MAX_PATTERN */
    HC_ENODEV = -7     /* no CUDA device / device is not sm_100 */
} hc_status;

#define HC_WORD_BITS 32                  /* w */
#define HC_MAX_ALPHA 15
#define HC_MAX_PATTERN 65536u            /* m: x and F are kept in shared memory */
#define HC_MAX_TEXT 0xFFFF0000ull        /* n: positions are 32-bit inside the kernels */

typedef struct hc_handle hc_handle;

/* Preprocessing(x, m, q, alpha) — Fig. 3, Eq. 1-5.
 *   x     : HOST pointer to the m pattern bytes; copied, the caller keeps ownership.
 *   m     : pattern length, 1 <= m <= HC_MAX_PATTERN.
 *   q     : q-gram length, 1 <= q <= min(m, 8).  (q > m -> HC_ETOOSHORT; q > 8 -> HC_EINVAL.)
 *   alpha : F has 2^alpha words, 1 <= alpha <= 15; s = floor(alpha/q) (Eq. 4).
 * Builds F (w = 32) and H_v on the host in Fig. 3 order (including optimisation 1,
 * P:330-335) and uploads F and x synchronously to the CURRENT device.
 * Returns a new handle (free with hc_destroy) or NULL (see hc_last_error()). */
hc_handle *hc_prepare(const uint8_t *x, size_t m, int q, int alpha);

/* Preprocessing of P patterns at once (the paper times Preprocessing with every search,
 * P:380; a batch of searches amortises its uploads): Fig. 3 for each xs[i] (length
 * ms[i], HOST memory, copied) with the same q and alpha, then ONE device allocation and
 * ONE host-to-device copy for all the tables and patterns.  hs_out[i] receives the
 * handle of xs[i]; each is used and destroyed like an hc_prepare handle (the shared
 * device block is freed with the last of them).  Returns HC_OK, or a negative
 * hc_status (parameter checks as hc_prepare, per pattern) with no handle created. */
int hc_prepare_batch(const uint8_t *const *xs, const size_t *ms, size_t P, int q, int alpha,
                     hc_handle **hs_out);

/* Code of the last failure on this host thread (HC_OK if none). */
int hc_last_error(void);

/* Static description of a status code (never NULL). */
const char *hc_strerror(int code);

/* Searching phase of HC (Fig. 5 left) on the device.
 *   y_dev   : DEVICE pointer to the n text bytes; caller-owned, any alignment, never written.
 *   n       : text length; n < m (including n == 0) returns 0, not an error.
 *   pos_out : DEVICE pointer to int64_t[max_out], caller-owned; receives the min(count, max_out)
 *             SMALLEST occurrence start positions, ascending.  NULL or max_out == 0: count only.
 *   stream  : all device work is enqueued on this stream (ordered after the caller's fill of
 *             y_dev).  The call returns once the count is known (it synchronises on the count
 *             read-back); the writes to pos_out are enqueued on `stream` and complete in
 *             stream order.
 * Returns the total number of occurrences (>= 0), or a negative hc_status. */
int64_t hc_search(const hc_handle *h, const uint8_t *y_dev, size_t n, int64_t *pos_out,
                  size_t max_out, cudaStream_t stream);

/* Tuning knobs and statistics for hc_search_ex (tests and the benchmark). */
typedef enum hc_path {
    HC_PATH_AUTO = 0,   /* chosen from m, q */
    HC_PATH_STAGED = 1, /* text tiles staged in shared memory by TMA bulk copies */
    HC_PATH_GATHER = 2, /* no staging: lanes read only the q-grams they hash, from global memory */
    HC_PATH_STREAM = 3, /* per-warp chunks staged in shared memory by 1-D TMA bulk copies */
    HC_PATH_SHC = 4,    /* Sentinel Hash Chain (Fig. 5 right): per-lane ranges copied into shared-
                           memory boxes followed by a copy of x, SHC's fast loop per lane */
    HC_PATH_SCAN = 5    /* hash every position of staged pieces once into filter / link bitmaps,
                           then Fig. 5's loop per segment with O(1) walks (walk-heavy texts) */
} hc_path;

typedef struct hc_search_opts {
    int path;         /* hc_path */
    int tile_bytes;   /* staged: text bytes per shared-memory stage; stream: target text bytes
                         per warp chunk (0 = default) */
    int stages;       /* staged: TMA pipeline depth (the stream kernels always use 2 buffers per warp) */
    int seg_per_lane; /* gather: segments handed to each lane per chunk (0 = default);
                         stream: < 0 = final drain on global text (no private boxes) */
    int max_ctas;     /* cap on the persistent grid (0 = no cap; tests use 1..3 for many tiles per CTA) */
    int time_kernel;  /* 1: record CUDA events around this call's device work (stats->kernel_ms);
                         2: also around the search kernel alone (stats->search_ms; the extra
                         event sits between the search and finish kernels) */
    int ctas_per_sm;  /* cap on resident CTAs per SM for the persistent grid (0 = occupancy max) */
    int debug;        /* must be 0.  Measurement-only modes (1 = copy pipeline alone, 3 = phase A
                         only, 5 = phase-B counters, 6 = filter on stale stage data; results NOT
                         valid) exist only in the instrumented build libhc_instr.so
                         (HC_INSTRUMENT=1, tools/); this library returns HC_EINVAL if set */
    int tma_chunk;    /* staged: bytes per TMA bulk copy (0 = one copy per tile stage);
                         (the stream path always moves a chunk by one 1-D TMA bulk copy) */
    unsigned long long *trace; /* must be NULL (instrumented build only: DEVICE buffer of
                                  grid x trace_tiles x 4 %globaltimer stamps per (CTA, tile)) */
    int trace_tiles;
    int surv_warps;   /* staged: survivor/producer warps per CTA (0 = default) */
    int block_warps;  /* stream: warps per CTA, 1..24 (0 = default: up to 24, one CTA per SM) */
    int no_multi;     /* hc_search_batch: 0 = multi-pattern launches for shifts 9..256 (measured
                         faster there), 1 = never (each pattern alone), 2 = whenever the
                         patterns' shapes allow (shifts <= 256) */
} hc_search_opts;

typedef struct hc_search_stats {
    int path;          /* path used */
    int grid;          /* CTAs launched by the search kernel */
    int block;         /* threads per CTA */
    int smem_bytes;    /* dynamic shared memory per CTA */
    int64_t tiles;     /* staged: text tiles; gather: lane chunks */
    int launches;      /* kernels launched by this call (search, re-run, sort, copy) */
    int reruns;        /* search re-runs after the position scratch overflowed */
    float kernel_ms;   /* if time_kernel: device time from the first search launch to the end
                          of the call's last kernel (search, finish, re-runs, ordering) */
    uint32_t dbg[2];   /* instrumented build, debug == 5: phase-B loop iterations and calls */
    float search_ms;   /* if time_kernel == 2: device time of the first search kernel alone */
} hc_search_stats;

/* hc_search with explicit options (NULL = defaults) and optional statistics (NULL = none). */
int64_t hc_search_ex(const hc_handle *h, const uint8_t *y_dev, size_t n, int64_t *pos_out,
                     size_t max_out, cudaStream_t stream, const hc_search_opts *opts,
                     hc_search_stats *stats);

/* Batch of independent searches over the same text (multi-pattern
 * batching): the result of pattern i is exactly hc_search(hs[i], y_dev, n, pos_out[i],
 * max_out[i], stream) (Fig. 5, per pattern).  Consecutive patterns of
 * equal (m, q, alpha) with shifts 9 <= m - q + 1 <= 256 are searched up to 4 per launch by
 * the multi-pattern kernel: one pass over the text, each lattice q-gram hashed once
 * and tested against every pattern's F (opts->no_multi = 1 disables it).  Launches
 * are spread over 8 library-owned streams so that one launch's tail and launch
 * latency overlap the next one's work; the call is ordered after prior work on
 * `stream`, and returns after all of them completed (stream order is preserved for
 * later work).
 *   hs      : npat handles (same device), read-only.
 *   y_dev   : DEVICE text, n bytes, caller-owned, read-only.
 *   counts  : HOST int64[npat], receives each pattern's occurrence count.
 *   pos_out : HOST array of npat DEVICE int64 pointers (entries may be NULL), or NULL:
 *             min(count, max_out[i]) smallest positions of pattern i, ascending.
 *   max_out : HOST size_t[npat], or NULL (count only).
 *   opts    : path/tuning knobs as for hc_search_ex (debug and trace are ignored);
 *             time_kernel = 1 puts the device time of the whole batch in stats->kernel_ms.
 * Patterns whose positions need more room than the scratch or the large sort are
 * re-run alone (stats->reruns).  Returns HC_OK or a negative hc_status. */
int hc_search_batch(const hc_handle *const *hs, size_t npat, const uint8_t *y_dev, size_t n,
                    int64_t *counts, int64_t *const *pos_out, const size_t *max_out,
                    cudaStream_t stream, const hc_search_opts *opts, hc_search_stats *stats);

/* End-to-end convenience: y_host and pos_out_host are HOST pointers.  Copies y to the
 * device (staged through pinned buffers when y_host is pageable), searches, and copies
 * min(count, max_out) positions back.  Synchronous.  Returns the count or a negative
 * hc_status. */
int64_t hc_search_host(const hc_handle *h, const uint8_t *y_host, size_t n,
                       int64_t *pos_out_host, size_t max_out, cudaStream_t stream);

/* End-to-end batch: hc_search_batch with HOST buffers.  Copies the n text bytes at y_host
 * (pinned or pageable HOST memory) to a device buffer the call owns, runs
 * hc_search_batch(hs, npat, ...) on it, and copies each pattern's min(count, max_out[i])
 * positions back into pos_out_host[i] (HOST int64 buffers, or NULL entries / NULL array for
 * counts only).  Synchronous; every copy and kernel is enqueued on `stream`.
 * counts: HOST int64[npat].  Returns HC_OK or a negative hc_status. */
int hc_search_batch_host(const hc_handle *const *hs, size_t npat, const uint8_t *y_host, size_t n,
                         int64_t *counts, int64_t *const *pos_out_host, const size_t *max_out,
                         cudaStream_t stream, const hc_search_opts *opts, hc_search_stats *stats);

/* Frees the handle's host and device state.  No search on the handle may be in flight. */
void hc_destroy(hc_handle *h);

/* Test introspection: the handle's host copy of the table the kernels use.
 *   *F receives a pointer to 2^alpha uint32_t words owned by the handle (valid until
 *   hc_destroy); alpha, s (Eq. 4), w (= 32) and H_v are written when non-NULL.
 * Returns HC_OK or HC_EINVAL. */
int hc_table(const hc_handle *h, const uint32_t **F, int *alpha, int *s, int *w,
             uint32_t *h_v);

/* Host-only Preprocessing (no device needed): the same table hc_prepare builds.
 *   F_out : HOST uint32_t[2^alpha], written in full.  s_out, hv_out: written when non-NULL.
 * Returns HC_OK or a negative hc_status (same parameter checks as hc_prepare). */
int hc_build_table(const uint8_t *x, size_t m, int q, int alpha, uint32_t *F_out,
                   int *s_out, uint32_t *hv_out);

/* Library version string. */
const char *hc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HC_H_ */
