// Internal interface between the host side (hc_api.cpp) and the device side
// (hc_*.cu, one translation unit per search path) of libhc.  Not part of the C-ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace hc {

// Everything one search kernel launch needs (passed by value).
struct KParams {
    const uint8_t *y;    // text, device, any alignment
    uint32_t n;          // text length (n >= m, n <= HC_MAX_TEXT)
    const uint32_t *F;   // filter table, device, 2^alpha words
    const uint8_t *x;    // pattern, device
    uint32_t m, q, s, mask, hv;
    uint32_t S;          // shift m - q + 1: also the segment length
    uint32_t alpha;
    uint32_t K;          // number of segments: ceil((n - m + 1) / S)
    // staged path
    uint32_t seg_per_tile;  // segments per shared-memory tile
    uint32_t ntiles;
    uint32_t stage_bytes;   // bytes per stage buffer (multiple of 16)
    uint32_t stages;
    uint32_t slot_bytes;    // survivor box slot size (>= S + m + 30, multiple of 16)
    uint32_t nbox;          // survivor boxes (32 slots each) per CTA
    // gather path
    uint32_t seg_per_chunk; // segments per warp chunk
    uint32_t nchunks;
    uint32_t block_warps;   // stream / SHC paths: warps per CTA
    uint32_t shc;           // SHC path (chunk geometry: whole segments)
    uint32_t mgather;       // multi-pattern kernel without staging (gather access)
    // output
    uint32_t *out;       // positions (window starts), unordered; NULL = count only
    uint32_t cap;        // capacity of out
    uint32_t *counter;   // [0] = total occurrences (may exceed cap)
    uint32_t debug;      // 1: staged kernel skips the search (pipeline measurement only)
    uint32_t tma_chunk;  // staged: split each tile's bulk copy into pieces of this size (0 = one)
    unsigned long long *trace;  // staged: per-(CTA, tile) %globaltimer events (debugging), or NULL
    uint32_t trace_tiles;       // tiles per CTA recorded
};

// Per-pattern parameters of a multi-pattern launch (stream path, patterns sharing
// m, q, alpha): the text is staged once and filtered for every pattern.
constexpr int kMaxPatterns = 4;
struct MParams {
    uint32_t npat;
    const uint32_t *F[kMaxPatterns];
    const uint8_t *x[kMaxPatterns];
    uint32_t hv[kMaxPatterns];
    uint32_t *counter[kMaxPatterns];
    uint32_t *out[kMaxPatterns];
    uint32_t cap[kMaxPatterns];
};

struct LaunchInfo {
    int grid = 0, block = 0, smem = 0;
};

// Device-side entry points (hc_stream.cu, hc_gather.cu, ...).  All enqueue on `st`.
cudaError_t launch_staged(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li);
cudaError_t launch_stream(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li);
cudaError_t launch_shc(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                       LaunchInfo *li);
cudaError_t launch_mstream(const KParams &p, const MParams &mp, cudaStream_t st, int max_ctas,
                           int ctas_per_sm, LaunchInfo *li);
int mstream_smem_bytes(uint32_t alpha, uint32_t m, uint32_t buf_bytes, uint32_t nwarps, uint32_t npat,
                       uint32_t bufs);
cudaError_t launch_gather(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li);
// One CTA after the search kernel: count -> host_count (mapped pinned), counter reset,
// ordering of <= kSmallSort positions into dst (first min(count, max_out), int64).
cudaError_t launch_finish(uint32_t *counter, const uint32_t *pos, uint32_t cap, int64_t *dst,
                          uint32_t max_out, uint32_t n_bound, uint32_t *host_count_dev,
                          cudaStream_t st,
                          unsigned long long *trace = nullptr);
// Ordering of count > kSmallSort positions (CUB radix sort), first k written as int64.
cudaError_t sort_large(const uint32_t *pos, uint32_t count, uint32_t n_bound, int64_t *dst,
                       uint32_t k, cudaStream_t st, int *launches);
constexpr uint32_t kSmallSort = 8192;

int staged_smem_bytes(uint32_t alpha, uint32_t m, uint32_t stage_bytes, uint32_t stages,
                      uint32_t slot_bytes, uint32_t nbox);
int gather_smem_bytes(uint32_t alpha, uint32_t m);
int shc_smem_bytes(uint32_t alpha, uint32_t m, uint32_t buf_bytes, uint32_t box_bytes,
                   uint32_t nwarps);
int stream_smem_bytes(uint32_t alpha, uint32_t m, uint32_t buf_bytes, uint32_t bufs, uint32_t nwarps);

constexpr int kStagedThreads = 256;
constexpr int kGatherThreads = 256;
constexpr int kStreamMaxThreads = 256;
constexpr int kWarpBuf = 64;  // per-warp match buffer entries (shared memory)

}  // namespace hc
