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
    const uint32_t *Fbits;  // filter bitmap, device, 2^alpha bits (bit v = F[v] != 0), >= 16 B
    const uint8_t *x;    // pattern, device, followed by >= 24 zero bytes (16-byte aligned)
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
    uint32_t lane_bits;     // stream: filter bitmap replicated per lane in shared memory
    uint32_t shc;           // SHC path (chunk geometry: whole segments)
    uint32_t mgather;       // multi-pattern kernel without staging (gather access)
    // output
    uint32_t *out;       // positions (window starts), unordered; NULL = count only
    uint32_t cap;        // capacity of out
    uint32_t *counter;   // kCtr words: [0] = total occurrences (may exceed cap), [1] = staged
                         // tile counter, [2] = CTAs done (epilogue ticket), [3] = give-up
                         // flag (gather); zero between calls.  [4] = the position in slot 0
                         // of out (read by the epilogue with the count)
    // fused epilogue (the last CTA to finish): count publication + ordering
    uint32_t *host_count;  // mapped pinned [2]: count, then 1 if the positions were ordered
                           // into dst by the epilogue (else the host orders them)
    int64_t *dst;        // caller's pos_out (device), NULL = count only
    uint32_t k_out;      // min(max_out, windows)
    uint32_t epi_cap;    // largest count the epilogue orders in its CTA's shared memory
    uint32_t nbits;      // positions are < 2^nbits
    uint32_t allow_abort;  // gather path: may give up on walk-heavy text (host_count[1] = 2)
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
    uint32_t *host_count[kMaxPatterns];
    int64_t *dst[kMaxPatterns];
    uint32_t k_out[kMaxPatterns];
};
constexpr int kCtr = 8;   // counter words per search (KParams::counter)

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
cudaError_t launch_scan(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                        LaunchInfo *li);
int scan_smem_bytes(uint32_t alpha, uint32_t m, uint32_t q, uint32_t buf_bytes);
// Ordering of `count` distinct positions (u32, unordered) into dst: the smallest k,
// ascending, as int64.  Used when the search kernel's epilogue did not order them
// (count above its shared-memory capacity, or skewed).  count <= kSmallSort: one CTA
// (bucket pass / block radix sort); larger: an n-bit bitmap and a popcount-prefix
// compaction (no comparison sort).  Adds the launches it made to *launches.
cudaError_t order_positions(const uint32_t *pos, uint32_t count, uint32_t n, int64_t *dst,
                            uint32_t k, cudaStream_t st, int *launches);
constexpr uint32_t kSmallSort = 8192;
#if defined(HC_INSTRUMENT) && HC_INSTRUMENT
cudaError_t read_epi_ts(unsigned long long *host16);  // hc_stream.cu, debug 10
#endif
inline uint32_t bits_for(uint32_t n) {   // positions < n fit in bits_for(n) bits
    uint32_t b = 1;
    while (b < 32 && (static_cast<uint64_t>(1) << b) < n) ++b;
    return b;
}
// shared-memory bytes the epilogue needs to order `count` positions (keys + bucket array)
constexpr uint32_t epi_bytes(uint32_t count) { return 12u * count + 544u; }

int staged_smem_bytes(uint32_t alpha, uint32_t m, uint32_t stage_bytes, uint32_t stages,
                      uint32_t slot_bytes, uint32_t nbox);
int gather_smem_bytes(uint32_t alpha, uint32_t m);
int shc_smem_bytes(uint32_t alpha, uint32_t m, uint32_t buf_bytes, uint32_t box_bytes,
                   uint32_t nwarps);
int stream_smem_bytes(uint32_t alpha, uint32_t m, uint32_t buf_bytes, uint32_t bufs, uint32_t nwarps,
                      uint32_t lane_bits);

constexpr int kStagedThreads = 256;
constexpr int kGatherThreads = 256;
constexpr int kStreamMaxThreads = 256;   // SHC and (x2) multi-pattern kernels
constexpr int kStreamFatThreads = 768;   // stream kernel: one CTA per SM, up to 24 warps (<= 85 registers)
constexpr int kStreamRegThreads = 640;   // ... or up to 20 warps with <= 102 registers
constexpr int kWarpBuf = 64;  // per-warp match buffer entries (shared memory)

}  // namespace hc
