// Internal interface between the host side (hc_api.cpp) and the device side
// (hc_kernels.cu) of libhc.  Not part of the C-ABI.
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
    uint32_t S;          // HC shift m - q + 1
    uint32_t alpha;
    // lattice: segments of L <= S window ends starting at a0; (y + a0) is
    // congruent to Wd - 1 mod Wd so every lattice q-gram sits in one aligned Wd-byte word.
    // Window ends [m-1, a0) form the head segment.
    uint32_t a0, L, Wd;
    uint32_t K;          // lattice segments: ceil((n - a0) / L), 0 if a0 >= n
    // staged path
    uint32_t seg_per_tile;  // segments per shared-memory tile
    uint32_t ntiles;
    uint32_t stage_bytes;   // bytes per stage buffer (multiple of 16)
    uint32_t stages;
    uint32_t surv_warps;    // survivor/producer warps per CTA (1..4)
    // gather path
    uint32_t seg_per_chunk; // segments per warp chunk
    uint32_t nchunks;
    // output
    uint32_t *out;       // positions (window starts), unordered; NULL = count only
    uint32_t cap;        // capacity of out
    uint32_t *counter;   // [0] = total occurrences (may exceed cap), [1] = CTA exit ticket
    // fused finish (last CTA): order <= sort_cap positions into dst, publish the count
    int64_t *dst;        // caller's int64 positions (NULL: none)
    uint32_t k_out;      // positions wanted (min(max_out, windows))
    uint32_t sort_cap;   // largest count the last CTA sorts in shared memory (power of 2)
    uint32_t *host_count;   // mapped pinned word (device alias) receiving the count
    uint32_t debug;      // 1: staged kernel skips the search (pipeline measurement only)
    uint32_t tma_chunk;  // staged: split each tile's bulk copy into pieces of this size (0 = one)
    unsigned long long *trace;  // staged: per-(CTA, tile) %globaltimer events (debugging), or NULL
    uint32_t trace_tiles;       // tiles per CTA recorded
};

using KernFn = void (*)(const KParams);
// per-q instantiation units (hc_inst.cu compiled with -DHC_Q=q): kernel for (s, WD) or NULL
#define HC_DECL_Q(Q) KernFn staged_kernel_q##Q(uint32_t s, uint32_t wd); \
                     KernFn gather_kernel_q##Q(uint32_t s, uint32_t wd);
HC_DECL_Q(1) HC_DECL_Q(2) HC_DECL_Q(3) HC_DECL_Q(4) HC_DECL_Q(5) HC_DECL_Q(6) HC_DECL_Q(7) HC_DECL_Q(8)
#undef HC_DECL_Q

struct LaunchInfo {
    int grid = 0, block = 0, smem = 0;
};

// Device-side entry points (hc_kernels.cu).  All enqueue on `st`.
cudaError_t launch_staged(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li);
cudaError_t launch_gather(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li);
// Ordering of count > kSmallSort positions (CUB radix sort), first k written as int64.
cudaError_t sort_large(const uint32_t *pos, uint32_t count, uint32_t n_bound, int64_t *dst,
                       uint32_t k, cudaStream_t st, int *launches);
constexpr uint32_t kSmallSort = 8192;

int staged_smem_bytes(uint32_t alpha, uint32_t m, uint32_t stage_bytes, uint32_t stages,
                      uint32_t slot_bytes, uint32_t nbox);
int gather_smem_bytes(uint32_t alpha, uint32_t m);

constexpr int kStagedThreads = 256;
constexpr int kGatherThreads = 256;
constexpr int kWarpBuf = 64;  // per-warp match buffer entries (shared memory)

}  // namespace hc
