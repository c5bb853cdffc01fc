// hc_finish.cu — ordering of the positions the search kernels' fused epilogue could not
// order itself: up to kSmallSort in one CTA, more through an n-bit
// bitmap (positions are distinct and < n) and a popcount-prefix compaction, which
// yields them ascending without a comparison sort.
#include <cub/block/block_radix_sort.cuh>

#include <mutex>

#include "hc_device.cuh"

namespace hc {

// One CTA of 1024 threads: orders 2 <= count <= kSmallSort positions (distinct keys)
// that the search kernel's epilogue could not (above its shared-memory capacity, or
// clustered) and writes the first min(count, max_out) as int64:
//   count <= kRankSort : rank counting (key i goes to #{j : key_j < key_i});
//   otherwise          : a bucket pass on the top 11 of the ceil(log2 n) bits
//                        (shared counters, scan, scatter), then each key's rank inside
//                        its bucket by counting; a bucket larger than kBucketMax
//                        (skewed positions) sends the whole set to a block radix sort.
constexpr uint32_t kRankSort = 256;
constexpr int kFinishThreads = 1024;
constexpr int kFinishItems = kSmallSort / kFinishThreads;
constexpr uint32_t kBucketBits = 11;
constexpr uint32_t kBuckets = 1u << kBucketBits;
constexpr uint32_t kBucketMax = 32;
using FinishSort = cub::BlockRadixSort<uint32_t, kFinishThreads, kFinishItems>;
__global__ void __launch_bounds__(kFinishThreads) order_small_kernel(const uint32_t *pos, uint32_t count,
                                                                     int64_t *dst, uint32_t max_out,
                                                                     uint32_t nbits) {
    __shared__ union {
        typename FinishSort::TempStorage sort;
        struct {
            uint32_t cnt[kBuckets];     // keys per bucket, then bucket starts
            uint32_t keys[kSmallSort];  // keys grouped by bucket
            uint32_t warp_sum[32];
            uint32_t maxcnt;
        } b;
    } sm;
    if (dst == nullptr || max_out == 0 || count == 0 || count > kSmallSort) return;
    const uint32_t k = min(count, max_out);
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (count == 1) {
        if (t == 0) dst[0] = static_cast<int64_t>(pos[0]);
        return;
    }
    if (count <= kRankSort) {
        if (t < count) sm.b.keys[t] = pos[t];
        __syncthreads();
        if (t < count) {
            const uint32_t key = sm.b.keys[t];
            uint32_t r = 0;
            for (uint32_t i = 0; i < count; ++i) r += sm.b.keys[i] < key;
            if (r < k) dst[r] = static_cast<int64_t>(key);
        }
        return;
    }
    // bucket pass: key -> bucket key >> shift (< kBuckets since key < 2^nbits)
    const uint32_t shift = nbits > kBucketBits ? nbits - kBucketBits : 0u;
    for (uint32_t i = t; i < kBuckets; i += kFinishThreads) sm.b.cnt[i] = 0;
    if (t == 0) sm.b.maxcnt = 0;
    __syncthreads();
    uint32_t key[kFinishItems], slot[kFinishItems];
#pragma unroll
    for (int i = 0; i < kFinishItems; ++i) {
        const uint32_t g = t + i * kFinishThreads;
        key[i] = g < count ? pos[g] : 0u;
        slot[i] = g < count ? atomicAdd(&sm.b.cnt[key[i] >> shift], 1u) : 0u;
    }
    __syncthreads();
    // exclusive scan of the 2048 counters: 2 per thread, warp shuffles, warp totals
    const uint32_t c0 = sm.b.cnt[2 * t], c1 = sm.b.cnt[2 * t + 1];
    uint32_t incl = c0 + c1;
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(HC_FULL, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) sm.b.warp_sum[warp] = incl;
    const uint32_t mx = __reduce_max_sync(HC_FULL, max(c0, c1));
    if (lane == 0) atomicMax(&sm.b.maxcnt, mx);
    __syncthreads();
    if (warp == 0) {
        uint32_t w = sm.b.warp_sum[lane];
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(HC_FULL, w, o);
            if (lane >= o) w += v;
        }
        sm.b.warp_sum[lane] = w - sm.b.warp_sum[lane];   // exclusive warp offsets
    }
    __syncthreads();
    const uint32_t base = sm.b.warp_sum[warp] + incl - (c0 + c1);
    const bool skewed = sm.b.maxcnt > kBucketMax;
    __syncthreads();
    if (!skewed) {
        sm.b.cnt[2 * t] = base;              // bucket starts
        sm.b.cnt[2 * t + 1] = base + c0;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kFinishItems; ++i)
            if (t + i * kFinishThreads < count) sm.b.keys[sm.b.cnt[key[i] >> shift] + slot[i]] = key[i];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kFinishItems; ++i) {
            if (t + i * kFinishThreads >= count) continue;
            const uint32_t bk = key[i] >> shift;
            const uint32_t lo = sm.b.cnt[bk];
            const uint32_t hi = bk + 1 < kBuckets ? sm.b.cnt[bk + 1] : count;
            uint32_t r = lo;
            for (uint32_t j = lo; j < hi; ++j) r += sm.b.keys[j] < key[i];
            if (r < k) dst[r] = static_cast<int64_t>(key[i]);
        }
        return;
    }
    // skewed positions: block radix sort (blocked arrangement, all-ones pads)
    uint32_t keys[kFinishItems];
#pragma unroll
    for (int i = 0; i < kFinishItems; ++i) {
        const uint32_t g = t * kFinishItems + i;
        keys[i] = g < count ? pos[g] : 0xffffffffu;
    }
    // real keys are < 2^nbits, the all-ones pads have bit nbits set: sorting bits
    // [0, nbits] puts the pads last
    const uint32_t hb = nbits < 32 ? nbits + 1 : 32;
    FinishSort(sm.sort).SortBlockedToStriped(keys, 0, static_cast<int>(hb));
#pragma unroll
    for (int i = 0; i < kFinishItems; ++i) {
        const uint32_t r = t + i * kFinishThreads;  // striped: rank r
        if (r < k) dst[r] = static_cast<int64_t>(keys[i]);
    }
}


// ------------------------------------------------------------------ bitmap ordering
// count > kSmallSort: every position sets its bit in an n-bit bitmap (scatter), the
// bits per tile of kTileWords words are counted on the way (warp-aggregated atomics),
// one CTA scans the tile counts, and each tile writes its positions in bit order at its
// offset (emit).  The bitmap and the tile counts are left zero for the next call (emit
// clears the words it read, the scan clears the counts), so nothing is memset per call.
constexpr uint32_t kTileWords = 2048;           // 64 Ki positions per emit tile
constexpr int kEmitThreads = 256;
constexpr uint32_t kEmitWords = kTileWords / kEmitThreads;   // 8 words per thread

__global__ void __launch_bounds__(256) bitmap_scatter_kernel(const uint32_t *pos, uint32_t count,
                                                             uint32_t *bm, uint32_t *tile_cnt) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; i0 < count;
         i0 += gridDim.x * blockDim.x) {
        const uint32_t i = i0 + lane;
        const bool in = i < count;
        const uint32_t p = in ? __ldcs(pos + i) : 0xffffffffu;
        const uint32_t w = p >> 5;
        // lanes hitting the same word OR their bits first: one atomic per distinct word
        const uint32_t same = __match_any_sync(HC_FULL, w);
        const uint32_t bits = __reduce_or_sync(same, in ? 1u << (p & 31) : 0u);
        if (in && lane == __ffs(same) - 1) atomicOr(bm + w, bits);
        const uint32_t t = in ? w / kTileWords : 0xffffffffu;
        const uint32_t st = __match_any_sync(HC_FULL, t);
        if (in && lane == __ffs(st) - 1) atomicAdd(tile_cnt + t, static_cast<uint32_t>(__popc(st)));
    }
}

// one CTA: exclusive scan of the tile counts into tile_off, counts cleared
__global__ void __launch_bounds__(1024) bitmap_scan_kernel(uint32_t *tile_cnt, uint32_t *tile_off,
                                                           uint32_t ntiles) {
    __shared__ uint32_t tmp[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t b = 0; b < ntiles; b += blockDim.x) {
        const uint32_t i = b + threadIdx.x;
        const uint32_t v = i < ntiles ? tile_cnt[i] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(HC_FULL, incl, o);
            if (lane >= o) incl += x;
        }
        if (lane == 31) tmp[warp] = incl;
        __syncthreads();
        uint32_t wb = 0, tot = 0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
            if (w < warp) wb += tmp[w];
            tot += tmp[w];
        }
        const uint32_t c0 = carry;
        if (i < ntiles) {
            tile_off[i] = c0 + wb + incl - v;
            tile_cnt[i] = 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry = c0 + tot;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kEmitThreads) bitmap_emit_kernel(uint32_t *bm, const uint32_t *tile_off,
                                                                   int64_t *dst, uint32_t k) {
    __shared__ uint32_t tmp[32];
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const size_t w0 = static_cast<size_t>(blockIdx.x) * kTileWords + t * kEmitWords;
    uint4 *src = reinterpret_cast<uint4 *>(bm + w0);
    uint4 a = src[0], b = src[1];
    const uint32_t wv[kEmitWords] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t loc = 0;
#pragma unroll
    for (uint32_t i = 0; i < kEmitWords; ++i) loc += __popc(wv[i]);
    if (loc) {                                  // leave the bitmap zero for the next call
        src[0] = make_uint4(0, 0, 0, 0);
        src[1] = make_uint4(0, 0, 0, 0);
    }
    uint32_t incl = loc;
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(HC_FULL, incl, o);
        if (lane >= o) incl += x;
    }
    if (lane == 31) tmp[warp] = incl;
    __syncthreads();
    uint32_t wb = 0;
    for (uint32_t w = 0; w < warp; ++w) wb += tmp[w];
    uint32_t r = tile_off[blockIdx.x] + wb + incl - loc;     // rank of this thread's first bit
#pragma unroll
    for (uint32_t i = 0; i < kEmitWords; ++i) {
        uint32_t x = wv[i];
        const int64_t base = static_cast<int64_t>(w0 + i) * 32;
        while (x && r < k) {
            const uint32_t bit = __ffs(x) - 1;
            x &= x - 1;
            dst[r++] = base + bit;
        }
    }
}

namespace {
// per (host thread, device) bitmap and tile arrays, grown on demand and zeroed once
struct Bitmap {
    uint32_t *bm = nullptr;        // nwords words, then 2 x ntiles tile counts / offsets
    size_t nwords = 0, ntiles = 0;
};
thread_local Bitmap g_bitmap[16];
}  // namespace

cudaError_t order_positions(const uint32_t *pos, uint32_t count, uint32_t n, int64_t *dst, uint32_t k,
                            cudaStream_t st, int *launches) {
    if (count < 2 || k == 0 || dst == nullptr) return cudaSuccess;
    if (count <= kSmallSort) {
        order_small_kernel<<<1, kFinishThreads, 0, st>>>(pos, count, dst, k, bits_for(n));
        if (launches) *launches += 1;
        return cudaGetLastError();
    }
    int dev = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return err;
    if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
    Bitmap &B = g_bitmap[dev];
    const size_t ntiles = (static_cast<size_t>(n) + 32 * kTileWords - 1) / (32 * kTileWords);
    const size_t nwords = ntiles * kTileWords;
    if (B.nwords < nwords) {
        if (B.bm) cudaFree(B.bm);   // synchronises: no earlier ordering still uses it
        B.bm = nullptr;
        B.nwords = B.ntiles = 0;
        const size_t bytes = (nwords + 2 * ntiles) * sizeof(uint32_t);
        err = cudaMalloc(&B.bm, bytes);
        if (err != cudaSuccess) return err;
        err = cudaMemsetAsync(B.bm, 0, bytes, st);
        if (err != cudaSuccess) return err;
        B.nwords = nwords;
        B.ntiles = ntiles;
    }
    uint32_t *tile_cnt = B.bm + B.nwords, *tile_off = tile_cnt + B.ntiles;
    const uint32_t sblocks = std::min<uint32_t>((count + 255) / 256, 148u * 16u);
    bitmap_scatter_kernel<<<sblocks, 256, 0, st>>>(pos, count, B.bm, tile_cnt);
    bitmap_scan_kernel<<<1, 1024, 0, st>>>(tile_cnt, tile_off, static_cast<uint32_t>(ntiles));
    bitmap_emit_kernel<<<static_cast<unsigned>(ntiles), kEmitThreads, 0, st>>>(B.bm, tile_off, dst, k);
    if (launches) *launches += 3;
    return cudaGetLastError();
}

}  // namespace hc
