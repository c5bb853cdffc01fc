// hc_finish.cu — count publication and ordering of the positions.
#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_radix_sort.cuh>

#include "hc_device.cuh"

namespace hc {

// ------------------------------------------------------------------ ordering
__global__ void widen_kernel(const uint32_t *src, int64_t *dst, uint32_t k) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
        dst[i] = static_cast<int64_t>(src[i]);
}


// Runs right after the search kernel, one CTA: publishes the count to the host
// (mapped pinned word), resets the device counter for the next call, and when
// 1 <= count <= kSmallSort orders the positions (distinct keys) and writes the first
// min(count, max_out) as int64:
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
__global__ void __launch_bounds__(kFinishThreads) finish_kernel(uint32_t *counter, const uint32_t *pos,
                                                                uint32_t cap, int64_t *dst,
                                                                uint32_t max_out, uint32_t nbits,
                                                                volatile uint32_t *host_count,
                                                                unsigned long long *trace) {
    __shared__ union {
        typename FinishSort::TempStorage sort;
        struct {
            uint32_t cnt[kBuckets];     // keys per bucket, then bucket starts
            uint32_t keys[kSmallSort];  // keys grouped by bucket
            uint32_t warp_sum[32];
            uint32_t maxcnt;
        } b;
    } sm;
    if (kInstrument && trace && threadIdx.x == 0) trace[0] = gtimer();
    pdl_wait();   // the search grid has completed and its writes are visible
    if (kInstrument && trace && threadIdx.x == 0) trace[1] = gtimer();
    const uint32_t count = *counter;
    __syncthreads();
    if (threadIdx.x == 0) {
        *host_count = count;
        counter[0] = 0;
        counter[1] = 0;   // staged path: dynamic tile counter
    }
    if (dst == nullptr || max_out == 0 || count == 0 || count > cap || count > kSmallSort) return;
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

cudaError_t launch_finish(uint32_t *counter, const uint32_t *pos, uint32_t cap, int64_t *dst,
                          uint32_t max_out, uint32_t n_bound, uint32_t *host_count_dev,
                          cudaStream_t st, unsigned long long *trace) {
    uint32_t nbits = 1;
    while (nbits < 32 && (static_cast<uint64_t>(1) << nbits) <= n_bound) ++nbits;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(kFinishThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, finish_kernel, counter, pos, cap, dst, max_out, nbits,
                              host_count_dev, trace);
}

// count > kSmallSort: CUB radix sort on ceil(log2 n) bits, then widen the first k.
cudaError_t sort_large(const uint32_t *pos, uint32_t count, uint32_t n_bound, int64_t *dst,
                       uint32_t k, cudaStream_t st, int *launches) {
    int end_bit = 1;
    while (end_bit < 32 && (static_cast<uint64_t>(1) << end_bit) <= n_bound) ++end_bit;
    uint32_t *alt = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t err = cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, pos, alt,
                                                     static_cast<int>(count), 0, end_bit, st);
    if (err != cudaSuccess) return err;
    err = cudaMallocAsync(reinterpret_cast<void **>(&alt),
                          static_cast<size_t>(count) * 4 + tmp_bytes + 256, st);
    if (err != cudaSuccess) return err;
    void *tmp = reinterpret_cast<void *>(
        (reinterpret_cast<uintptr_t>(alt) + static_cast<size_t>(count) * 4 + 255) &
        ~static_cast<uintptr_t>(255));
    err = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, pos, alt, static_cast<int>(count), 0,
                                         end_bit, st);
    if (err == cudaSuccess) {
        const uint32_t blocks = min((k + 255) / 256, 148u * 8u);
        widen_kernel<<<blocks, 256, 0, st>>>(alt, dst, k);
        err = cudaGetLastError();
        if (launches) *launches += 1 + (end_bit + 7) / 8 + 1;  // histogram + onesweep passes + widen
    }
    cudaError_t e2 = cudaFreeAsync(alt, st);
    return err != cudaSuccess ? err : e2;
}

}  // namespace hc
