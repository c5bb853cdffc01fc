// hc_launch.cu — host-side launchers of libhc's kernels (grid sizing, attribute and
// occupancy caches) and the result-ordering kernels.
#include <cub/device/device_radix_sort.cuh>

#include <cstdio>
#include <cstdlib>

#include "hc_internal.h"
#include "hc_device.cuh"

namespace hc {

int staged_smem_bytes(uint32_t alpha, uint32_t m, uint32_t stage_bytes, uint32_t stages,
                      uint32_t slot_bytes, uint32_t nbox) {
    return static_cast<int>(
        staged_layout(alpha, m, stage_bytes, stages, kStagedThreads / 32, slot_bytes, nbox).total);
}
int gather_smem_bytes(uint32_t alpha, uint32_t m) {
    return static_cast<int>(gather_layout(alpha, m, kGatherThreads / 32).total);
}

// ------------------------------------------------------------------ launchers
static KernFn pick_kernel(bool staged, uint32_t q, uint32_t s, uint32_t wd) {
    switch (q) {
#define HC_Q_CASE(Q) \
    case Q: return staged ? staged_kernel_q##Q(s, wd) : gather_kernel_q##Q(s, wd);
        HC_Q_CASE(1) HC_Q_CASE(2) HC_Q_CASE(3) HC_Q_CASE(4)
        HC_Q_CASE(5) HC_Q_CASE(6) HC_Q_CASE(7) HC_Q_CASE(8)
#undef HC_Q_CASE
        default: return nullptr;
    }
}

struct KernCache {
    KernFn fn;
    int smem;
    int occ;
};

static cudaError_t launch_common(KernFn kern, const KParams &p, int threads, int smem,
                                 int work_units, int max_ctas, int ctas_per_sm, cudaStream_t st,
                                 LaunchInfo *li) {
    // per-thread caches of the driver queries (they cost more than a whole large-m
    // search): the dynamic shared-memory limit is raised once per kernel to the
    // device maximum (so any later smem size is allowed), occupancy per (kernel, smem)
    static thread_local KernFn attr_set[128];
    static thread_local int nattr = 0;
    static thread_local KernCache cache[256];
    static thread_local int ncache = 0;
    static thread_local int sms = 0, smem_max = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    }
    bool have_attr = false;
    for (int c = 0; c < nattr; ++c) have_attr |= attr_set[c] == kern;
    if (!have_attr) {
        cudaFuncAttributes fa;
        cudaError_t err = cudaFuncGetAttributes(&fa, kern);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_max - static_cast<int>(fa.sharedSizeBytes));
        if (err != cudaSuccess) {
            if (std::getenv("HC_DEBUG"))
                std::fprintf(stderr, "libhc: cudaFuncSetAttribute: %s\n", cudaGetErrorName(err));
            return err;
        }
        if (nattr < 128) attr_set[nattr++] = kern;
    }
    if (smem > smem_max) return cudaErrorInvalidValue;
    int occ = -1;
    for (int c = 0; c < ncache; ++c)
        if (cache[c].fn == kern && cache[c].smem == smem) occ = cache[c].occ;
    if (occ < 0) {
        cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        if (err != cudaSuccess) {
            if (std::getenv("HC_DEBUG"))
                std::fprintf(stderr, "libhc: occupancy(smem=%d): %s\n", smem, cudaGetErrorName(err));
            return err;
        }
        if (ncache < 256) cache[ncache++] = KernCache{kern, smem, occ};
    }
    if (occ < 1) return cudaErrorInvalidConfiguration;
    if (ctas_per_sm > 0 && occ > ctas_per_sm) occ = ctas_per_sm;
    long grid = static_cast<long>(sms) * occ;
    if (grid > work_units) grid = work_units;
    if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
    if (grid < 1) grid = 1;
    kern<<<static_cast<unsigned>(grid), threads, smem, st>>>(p);
    if (li) {
        li->grid = static_cast<int>(grid);
        li->block = threads;
        li->smem = smem;
    }
    return cudaGetLastError();
}

cudaError_t launch_staged(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li) {
    KernFn kern = pick_kernel(true, p.q, p.s, p.Wd);
    if (!kern) return cudaErrorInvalidValue;
    const int smem = staged_smem_bytes(p.alpha, p.m, p.stage_bytes, p.stages, 0, 0);
    return launch_common(kern, p, kStagedThreads, smem, static_cast<int>(p.ntiles), max_ctas,
                         ctas_per_sm, st, li);
}

cudaError_t launch_gather(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li) {
    KernFn kern = pick_kernel(false, p.q, p.s, p.Wd);
    if (!kern) return cudaErrorInvalidValue;
    const int smem = gather_smem_bytes(p.alpha, p.m);
    const int warps_needed = static_cast<int>(p.nchunks);
    const int ctas = (warps_needed + kGatherThreads / 32 - 1) / (kGatherThreads / 32);
    return launch_common(kern, p, kGatherThreads, smem, ctas, max_ctas, ctas_per_sm, st, li);
}

// ------------------------------------------------------------------ ordering
__global__ void widen_kernel(const uint32_t *src, int64_t *dst, uint32_t k) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
        dst[i] = static_cast<int64_t>(src[i]);
}


// One-CTA bitonic sort of sort_cap < count <= kSmallSort distinct positions (1024 threads).
__global__ void __launch_bounds__(1024) small_sort_kernel(const uint32_t *src, uint32_t count,
                                                          int64_t *dst, uint32_t k) {
    __shared__ uint32_t s[kSmallSort];
    uint32_t P = 1;
    while (P < count) P <<= 1;
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) s[i] = i < count ? src[i] : 0xffffffffu;
    __syncthreads();
    for (uint32_t size = 2; size <= P; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                const uint32_t pr = i ^ stride;
                if (pr > i) {
                    const bool asc = (i & size) == 0;
                    const uint32_t a = s[i], b = s[pr];
                    if ((a > b) == asc) {
                        s[i] = b;
                        s[pr] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) dst[i] = static_cast<int64_t>(s[i]);
}

// count > kSmallSort: CUB radix sort on ceil(log2 n) bits, then widen the first k.
cudaError_t sort_large(const uint32_t *pos, uint32_t count, uint32_t n_bound, int64_t *dst,
                       uint32_t k, cudaStream_t st, int *launches) {
    if (count <= kSmallSort) {
        small_sort_kernel<<<1, 1024, 0, st>>>(pos, count, dst, k);
        if (launches) ++*launches;
        return cudaGetLastError();
    }
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
