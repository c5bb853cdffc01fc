// Fixed-cost probes (not part of libhc): what does an event-timed launch cost on this box
// for (a) an empty kernel, (b) an empty kernel with 72 KB of dynamic shared memory on a
// 444-CTA grid, (c) the same ending with a last-CTA ticket, (d) ... plus a write to mapped
// pinned host memory (the way the search kernels publish their count)?
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_empty(uint32_t *ctr, uint32_t *host, int mode) {
    extern __shared__ uint8_t sm[];
    if (mode >= 1) {
        __shared__ uint32_t last;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) last = atomicAdd(ctr, 1u) == gridDim.x - 1;
        __syncthreads();
        if (last && threadIdx.x == 0) {
            ctr[0] = 0;
            if (mode >= 2) host[0] = 1;
            if (mode == 3) ctr[1] = 1;
        }
    }
}

extern "C" int probe_launch(int blocks, int smem, int mode, uint32_t *ctr, uint32_t *host_dev,
                            cudaStream_t st) {
    static bool set = false;
    if (!set) {
        cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        set = true;
    }
    k_empty<<<blocks, 256, smem, st>>>(ctr, host_dev, mode);
    return (int)cudaGetLastError();
}
extern "C" uint32_t *probe_host_alloc(uint32_t **dev) {
    void *h = nullptr, *d = nullptr;
    cudaHostAlloc(&h, 64, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&d, h, 0);
    *dev = (uint32_t *)d;
    return (uint32_t *)h;
}
