// Isolated timing of the epilogue's block_order (hc_device.cuh): one CTA orders `count`
// keys; compared with the same call inside the search kernel's last CTA.
#include "hc_device.cuh"

__global__ void probe_kernel(const uint32_t *pos, uint32_t count, int64_t *dst, unsigned long long *t) {
    extern __shared__ __align__(128) uint8_t smem[];
    unsigned long long t0 = clock64();
    bool ok = hc::block_order(pos, count, dst, count, smem);
    __syncthreads();
    if (threadIdx.x == 0) { t[0] = clock64() - t0; t[1] = ok; }
}

extern "C" int probe_order(const uint32_t *pos, uint32_t count, int64_t *dst, unsigned long long *t,
                           int threads, int smem) {
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe_kernel<<<1, threads, smem>>>(pos, count, dst, t);
    return (int)cudaDeviceSynchronize();
}
