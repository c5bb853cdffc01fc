// hc_launch.cu — persistent-grid launches of the search kernels.
#include <mutex>

#include "hc_device.cuh"

namespace hc {

namespace {

// Driver queries cached per (device, kernel): they cost more than a whole large-m search.
// cudaFuncSetAttribute applies to the current device only, so the "limit raised" flag,
// the SM count, the shared-memory limit and the occupancy are all keyed by device.
constexpr int kMaxDev = 16;
struct DevInfo {
    int sms = 0, smem_max = 0;
};
struct AttrKey {
    int dev;
    const void *kern;
};
struct OccKey {
    int dev;
    const void *kern;
    int threads, smem, occ;
};

std::mutex g_mu;
DevInfo g_dev[kMaxDev];
AttrKey g_attr[512];
int g_nattr = 0;
OccKey g_occ[2048];
int g_nocc = 0;

}  // namespace

cudaError_t launch_kernel(const void *kern, void **args, int threads, int smem, long work_units,
                          int max_ctas, int ctas_per_sm, cudaStream_t st, LaunchInfo *li) {
    int dev = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return err;
    if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
    int occ = -1;
    DevInfo di;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        DevInfo &d = g_dev[dev];
        if (d.sms == 0) {
            cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
            cudaDeviceGetAttribute(&d.smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            if (d.sms <= 0) d.sms = 1;
        }
        di = d;
        bool have_attr = false;
        for (int c = 0; c < g_nattr && !have_attr; ++c)
            have_attr = g_attr[c].dev == dev && g_attr[c].kern == kern;
        if (!have_attr) {
            // raise the dynamic shared-memory limit once to the device maximum (less the
            // kernel's static shared memory), so any later size is allowed
            cudaFuncAttributes fa;
            err = cudaFuncGetAttributes(&fa, kern);
            if (err == cudaSuccess)
                err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           d.smem_max - static_cast<int>(fa.sharedSizeBytes));
            if (err != cudaSuccess) {
                if (std::getenv("HC_DEBUG"))
                    std::fprintf(stderr, "libhc: cudaFuncSetAttribute: %s\n", cudaGetErrorName(err));
                return err;
            }
            if (g_nattr < 512) g_attr[g_nattr++] = AttrKey{dev, kern};
        }
        for (int c = 0; c < g_nocc; ++c)
            if (g_occ[c].dev == dev && g_occ[c].kern == kern && g_occ[c].threads == threads &&
                g_occ[c].smem == smem)
                occ = g_occ[c].occ;
    }
    if (smem > di.smem_max) return cudaErrorInvalidValue;
    if (occ < 0) {
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        if (err != cudaSuccess) {
            if (std::getenv("HC_DEBUG"))
                std::fprintf(stderr, "libhc: occupancy(smem=%d): %s\n", smem, cudaGetErrorName(err));
            return err;
        }
        std::lock_guard<std::mutex> lk(g_mu);
        if (g_nocc < 2048) g_occ[g_nocc++] = OccKey{dev, kern, threads, smem, occ};
    }
    if (occ < 1) return cudaErrorInvalidConfiguration;
    if (ctas_per_sm > 0 && occ > ctas_per_sm) occ = ctas_per_sm;
    long grid = static_cast<long>(di.sms) * occ;
    if (grid > work_units) grid = work_units;
    if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
    if (grid < 1) grid = 1;
    err = cudaLaunchKernel(kern, dim3(static_cast<unsigned>(grid)), dim3(threads), args,
                           static_cast<size_t>(smem), st);
    if (li) {
        li->grid = static_cast<int>(grid);
        li->block = threads;
        li->smem = smem;
    }
    return err;
}

}  // namespace hc
