// hc_gather.cu — gather path (HC_PATH_GATHER, the default for shifts S > 32): no
// staging; lanes read only the aligned 8-byte words holding the q-grams they hash
// (ld.global.nc), so HC's sublinear reads stay sublinear in DRAM sectors.
// DESIGN.md 5.
#include "hc_device.cuh"

namespace hc {

struct GatherLayout {
    uint32_t f_off, x_off, q_off, q2_off, wbuf_off, total;
};
__host__ __device__ inline GatherLayout gather_layout(uint32_t alpha, uint32_t m,
                                                      uint32_t nwarps) {
    GatherLayout L;
    L.f_off = 0;
    L.x_off = round_up((1u << alpha) * 4u, 16);
    L.q_off = L.x_off + round_up(m + 8, 16);
    L.q2_off = L.q_off + nwarps * kWarpBuf * 4u;
    L.wbuf_off = L.q2_off + nwarps * kWarpBuf * 4u;
    L.total = L.wbuf_off + nwarps * kWarpBuf * 4u;
    return L;
}

int gather_smem_bytes(uint32_t alpha, uint32_t m) {
    return static_cast<int>(gather_layout(alpha, m, kGatherThreads / 32).total);
}

template <int Q, int SH>
__global__ void __launch_bounds__(kGatherThreads) gather_kernel(const KParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr uint32_t NW = kGatherThreads / 32;
    const GatherLayout L = gather_layout(p.alpha, p.m, NW);
    uint32_t *sFp = reinterpret_cast<uint32_t *>(smem + L.f_off);
    uint8_t *sx = smem + L.x_off;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (kInstrument && tid == 0) trace_cta(p, 0);
    pdl_launch_dependents();
    load_table(p, sFp, sx);
    if (tid == 0) s_params[0] = p;
    __syncthreads();
    const FTable sF{fence_value(smem_u32(sFp))};
    WarpOut wo{reinterpret_cast<uint32_t *>(smem + L.wbuf_off) + warp * kWarpBuf, 0u};
    const GlobalText txt{p.y};
    WarpQueueSink<Q, SH, GlobalText> sink{p, txt, sF, sx,
                                          reinterpret_cast<uint32_t *>(smem + L.q_off) + warp * kWarpBuf,
                                          reinterpret_cast<uint32_t *>(smem + L.q2_off) + warp * kWarpBuf,
                                          0u, 0u, wo, lane};
    const uint32_t total_warps = gridDim.x * NW;
    if (kInstrument && warp == 0 && lane == 0) trace_event(p, 0, 0);          // table loaded
    for (uint32_t c = blockIdx.x * NW + warp; c < p.nchunks; c += total_warps) {
        const uint32_t seg_lo = c * p.seg_per_chunk;
        const uint32_t seg_hi = min(seg_lo + p.seg_per_chunk, p.K);
        filter_lattice<Q, SH>(p, txt, sF, seg_lo, seg_hi, lane, sink);
    }
    if (kInstrument && warp == 0 && lane == 0) trace_event(p, 0, 1);          // lattice filtered
    sink.drain();
    if (kInstrument && warp == 0 && lane == 0) trace_event(p, 0, 2);          // survivors done
    wo.flush(p, lane);
    if (kInstrument && lane == 0) trace_cta(p, 1);   // last warp to get here wins
}

template <int Q, int SH>
struct PickGather {
    using Fn = KernFn;
    static KernFn fn() { return gather_kernel<Q, SH>; }
};

cudaError_t launch_gather(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li) {
    KernFn kern = pick<PickGather>(p.q, p.s);
    if (!kern) return cudaErrorInvalidValue;
    const int smem = gather_smem_bytes(p.alpha, p.m);
    const long ctas = (static_cast<long>(p.nchunks) + kGatherThreads / 32 - 1) / (kGatherThreads / 32);
    KParams a = p;
    void *args[] = {&a};
    return launch_kernel(reinterpret_cast<const void *>(kern), args, kGatherThreads, smem, ctas,
                         max_ctas, ctas_per_sm, st, li);
}

}  // namespace hc
