// hc_gather.cu — gather path (HC_PATH_GATHER, the default for shifts S > 32): no
// staging; lanes read only the aligned 8-byte words holding the q-grams they hash
// (ld.global.nc), so HC's sublinear reads stay sublinear in DRAM sectors.
// DESIGN.md 5.
#include "hc_device.cuh"

namespace hc {

struct GatherLayout {
    uint32_t f_off, x_off, bits_off, q_off, q2_off, wbuf_off, bar_off, total;
    uint32_t f_bytes, x_bytes, bits_words;   // bulk-copied F and x, bitmap words
};
__host__ __device__ inline GatherLayout gather_layout(uint32_t alpha, uint32_t m,
                                                      uint32_t nwarps) {
    GatherLayout L;
    L.f_bytes = round_up((1u << alpha) * 4u, 16);
    L.x_bytes = round_up(m + 8, 16);
    L.bits_words = (1u << alpha) / 32 > 4 ? (1u << alpha) / 32 : 4u;
    L.f_off = 0;
    L.x_off = L.f_bytes;
    L.bits_off = L.x_off + L.x_bytes;
    L.q_off = L.bits_off + 4 * L.bits_words;
    L.q2_off = L.q_off + nwarps * kWarpBuf * 4u;
    L.wbuf_off = L.q2_off + nwarps * kWarpBuf * 4u;
    L.bar_off = L.wbuf_off + nwarps * kWarpBuf * 4u;
    L.total = L.bar_off + 16;
    return L;
}

int gather_smem_bytes(uint32_t alpha, uint32_t m) {
    return static_cast<int>(gather_layout(alpha, m, kGatherThreads / 32).total);
}

// One warp's lattice loop.  Chunk c holds the lattice points [c*32L, (c+1)*32L); lane l
// takes points c*32L + u*32 + l, u < L.  The L q-gram loads of a chunk are issued
// together (one DRAM round trip per chunk instead of one per round), and the next
// chunk's loads are issued before this chunk's survivors are handed to the sink
// (first steps / phase B round trips), so they overlap.  The first chunk's loads are
// issued before the table load (`W` comes in loaded).
template <int Q, int SH, class Sink>
__device__ __forceinline__ void gather_loop(const KParams &p, const GlobalText &txt, const FBits &fb,
                                            uint32_t c, uint32_t total_warps, uint32_t lane,
                                            uint32_t L, uint64_t (&W)[4], Sink &sink, uint64_t *bar,
                                            bool &ready) {
    // ONE copy of the loop for L = 1, 2, 4 (rounds u >= L are skipped by warp-uniform tests):
    // three specialised copies tripled the kernel's code, and code size is time here (the
    // kernel runs for 30-60 us and fetches most of its instructions exactly once).
    const uint32_t step = 32 * p.S;
    while (c < p.nchunks) {
        const uint32_t k0 = c * 32 * L;
        const uint32_t pos0 = p.m - 1 + (k0 + lane) * p.S;
        uint32_t pm = 0;                           // bit u: round u's lattice point passes
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u)
            pm |= static_cast<uint32_t>(u < L && k0 + u * 32 + lane < p.K &&
                                        fb.pass(qhash<Q, SH>(W[u], p.mask))) << u;   // l.4-6
        c += total_warps;
        if (c < p.nchunks) {                       // next chunk's loads, before the survivors
            const uint32_t kn = c * 32 * L + lane;
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u)
                if (u < L) W[u] = kn + u * 32 < p.K ? end8<Q>(txt, p.m - 1 + (kn + u * 32) * p.S) : 0ull;
        }
        if (__any_sync(HC_FULL, pm != 0)) {
            if (!ready) {                          // F and x (TMA bulk copy) are needed now
                mbar_wait(bar, 0);
                ready = true;
            }
#pragma unroll 1
            for (uint32_t u = 0; u < L; ++u) {     // one copy of the sink's code
                const bool pass = (pm >> u) & 1u;
                const uint32_t bm = __ballot_sync(HC_FULL, pass);
                if (bm) sink(bm, pass, pos0 + u * step);
            }
        }
    }
}

// Table load: thread 0 starts ONE TMA bulk copy of F and x (complete_tx on an mbarrier),
// the filter bitmap (2^alpha bits) is loaded by the threads in one round trip, and the
// lattice filter runs on the bitmap while F is still in flight; a warp waits for F only
// when it first has survivors.  Every warp waits before the end, so the copy has landed
// before the epilogue reuses the shared memory.
template <int Q, int SH>
// Registers: q-grams of up to 4 bytes hash from one 32-bit half and fit 64 registers, i.e. 4
// CTAs per SM (A/B: C3/C4 m = 128..1024, q = 3 or 4: 7-8% faster than at 80 registers and 3
// CTAs); longer q-grams spill there (C2, q = 6 or 8: 5-11% slower) and get up to 85 (3 CTAs).
__global__ void __launch_bounds__(kGatherThreads, Q <= 4 ? 4 : 3) gather_kernel(const KParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr uint32_t NW = kGatherThreads / 32;
    const GatherLayout Lo = gather_layout(p.alpha, p.m, NW);
    uint32_t *sFp = reinterpret_cast<uint32_t *>(smem + Lo.f_off);
    uint8_t *sx = smem + Lo.x_off;
    uint32_t *sbits = reinterpret_cast<uint32_t *>(smem + Lo.bits_off);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + Lo.bar_off);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (kInstrument && tid == 0) trace_cta(p, 0);
    path_ts(p, 0);
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar, Lo.f_bytes + Lo.x_bytes);
        bulk_g2s(smem_u32(sFp), p.F, Lo.f_bytes, bar);
        bulk_g2s(smem_u32(sx), p.x, Lo.x_bytes, bar);   // x is followed by >= 24 zero bytes
    }
    // the filter bitmap first (its loads must not queue behind the lattice's DRAM misses)
    uint32_t bw = 0;
    if (tid < Lo.bits_words) bw = __ldg(p.Fbits + tid);
    const GlobalText txt = global_text(p);
    const uint32_t total_warps = gridDim.x * NW;
    const uint32_t c0 = blockIdx.x * NW + warp;
    const uint32_t L = p.seg_per_chunk / 32;   // lattice points per lane per chunk: 1, 2 or 4
    // then the first chunk's lattice loads (they overlap the bitmap's round trip)
    uint64_t W[4] = {0ull, 0ull, 0ull, 0ull};
    if (c0 < p.nchunks) {
        const uint32_t kn = c0 * p.seg_per_chunk + lane;
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u)
            if (u < L && kn + u * 32 < p.K) W[u] = end8<Q>(txt, p.m - 1 + (kn + u * 32) * p.S);
    }
    if (tid < Lo.bits_words) sbits[tid] = bw;
    for (uint32_t w = tid + blockDim.x; w < Lo.bits_words; w += blockDim.x) sbits[w] = __ldg(p.Fbits + w);
    if (tid == 0) s_params[0] = p;
    __syncthreads();
    const FTable sF{fence_value(smem_u32(sFp))};
    const FBits fb{fence_value(smem_u32(sbits))};
    WarpOut wo{reinterpret_cast<uint32_t *>(smem + Lo.wbuf_off) + warp * kWarpBuf, 0u};
    WarpQueueSink<Q, SH, GlobalText> sink{p, txt, sF, sx,
                                          reinterpret_cast<uint32_t *>(smem + Lo.q_off) + warp * kWarpBuf,
                                          reinterpret_cast<uint32_t *>(smem + Lo.q2_off) + warp * kWarpBuf,
                                          0u, 0u, wo, lane};
    bool ready = false;
    path_ts(p, 1);
    if (kInstrument && lane == 0) trace_event(p, warp, 0);          // bitmap loaded
    gather_loop<Q, SH>(p, txt, fb, c0, total_warps, lane, L, W, sink, bar, ready);
    path_ts(p, 3);
    if (!ready) mbar_wait(bar, 0);
    path_ts(p, 4);
    if (kInstrument && lane == 0) trace_event(p, warp, 1);          // lattice filtered
    sink.drain();
    path_ts(p, 5);
    if (kInstrument && lane == 0) trace_event(p, warp, 2);          // survivors done
    wo.flush(p, lane);
    path_ts(p, 6);
    if (kInstrument && lane == 0) trace_event(p, warp, 3);          // flushed
    if (kInstrument && lane == 0) trace_cta(p, 1);   // last warp to get here wins
    __syncthreads();
    if (tid == 0) mbar_inval(bar);                 // the epilogue may reuse this memory
    search_epilogue(p, smem);
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
    a.epi_cap = epi_cap_for(smem);
    void *args[] = {&a};
    return launch_kernel(reinterpret_cast<const void *>(kern), args, kGatherThreads, smem, ctas,
                         max_ctas, ctas_per_sm, st, li);
}

}  // namespace hc
