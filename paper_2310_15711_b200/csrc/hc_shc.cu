// hc_shc.cu — SHC path (HC_PATH_SHC): the Sentinel Hash Chain of Fig. 5
// right run per lane on shared-memory boxes that carry their own sentinel.
#include "hc_device.cuh"

namespace hc {

int shc_smem_bytes(uint32_t alpha, uint32_t m, uint32_t buf_bytes, uint32_t box_bytes,
                   uint32_t nwarps) {
    const uint32_t x_off = round_up((1u << alpha) * 4u, 16);
    const uint32_t ring_off = round_up(x_off + round_up(m + 8, 16) + 16, 128);
    return static_cast<int>(ring_off + nwarps * 2 * buf_bytes + nwarps * 32 * box_bytes);
}

// ------------------------------------------------------------------ SHC kernel
// Sentinel Hash Chain (Fig. 5 right; optimisation 3) on the GPU.
// SHC copies x after the end of y (l.2-3) so that its fast loop (l.6-7: shift while
// F[v] == 0) needs no position test; the test moves after the loop (l.8).  Here the
// "text" of each lane is its own range of c = seg_per_chunk / 32 consecutive segments
// (window ends [a_kL, b_L), b_L = min(a_{kL+c}, n)): the lane copies the bytes
// [a_kL - m + 1, b_L - 1] from the warp's staged chunk into its own shared-memory box
// and writes x right after them (its sentinel), then runs SHC on the box with b_L in
// the role of n.  By R11 (segmented runs are exact) the lane reports exactly the
// occurrences ending in [a_kL, b_L).  Termination of the fast loop: the window ends it
// visits past b_L - 1 step by S, so one of them falls in [b_L + q - 1, b_L + m - 1]
// (an interval of S ends); that window's q-gram lies inside the sentinel copy of x,
// and every q-gram of x has F != 0 (Fig. 3), so the loop stops there at the latest.
// Every lane runs its own loop (divergent, one window at a time): this is the
// per-lane sequential skip loop of SURVEY 8(a) "window scan", measured against the
// lattice filter of the stream path.  Matches: one global atomicAdd each.
__device__ __forceinline__ void shc_output(const KParams &p, uint32_t pos) {
    const uint32_t slot = atomicAdd(p.counter, 1u);
    if (slot < p.cap) p.out[slot] = pos;
    if (slot == 0) p.counter[4] = pos;   // the first slot's position (epilogue)
}

template <int Q, int SH>
__device__ __forceinline__ void shc_lane(const KParams &p, const SmemText &bx, const FTable &sF,
                                         const uint8_t *sx, uint32_t j, uint32_t b) {
    const uint32_t S = p.S;
    while (true) {
        // l.6-7: the fast loop, no position test (the sentinel stops it)
        uint32_t v = qhash<Q, SH>(end8<Q>(bx, j), p.mask);
        uint32_t z = sF[v];
        while (z == 0u) {
            j += S;
            v = qhash<Q, SH>(end8<Q>(bx, j), p.mask);
            z = sF[v];
        }
        if (j >= b) return;                                  // l.8
        const uint32_t e = j;                                // l.9-10: v, z of window e
        const uint32_t i = j + 2 * Q - p.m;                  // l.11 (j >= m - 1 >= ... )
        bool broke = false;
        while (j >= i) {                                     // l.12
            j -= Q;                                          // l.13
            v = qhash<Q, SH>(end8<Q>(bx, j), p.mask);         // l.14
            if ((z & (1u << (v & (kWordBits - 1)))) == 0u) { // l.15-16
                broke = true;
                break;
            }
            z = sF[v];                                       // l.17
        }
        if (!broke) {                                        // l.18-21, index per R1
            j = e + Q - p.m;   // = i - q (then j + S = e + 1)
            if (v == p.hv && verify(bx, sx, e + 1 - p.m, p.m)) shc_output(p, e + 1 - p.m);
        }
        j += S;                                              // l.22
    }
}

template <int Q, int SH>
__global__ void __launch_bounds__(kStreamMaxThreads) shc_kernel(const KParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t NW = blockDim.x / 32;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // F | x | per-warp stage ring | per-lane boxes
    const uint32_t x_off = round_up((1u << p.alpha) * 4u, 16);
    const uint32_t ring_off = round_up(x_off + round_up(p.m + 8, 16) + 16, 128);
    const uint32_t box_off = ring_off + NW * p.stages * p.stage_bytes;
    uint32_t *sFp = reinterpret_cast<uint32_t *>(smem);
    uint8_t *sx = smem + x_off;
    pdl_launch_dependents();
    const uint32_t total_warps = gridDim.x * NW;
    const uint32_t gw = blockIdx.x * NW + warp;
    const uint32_t bufs0 = smem_u32(smem + ring_off) + warp * p.stages * p.stage_bytes;
    const uint32_t box = smem_u32(smem + box_off) + (warp * 32 + lane) * p.slot_bytes;
    load_table(p, sFp, sx);
    if (tid == 0) s_params[0] = p;
    __syncthreads();
    const FTable sF{fence_value(smem_u32(sFp))};
    const uint32_t y32 = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p.y));
    const uint32_t c_lane = p.seg_per_chunk / 32;             // segments per lane
    constexpr int NB = 2;
    stream_issue(p, gw, bufs0, lane);
    uint32_t bsel = 0;
    for (uint32_t c = gw; c < p.nchunks; c += total_warps) {
        const uint32_t bn = bsel ^ 1u;
        stream_issue(p, c + total_warps, bufs0 + bn * p.stage_bytes, lane);
        cp_async_wait<NB - 1>();
        __syncwarp();
        const StreamChunk g = stream_chunk(p, c);
        const uint32_t buf = fence_value(bufs0 + bsel * p.stage_bytes);
        const uint32_t base = buf + ((y32 + g.first) & 15u) - g.first;   // text p at base + p
        const uint32_t kL = g.k0 + lane * c_lane;
        if (kL < g.k1) {
            const uint32_t aL = p.m - 1 + kL * p.S;
            const uint32_t bL = min(p.m - 1 + min(kL + c_lane, g.k1) * p.S, p.n);
            // box: bytes [aL - m + 1, bL) in whole 16-byte words (alignment kept), then x
            const uint32_t lo = aL + 1 - p.m;
            const uint32_t s0 = (base + lo) & ~15u, s1 = (base + bL + 15) & ~15u;
            for (uint32_t a = s0, d = box; a < s1; a += 16, d += 16) sts128(d, lds128(a));
            const uint32_t bbase = box - (s0 - base);                        // text p at bbase + p
            for (uint32_t t = 0; t < p.m; ++t)                                 // l.2-3: the sentinel
                asm volatile("st.shared.u8 [%0], %1;" ::"r"(bbase + bL + t), "r"(static_cast<uint32_t>(sx[t]))
                             : "memory");
            shc_lane<Q, SH>(p, SmemText{bbase}, sF, sx, aL, bL);
        }
        __syncwarp();
        bsel = bn;
    }
    cp_async_wait<0>();
    search_epilogue(p, smem);
}

template <int Q, int SH>
struct PickShc {
    using Fn = KernFn;
    static KernFn fn() { return shc_kernel<Q, SH>; }
};

cudaError_t launch_shc(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                       LaunchInfo *li) {
    KernFn kern = pick<PickShc>(p.q, p.s);
    if (!kern) return cudaErrorInvalidValue;
    const uint32_t nw = p.block_warps;
    const int smem = shc_smem_bytes(p.alpha, p.m, p.stage_bytes, p.slot_bytes, nw);
    const long ctas = (p.nchunks + nw - 1) / nw;
    KParams a = p;
    a.epi_cap = epi_cap_for(smem);
    void *args[] = {&a};
    return launch_kernel(reinterpret_cast<const void *>(kern), args, static_cast<int>(32 * nw), smem,
                         ctas, max_ctas, ctas_per_sm, st, li);
}

}  // namespace hc
