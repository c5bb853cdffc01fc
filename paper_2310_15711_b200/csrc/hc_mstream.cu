// hc_mstream.cu — multi-pattern launches of hc_search_batch.
#include "hc_device.cuh"

namespace hc {

// ------------------------------------------------------------------ multi-pattern stream
// one pass over the text for P <= kMaxPat patterns that share (m, q,
// alpha), hence the lattice a_k and the hash of every lattice q-gram (Eq. 3 depends on
// q, s and alpha only).  Each warp stages a chunk once (as on the stream path), hashes
// each lattice q-gram once, and tests it against every pattern's filter (l.6): a
// the patterns' F tables in shared memory.  Each pattern has its own survivor queues,
// output buffer, counter and positions; first steps run on the stage, phase B on
// global text, with pattern i's launch parameters from s_params[i].  (F read through
// L1 from global memory instead measured no faster than separate searches: every
// chunk's survivors then wait on L2 latency, pattern after pattern.)  Every pattern's result is
// exactly its single-pattern search's (each pattern runs Fig. 5 on the same
// segments, R11).
struct MStreamLayout {
    uint32_t f_off, f_words, x_off, x_stride, warp_off, warp_bytes, ring_off, total;
    // per-warp region: [P][kStreamQ1] q1 | [P][kWarpBuf] q2 | [P][kWarpBuf] wbuf |
    //                  [P] ctr | [P][2] state (n2, wcnt)
};
__host__ __device__ inline MStreamLayout mstream_layout(uint32_t alpha, uint32_t m, uint32_t nwarps,
                                                        uint32_t buf_bytes, uint32_t P) {
    MStreamLayout L;
    L.f_off = 0;
    L.f_words = 1u << alpha;
    L.x_off = round_up(P * L.f_words * 4u, 16);
    L.x_stride = round_up(m + 8, 16);
    L.warp_off = round_up(L.x_off + P * L.x_stride, 16);
    L.warp_bytes = round_up(P * (kStreamQ1 + 2 * kWarpBuf) * 4u + P * 12u, 16);
    L.ring_off = round_up(L.warp_off + nwarps * L.warp_bytes + 16, 128);
    L.total = L.ring_off + nwarps * 2 * buf_bytes;   // (host adds the third buffer per warp)
    return L;
}
int mstream_smem_bytes(uint32_t alpha, uint32_t m, uint32_t buf_bytes, uint32_t nwarps, uint32_t npat,
                       uint32_t bufs) {
    return static_cast<int>(mstream_layout(alpha, m, nwarps, buf_bytes, npat).total +
                            (bufs - 2) * nwarps * buf_bytes);
}

template <int Q, int SH>
struct MWarp {   // one warp's per-pattern queues and output state (shared memory)
    uint32_t *q1, *q2, *wbuf, *ctr, *state;
    uint32_t f0, fbytes;   // shared address of pattern 0's F, bytes per F
    __device__ __forceinline__ uint32_t *q1_of(uint32_t i) const { return q1 + i * kStreamQ1; }
    __device__ __forceinline__ uint32_t *q2_of(uint32_t i) const { return q2 + i * kWarpBuf; }
    __device__ __forceinline__ uint32_t *wbuf_of(uint32_t i) const { return wbuf + i * kWarpBuf; }
    // first steps of `cnt` (<= 32) queued survivors of pattern i (entries q1[from ..]) on
    // global text (the queue spans chunks: survivors are drained 32 at a time, so each
    // pattern costs one L2 round trip per 32 survivors, not one per chunk); continuing
    // segments to pattern i's q2 (phase B on global text)
    template <class T>
    __device__ __forceinline__ void steps(uint32_t i, const T &, uint32_t from,
                                          uint32_t cnt, const uint8_t *sx, uint32_t lane) const {
        __syncwarp();
        const bool act = lane < cnt;
        const uint32_t e = act ? q1_of(i)[from + lane] : 0u;
        __syncwarp();
        const KParams &pp = s_params[i];
        const FTable ft{f0 + i * fbytes};
        const GlobalText gtxt = global_text(pp);
        WarpOut wo{wbuf_of(i), state[2 * i + 1]};
        WarpQueueSink<Q, SH, GlobalText> sink{pp, gtxt, ft, sx, nullptr, q2_of(i),
                                              0u, state[2 * i], wo, lane, i};
        sink.steps_e_on(gtxt, act, e);
        __syncwarp();
        if (lane == 0) {
            state[2 * i] = sink.n2;
            state[2 * i + 1] = wo.cnt;
        }
        __syncwarp();
    }
};

template <int Q, int SH, class T>
__device__ __forceinline__ void mstream_filter(const KParams &p, const T &txt, uint32_t P,
                                               uint32_t k0, uint32_t k1, uint32_t lane,
                                               const MWarp<Q, SH> &mw, const uint8_t *sx0,
                                               uint32_t xs) {
    const uint32_t step = 32 * p.S;
    const uint32_t pos0 = p.m - 1 + k0 * p.S;         // a_k0: readable in this chunk
    uint32_t pos = pos0 + lane * p.S;                 // a_k of lattice point k0 + lane
    uint32_t k = k0;
    while (k < k1) {
        // trips until some pattern's queue holds 32; past k1 (the last trip) the loads
        // are redirected to a_k0 and the tests masked, so no load sits in a branch
        uint32_t full = 0;
        while (k < k1 && !full) {
            uint32_t v[kStreamUnroll];
            bool in[kStreamUnroll];
#pragma unroll
            for (int u = 0; u < kStreamUnroll; ++u) {
                in[u] = k + u * 32 + lane < k1;
                v[u] = qhash<Q, SH>(end8<Q>(txt, in[u] ? pos + u * step : pos0), p.mask);
            }
#pragma unroll
            for (int i = 0; i < kMaxPat; ++i) {
                if (i < static_cast<int>(P)) {
                    const FTable ft{mw.f0 + i * mw.fbytes};
                    uint32_t pm = 0;
#pragma unroll
                    for (int u = 0; u < kStreamUnroll; ++u)
                        pm |= static_cast<uint32_t>(in[u] && ft.pass(v[u])) << u;
                    const uint32_t c = __popc(pm);
                    if (__reduce_add_sync(HC_FULL, c)) {
                        if (c) {
                            uint32_t slot = atomicAdd(mw.ctr + i, c);
#pragma unroll
                            for (int u = 0; u < kStreamUnroll; ++u)
                                if ((pm >> u) & 1u) mw.q1_of(i)[slot++] = pos + u * step;
                        }
                        __syncwarp();
                        full |= static_cast<uint32_t>(ld_volatile_shared(mw.ctr + i) >= 32) << i;
                    }
                }
            }
            k += 32 * kStreamUnroll;
            pos += kStreamUnroll * step;
        }
        // drain the full queues, 32 survivors at a time (first steps on the stage)
#pragma unroll
        for (int i = 0; i < kMaxPat; ++i) {
            if ((full >> i) & 1u) {
                uint32_t n1 = ld_volatile_shared(mw.ctr + i);
                while (n1 >= 32) {
                    n1 -= 32;
                    mw.steps(i, txt, n1, 32, sx0 + i * xs, lane);
                    if (lane == 0) st_volatile_shared(mw.ctr + i, n1);
                    __syncwarp();
                }
            }
        }
    }
}

template <int Q, int SH, int NB>
__device__ __forceinline__ void mstream_loop(const KParams &p, uint32_t P, const MWarp<Q, SH> &mw,
                                             const uint8_t *sx0, uint32_t xs, uint32_t bufs0,
                                             uint32_t gw, uint32_t total_warps, uint32_t lane) {
    const uint32_t y32 = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p.y));
#pragma unroll
    for (int b = 0; b < NB - 1; ++b) stream_issue(p, gw + b * total_warps, bufs0 + b * p.stage_bytes, lane);
    uint32_t b = 0;
    for (uint32_t c = gw; c < p.nchunks; c += total_warps) {
        const uint32_t bn = b == 0 ? NB - 1 : b - 1;
        stream_issue(p, c + (NB - 1) * total_warps, bufs0 + bn * p.stage_bytes, lane);
        cp_async_wait<NB - 1>();
        __syncwarp();
        const StreamChunk g = stream_chunk(p, c);
        const uint32_t buf = fence_value(bufs0 + b * p.stage_bytes);
        const SmemText txt{buf + ((y32 + g.first) & 15u) - g.first};
        mstream_filter<Q, SH, SmemText>(p, txt, P, g.k0, g.k1, lane, mw, sx0, xs);
        __syncwarp();
        b = b + 1 == NB ? 0 : b + 1;
    }
    cp_async_wait<0>();
}

template <int Q, int SH>
// Shared memory limits this kernel to <= 512 threads per SM (one 16-warp CTA, or two 8-warp
// CTAs), so it may use up to 128 registers: at the default 64 it spilled 260 B per thread.
__global__ void __launch_bounds__(2 * kStreamMaxThreads, 1) mstream_kernel(const KParams p, const MParams mp) {
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t NW = blockDim.x / 32;
    const uint32_t P = mp.npat;
    const MStreamLayout L = mstream_layout(p.alpha, p.m, NW, p.stage_bytes, P);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    pdl_launch_dependents();
    if (tid < P) {
        KParams q = p;
        q.F = mp.F[tid];
        q.x = mp.x[tid];
        q.hv = mp.hv[tid];
        q.counter = mp.counter[tid];
        q.out = mp.out[tid];
        q.cap = mp.cap[tid];
        s_params[tid] = q;
    }
    // every pattern's F and x
    uint32_t *sF = reinterpret_cast<uint32_t *>(smem + L.f_off);
    if (L.f_words >= 4) {
        // 16-byte loads, four in flight per thread (F of every pattern)
        const uint32_t per = L.f_words / 4, tot4 = P * per;
        uint4 *dst = reinterpret_cast<uint4 *>(sF);
        for (uint32_t w0 = tid; w0 < tot4; w0 += 4 * blockDim.x) {
            uint4 v[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint32_t w = w0 + r * blockDim.x;
                if (w < tot4) v[r] = __ldg(reinterpret_cast<const uint4 *>(mp.F[w / per]) + w % per);
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint32_t w = w0 + r * blockDim.x;
                if (w < tot4) dst[w] = v[r];
            }
        }
    } else {
        for (uint32_t w = tid; w < P * L.f_words; w += blockDim.x)
            sF[w] = __ldg(mp.F[w / L.f_words] + w % L.f_words);
    }
    uint8_t *sx0 = smem + L.x_off;
    for (uint32_t i = 0; i < P; ++i) {
        for (uint32_t t = tid; t < p.m; t += blockDim.x) sx0[i * L.x_stride + t] = __ldg(mp.x[i] + t);
        if (tid < 8) sx0[i * L.x_stride + p.m + tid] = 0;
    }
    uint8_t *wr = smem + L.warp_off + warp * L.warp_bytes;
    MWarp<Q, SH> mw;
    mw.q1 = reinterpret_cast<uint32_t *>(wr);
    mw.q2 = mw.q1 + P * kStreamQ1;
    mw.wbuf = mw.q2 + P * kWarpBuf;
    mw.ctr = mw.wbuf + P * kWarpBuf;
    mw.state = mw.ctr + P;
    mw.f0 = smem_u32(sF);
    mw.fbytes = L.f_words * 4u;
    if (lane < P) {
        mw.ctr[lane] = 0;
        mw.state[2 * lane] = 0;
        mw.state[2 * lane + 1] = 0;
    }
    __syncthreads();
    mw.f0 = fence_value(mw.f0);
    const uint32_t total_warps = gridDim.x * NW;
    const uint32_t gw = blockIdx.x * NW + warp;
    const uint32_t bufs0 = smem_u32(smem + L.ring_off) + warp * p.stages * p.stage_bytes;
    if (p.mgather) {
        // large shifts: no staging, the lattice q-grams are read from global memory (the
        // gather path's access), hashed once and tested against every pattern: the
        // patterns share the DRAM sectors the lattice touches
        const GlobalText gtxt = global_text(p);
        for (uint32_t c = gw; c < p.nchunks; c += total_warps) {
            const uint32_t k0 = c * p.seg_per_chunk;
            mstream_filter<Q, SH, GlobalText>(p, gtxt, P, k0, min(k0 + p.seg_per_chunk, p.K), lane, mw,
                                              sx0, L.x_stride);
        }
    } else   // two buffers per warp (one loop variant: code size is time)
        mstream_loop<Q, SH, 2>(p, P, mw, sx0, L.x_stride, bufs0, gw, total_warps, lane);
    // queued survivors, phase B leftovers and output buffers of every pattern
    __syncwarp();
    for (uint32_t i = 0; i < P; ++i) {
        const uint32_t n1 = ld_volatile_shared(mw.ctr + i);
        if (n1) mw.steps(i, SmemText{0u}, 0, n1, sx0 + i * L.x_stride, lane);
    }
    for (uint32_t i = 0; i < P; ++i) {
        const KParams &pp = s_params[i];
        const FTable ft{mw.f0 + i * mw.fbytes};
        const GlobalText gtxt = global_text(pp);
        WarpOut wo{mw.wbuf_of(i), mw.state[2 * i + 1]};
        WarpQueueSink<Q, SH, GlobalText> sink{pp, gtxt, ft, sx0 + i * L.x_stride, nullptr,
                                              mw.q2_of(i), 0u, mw.state[2 * i], wo, lane, i};
        sink.drain();
        wo.flush(pp, lane);
    }
    // fused epilogue: the last CTA publishes and orders every pattern's positions
    if (cta_is_last(mp.counter[0] + 2)) {
        for (uint32_t i = 0; i < P; ++i) {
            const uint32_t cnt_i = *reinterpret_cast<volatile uint32_t *>(mp.counter[i]);
            const uint32_t pos0_i = *reinterpret_cast<volatile uint32_t *>(mp.counter[i] + 4);
            publish_search(mp.counter[i], mp.out[i], mp.cap[i], mp.host_count[i], mp.dst[i],
                           mp.k_out[i], p.epi_cap, smem, p.debug == 9, p.nbits, cnt_i, pos0_i);
            __syncthreads();
        }
        if (tid == 0) mp.counter[0][2] = 0;
    }
}

template <int Q, int SH>
struct PickMStream {
    using Fn = void (*)(const KParams, const MParams);
    static Fn fn() { return mstream_kernel<Q, SH>; }
};

cudaError_t launch_mstream(const KParams &p, const MParams &mp, cudaStream_t st, int max_ctas,
                           int ctas_per_sm, LaunchInfo *li) {
    auto kern = pick<PickMStream>(p.q, p.s);
    if (!kern) return cudaErrorInvalidValue;
    const uint32_t nw = p.block_warps;
    const int smem = mstream_smem_bytes(p.alpha, p.m, p.stage_bytes, nw, mp.npat, p.stages);
    const long ctas = (p.nchunks + nw - 1) / nw;
    KParams a = p;
    a.epi_cap = epi_cap_for(smem);
    MParams b = mp;
    void *args[] = {&a, &b};
    return launch_kernel(reinterpret_cast<const void *>(kern), args, static_cast<int>(32 * nw), smem,
                         ctas, max_ctas, ctas_per_sm, st, li);
}

}  // namespace hc
