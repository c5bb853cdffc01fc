// hc_stream.cu — stream path (HC_PATH_STREAM, the default for shifts S <= 32): one CTA of
// up to 24 warps per SM; per-warp chunks staged in shared memory by one 1-D TMA bulk copy
// each; lattice filter on the stage against per-lane copies of the filter bitmap; survivors
// through first steps and phase B on global text; final drain on private boxes.  DESIGN.md 5.
#include "hc_device.cuh"

namespace hc {

// ------------------------------------------------------------------ stream kernel
// Small shifts (S <= 32), every text sector is read (f(m) = 1).  Each warp
// owns a contiguous run of segments per chunk and stages the chunk's lattice q-gram bytes
// (plus those of the first steps) into its own shared-memory buffer, one chunk ahead of the
// one it filters: no CTA-wide barrier, no hand-off between warps.  Phase A reads the
// buffer; the lattice survivors go through first_steps and phase B on global text
// (the chunk was just streamed through L2), exactly as on the gather path.
struct StreamLayout {
    uint32_t f_off, bits_off, x_off, q_off, q2_off, wbuf_off, ctr_off, buf_off, total;
};
__host__ __device__ inline StreamLayout stream_layout(uint32_t alpha, uint32_t m, uint32_t nwarps,
                                                      uint32_t buf_bytes, uint32_t bufs,
                                                      uint32_t lane_bits) {
    StreamLayout L;
    L.f_off = 0;
    L.bits_off = round_up((1u << alpha) * 4u, 16);
    // the filter bitmap: one copy per lane (2^alpha words, at least one word each) or one copy
    L.x_off = L.bits_off + (lane_bits ? max((1u << alpha) * 4u, 128u) : max((1u << alpha) / 8u, 16u));
    L.q_off = L.x_off + round_up(m + 8, 16);
    L.q2_off = L.q_off + nwarps * kStreamQ1 * 4u;
    L.wbuf_off = L.q2_off + nwarps * kWarpBuf * 4u;
    L.ctr_off = L.wbuf_off + nwarps * kWarpBuf * 4u;
    // per-warp counters, then 4 mbarriers per warp (TMA variant)
    L.buf_off = round_up(round_up(L.ctr_off + nwarps * 4u, 8) + nwarps * 32u + 16, 128);
    L.total = L.buf_off + nwarps * bufs * buf_bytes;
    return L;
}
int stream_smem_bytes(uint32_t alpha, uint32_t m, uint32_t buf_bytes, uint32_t bufs,
                      uint32_t nwarps, uint32_t lane_bits) {
    return static_cast<int>(stream_layout(alpha, m, nwarps, buf_bytes, bufs, lane_bits).total);
}

// Phase A of the stream path over lattice points [k0, k1) of a staged chunk: the same
// l.4-6 test as filter_lattice, but the survivors are appended to a per-warp queue
// (q1, count n1, shared slot counter ctr) with one shared atomic per lane that has
// any, and the queue is drained (first_steps, phase B: calls) only between runs of
// trips, so the trip loop has no call in it and keeps its state in registers.
template <int Q, int SH>
struct StreamQueue {
    uint32_t *q1;     // kStreamQ1 window ends a_k
    uint32_t *ctr;    // shared slot counter (= n1 between trips)
    uint32_t n1;      // warp-uniform count
    // first steps of up to 32 queued survivors (the last ones queued), on global text (the
    // chunk was just streamed through L2; the queue spans chunks, so every batch but the
    // last is full)
    __device__ __forceinline__ void drain32(WarpQueueSink<Q, SH, GlobalText, FTable> &sink,
                                            uint32_t lane) {
        __syncwarp();
        const uint32_t cnt = min(n1, 32u);
        const bool act = lane < cnt;
        const uint32_t e = act ? q1[n1 - cnt + lane] : 0u;
        n1 -= cnt;
        __syncwarp();
        if (lane == 0) *ctr = n1;
        __syncwarp();
        sink.steps_e(act, e);
    }
    __device__ __forceinline__ void drain_all(WarpQueueSink<Q, SH, GlobalText, FTable> &sink,
                                              uint32_t lane) {
#pragma unroll 1
        while (n1) drain32(sink, lane);
    }
};

template <int Q, int SH>
__device__ __forceinline__ void stream_filter(const KParams &p, const SmemText &txt, const PassBits &sF,
                                              uint32_t k0, uint32_t k1, uint32_t lane,
                                              StreamQueue<Q, SH> &qu,
                                              WarpQueueSink<Q, SH, GlobalText, FTable> &sink) {
    const uint32_t step = 32 * p.S;
    uint32_t pos = p.m - 1 + (k0 + lane) * p.S;   // window end a_k of lattice point k0 + lane
    uint32_t k = k0;
    while (true) {
        while (k + 32 * kStreamUnroll <= k1 && qu.n1 < 32) {
            uint64_t W[kStreamUnroll];
#pragma unroll
            for (int u = 0; u < kStreamUnroll; ++u) W[u] = end8<Q>(txt, pos + u * step);
            uint32_t pm = 0;
#pragma unroll
            for (int u = 0; u < kStreamUnroll; ++u)
                pm |= static_cast<uint32_t>(sF.pass(qhash<Q, SH>(W[u], p.mask))) << u;
            if (kInstrument && p.debug == 3) pm = 0;   // phase A alone (measurement)
            if (__any_sync(HC_FULL, pm != 0)) {
                const uint32_t c = __popc(pm);
                const uint32_t tot = __reduce_add_sync(HC_FULL, c);
                if (c) {
                    // one store in the common case (a lane rarely has two passes in a trip)
                    uint32_t slot = atomicAdd(qu.ctr, c);
                    uint32_t rest = pm;
#pragma unroll 1
                    do {
                        const uint32_t u = __ffs(rest) - 1;
                        qu.q1[slot++] = pos + u * step;
                        rest &= rest - 1;
                    } while (rest);
                }
                qu.n1 += tot;
            }
            k += 32 * kStreamUnroll;
            pos += kStreamUnroll * step;
        }
        if (qu.n1 < 32) break;
        qu.drain32(sink, lane);
    }
    // ragged tail, one round at a time; no drain here (the queue holds 32 * (unroll + 1):
    // < 32 on entry plus fewer than `unroll` rounds), the next chunk's loop drains first
    for (; k < k1; k += 32, pos += step) {
        const bool in = k + lane < k1;
        const bool pass = in && sF.pass(qhash<Q, SH>(end8<Q>(txt, pos), p.mask));
        const uint32_t bm = __ballot_sync(HC_FULL, pass);
        if (bm) {
            if (pass) qu.q1[qu.n1 + __popc(bm & lanemask_lt())] = pos;
            qu.n1 += __popc(bm);
            __syncwarp();
            if (lane == 0) *qu.ctr = qu.n1;
        }
    }
}

// Each chunk is moved by ONE 1-D bulk copy (cp.async.bulk, issued
// by lane 0, completion on the buffer's mbarrier).  Interior chunks (all but the first and
// the last few of the text) have a fixed geometry: chunk c holds lattice points
// [c spc, (c+1) spc) and text bytes [first, first + D + max(q, 2q - S)), first = c D + m - 2q,
// D = spc S (stream_chunk's range, unclipped), so the loop only advances `first`; their 16-byte words lie wholly inside y.  Edge chunks
// take the general route (stream_chunk; the partial 16-byte words at the two ends of an
// unaligned text are stored by the lanes).
struct TmaStream {
    uintptr_t y;
    uint32_t y32, D, len, bufs0, stage_bytes;
    uint64_t *bar;
};
__device__ __forceinline__ bool chunk_interior(const KParams &p, const TmaStream &ts, uint32_t c,
                                               uint32_t first) {
    return c >= 1 && first + ts.len + 15 <= p.n;
}
__device__ __forceinline__ void tma_issue(const KParams &p, const TmaStream &ts, uint32_t c,
                                          uint32_t first, uint32_t b, uint32_t lane) {
    if (c >= p.nchunks) return;
    const uint32_t buf = ts.bufs0 + b * ts.stage_bytes;
    if (chunk_interior(p, ts, c, first)) {
        if (lane == 0) {
            const uintptr_t A = (ts.y + first) & ~static_cast<uintptr_t>(15);
            const uint32_t bytes = (((ts.y32 + first) & 15u) + ts.len + 15u) & ~15u;
            chk_text_range(p.y, p.n, A, bytes);
            mbar_arrive_expect_tx(&ts.bar[b], bytes);
            bulk_g2s(buf, reinterpret_cast<const void *>(A), bytes, &ts.bar[b]);
        }
        return;
    }
    const uintptr_t y = ts.y, ye = y + p.n;
    const StreamChunk g = stream_chunk(p, c);
    const uintptr_t A = (y + g.first) & ~static_cast<uintptr_t>(15);
    const uint32_t nbytes = static_cast<uint32_t>(((y + g.last + 16) & ~static_cast<uintptr_t>(15)) - A);
    const uintptr_t lo = max(A, (y + 15) & ~static_cast<uintptr_t>(15));
    const uintptr_t hi = min(A + nbytes, ye & ~static_cast<uintptr_t>(15));
    if (A < lo || A + nbytes > hi) {                 // bytes outside [lo, hi)
        for (uintptr_t a = A + lane; a < A + nbytes; a += 32)
            if ((a < lo || a >= hi) && a >= y && a < ye)
                asm volatile("st.shared.u8 [%0], %1;" ::"r"(buf + static_cast<uint32_t>(a - A)),
                             "r"(static_cast<uint32_t>(__ldg(reinterpret_cast<const uint8_t *>(a))))
                             : "memory");
    }
    __syncwarp();
    if (lane == 0) {
        fence_proxy_async();                         // the lanes' stores above
        if (hi > lo) {
            chk_text_range(p.y, p.n, lo, static_cast<uint32_t>(hi - lo));
            mbar_arrive_expect_tx(&ts.bar[b], static_cast<uint32_t>(hi - lo));
            bulk_g2s(buf + static_cast<uint32_t>(lo - A), reinterpret_cast<const void *>(lo),
                     static_cast<uint32_t>(hi - lo), &ts.bar[b]);
        } else {
            mbar_arrive(&ts.bar[b]);
        }
    }
}
template <int NB>
__device__ __forceinline__ void stream_prologue_tma(const KParams &p, const TmaStream &ts, uint32_t gw,
                                                    uint32_t total_warps, uint32_t lane) {
    if (lane == 0) {
        for (int b = 0; b < NB; ++b) mbar_init(&ts.bar[b], 1);
        fence_mbar_init();
    }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < NB - 1; ++b) {
        const uint32_t c = gw + b * total_warps;
        tma_issue(p, ts, c, c * ts.D + p.m - 2 * p.q, b, lane);
    }
}
template <int Q, int SH, int NB>
__device__ __forceinline__ void stream_loop_tma(const KParams &p, const PassBits &sF,
                                                WarpQueueSink<Q, SH, GlobalText, FTable> &sink,
                                                StreamQueue<Q, SH> &qu, const TmaStream &ts,
                                                uint32_t gw, uint32_t total_warps, uint32_t lane) {
    const uint32_t stride = total_warps * ts.D;
    uint32_t first = gw * ts.D + p.m - 2 * p.q;       // of chunk c when interior (mod 2^32)
    uint32_t b = 0, par = 0;   // par: bit b = phase parity of buffer b's next completion
    for (uint32_t c = gw; c < p.nchunks; c += total_warps, first += stride) {
        const uint32_t bn = b == 0 ? NB - 1 : b - 1;
        tma_issue(p, ts, c + (NB - 1) * total_warps, first + (NB - 1) * stride, bn, lane);
        mbar_wait(&ts.bar[b], (par >> b) & 1u);
        par ^= 1u << b;
        const uint32_t buf = fence_value(ts.bufs0 + b * ts.stage_bytes);
        if (!(kInstrument && p.debug == 1)) {   // debug 1: copy pipeline alone
            uint32_t k0 = c * p.seg_per_chunk, k1 = k0 + p.seg_per_chunk, f = first;
            if (!chunk_interior(p, ts, c, first)) {
                const StreamChunk g = stream_chunk(p, c);
                k1 = g.k1;
                f = g.first;
            }
            const SmemText txt{buf + ((ts.y32 + f) & 15u) - f};
            stream_filter<Q, SH>(p, txt, sF, k0, k1, lane, qu, sink);
        }
        __syncwarp();              // every lane is done with buffer b before its refill
        b = b + 1 == NB ? 0 : b + 1;
    }
    __syncwarp();
    if (lane == 0)
        for (int i = 0; i < NB; ++i) mbar_inval(&ts.bar[i]);   // the epilogue reuses this memory
}

// Final drain on private copies.  When a warp runs out of chunks its queues still hold
// < 32 lattice survivors (q1) and < 32 continuing segments (q2).  Running them through
// first steps and phase B on global text is a chain of dependent L2 round trips (one per
// window visited, up to ~10 for the slowest warp: 5-6 us at the end of every search, when
// nothing else is left to overlap it).  Instead each lane copies the text its segment can
// ever touch, y[a_k - m + 1 .. a_k + S - 1] (R11), into a private box in the warp's now
// idle chunk buffers (one round trip for all of them), and Fig. 5 continues on the box at
// shared-memory latency.  A lattice survivor starts at its window end a_k (first_steps is
// only a shortcut of the same loop).  p.slot_bytes = box size (0: boxes do not fit).
template <int Q, int SH>
__device__ __forceinline__ void final_drain_boxes(const KParams &p, const FTable &sF, const uint8_t *sx,
                                                  const uint32_t *q1, uint32_t n1, const uint32_t *q2,
                                                  uint32_t n2, uint32_t boxes, WarpOut &wo, uint32_t lane) {
    const uintptr_t y = reinterpret_cast<uintptr_t>(p.y), ye = y + p.n;
    const uint32_t total = n1 + n2;
    for (uint32_t base = 0; base < total; base += 32) {
        const uint32_t idx = base + lane;
        const bool act = idx < total;
        const uint32_t start = act ? (idx < n1 ? q1[idx] : q2[idx - n1]) : p.m - 1;
        const uint32_t ak = p.m - 1 + (start - (p.m - 1)) / p.S * p.S;
        const uint32_t lo = ak + 1 - p.m, hi = min(ak + p.S, p.n) - 1;
        const uint32_t box = boxes + lane * p.slot_bytes + 16;   // 16 bytes of slack below (end8)
        const uintptr_t A = (y + lo) & ~static_cast<uintptr_t>(15);
        const uintptr_t B = (y + hi + 16) & ~static_cast<uintptr_t>(15);
        if (act) {
            for (uintptr_t w = A; w < B; w += 16) {
                const uint32_t d = box + static_cast<uint32_t>(w - A);
                if (w >= y && w + 16 <= ye) {
                    chk_text_range(p.y, p.n, w, 16);
                    cp_async16(d, reinterpret_cast<const void *>(w));
                } else {
                    for (uint32_t b = 0; b < 16; ++b)
                        if (w + b >= y && w + b < ye)
                            asm volatile("st.shared.u8 [%0], %1;" ::"r"(d + b),
                                         "r"(static_cast<uint32_t>(__ldg(reinterpret_cast<const uint8_t *>(w + b))))
                                         : "memory");
                }
            }
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        const SmemText txt{fence_value(box + static_cast<uint32_t>((y + lo) - A)) - lo};
        run_segments<Q, SH>(p, txt, sF, sx, act, start, wo, lane);
        __syncwarp();
    }
}

// The stream kernel's tables: the filter bitmap (replicated per lane or not), F and x.  Every
// thread issues ALL its global loads (one bitmap word, two 16-byte vectors of F, one of x)
// before its first shared store: one DRAM round trip for the lot (after the L2 flush of the
// bench every one of them is a miss), where load_pass_bits + load_table took three in a row.
// What a 768-thread block cannot cover that way (alpha > 13 at fewer warps, m > 12 K) follows
// in plain loops.
__device__ __forceinline__ void stream_load_tables(const KParams &p, uint32_t *bits, uint32_t *sF,
                                                   uint8_t *sx) {
    const uint32_t T = blockDim.x, t = threadIdx.x, lane = t & 31, warp = t >> 5, NW = T >> 5;
    const uint32_t nF = 1u << p.alpha;
    const uint32_t nw = nF > 32 ? nF / 32 : 1u;          // bitmap words
    if (nF < 8) {                                        // tiny tables: the plain loaders
        load_pass_bits(p, bits);
        load_table(p, sF, sx);
        return;
    }
    const uint32_t n4 = nF / 4;                          // 16-byte vectors of F
    const uint32_t n16 = (p.m + 8 + 15) / 16;            // ... and of x (zero-padded past m)
    const uint4 *F4 = reinterpret_cast<const uint4 *>(p.F);
    const uint4 *x4 = reinterpret_cast<const uint4 *>(p.x);
    // loads
    uint32_t bw = 0;
    if (p.lane_bits) {
        if (warp * 32 + lane < nw) bw = __ldg(p.Fbits + warp * 32 + lane);
    } else if (t < nw) {
        bw = __ldg(p.Fbits + t);
    }
    uint4 fv[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
#pragma unroll
    for (uint32_t r = 0; r < 2; ++r)
        if (t + r * T < n4) fv[r] = __ldg(F4 + t + r * T);
    uint4 xv = make_uint4(0, 0, 0, 0);
    if (t < n16 && 16 * t < p.m) xv = __ldg(x4 + t);
    // stores
    if (p.lane_bits) {
        if (warp * 32 < nw) {
            const uint32_t cnt = min(32u, nw - warp * 32);
            for (uint32_t k = 0; k < cnt; ++k) bits[(warp * 32 + k) * 32 + lane] = __shfl_sync(HC_FULL, bw, k);
        }
        for (uint32_t base = (warp + NW) * 32; base < nw; base += NW * 32) {   // alpha > 10 + log2(NW)
            const uint32_t v = base + lane < nw ? __ldg(p.Fbits + base + lane) : 0u;
            const uint32_t cnt = min(32u, nw - base);
            for (uint32_t k = 0; k < cnt; ++k) bits[(base + k) * 32 + lane] = __shfl_sync(HC_FULL, v, k);
        }
    } else {
        if (t < nw) bits[t] = bw;
        for (uint32_t i = t + T; i < nw; i += T) bits[i] = __ldg(p.Fbits + i);
    }
    uint4 *dF = reinterpret_cast<uint4 *>(sF);
#pragma unroll
    for (uint32_t r = 0; r < 2; ++r)
        if (t + r * T < n4) dF[t + r * T] = fv[r];
    for (uint32_t w = t + 2 * T; w < n4; w += T) dF[w] = __ldg(F4 + w);
    for (uint32_t w = t; w < n16; w += T) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (w == t) v = xv;
        else if (16 * w < p.m) v = __ldg(x4 + w);
        uint32_t *vw = reinterpret_cast<uint32_t *>(&v);
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {               // zero from byte m on (8-byte compares of x)
            const uint32_t b = 16 * w + 4 * j;
            if (b >= p.m) vw[j] = 0;
            else if (b + 4 > p.m) vw[j] &= (1u << (8 * (p.m - b))) - 1u;
        }
        reinterpret_cast<uint4 *>(sx)[w] = v;
    }
}

// The kernel body; two entry points compile it for two register budgets (below).
template <int Q, int SH>
__device__ __forceinline__ void stream_body(const KParams &p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t NW = blockDim.x / 32;
    const StreamLayout L = stream_layout(p.alpha, p.m, NW, p.stage_bytes, p.stages, p.lane_bits);
    uint32_t *sFp = reinterpret_cast<uint32_t *>(smem + L.f_off);
    uint8_t *sx = smem + L.x_off;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (kInstrument && tid == 0) trace_cta(p, 0);
    path_ts(p, 0);
    pdl_launch_dependents();
    const uint32_t total_warps = gridDim.x * NW;
    const uint32_t gw = blockIdx.x * NW + warp;
    const uint32_t bufs0 = smem_u32(smem + L.buf_off) + warp * p.stages * p.stage_bytes;
    // the first chunks' copies go out before the table load: both DRAM round trips overlap
    const uintptr_t yaddr = reinterpret_cast<uintptr_t>(p.y);
    const TmaStream ts{yaddr, static_cast<uint32_t>(yaddr), p.seg_per_chunk * p.S,
                       p.seg_per_chunk * p.S + max(p.q, 2 * p.q - min(p.S, 2 * p.q)), bufs0, p.stage_bytes,
                       reinterpret_cast<uint64_t *>(smem + L.ctr_off + round_up(NW * 4u, 8)) + warp * 4};
    stream_prologue_tma<2>(p, ts, gw, total_warps, lane);
    stream_load_tables(p, reinterpret_cast<uint32_t *>(smem + L.bits_off), sFp, sx);
    if (tid == 0) s_params[0] = p;
    __syncthreads();
    path_ts(p, 1);
    const FTable sF{fence_value(smem_u32(sFp))};
    const PassBits pb{fence_value(smem_u32(smem + L.bits_off)) + (p.lane_bits ? 4 * lane : 0u),
                      p.lane_bits ? 7u : 2u};
    WarpOut wo{reinterpret_cast<uint32_t *>(smem + L.wbuf_off) + warp * kWarpBuf, 0u};
    const GlobalText gtxt = global_text(p);
    WarpQueueSink<Q, SH, GlobalText, FTable> sink{p, gtxt, sF, sx, nullptr,
                                          reinterpret_cast<uint32_t *>(smem + L.q2_off) + warp * kWarpBuf,
                                          0u, 0u, wo, lane};
    uint32_t *ctr = reinterpret_cast<uint32_t *>(smem + L.ctr_off) + warp;
    if (lane == 0) *ctr = 0;
    __syncwarp();
    StreamQueue<Q, SH> qu{reinterpret_cast<uint32_t *>(smem + L.q_off) + warp * kStreamQ1, ctr, 0u};
    // two buffers per warp (3 and 4 measured slower at every m: DESIGN.md 5; fewer loop
    // variants also keep the kernel's code small)
    stream_loop_tma<Q, SH, 2>(p, pb, sink, qu, ts, gw, total_warps, lane);
    path_ts(p, 3);
#ifndef HC_NO_BOXES
    if (p.slot_bytes) {
        __syncwarp();
        final_drain_boxes<Q, SH>(p, sF, sx, qu.q1, qu.n1, sink.q2, sink.n2, bufs0, wo, lane);
        qu.n1 = 0;
        sink.n2 = 0;
    } else
#endif
    {
        qu.drain_all(sink, lane);
        path_ts(p, 4);
        sink.drain();
    }
    path_ts(p, 5);
    wo.flush(p, lane);
    path_ts(p, 6);
    if (kInstrument && lane == 0) trace_cta(p, 1);
    search_epilogue(p, smem);
}

#if HC_INSTRUMENT
cudaError_t read_epi_ts(unsigned long long *host8) {   // debug 10 (this TU's stamps)
    return cudaMemcpyFromSymbol(host8, g_epi_ts, sizeof(unsigned long long) * 16);
}
#endif

// One CTA per SM (F and the per-lane filter bitmaps are held once per SM), two builds:
//  - up to 24 warps at <= 85 registers (12 B of spills): dense lattices, S <= 8, where the
//    filter loop is issue-bound and every warp counts (C2 m = 8, C3/C4 m <= 8: 2-3.5%
//    faster than the other build);
//  - up to 20 warps at <= 102 registers (96 used, no spills): every other shift (C2 m = 16
//    and 32 3.5% faster, C3/C4 m = 16 7%: A/B).
template <int Q, int SH>
__global__ void __launch_bounds__(kStreamFatThreads, 1) stream_kernel(const KParams p) {
    stream_body<Q, SH>(p);
}
template <int Q, int SH>
__global__ void __launch_bounds__(kStreamRegThreads, 1) stream_kernel_r(const KParams p) {
    stream_body<Q, SH>(p);
}

template <int Q, int SH>
struct PickStream {
    using Fn = KernFn;
    static KernFn fn() { return stream_kernel<Q, SH>; }
};
template <int Q, int SH>
struct PickStreamR {
    using Fn = KernFn;
    static KernFn fn() { return stream_kernel_r<Q, SH>; }
};

cudaError_t launch_stream(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li) {
    const uint32_t nw = p.block_warps;
    KernFn kern = 32 * nw <= static_cast<uint32_t>(kStreamRegThreads) ? pick<PickStreamR>(p.q, p.s)
                                                                       : pick<PickStream>(p.q, p.s);
    if (!kern) return cudaErrorInvalidValue;
    const int smem = stream_smem_bytes(p.alpha, p.m, p.stage_bytes, p.stages, nw, p.lane_bits);
    const long ctas = (p.nchunks + nw - 1) / nw;
    KParams a = p;
    a.epi_cap = epi_cap_for(smem);
    void *args[] = {&a};
    return launch_kernel(reinterpret_cast<const void *>(kern), args, static_cast<int>(32 * nw), smem,
                         ctas, max_ctas, ctas_per_sm, st, li);
}

}  // namespace hc
