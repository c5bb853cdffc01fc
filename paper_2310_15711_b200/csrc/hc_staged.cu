// hc_staged.cu — staged path (HC_PATH_STAGED, an option, not a default): persistent
// warp-specialised CTAs stream 24 KiB text tiles into a shared-memory ring with 1-D TMA
// bulk copies (cp.async.bulk + mbarrier complete_tx).  Measured slower than the stream
// path at every m it applies to; kept as the TMA-ring design point.
#include "hc_device.cuh"

namespace hc {

// Staged path sink.  Lattice survivors (segment k) are collected per warp (q1) and
// run 32 at a time through first_steps_eval.  The rest go, as the window end to
// continue from, to the warp's region of the stage's queue, which the survivor warp
// runs in batches of 32 taken across all regions (a full region is run by its warp
// first).
template <int Q, int SH, class T>
struct RegionSink {
    const KParams &p;
    const T &txt;
    const FTable &sF;
    const uint8_t *sx;
    uint32_t *region;   // kRegion entries (window ends)
    uint32_t cnt;       // warp-uniform
    uint32_t *q1;       // kWarpBuf lattice survivors (a_k)
    uint32_t n1;        // warp-uniform
    WarpOut &wo;
    uint32_t lane;
    __device__ __forceinline__ void push(bool keep, uint32_t start) {
        const uint32_t bm = __ballot_sync(HC_FULL, keep);
        const uint32_t nb = __popc(bm);
        if (cnt + nb > kRegion) {
            __syncwarp();
            for (uint32_t b = 0; b < cnt; b += 32)
                run_survivors<Q, SH>(p, txt, sF, sx, region + b, min(32u, cnt - b), wo, lane);
            __syncwarp();
            cnt = 0;
        }
        if (keep) region[cnt + __popc(bm & lanemask_lt())] = start;
        cnt += nb;
    }
    __device__ __forceinline__ void first_steps(uint32_t c) {
        const bool act = lane < c;
        uint32_t start;
        const bool keep = first_steps_eval<Q, SH>(p, txt, sF, act, act ? q1[lane] : 0u, start);
        push(keep, start);
    }
    __device__ __forceinline__ void operator()(uint32_t bm, bool pass, uint32_t e) {
        if (kInstrument && p.debug == 3) return;         // phase A only (measurement)
        if (pass) q1[n1 + __popc(bm & lanemask_lt())] = e;
        n1 += __popc(bm);
        if (n1 >= 32) {
            __syncwarp();
            first_steps(32);
            const uint32_t rest = n1 - 32;
            const uint32_t mv = lane < rest ? q1[32 + lane] : 0u;
            __syncwarp();
            if (lane < rest) q1[lane] = mv;
            __syncwarp();
            n1 = rest;
        }
    }
    __device__ __forceinline__ void finish() {           // before the stage is handed on
        if (n1) {
            __syncwarp();
            first_steps(n1);
            n1 = 0;
        }
    }
};

// ------------------------------------------------------------------ shared layout
// Staged CTA: NF = NW - kSurvWarps filter warps + kSurvWarps survivor warps.
// Shared memory: F | x | per-warp queue | per-warp out buffer | survivor regions
// [stages][NW][kRegion] | region counts [stages][NW] | full[stages] + filtered[stages]
// mbarriers | tile id per stage | survivor-warp box meta [kSurvWarps][nbox][2] |
// survivor boxes [kSurvWarps][nbox][slot_bytes] | stage ring.
struct StagedLayout {
    uint32_t f_off, x_off, q_off, wbuf_off, sq_off, cnt_off, full_off, filt_off, tile_off, meta_off,
        box_off, stage_off, total;
};
__host__ __device__ inline StagedLayout staged_layout(uint32_t alpha, uint32_t m,
                                                      uint32_t stage_bytes, uint32_t stages,
                                                      uint32_t nwarps, uint32_t slot_bytes,
                                                      uint32_t nbox) {
    StagedLayout L;
    L.f_off = 0;
    L.x_off = round_up((1u << alpha) * 4u, 16);
    L.q_off = L.x_off + round_up(m + 8, 16);
    L.wbuf_off = L.q_off + nwarps * kWarpBuf * 4u;
    L.sq_off = L.wbuf_off + nwarps * kWarpBuf * 4u;
    L.cnt_off = L.sq_off + stages * nwarps * kRegion * 4u;
    L.full_off = round_up(L.cnt_off + stages * nwarps * 4u, 8);
    L.filt_off = L.full_off + stages * 8u;
    L.tile_off = L.filt_off + stages * 8u;
    L.meta_off = L.tile_off + stages * 4u;
    L.box_off = round_up(L.meta_off + kSurvWarps * nbox * 8u, 16);
    L.stage_off = round_up(L.box_off + kSurvWarps * nbox * slot_bytes, 128);
    L.total = L.stage_off + stages * stage_bytes;
    return L;
}

int staged_smem_bytes(uint32_t alpha, uint32_t m, uint32_t stage_bytes, uint32_t stages,
                      uint32_t slot_bytes, uint32_t nbox) {
    return static_cast<int>(
        staged_layout(alpha, m, stage_bytes, stages, kStagedThreads / 32, slot_bytes, nbox).total);
}

// Geometry of staged tile t: segments [k0, k1), text bytes [lo, hi).
struct TileGeom {
    uint32_t k0, k1;
    uint64_t lo, hi;           // byte indices into y
    uintptr_t gbase;           // 16-aligned global address mapped to stage offset 0
    uintptr_t A, B;            // bulk-copied global range [A, B) (16-aligned, inside y)
};
__device__ __forceinline__ TileGeom tile_geom(const KParams &p, uint32_t t) {
    TileGeom g;
    g.k0 = t * p.seg_per_tile;
    g.k1 = min(g.k0 + p.seg_per_tile, p.K);
    g.lo = static_cast<uint64_t>(g.k0) * p.S;
    g.hi = min(static_cast<uint64_t>(p.m) - 1 + static_cast<uint64_t>(g.k1) * p.S,
               static_cast<uint64_t>(p.n));
    const uintptr_t y = reinterpret_cast<uintptr_t>(p.y);
    const uintptr_t ga = y + g.lo;
    g.gbase = ga & ~static_cast<uintptr_t>(15);
    const uintptr_t ybeg = (y + 15) & ~static_cast<uintptr_t>(15);
    const uintptr_t yend = (y + p.n) & ~static_cast<uintptr_t>(15);
    g.A = max(g.gbase, ybeg);
    g.B = min((y + g.hi + 15) & ~static_cast<uintptr_t>(15), yend);
    return g;
}

__device__ __forceinline__ void issue_tile(const KParams &p, uint32_t t, uint8_t *stage,
                                           uint64_t *bar) {
    const TileGeom g = tile_geom(p, t);
    if (g.B > g.A) {
        const uint32_t bytes = static_cast<uint32_t>(g.B - g.A);
        mbar_arrive_expect_tx(bar, bytes);
        const uint32_t chunk = p.tma_chunk ? p.tma_chunk : bytes;
        for (uint32_t o = 0; o < bytes; o += chunk)
            bulk_g2s(smem_u32(stage) + static_cast<uint32_t>(g.A - g.gbase) + o,
                     reinterpret_cast<const void *>(g.A + o), min(chunk, bytes - o), bar);
    } else {
        mbar_arrive(bar);
    }
}

// Loads tile t into `stage` (one warp): bytes outside the 16-aligned interior the bulk
// copy can move (only at the two ends of an unaligned text, or tiny texts) are
// stored by the lanes first; then lane 0 arms `bar` and issues the bulk copy.  The
// lanes' stores are ordered before the arrive (syncwarp + release of the arrive).
__device__ __forceinline__ void load_tile_warp(const KParams &p, uint32_t t, uint8_t *stage,
                                               uint64_t *bar, uint32_t lane) {
    if (t == 0 || t + 2 >= p.ntiles) {
        const TileGeom g = tile_geom(p, t);
        const uintptr_t y = reinterpret_cast<uintptr_t>(p.y);
        const uintptr_t ga = y + g.lo, gh = y + g.hi;
        if (g.B <= g.A) {
            for (uintptr_t a = ga + lane; a < gh; a += 32)
                stage[a - g.gbase] = __ldg(reinterpret_cast<const uint8_t *>(a));
        } else {
            for (uintptr_t a = ga + lane; a < g.A; a += 32)
                stage[a - g.gbase] = __ldg(reinterpret_cast<const uint8_t *>(a));
            for (uintptr_t a = g.B + lane; a < gh; a += 32)
                stage[a - g.gbase] = __ldg(reinterpret_cast<const uint8_t *>(a));
        }
    }
    __syncwarp();
    if (lane == 0) {
        fence_proxy_async();
        issue_tile(p, t, stage, bar);
    }
    __syncwarp();
}

// Warp-specialised staged kernel.  Per stage s of the ring:
//   full[s]     armed by the producer (expect_tx), completed by the TMA bulk copy;
//               tile[s] (written before the arm) says which tile, >= ntiles = none;
//   filtered[s] one arrival per filter warp once its slice of the tile is filtered
//               (first_steps included) and its survivors are in its region of s;
// the survivor warp owning the iteration waits filtered[s], takes the survivors'
// window ends out of the regions, refills stage s at once with the next tile of a
// global counter (dynamic scheduling: CTAs that run ahead take more tiles, so the
// grid finishes together), and then runs phase B on them reading the text from
// global memory (the tile was just streamed through L2): survivors never hold a
// stage.  Filter warps never wait for survivor work, only for data.
template <int Q, int SH>
__global__ void __launch_bounds__(kStagedThreads, 3) staged_kernel(const KParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr uint32_t NW = kStagedThreads / 32;
    constexpr uint32_t NF = NW - kSurvWarps;
    const StagedLayout L = staged_layout(p.alpha, p.m, p.stage_bytes, p.stages, NW, p.slot_bytes,
                                         p.nbox);
    uint32_t *sFp = reinterpret_cast<uint32_t *>(smem + L.f_off);
    uint8_t *sx = smem + L.x_off;
    uint32_t *sq = reinterpret_cast<uint32_t *>(smem + L.sq_off);
    uint32_t *qcnt = reinterpret_cast<uint32_t *>(smem + L.cnt_off);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + L.full_off);
    uint64_t *filt = reinterpret_cast<uint64_t *>(smem + L.filt_off);
    volatile uint32_t *tile = reinterpret_cast<volatile uint32_t *>(smem + L.tile_off);
    uint8_t *stages = smem + L.stage_off;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (kInstrument && tid == 0) trace_cta(p, 0);
    pdl_launch_dependents();

    // loads tile t (or nothing, t >= ntiles) into stage st: the tile id is published
    // before the barrier is armed (the arm releases it to the waiters)
    auto produce = [&](uint32_t st, uint32_t t) {
        if (lane == 0) tile[st] = t;
        __syncwarp();
        if (t < p.ntiles) {
            load_tile_warp(p, t, stages + st * p.stage_bytes, &full[st], lane);
        } else if (lane == 0) {
            mbar_arrive(&full[st]);
        }
        __syncwarp();
    };
    // the producer warp starts the first tiles' copies before the table load
    if (warp == NF) {
        if (lane == 0) {
            for (uint32_t st = 0; st < p.stages; ++st) {
                mbar_init(&full[st], 1);
                mbar_init(&filt[st], NF);
            }
            fence_mbar_init();
        }
        __syncwarp();
        for (uint32_t st = 0; st < p.stages; ++st) produce(st, blockIdx.x + st * gridDim.x);
    }
    load_table(p, sFp, sx);
    if (tid == 0) s_params[0] = p;
    __syncthreads();
    const FTable sF{smem_u32(sFp)};
    WarpOut wo{reinterpret_cast<uint32_t *>(smem + L.wbuf_off) + warp * kWarpBuf, 0u};
    const uint32_t y32 = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p.y));
    const uint32_t stage0 = smem_u32(stages);
    const bool dynamic = !(kInstrument && p.debug == 6);

    if (warp < NF) {
        // Each stage carries a chain of tiles (produced in order by the survivor warp
        // owning the stage's iterations) that ends with the first "no tile"; the filter
        // warps go round the stages until every chain has ended.
        const uint32_t all = (1u << p.stages) - 1u;
        uint32_t ended = 0, st = 0, par = 0;
        for (uint32_t it = 0; ended != all; ++it) {
            if (((ended >> st) & 1u) == 0) {
            // debug 6: filter compute alone (stale stage data, static tiles, no refills)
            if (dynamic || it < p.stages) mbar_wait(&full[st], par);
            const uint32_t t = dynamic ? fence_value(tile[st]) : blockIdx.x + it * gridDim.x;
            uint32_t *q = sq + st * (NF * kRegion);     // NF regions of kRegion entries
            uint32_t *qc = qcnt + st * NF;              // entries used per region
            if (t >= p.ntiles) {
                ended |= 1u << st;
                if (lane == 0) {
                    qc[warp] = 0;
                    mbar_arrive(&filt[st]);             // lets the survivor warp see the end
                }
            } else {
            if (warp == 0 && lane == 0) trace_event(p, it, 0);
            const uint32_t k0 = t * p.seg_per_tile;
            const uint32_t k1 = min(k0 + p.seg_per_tile, p.K);
            const uint32_t lo = k0 * p.S;               // first text byte of the tile
            // shared address of text byte p: stage + ((y + lo) & 15) + (p - lo)
            const SmemText txt{stage0 + st * p.stage_bytes + ((y32 + lo) & 15u) - lo};
            RegionSink<Q, SH, SmemText> sink{p,  txt, sF, sx, q + warp * kRegion, 0u,
                                             reinterpret_cast<uint32_t *>(smem + L.q_off) + warp * kWarpBuf,
                                             0u, wo, lane};
            if (!(kInstrument && p.debug == 1)) {
                const uint32_t nseg = k1 - k0;
                const uint32_t seg_lo = k0 + (warp * nseg) / NF;
                const uint32_t seg_hi = k0 + ((warp + 1) * nseg) / NF;
                filter_lattice<Q, SH>(p, txt, sF, seg_lo, seg_hi, lane, sink);
                sink.finish();
            }
            __syncwarp();
            if (warp == 0 && lane == 0) trace_event(p, it, 1);
            if (lane == 0) {
                qc[warp] = sink.cnt;
                mbar_arrive(&filt[st]);                 // release: region + count visible
            }
            }
            }
            if (++st == p.stages) {
                st = 0;
                par ^= 1u;
            }
        }
    } else if (dynamic) {
        // survivor warp NF + i owns the iterations it = i, i + kSurvWarps, ...; it
        // grabs the tile it will produce next one iteration ahead (hides the atomic)
        uint32_t nt = 0;
        if (lane == 0) nt = p.stages * gridDim.x + atomicAdd(p.counter + 1, 1u);
        for (uint32_t it = warp - NF;; it += kSurvWarps) {
            const uint32_t st = it % p.stages, par = (it / p.stages) & 1u;
            mbar_wait(&filt[st], par);
            const uint32_t t = fence_value(tile[st]);
            if (t >= p.ntiles) break;
            const uint32_t lo = t * p.seg_per_tile * p.S;
            uint32_t *q = sq + st * (NF * kRegion);
            const uint32_t *qc = qcnt + st * NF;
            const SmemText txt{stage0 + st * p.stage_bytes + ((y32 + lo) & 15u) - lo};
            // inclusive prefix of the region counts (lanes < NF), total in every lane
            uint32_t incl = lane < NF ? qc[lane] : 0u;
#pragma unroll
            for (uint32_t o = 1; o < NF; o <<= 1) {
                const uint32_t t2 = __shfl_up_sync(HC_FULL, incl, o);
                if (lane >= o) incl += t2;
            }
            const uint32_t total = (kInstrument && p.debug == 3) ? 0u : __shfl_sync(HC_FULL, incl, NF - 1);
            if (lane == 0) trace_event(p, it, 3);
            // entry g lives in region r with excl(r) <= g < incl(r)
            auto entry = [&](uint32_t g) -> uint32_t {
                uint32_t r = 0, base = 0;
#pragma unroll
                for (uint32_t w = 0; w < NF; ++w) {
                    const uint32_t iw = __shfl_sync(HC_FULL, incl, w);
                    if (g >= iw) {
                        r = w + 1;
                        base = iw;
                    }
                }
                return g < total ? q[r * kRegion + (g - base)] : 0u;
            };
            // The survivors are taken out of the stage before it is refilled: the first
            // nbox as boxes (their segment's text copied in 16-byte chunks to this
            // warp's box area, based so that text p is at base + p), the next kWarpBuf
            // as window ends only (phase B reads them from global memory), the rest
            // (rare after first_steps) are run on the stage first.
            uint32_t *meta = reinterpret_cast<uint32_t *>(smem + L.meta_off) + (warp - NF) * 2 * p.nbox;
            const uint32_t box0 = smem_u32(smem + L.box_off) + (warp - NF) * p.nbox * p.slot_bytes;
            uint32_t *mine = reinterpret_cast<uint32_t *>(smem + L.q_off) + warp * kWarpBuf;
            const uint32_t nb = min(total, p.nbox);
            const uint32_t nm = min(total - nb, static_cast<uint32_t>(kWarpBuf));
            for (uint32_t b = nb + nm; b < total; b += 32) {
                const uint32_t start = entry(b + lane);
                run_segments<Q, SH>(p, txt, sF, sx, b + lane < total, start, wo, lane);
            }
            for (uint32_t b = 0; b < nb + nm; b += 32) {
                const uint32_t g = b + lane;
                const uint32_t start = entry(g);
                if (g < nb) {
                    const uint32_t k = (start - (p.m - 1)) / p.S;
                    const uint32_t hi = min(p.m - 1 + (k + 1) * p.S, p.n);
                    const uint32_t a0 = (txt.base + start + 1 - p.m) & ~15u;
                    const uint32_t a1 = (txt.base + hi - 1) & ~15u;
                    const uint32_t d0 = box0 + g * p.slot_bytes;
                    for (uint32_t a = a0, d = d0; a <= a1; a += 16, d += 16) sts128(d, lds128(a));
                    meta[2 * g] = start;
                    meta[2 * g + 1] = d0 - (a0 - txt.base);
                } else if (g < nb + nm) {
                    mine[g - nb] = start;
                }
            }
            __syncwarp();
            produce(st, __shfl_sync(HC_FULL, nt, 0));
            if (lane == 0) nt = p.stages * gridDim.x + atomicAdd(p.counter + 1, 1u);
            for (uint32_t b = 0; b < nb; b += 32) {
                const bool act = b + lane < nb;
                const SmemText btxt{act ? meta[2 * (b + lane) + 1] : txt.base};
                run_segments<Q, SH>(p, btxt, sF, sx, act, act ? meta[2 * (b + lane)] : 0u, wo, lane);
            }
            const GlobalText gtxt = global_text(p);
            for (uint32_t b = 0; b < nm; b += 32) {
                const bool act = b + lane < nm;
                run_segments<Q, SH>(p, gtxt, sF, sx, act, act ? mine[b + lane] : 0u, wo, lane);
            }
            __syncwarp();
            if (lane == 0) trace_event(p, it, 2);
        }
    }
    wo.flush(p, lane);
    if (kInstrument && lane == 0) trace_cta(p, 1);   // last warp to get here wins
    search_epilogue(p, smem);
}

template <int Q, int SH>
struct PickStaged {
    using Fn = KernFn;
    static KernFn fn() { return staged_kernel<Q, SH>; }
};

cudaError_t launch_staged(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li) {
    KernFn kern = pick<PickStaged>(p.q, p.s);
    if (!kern) return cudaErrorInvalidValue;
    const int smem = staged_smem_bytes(p.alpha, p.m, p.stage_bytes, p.stages, p.slot_bytes, p.nbox);
    KParams a = p;
    a.epi_cap = epi_cap_for(smem);
    void *args[] = {&a};
    return launch_kernel(reinterpret_cast<const void *>(kern), args, kStagedThreads, smem,
                         static_cast<long>(p.ntiles), max_ctas, ctas_per_sm, st, li);
}

}  // namespace hc
