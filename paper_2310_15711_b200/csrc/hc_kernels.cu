// hc_kernels.cu — sm_100a device side of libhc: the Hash Chain searching phase
// (Fig. 5 left) as data-parallel CUDA kernels.
//
// Data parallelism (reading R11): the window ends
// [m-1, n) are cut into K segments of S = m-q+1 ends, a_k = m-1 + k*S.  HC
// started at a_k with loop bound b = min(a_k + S, n) reports exactly the
// occurrences ending in [a_k, b) and reads only y[a_k-m+1 .. b-1].  A segment
// whose first window is rejected by the F[v] == 0 fast path is done
// after one hash; the others continue the paper's loop inside the segment.
//
// Each lane runs the loop of Fig. 5 as a flat state machine doing ONE q-gram
// hash per iteration (window-end hash, l.4-6, or one walk step, l.9-13), so the
// 32 lanes of a warp stay converged; a lane whose segment is finished takes
// the next segment of the warp's range in the same iteration (ballot/popc).
//
// Two text access paths:
//   staged : persistent CTAs stream tiles of the text into shared memory with
//            TMA bulk copies (cp.async.bulk + mbarrier), NSTAGE-deep ring; every
//            hash reads shared memory.  For small shifts (every 32-B sector of
//            the text is touched anyway).
//   gather : no staging; each lane reads only the aligned 8-byte words holding
//            the q-grams it hashes (ld.global.nc).  For large shifts, where HC
//            touches a small fraction of the text (sublinear search).
// F (2^alpha u32 words) and x live in shared memory in both paths.
// Matches go to a per-warp shared buffer and are flushed 32 at a time with one
// atomicAdd per flush (ballot/popc ranks); the host sorts them afterwards.

#include <cub/device/device_radix_sort.cuh>

#include "hc_internal.h"

namespace hc {

#define HC_FULL 0xffffffffu
constexpr uint32_t kWordBits = 32;  // w (R2)

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(tx)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "HC_WAIT%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra HC_DONE%=;\n\t"
        "bra HC_WAIT%=;\n"
        "HC_DONE%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D TMA bulk copy global -> shared, completion signalled on `bar` (tx bytes).
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// ------------------------------------------------------------------ text access
// Text byte p (0 <= p < n) of y, read from global memory (read-only path).
struct GlobalText {
    const uint8_t *y;
    __device__ __forceinline__ uintptr_t addr(uint32_t p) const {
        return reinterpret_cast<uintptr_t>(y) + p;
    }
    __device__ __forceinline__ uint64_t word(uintptr_t aligned) const {
        return __ldg(reinterpret_cast<const unsigned long long *>(aligned));
    }
    __device__ __forceinline__ uint32_t byte(uint32_t p) const { return __ldg(y + p); }
    static constexpr bool kLoSafe = false;  // the word before may be outside y
};

// Text byte p read from a shared-memory stage: byte p is at smem[base + p]
// (offsets mod 2^32; the stage is 16-aligned so offsets keep y's alignment mod 16).
struct SmemText {
    const uint8_t *s;  // start of the dynamic shared-memory array
    uint32_t base;
    __device__ __forceinline__ uint32_t addr(uint32_t p) const { return base + p; }
    __device__ __forceinline__ uint64_t word(uint32_t aligned) const {
        return *reinterpret_cast<const uint64_t *>(s + aligned);
    }
    __device__ __forceinline__ uint32_t byte(uint32_t p) const { return s[base + p]; }
    static constexpr bool kLoSafe = true;   // stages never start at shared offset 0
};

// The 8 text bytes y[p-7 .. p] as a little-endian u64 (byte 7 = y[p]).  Only the
// top Q bytes are meaningful: reads just the aligned 8-byte words holding y[p]
// and y[p-Q+1] (both inside the text), so no byte outside [0, n) is touched.
template <int Q, class T>
__device__ __forceinline__ uint64_t end8(const T &t, uint32_t p) {
    auto a = t.addr(p);
    using A = decltype(a);
    const A ah = a & ~static_cast<A>(7);
    const uint32_t off = static_cast<uint32_t>(a & 7);
    const uint64_t hi = t.word(ah);
    uint64_t lo = 0;
    if (Q > 1) {
        if (T::kLoSafe || off < static_cast<uint32_t>(Q - 1)) lo = t.word(ah - 8);
    }
    return off == 7 ? hi : ((lo >> (8 * (off + 1))) | (hi << (56 - 8 * off)));
}

// Eq. 3 / Fig. 3 Hash: v = 0; for i = p downto p-q+1:
// v = (v << s) + y[i]; return v & mask.  W holds y[p-7..p], byte 7 = y[p].
template <int Q>
__device__ __forceinline__ uint32_t qhash(uint64_t W, uint32_t s, uint32_t mask) {
    const uint32_t whi = static_cast<uint32_t>(W >> 32), wlo = static_cast<uint32_t>(W);
    uint32_t v = 0;
#pragma unroll
    for (int t = 0; t < Q; ++t) {
        const int b = 7 - t;
        const uint32_t c = b >= 4 ? (whi >> (8 * (b - 4))) & 0xffu : (wlo >> (8 * b)) & 0xffu;
        v = (v << s) + c;
    }
    return v & mask;
}

// Fig. 5 l.16 verification: y[start .. start+m-1] == x (sx: x in shared memory,
// 16-aligned).  8 bytes per step, then a byte tail.
template <class T>
__device__ __noinline__ bool verify(const T &t, const uint8_t *sx, uint32_t start, uint32_t m) {
    uint32_t k = 0;
    for (; k + 8 <= m; k += 8) {
        const uint64_t a = end8<8>(t, start + k + 7);
        const uint64_t b = *reinterpret_cast<const uint64_t *>(sx + k);
        if (a != b) return false;
    }
    for (; k < m; ++k)
        if (t.byte(start + k) != sx[k]) return false;
    return true;
}

// Per-warp match buffer: positions are appended (ballot rank) and flushed to
// global memory 32 at a time with one atomicAdd.
struct WarpOut {
    uint32_t *buf;   // shared, kWarpBuf entries
    uint32_t cnt;    // warp-uniform
    __device__ __forceinline__ void push(bool found, uint32_t pos, const KParams &p,
                                         uint32_t lane) {
        const uint32_t fm = __ballot_sync(HC_FULL, found);
        if (fm == 0) return;
        if (found) buf[cnt + __popc(fm & lanemask_lt())] = pos;
        cnt += __popc(fm);
        if (cnt >= 32) {
            __syncwarp();
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(p.counter, 32u);
            base = __shfl_sync(HC_FULL, base, 0);
            const uint32_t v = buf[lane];
            if (base + lane < p.cap) p.out[base + lane] = v;
            const uint32_t rest = cnt - 32;
            const uint32_t nv = lane < rest ? buf[32 + lane] : 0u;
            __syncwarp();
            if (lane < rest) buf[lane] = nv;
            __syncwarp();
            cnt = rest;
        }
    }
    __device__ __forceinline__ void flush(const KParams &p, uint32_t lane) {
        __syncwarp();
        if (cnt == 0) return;
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(p.counter, cnt);
        base = __shfl_sync(HC_FULL, base, 0);
        if (lane < cnt && base + lane < p.cap) p.out[base + lane] = buf[lane];
        __syncwarp();
        cnt = 0;
    }
};

// Runs HC on segments [seg_lo, seg_hi) with the 32 lanes of the calling warp.
// Every lane of the warp must call it (warp-synchronous).
template <int Q, bool COUNT_ONLY, class T>
__device__ __forceinline__ void run_segments(const KParams &p, const T &txt, const uint32_t *sF,
                                             const uint8_t *sx, uint32_t seg_lo, uint32_t seg_hi,
                                             WarpOut &wo, uint32_t &nfound, uint32_t lane) {
    const uint32_t lt = lanemask_lt();
    uint32_t cursor = seg_lo;
    bool active = false, walk = false;
    uint32_t j = 0, e = 0, i = 0, b = 0, z = 0;
    while (true) {
        const uint32_t idle = __ballot_sync(HC_FULL, !active);
        if (idle != 0 && cursor < seg_hi) {
            const uint32_t k = cursor + __popc(idle & lt);
            if (!active && k < seg_hi) {
                active = true;
                walk = false;
                j = p.m - 1 + k * p.S;                 // lattice window end a_k
                b = min(j + p.S, p.n);                 // segment bound
            }
            cursor += __popc(idle);
        }
        if (__ballot_sync(HC_FULL, active) == 0) break;
        bool found = false;
        uint32_t fpos = 0;
        if (active) {
            const uint32_t pos = walk ? j - p.q : j;
            const uint32_t v = qhash<Q>(end8<Q>(txt, pos), p.s, p.mask);
            bool complete = false;
            if (!walk) {                               // Fig. 5 l.4-7
                e = j;
                z = sF[v];
                if (z == 0) {
                    j += p.S;                          // l.18 fast path
                } else {
                    i = j + 2 * p.q - p.m;             // l.7: i = j - m + 2q (> 0)
                    if (j >= i) walk = true;           // l.8
                    else complete = true;              // m < 2q: while-else (R7)
                }
            } else {                                   // l.9-13
                j -= p.q;
                if (((z >> (v & (kWordBits - 1))) & 1u) == 0) {
                    walk = false;                      // l.12 break
                    j += p.S;                          // l.18
                } else {
                    z = sF[v];                         // l.13
                    if (j < i) {
                        walk = false;
                        complete = true;
                    }
                }
            }
            if (complete) {                            // l.14-18, index per R1
                if (v == p.hv && verify(txt, sx, e + 1 - p.m, p.m)) {
                    found = true;
                    fpos = e + 1 - p.m;
                }
                j = e + 1;                             // (i - q) + (m - q + 1)
            }
            if (!walk && j >= b) active = false;
        }
        if (COUNT_ONLY) {
            nfound += found ? 1u : 0u;
        } else {
            wo.push(found, fpos, p, lane);
        }
    }
}

// ------------------------------------------------------------------ shared layout
struct StagedLayout {
    uint32_t f_off, x_off, wbuf_off, mbar_off, stage_off, total;
};
__host__ __device__ inline uint32_t round_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }
__host__ __device__ inline StagedLayout staged_layout(uint32_t alpha, uint32_t m,
                                                      uint32_t stage_bytes, uint32_t stages,
                                                      uint32_t nwarps) {
    StagedLayout L;
    L.f_off = 0;
    L.x_off = round_up((1u << alpha) * 4u, 16);
    L.wbuf_off = L.x_off + round_up(m + 8, 16);
    L.mbar_off = L.wbuf_off + nwarps * kWarpBuf * 4u;
    L.stage_off = round_up(L.mbar_off + stages * 8u, 128);
    L.total = L.stage_off + stages * stage_bytes;
    return L;
}
struct GatherLayout {
    uint32_t f_off, x_off, wbuf_off, total;
};
__host__ __device__ inline GatherLayout gather_layout(uint32_t alpha, uint32_t m,
                                                      uint32_t nwarps) {
    GatherLayout L;
    L.f_off = 0;
    L.x_off = round_up((1u << alpha) * 4u, 16);
    L.wbuf_off = L.x_off + round_up(m + 8, 16);
    L.total = L.wbuf_off + nwarps * kWarpBuf * 4u;
    return L;
}

int staged_smem_bytes(uint32_t alpha, uint32_t m, uint32_t stage_bytes, uint32_t stages) {
    return static_cast<int>(staged_layout(alpha, m, stage_bytes, stages, kStagedThreads / 32).total);
}
int gather_smem_bytes(uint32_t alpha, uint32_t m) {
    return static_cast<int>(gather_layout(alpha, m, kGatherThreads / 32).total);
}

__device__ __forceinline__ void load_table(const KParams &p, uint32_t *sF, uint8_t *sx) {
    const uint32_t nF = 1u << p.alpha;
    for (uint32_t w = threadIdx.x; w < nF; w += blockDim.x) sF[w] = __ldg(p.F + w);
    for (uint32_t k = threadIdx.x; k < p.m; k += blockDim.x) sx[k] = __ldg(p.x + k);
    // zero the 8-byte tail so 8-byte compares of x never read uninitialised bytes
    if (threadIdx.x < 8) sx[p.m + threadIdx.x] = 0;
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
        bulk_g2s(smem_u32(stage) + static_cast<uint32_t>(g.A - g.gbase),
                 reinterpret_cast<const void *>(g.A), bytes, bar);
    } else {
        mbar_arrive(bar);
    }
}

template <int Q, bool COUNT_ONLY>
__global__ void __launch_bounds__(kStagedThreads) staged_kernel(const KParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr uint32_t NW = kStagedThreads / 32;
    const StagedLayout L = staged_layout(p.alpha, p.m, p.stage_bytes, p.stages, NW);
    uint32_t *sF = reinterpret_cast<uint32_t *>(smem + L.f_off);
    uint8_t *sx = smem + L.x_off;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + L.mbar_off);
    uint8_t *stages = smem + L.stage_off;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    load_table(p, sF, sx);
    if (tid == 0) {
        for (uint32_t st = 0; st < p.stages; ++st) mbar_init(&mbar[st], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        for (uint32_t st = 0; st < p.stages; ++st) {
            const uint32_t t = blockIdx.x + st * gridDim.x;
            if (t < p.ntiles) issue_tile(p, t, stages + st * p.stage_bytes, &mbar[st]);
        }
    }
    WarpOut wo{reinterpret_cast<uint32_t *>(smem + L.wbuf_off) + warp * kWarpBuf, 0u};
    uint32_t nfound = 0;
    const uintptr_t y = reinterpret_cast<uintptr_t>(p.y);

    for (uint32_t it = 0;; ++it) {
        const uint32_t t = blockIdx.x + it * gridDim.x;
        if (t >= p.ntiles) break;
        const uint32_t st = it % p.stages;
        const uint32_t par = (it / p.stages) & 1u;
        uint8_t *sbuf = stages + st * p.stage_bytes;
        const TileGeom g = tile_geom(p, t);
        mbar_wait(&mbar[st], par);
        // bytes of the tile outside the bulk-copied 16-aligned interior (only at the
        // two ends of an unaligned text, or for tiny texts): plain byte loads
        const uintptr_t ga = y + g.lo, gh = y + g.hi;
        const bool edges = (g.B <= g.A) || (g.A > ga) || (g.B < gh);
        if (edges) {
            if (g.B <= g.A) {
                for (uintptr_t a = ga + tid; a < gh; a += blockDim.x)
                    sbuf[a - g.gbase] = __ldg(reinterpret_cast<const uint8_t *>(a));
            } else {
                for (uintptr_t a = ga + tid; a < g.A; a += blockDim.x)
                    sbuf[a - g.gbase] = __ldg(reinterpret_cast<const uint8_t *>(a));
                for (uintptr_t a = g.B + tid; a < gh; a += blockDim.x)
                    sbuf[a - g.gbase] = __ldg(reinterpret_cast<const uint8_t *>(a));
            }
            __syncthreads();
        }
        // shared address of text byte p: smem(sbuf) + (y + p - gbase)
        const SmemText txt{smem, static_cast<uint32_t>(sbuf - smem) + static_cast<uint32_t>(y - g.gbase)};
        const uint32_t nseg = g.k1 - g.k0;
        const uint32_t seg_lo = g.k0 + (warp * nseg) / NW;
        const uint32_t seg_hi = g.k0 + ((warp + 1) * nseg) / NW;
        run_segments<Q, COUNT_ONLY>(p, txt, sF, sx, seg_lo, seg_hi, wo, nfound, lane);
        __syncthreads();  // every warp is done with this stage
        if (tid == 0) {
            const uint32_t tn = t + p.stages * gridDim.x;
            if (tn < p.ntiles) {
                fence_proxy_async();
                issue_tile(p, tn, sbuf, &mbar[st]);
            }
        }
    }
    if (COUNT_ONLY) {
        for (int o = 16; o > 0; o >>= 1) nfound += __shfl_xor_sync(HC_FULL, nfound, o);
        if (lane == 0 && nfound) atomicAdd(p.counter, nfound);
    } else {
        wo.flush(p, lane);
    }
}

template <int Q, bool COUNT_ONLY>
__global__ void __launch_bounds__(kGatherThreads) gather_kernel(const KParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr uint32_t NW = kGatherThreads / 32;
    const GatherLayout L = gather_layout(p.alpha, p.m, NW);
    uint32_t *sF = reinterpret_cast<uint32_t *>(smem + L.f_off);
    uint8_t *sx = smem + L.x_off;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    load_table(p, sF, sx);
    __syncthreads();
    WarpOut wo{reinterpret_cast<uint32_t *>(smem + L.wbuf_off) + warp * kWarpBuf, 0u};
    uint32_t nfound = 0;
    const GlobalText txt{p.y};
    const uint32_t total_warps = gridDim.x * NW;
    for (uint32_t c = blockIdx.x * NW + warp; c < p.nchunks; c += total_warps) {
        const uint32_t seg_lo = c * p.seg_per_chunk;
        const uint32_t seg_hi = min(seg_lo + p.seg_per_chunk, p.K);
        run_segments<Q, COUNT_ONLY>(p, txt, sF, sx, seg_lo, seg_hi, wo, nfound, lane);
    }
    if (COUNT_ONLY) {
        for (int o = 16; o > 0; o >>= 1) nfound += __shfl_xor_sync(HC_FULL, nfound, o);
        if (lane == 0 && nfound) atomicAdd(p.counter, nfound);
    } else {
        wo.flush(p, lane);
    }
}

// ------------------------------------------------------------------ launchers
template <class K>
static cudaError_t launch_common(K kern, const KParams &p, int threads, int smem, int work_units,
                                 int max_ctas, cudaStream_t st, LaunchInfo *li) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
    if (err != cudaSuccess) return err;
    if (occ < 1) return cudaErrorInvalidConfiguration;
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

#define HC_DISPATCH_Q(Q_, KERNEL, CO)                                          \
    switch (Q_) {                                                              \
        case 1: kern = CO ? KERNEL<1, true> : KERNEL<1, false>; break;         \
        case 2: kern = CO ? KERNEL<2, true> : KERNEL<2, false>; break;         \
        case 3: kern = CO ? KERNEL<3, true> : KERNEL<3, false>; break;         \
        case 4: kern = CO ? KERNEL<4, true> : KERNEL<4, false>; break;         \
        case 5: kern = CO ? KERNEL<5, true> : KERNEL<5, false>; break;         \
        case 6: kern = CO ? KERNEL<6, true> : KERNEL<6, false>; break;         \
        case 7: kern = CO ? KERNEL<7, true> : KERNEL<7, false>; break;         \
        case 8: kern = CO ? KERNEL<8, true> : KERNEL<8, false>; break;         \
        default: return cudaErrorInvalidValue;                                 \
    }

cudaError_t launch_staged(const KParams &p, cudaStream_t st, int max_ctas, LaunchInfo *li) {
    void (*kern)(const KParams) = nullptr;
    const bool co = p.out == nullptr;
    HC_DISPATCH_Q(p.q, staged_kernel, co);
    const int smem = staged_smem_bytes(p.alpha, p.m, p.stage_bytes, p.stages);
    return launch_common(kern, p, kStagedThreads, smem, static_cast<int>(p.ntiles), max_ctas, st, li);
}

cudaError_t launch_gather(const KParams &p, cudaStream_t st, int max_ctas, LaunchInfo *li) {
    void (*kern)(const KParams) = nullptr;
    const bool co = p.out == nullptr;
    HC_DISPATCH_Q(p.q, gather_kernel, co);
    const int smem = gather_smem_bytes(p.alpha, p.m);
    const int warps_needed = static_cast<int>(p.nchunks);
    const int ctas = (warps_needed + kGatherThreads / 32 - 1) / (kGatherThreads / 32);
    return launch_common(kern, p, kGatherThreads, smem, ctas, max_ctas, st, li);
}

// ------------------------------------------------------------------ ordering
__global__ void widen_kernel(const uint32_t *src, int64_t *dst, uint32_t k) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
        dst[i] = static_cast<int64_t>(src[i]);
}

constexpr uint32_t kSmallSort = 8192;

// One-CTA bitonic sort of <= kSmallSort distinct keys in shared memory.
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

cudaError_t sort_and_widen(uint32_t *pos, uint32_t count, uint32_t n_bound, int64_t *dst,
                           uint32_t k, cudaStream_t st, int *launches) {
    if (k == 0) return cudaSuccess;
    if (count <= 1) {
        widen_kernel<<<1, 32, 0, st>>>(pos, dst, k);
        if (launches) ++*launches;
        return cudaGetLastError();
    }
    if (count <= kSmallSort) {
        small_sort_kernel<<<1, 1024, 0, st>>>(pos, count, dst, k);
        if (launches) ++*launches;
        return cudaGetLastError();
    }
    int end_bit = 1;
    while (end_bit < 32 && (static_cast<uint64_t>(1) << end_bit) <= n_bound) ++end_bit;
    uint32_t *alt = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t err = cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, pos, alt,
                                                     static_cast<int>(count), 0, end_bit, st);
    if (err != cudaSuccess) return err;
    err = cudaMallocAsync(reinterpret_cast<void **>(&alt), static_cast<size_t>(count) * 4 + tmp_bytes + 256, st);
    if (err != cudaSuccess) return err;
    tmp = reinterpret_cast<void *>(
        (reinterpret_cast<uintptr_t>(alt) + static_cast<size_t>(count) * 4 + 255) & ~static_cast<uintptr_t>(255));
    err = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, pos, alt, static_cast<int>(count), 0,
                                         end_bit, st);
    if (err == cudaSuccess) {
        const uint32_t blocks = min((k + 255) / 256, 148u * 8u);
        widen_kernel<<<blocks, 256, 0, st>>>(alt, dst, k);
        err = cudaGetLastError();
        if (launches) *launches += 4;  // CUB onesweep: histogram + passes; approximate
    }
    cudaError_t e2 = cudaFreeAsync(alt, st);
    return err != cudaSuccess ? err : e2;
}

}  // namespace hc
