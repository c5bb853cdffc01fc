// hc_kernels.cu — sm_100a device side of libhc: the Hash Chain searching phase
// (Fig. 5 left) as data-parallel CUDA kernels.
//
// Data parallelism (reading R11): the window ends
// [m-1, n) are cut into K segments of S = m-q+1 ends, a_k = m-1 + k*S (the
// "lattice").  HC started at a_k with loop bound b = min(a_k + S, n) reports
// exactly the occurrences ending in [a_k, b) and reads only y[a_k-m+1 .. b-1].
//
// Two phases per warp:
//   A. filter:   every lane hashes the q-gram ending at one lattice point a_k
//                (Fig. 5 l.4-5) and tests F[v] != 0 (l.6).  F[v] == 0 means the
//                segment is finished (the l.18 shift lands on a_{k+1});
//                on the paper's workloads 66-99% of segments end here.  The
//                survivors are compacted into a per-warp queue (ballot/popc).
//   B. survivor: 32 queued segments at a time, one per lane, continue the
//                paper's loop inside their segment as a flat state machine that
//                does ONE q-gram hash per iteration (window-end hash l.4-6 or
//                one walk step l.9-13), keeping the warp converged.  Long walks
//                (>= kLongWalk remaining steps) are done by the whole warp, 32
//                steps at a time (same link tests, same break point), and long
//                verifications (m > kCoopVerifyMin) compare 256 bytes per warp
//                step.
// Two text access paths:
//   staged : persistent CTAs stream tiles of the text into shared memory with
//            TMA bulk copies (cp.async.bulk + mbarrier ring); every hash reads
//            shared memory.  For small shifts, where every 32-B sector of the
//            text is touched anyway.
//   gather : no staging; lanes read only the aligned 8-byte words holding the
//            q-grams they hash (ld.global.nc).  For large shifts, where HC
//            touches a small fraction of the text (sublinear search).
// F (2^alpha u32 words) and x live in shared memory in both paths.
// Matches go to a per-warp shared buffer, flushed 32 at a time with one
// atomicAdd (ballot/popc ranks); the host orders them afterwards.

#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_radix_sort.cuh>

#include <cstdio>
#include <cstdlib>

#include "hc_internal.h"

namespace hc {

#define HC_FULL 0xffffffffu
constexpr uint32_t kWordBits = 32;       // w (R2)
constexpr uint32_t kLongWalk = 4;        // walks past this many links with as many left go warp-wide
constexpr uint32_t kCoopVerifyMin = 64;  // m above which verification is warp-wide
constexpr int kUnroll = 4;               // lattice rounds whose loads are issued together
constexpr int kWalkUnroll = 4;           // walk steps evaluated per phase-B iteration
constexpr uint32_t kSurvWarps = 2;       // staged: survivor/producer warps per CTA

// Launch parameters, copied to shared memory at kernel start so that the out-of-line
// phase-B routine can read them without a stack copy.
constexpr int kMaxPat = kMaxPatterns;   // patterns per multi-pattern launch (stream path)
__shared__ KParams s_params[kMaxPat];
constexpr uint32_t kRegion = 32;         // staged: survivor entries per filter warp per slot

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
// Programmatic dependent launch: the search kernels let the finish kernel launch
// early (its CTA then waits in griddepcontrol.wait for the search grid to complete
// and its memory to be visible), hiding the finish kernel's launch latency.
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_event(const KParams &p, uint32_t it, uint32_t ev) {
    if (p.trace && it < p.trace_tiles)
        p.trace[(static_cast<size_t>(blockIdx.x) * p.trace_tiles + it) * 4 + ev] = gtimer();
}
// CTA entry (ev 0) / exit (ev 1) stamps after the per-tile records (one thread)
__device__ __forceinline__ void trace_cta(const KParams &p, uint32_t ev) {
    if (p.trace)
        p.trace[static_cast<size_t>(gridDim.x) * p.trace_tiles * 4 + blockIdx.x * 2 + ev] = gtimer();
}
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}
// 64-bit shifts with PTX semantics: amounts >= 64 give 0 (clamped), no select needed.
__device__ __forceinline__ uint64_t shr64(uint64_t a, uint32_t s) {
    uint64_t r;
    asm("shr.b64 %0, %1, %2;" : "=l"(r) : "l"(a), "r"(s));
    return r;
}
__device__ __forceinline__ uint64_t shl64(uint64_t a, uint32_t s) {
    uint64_t r;
    asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(a), "r"(s));
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
    __device__ __forceinline__ GlobalText shfl(uint32_t) const { return *this; }  // same in all lanes
    static constexpr bool kLoSafe = false;  // the word before may be outside y
};

// Shared-memory loads by shared-space address.  Not volatile: callers make the
// address depend on a value produced after the mbarrier wait (see fence_value), so
// they cannot be hoisted above it.
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
    uint64_t r;
    asm("ld.shared.u64 %0, [%1];" : "=l"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t r;
    asm("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint32_t r;
    asm("ld.shared.u8 %0, [%1];" : "=r"(r) : "r"(a));
    return r;
}
// Opaque copy of v, ordered after every earlier volatile asm (e.g. an mbarrier wait).
__device__ __forceinline__ uint32_t fence_value(uint32_t v) {
    asm volatile("mov.b32 %0, %0;" : "+r"(v) :: "memory");
    return v;
}

// Text byte p read from a shared-memory stage: byte p is at shared address base + p
// (mod 2^32; the stage is 16-aligned so addresses keep y's alignment mod 16).
struct SmemText {
    uint32_t base;
    __device__ __forceinline__ uint32_t addr(uint32_t p) const { return base + p; }
    __device__ __forceinline__ uint64_t word(uint32_t aligned) const { return lds64(aligned); }
    __device__ __forceinline__ uint32_t byte(uint32_t p) const { return lds8(base + p); }
    // lane L's mapping (survivor boxes: every lane has its own)
    __device__ __forceinline__ SmemText shfl(uint32_t L) const {
        return SmemText{__shfl_sync(0xffffffffu, base, L)};
    }
    static constexpr bool kLoSafe = true;   // stages/boxes never start at shared offset 0
};

// F (2^alpha words) in shared memory, addressed by shared-space address.
struct FTable {
    uint32_t base;
    __device__ __forceinline__ uint32_t operator[](uint32_t v) const { return lds32(base + 4 * v); }
    __device__ __forceinline__ bool pass(uint32_t v) const { return (*this)[v] != 0u; }   // l.6
};
// The 8 text bytes y[p-7 .. p] as a little-endian u64 (byte 7 = y[p]).  Only the
// top Q bytes are meaningful.  Reads just the aligned 8-byte words holding y[p]
// and y[p-Q+1] (both inside the text), so no byte outside [0, n) is touched.
template <int Q, class T>
__device__ __forceinline__ uint64_t end8(const T &t, uint32_t p) {
    auto a = t.addr(p);
    using A = decltype(a);
    const A ah = a & ~static_cast<A>(7);
    const uint32_t off = static_cast<uint32_t>(a & 7);
    const uint64_t hi = t.word(ah);
    uint64_t lo = 0;
    if constexpr (Q > 1) {
        if (T::kLoSafe || off + 1 < static_cast<uint32_t>(Q)) lo = t.word(ah - 8);
    }
    return shr64(lo, 8 * (off + 1)) | shl64(hi, 56 - 8 * off);
}

// Eq. 3 / Fig. 3 Hash: v = 0; for i = p downto p-q+1:
// v = (v << s) + y[i]; return v & mask, i.e. v = sum_i c_i 2^(s i) with c_0 the
// first byte of the q-gram (reading R4).  With q and s compile-time, the sum is
// evaluated with dp4a: bytes of one 32-bit half whose weights 2^(s (i - i0)) fit
// in 8 bits form one group; v = sum_g dp4a(half_g, weights_g) << (s i0_g).
struct HashPlan {
    int n;
    int reg[8];
    uint32_t w[8];
    int sh[8];
};
template <int Q, int SH>
__host__ __device__ constexpr HashPlan make_plan() {
    HashPlan P{0, {0, 0, 0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0, 0, 0}};
    int i = 0;
    while (i < Q) {
        const int b = 8 - Q + i;  // byte of W holding c_i
        const int reg = b >= 4 ? 1 : 0;
        const int i0 = i;
        uint32_t w = 0;
        int j = i;
        while (j < Q) {
            const int bj = 8 - Q + j;
            if ((bj >= 4 ? 1 : 0) != reg || SH * (j - i0) > 7) break;
            w |= (1u << (SH * (j - i0))) << (8 * (bj & 3));
            ++j;
        }
        P.reg[P.n] = reg;
        P.w[P.n] = w;
        P.sh[P.n] = SH * i0;
        P.n++;
        i = j;
    }
    return P;
}
template <int Q, int SH>
__device__ __forceinline__ uint32_t qhash(uint64_t W, uint32_t mask) {
    constexpr HashPlan P = make_plan<Q, SH>();
    const uint32_t lo = static_cast<uint32_t>(W), hi = static_cast<uint32_t>(W >> 32);
    uint32_t v = 0;
#pragma unroll
    for (int g = 0; g < P.n; ++g) v += __dp4a(P.reg[g] ? hi : lo, P.w[g], 0u) << P.sh[g];
    return v & mask;
}

// Fig. 5 l.16 verification by one lane: y[start .. start+m-1] == x (sx: x in
// shared memory, 16-aligned).  8 bytes per step, then a byte tail.
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

// The same comparison done by the whole warp, 4 x 8 bytes per lane per round.
template <class T>
__device__ __forceinline__ bool verify_warp(const T &t, const uint8_t *sx, uint32_t start,
                                            uint32_t m, uint32_t lane) {
    for (uint32_t k0 = 0; k0 < m; k0 += 1024) {
        bool bad = false;
#pragma unroll
        for (uint32_t r = 0; r < 4; ++r) {
            const uint32_t k = k0 + 256 * r + 8 * lane;
            if (k + 8 <= m) {
                bad |= end8<8>(t, start + k + 7) != *reinterpret_cast<const uint64_t *>(sx + k);
            } else {
                for (uint32_t kk = k; kk < m; ++kk) bad |= t.byte(start + kk) != sx[kk];
            }
        }
        if (__any_sync(HC_FULL, bad)) return false;
    }
    return true;
}

// Fig. 5 l.8-13 for one lane's walk, done by the whole warp: lane l evaluates steps
// t = 4l .. 4l+3 of the next 128 (hash of the q-gram ending at j-(t+1)q, its word
// F[v_t]); the link test of step t uses the word of step t-1 (previous register, or
// the previous lane's last one).  The first failing step is the sequential loop's
// break (l.12).  On return j is the position of the last evaluated step (the
// failing one if broke) and v its hash.  On global text the window is prefetched
// into L2 first, so the rounds and the verification that follows hit L2.
template <int Q, int SH, class T, class FT>
__device__ __forceinline__ void walk_warp(const KParams &p, const T &txt, const FT &sF,
                                          uint32_t lane, uint32_t &j, uint32_t i, uint32_t z,
                                          uint32_t &v, bool &broke) {
    constexpr uint32_t PL = 4;                    // steps per lane per round
    uint32_t R = (j - i) / Q + 1;                 // steps while j >= i
    if constexpr (!T::kLoSafe) {
        const uintptr_t lo = (txt.addr(j - R * Q - 7)) & ~static_cast<uintptr_t>(127);
        const uintptr_t hi = txt.addr(j);
        for (uintptr_t a = lo + 128 * lane; a <= hi; a += 128 * 32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
    broke = false;
    while (true) {
        const uint32_t steps = min(R, 32u * PL);
        uint32_t vt[PL], zt[PL];
#pragma unroll
        for (uint32_t s = 0; s < PL; ++s) {
            const uint32_t t = PL * lane + s;
            vt[s] = t < steps ? qhash<Q, SH>(end8<Q>(txt, j - (t + 1) * Q), p.mask) : 0u;
        }
#pragma unroll
        for (uint32_t s = 0; s < PL; ++s) zt[s] = PL * lane + s < steps ? sF[vt[s]] : 0u;
        uint32_t zprev = __shfl_up_sync(HC_FULL, zt[PL - 1], 1);
        if (lane == 0) zprev = z;
        uint32_t first = 0xffffffffu;             // first failing step of this lane
#pragma unroll
        for (int s = PL - 1; s >= 0; --s) {
            const uint32_t zp = s == 0 ? zprev : zt[s - 1];
            const bool ok = (zp >> (vt[s] & (kWordBits - 1))) & 1u;
            if (PL * lane + s < steps && !ok) first = PL * lane + s;
        }
        const uint32_t tmin = __reduce_min_sync(HC_FULL, first);
        const uint32_t tv = tmin != 0xffffffffu ? tmin : steps - 1;   // step whose hash is v
        uint32_t vsel = vt[0], zsel = zt[0];
#pragma unroll
        for (uint32_t s = 1; s < PL; ++s)
            if ((tv & (PL - 1)) == s) {
                vsel = vt[s];
                zsel = zt[s];
            }
        v = __shfl_sync(HC_FULL, vsel, tv / PL);
        if (tmin != 0xffffffffu) {
            j -= (tmin + 1) * Q;
            broke = true;
            return;
        }
        z = __shfl_sync(HC_FULL, zsel, tv / PL);
        j -= steps * Q;
        R -= steps;
        if (R == 0) return;
    }
}

// Per-warp match buffer: positions are appended (ballot rank) and flushed to
// global memory 32 at a time with one atomicAdd.  Count-only calls have cap 0:
// the same counting, no position writes.
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

// Phase B: HC (Fig. 5) on one segment per active lane, from the window end `start`
// inside the segment (the lattice point a_k, or where first_steps left it), warp-
// synchronous.  Each iteration a lane evaluates its window-end hash (l.4-6) and up to
// kWalkUnroll walk steps (l.9-13): the hashes and F words of all positions it may
// need (j, j-q, ..., never below the window) are loaded in parallel, then the link
// tests run in registers in the paper's order, so the result is the sequential
// loop's; one iteration costs one shared/global round trip instead of one per step.
template <int Q, int SH, class T, class FT>
__device__ __noinline__ uint32_t run_segments_impl(const T txt, const FT sF, const uint8_t *sx,
                                                   bool active, uint32_t start, uint32_t *wbuf,
                                                   uint32_t wcnt, uint32_t lane, uint32_t pi) {
    // One out-of-line copy per kernel: phase B is cold relative to the filter loop and
    // inlining it at every call site multiplied the kernel's code size (I-cache misses).
    // The launch parameters of pattern pi are read from shared memory.
    const KParams &p = s_params[pi];
    WarpOut wo{wbuf, wcnt};
    constexpr int U = kWalkUnroll;
    uint32_t j = start;                        // a window end inside segment k
    const uint32_t k = (start - (p.m - 1)) / p.S;
    const uint32_t b = min(p.m - 1 + (k + 1) * p.S, p.n);   // segment bound
    uint32_t e = 0, i = 0, z = 0, v = 0, wsteps = 0;
    bool walk = false;
    const bool long_walks = p.m >= 2 * kLongWalk * Q;   // warp-wide walks can pay off
    if (p.debug == 5 && lane == 0) atomicAdd(p.counter + 3, 1u);
    while (__any_sync(HC_FULL, active)) {
        if (p.debug == 5 && lane == 0) atomicAdd(p.counter + 2, 1u);
        bool need_v = false, stepped = false;
        if (long_walks) {
            // walks that passed kLongWalk link tests and still have >= kLongWalk steps to
            // go (near-matches, true matches) finish warp-wide, one lane at a time
            uint32_t lm = __ballot_sync(HC_FULL, active && walk && wsteps >= kLongWalk &&
                                                     (j - i) >= kLongWalk * Q);
            while (lm) {
                const uint32_t L = __ffs(lm) - 1;
                lm &= lm - 1;
                uint32_t jL = __shfl_sync(HC_FULL, j, L);
                const uint32_t iL = __shfl_sync(HC_FULL, i, L);
                const uint32_t zL = __shfl_sync(HC_FULL, z, L);
                uint32_t vL = 0;
                bool broke = false;
                walk_warp<Q, SH>(p, txt.shfl(L), sF, lane, jL, iL, zL, vL, broke);
                if (lane == L) {
                    stepped = true;
                    walk = false;
                    v = vL;
                    if (broke) {
                        j = jL + p.S;                              // l.12 -> l.18
                    } else {
                        need_v = v == p.hv;                        // l.14-16
                        j = e + 1;                                 // (i - q) + (m - q + 1)
                    }
                    if (j >= b) active = false;
                }
            }
        }
        if (active && !stepped) {
            // positions this iteration may hash: j (window end, if not walking) and
            // j - t q for the walk steps t = 1..U still allowed (j - (t-1) q >= i)
            const uint32_t ii = walk ? i : j + 2 * Q - p.m;    // l.7
            const uint32_t R = j >= ii ? (j - ii) / Q + 1 : 0u;
            uint32_t vv[U + 1], zz[U + 1];
#pragma unroll
            for (int t = 0; t <= U; ++t) {
                const bool need = t == 0 ? !walk : static_cast<uint32_t>(t) <= R;
                vv[t] = need ? qhash<Q, SH>(end8<Q>(txt, j - t * Q), p.mask) : 0u;
            }
#pragma unroll
            for (int t = 0; t <= U; ++t) {
                const bool need = t == 0 ? !walk : static_cast<uint32_t>(t) <= R;
                zz[t] = need ? sF[vv[t]] : 0u;
            }
            bool complete = false;
            if (!walk) {                                       // l.4-7
                e = j;
                v = vv[0];
                z = zz[0];
                if (z == 0) {
                    j += p.S;                                  // l.18 fast path
                } else {
                    i = ii;
                    if (j >= i) {                              // l.8
                        walk = true;
                        wsteps = 0;
                    } else {
                        complete = true;                       // m < 2q: while-else (R7)
                    }
                }
            }
#pragma unroll
            for (int t = 1; t <= U; ++t) {                     // l.9-13, in order
                if (walk) {
                    j -= Q;
                    v = vv[t];
                    ++wsteps;
                    if (((z >> (v & (kWordBits - 1))) & 1u) == 0) {
                        walk = false;                          // l.12 break
                        j += p.S;                              // l.18
                    } else {
                        z = zz[t];                             // l.13
                        if (j < i) {
                            walk = false;
                            complete = true;
                        }
                    }
                }
            }
            if (complete) {                                    // l.14-16, index per R1
                need_v = v == p.hv;
                j = e + 1;
            }
            if (!walk && j >= b) active = false;
        }
        bool found = false;
        if (p.m > kCoopVerifyMin) {
            uint32_t vm = __ballot_sync(HC_FULL, need_v);
            while (vm) {
                const uint32_t L = __ffs(vm) - 1;
                vm &= vm - 1;
                const uint32_t st = __shfl_sync(HC_FULL, e + 1 - p.m, L);
                const bool ok = verify_warp(txt.shfl(L), sx, st, p.m, lane);
                if (lane == L) found = ok;
            }
        } else if (need_v) {
            found = verify(txt, sx, e + 1 - p.m, p.m);
        }
        wo.push(found, e + 1 - p.m, p, lane);                 // l.17
    }
    return wo.cnt;
}

template <int Q, int SH, class T, class FT>
__device__ __forceinline__ void run_segments(const KParams &, const T &txt, const FT &sF,
                                             const uint8_t *sx, bool active, uint32_t start,
                                             WarpOut &wo, uint32_t lane, uint32_t pi = 0) {
    wo.cnt = run_segments_impl<Q, SH, T, FT>(txt, sF, sx, active, start, wo.buf, wo.cnt, lane, pi);
}

// Phase B on `cnt` <= 32 queued segments (queue[lane]), one per lane.
template <int Q, int SH, class T, class FT>
__device__ __forceinline__ void run_survivors(const KParams &p, const T &txt, const FT &sF,
                                              const uint8_t *sx, const uint32_t *queue,
                                              uint32_t cnt, WarpOut &wo, uint32_t lane,
                                              uint32_t pi = 0) {
    const bool active = lane < cnt;
    const uint32_t k = active ? queue[lane] : 0u;
    __syncwarp();
    run_segments<Q, SH>(p, txt, sF, sx, active, k, wo, lane, pi);
}

// Phase A over lattice points [seg_lo, seg_hi), 32 * kUnroll per warp step: every
// lane hashes the q-gram ending at its lattice point a_k = m-1 + k S (Fig. 5 l.4)
// and tests F[v] != 0 (l.6).  Survivor segments are handed to `sink` (warp-uniform
// call, ballot mask + the lane's window end a_k).  Full steps run without bounds checks.
template <int Q, int SH, class T, class FT, class Sink>
__device__ __forceinline__ void filter_lattice(const KParams &p, const T &txt, const FT &sF,
                                               uint32_t seg_lo, uint32_t seg_hi, uint32_t lane,
                                               Sink &&sink) {
    const uint32_t step = 32 * p.S;
    uint32_t pos = p.m - 1 + (seg_lo + lane) * p.S;   // window end of lattice point seg_lo+lane
    uint32_t k0 = seg_lo;
    for (; k0 + 32 * kUnroll <= seg_hi; k0 += 32 * kUnroll, pos += kUnroll * step) {
        uint64_t W[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) W[u] = end8<Q>(txt, pos + u * step);
        bool pass[kUnroll];
        bool any = false;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            pass[u] = sF.pass(qhash<Q, SH>(W[u], p.mask));
            any |= pass[u];
        }
        if (__any_sync(HC_FULL, any)) {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const uint32_t bm = __ballot_sync(HC_FULL, pass[u]);
                if (bm) sink(bm, pass[u], pos + u * step);
            }
        }
    }
    for (; k0 < seg_hi; k0 += 32, pos += step) {       // ragged tail, one round at a time
        const bool in = k0 + lane < seg_hi;
        const bool pass = in && sF.pass(qhash<Q, SH>(end8<Q>(txt, pos), p.mask));
        const uint32_t bm = __ballot_sync(HC_FULL, pass);
        if (bm) sink(bm, pass, pos);
    }
}

// first_steps: the first steps of Fig. 5 for the window e = a_k of a lattice survivor
// (F[v_0] != 0 already, l.6), evaluated lane-parallel, when m >= 2q: the walk's first
// step (l.9-12) tests the link bit of v_1 = h(y[e-2q+1..e-q]) in F[v_0]; if it is
// clear the loop breaks and the next window ends at j = e - q + S (l.18); if
// F[h(j)] == 0 that window shifts by S again (l.6) to j + S >= a_k + S, out of
// the segment (R11), and the segment is finished (returns false).  Otherwise the
// segment continues at `start` = e (link set) or j.  Exact: these are the paper's
// steps in order, with the three hashes loaded in parallel.  On DNA this finishes
// ~90% of the lattice survivors for one memory round trip per 32.
template <int Q, int SH, class T, class FT>
__device__ __forceinline__ bool first_steps_eval(const KParams &p, const T &txt, const FT &sF,
                                                 bool act, uint32_t e, uint32_t &start) {
    start = e;
    if (!act) return false;
    if (p.m < 2 * Q) return true;                        // no walk step to test (R7)
    const uint32_t j = e - Q + p.S;
    const bool jin = j < p.n;                            // else the break leaves the text
    const uint64_t W0 = end8<Q>(txt, e), W1 = end8<Q>(txt, e - Q);
    const uint64_t W2 = end8<Q>(txt, jin ? j : e);
    const uint32_t v1 = qhash<Q, SH>(W1, p.mask);
    const uint32_t z0 = sF[qhash<Q, SH>(W0, p.mask)];
    const uint32_t z2 = sF[qhash<Q, SH>(W2, p.mask)];
    if (((z0 >> (v1 & (kWordBits - 1))) & 1u) != 0u) return true;   // link set: walk on
    start = j;                                           // break at the first step
    return jin && z2 != 0u;
}

// Gather path sink: lattice survivors (k) are queued per warp (q1) and run 32 at a
// time through first_steps_eval; the segments that continue go to a second queue
// (q2, window ends) that runs phase B whenever 32 are queued (both queues may span
// chunks, since the survivors read global memory).
template <int Q, int SH, class T, class FT = FTable>
struct WarpQueueSink {
    const KParams &p;
    const T &txt;
    const FT &sF;
    const uint8_t *sx;
    uint32_t *q1, *q2;     // kWarpBuf entries each: lattice survivors' a_k / window ends
    uint32_t n1, n2;       // warp-uniform
    WarpOut &wo;
    uint32_t lane;
    uint32_t pi = 0;       // pattern index (launch parameters s_params[pi])
    __device__ __forceinline__ void steps(uint32_t c) {  // first steps of q1[0..c) -> q2
        const bool act = lane < c;
        steps_e(act, act ? q1[lane] : 0u);
    }
    // first steps of the lattice survivor a_k = e of each active lane -> q2
    __device__ __forceinline__ void steps_e(bool act, uint32_t e) { steps_e_on(txt, act, e); }
    // the same, reading the first steps' q-grams from `t2` (e.g. a shared-memory stage)
    template <class T2>
    __device__ __forceinline__ void steps_e_on(const T2 &t2, bool act, uint32_t e) {
        uint32_t start;
        const bool keep = first_steps_eval<Q, SH>(p, t2, sF, act, e, start);
        const uint32_t bm = __ballot_sync(HC_FULL, keep);
        if (keep) q2[n2 + __popc(bm & lanemask_lt())] = start;
        n2 += __popc(bm);
        if (n2 >= 32) {
            __syncwarp();
            run_survivors<Q, SH>(p, txt, sF, sx, q2, 32, wo, lane, pi);
            const uint32_t rest = n2 - 32;
            const uint32_t nv = lane < rest ? q2[32 + lane] : 0u;
            __syncwarp();
            if (lane < rest) q2[lane] = nv;
            __syncwarp();
            n2 = rest;
        }
    }
    __device__ __forceinline__ void operator()(uint32_t bm, bool pass, uint32_t e) {
        if (pass) q1[n1 + __popc(bm & lanemask_lt())] = e;
        n1 += __popc(bm);
        if (n1 >= 32) {
            __syncwarp();
            steps(32);
            const uint32_t rest = n1 - 32;
            const uint32_t nv = lane < rest ? q1[32 + lane] : 0u;
            __syncwarp();
            if (lane < rest) q1[lane] = nv;
            __syncwarp();
            n1 = rest;
        }
    }
    __device__ __forceinline__ void drain() {
        if (n1) {
            __syncwarp();
            steps(n1);
            n1 = 0;
        }
        if (n2) {
            __syncwarp();
            run_survivors<Q, SH>(p, txt, sF, sx, q2, n2, wo, lane, pi);
            n2 = 0;
        }
    }
};

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
        if (p.debug == 3) return;                        // phase A only (measurement)
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
__host__ __device__ inline uint32_t round_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }
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

int staged_smem_bytes(uint32_t alpha, uint32_t m, uint32_t stage_bytes, uint32_t stages,
                      uint32_t slot_bytes, uint32_t nbox) {
    return static_cast<int>(
        staged_layout(alpha, m, stage_bytes, stages, kStagedThreads / 32, slot_bytes, nbox).total);
}
int gather_smem_bytes(uint32_t alpha, uint32_t m) {
    return static_cast<int>(gather_layout(alpha, m, kGatherThreads / 32).total);
}

__device__ __forceinline__ void load_table(const KParams &p, uint32_t *sF, uint8_t *sx) {
    const uint32_t nF = 1u << p.alpha;
    if (nF >= 4) {
        const uint4 *src = reinterpret_cast<const uint4 *>(p.F);
        uint4 *dst = reinterpret_cast<uint4 *>(sF);
        for (uint32_t w = threadIdx.x; w < nF / 4; w += blockDim.x) dst[w] = __ldg(src + w);
    } else {
        for (uint32_t w = threadIdx.x; w < nF; w += blockDim.x) sF[w] = __ldg(p.F + w);
    }
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

__device__ __forceinline__ uint32_t ld_volatile_shared(const uint32_t *a) {
    return *reinterpret_cast<const volatile uint32_t *>(a);
}
__device__ __forceinline__ void st_volatile_shared(uint32_t *a, uint32_t v) {
    *reinterpret_cast<volatile uint32_t *>(a) = v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(a));
    return r;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
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
    if (tid == 0) trace_cta(p, 0);
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
    const bool dynamic = p.debug != 6;

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
            if (p.debug != 1) {
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
            const uint32_t total = p.debug == 3 ? 0u : __shfl_sync(HC_FULL, incl, NF - 1);
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
            const GlobalText gtxt{p.y};
            for (uint32_t b = 0; b < nm; b += 32) {
                const bool act = b + lane < nm;
                run_segments<Q, SH>(p, gtxt, sF, sx, act, act ? mine[b + lane] : 0u, wo, lane);
            }
            __syncwarp();
            if (lane == 0) trace_event(p, it, 2);
        }
    }
    wo.flush(p, lane);
    if (lane == 0) trace_cta(p, 1);   // last warp to get here wins
}

template <int Q, int SH>
__global__ void __launch_bounds__(kGatherThreads) gather_kernel(const KParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr uint32_t NW = kGatherThreads / 32;
    const GatherLayout L = gather_layout(p.alpha, p.m, NW);
    uint32_t *sFp = reinterpret_cast<uint32_t *>(smem + L.f_off);
    uint8_t *sx = smem + L.x_off;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) trace_cta(p, 0);
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
    if (warp == 0 && lane == 0) trace_event(p, 0, 0);          // table loaded
    for (uint32_t c = blockIdx.x * NW + warp; c < p.nchunks; c += total_warps) {
        const uint32_t seg_lo = c * p.seg_per_chunk;
        const uint32_t seg_hi = min(seg_lo + p.seg_per_chunk, p.K);
        filter_lattice<Q, SH>(p, txt, sF, seg_lo, seg_hi, lane, sink);
    }
    if (warp == 0 && lane == 0) trace_event(p, 0, 1);          // lattice filtered
    sink.drain();
    if (warp == 0 && lane == 0) trace_event(p, 0, 2);          // survivors done
    wo.flush(p, lane);
    if (lane == 0) trace_cta(p, 1);   // last warp to get here wins
}

// ------------------------------------------------------------------ stream kernel
// Small shifts (S <= 32), every text sector is read (f(m) = 1).  Each warp
// owns a contiguous run of segments per chunk and stages exactly the chunk's lattice
// q-gram bytes [k0 S + S - 1, k1 S + q - 2] into its own shared-memory buffer with
// 16-byte cp.async copies (coalesced, L2-only), kStreamBufs - 1 chunks ahead of the
// one it filters: no CTA-wide barrier, no hand-off between warps.  Phase A reads the
// buffer; the lattice survivors go through first_steps and phase B on global text
// (the chunk was just streamed through L2), exactly as on the gather path.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

#ifndef HC_STREAM_UNROLL
#define HC_STREAM_UNROLL 4
#endif
constexpr int kStreamUnroll = HC_STREAM_UNROLL;        // stream: lattice rounds per trip
constexpr uint32_t kStreamQ1 = 32 * (kStreamUnroll + 1);   // lattice survivor queue per warp
struct StreamLayout {
    uint32_t f_off, x_off, q_off, q2_off, wbuf_off, ctr_off, buf_off, total;
};
__host__ __device__ inline StreamLayout stream_layout(uint32_t alpha, uint32_t m, uint32_t nwarps,
                                                      uint32_t buf_bytes, uint32_t bufs) {
    StreamLayout L;
    L.f_off = 0;
    L.x_off = round_up((1u << alpha) * 4u, 16);
    L.q_off = L.x_off + round_up(m + 8, 16);
    L.q2_off = L.q_off + nwarps * kStreamQ1 * 4u;
    L.wbuf_off = L.q2_off + nwarps * kWarpBuf * 4u;
    L.ctr_off = L.wbuf_off + nwarps * kWarpBuf * 4u;
    // per-warp counters, then 4 mbarriers per warp (TMA variant)
    L.buf_off = round_up(round_up(L.ctr_off + nwarps * 4u, 8) + nwarps * 32u + 16, 128);
    L.total = L.buf_off + nwarps * bufs * buf_bytes;
    return L;
}
int shc_smem_bytes(uint32_t alpha, uint32_t m, uint32_t buf_bytes, uint32_t box_bytes,
                   uint32_t nwarps) {
    const uint32_t x_off = round_up((1u << alpha) * 4u, 16);
    const uint32_t ring_off = round_up(x_off + round_up(m + 8, 16) + 16, 128);
    return static_cast<int>(ring_off + nwarps * 2 * buf_bytes + nwarps * 32 * box_bytes);
}
int stream_smem_bytes(uint32_t alpha, uint32_t m, uint32_t buf_bytes, uint32_t bufs,
                      uint32_t nwarps) {
    return static_cast<int>(stream_layout(alpha, m, nwarps, buf_bytes, bufs).total);
}

// Text bytes of chunk c: the q-grams ending at a_k, k in [k0, k1), and at a_k - q and
// a_k - q + S (the first steps of Fig. 5 for a lattice survivor).
struct StreamChunk {
    uint32_t k0, k1, first, last;   // bytes [first, last] of y
};
__device__ __forceinline__ StreamChunk stream_chunk(const KParams &p, uint32_t c) {
    StreamChunk g;
    g.k0 = c * p.seg_per_chunk;
    g.k1 = min(g.k0 + p.seg_per_chunk, p.K);
    if (p.shc) {
        // SHC path: whole segments, [a_k0 - m + 1, min(a_k1, n) - 1] (every window)
        g.first = g.k0 * p.S;
        g.last = min(p.m - 1 + g.k1 * p.S, p.n) - 1;
        return g;
    }
    // bytes [a_k0 - 2q + 1, a_{k1} - q]: the lattice q-grams plus those of the first
    // steps (first_steps_eval reads the q-grams ending at a_k - q and a_k - q + S)
    const uint32_t a0 = p.m - 1 + g.k0 * p.S;
    g.first = a0 + 1 >= 2 * p.q ? a0 + 1 - 2 * p.q : 0u;
    const uint32_t alast = p.m - 1 + (g.k1 - 1) * p.S;
    g.last = max(alast, min(alast + p.S - p.q, p.n - 1));
    return g;
}
// Issues chunk c's copies into the buffer at shared address `buf` (one warp).  The
// 16-byte words wholly inside y are copied with cp.async; the bytes of the partial
// words at the two ends of an unaligned text are stored directly (first/last chunk).
__device__ __forceinline__ void stream_issue(const KParams &p, uint32_t c, uint32_t buf,
                                             uint32_t lane) {
    if (c < p.nchunks) {
        const StreamChunk g = stream_chunk(p, c);
        const uintptr_t y = reinterpret_cast<uintptr_t>(p.y);
        const uintptr_t A = (y + g.first) & ~static_cast<uintptr_t>(15);
        const uint32_t nbytes =
            static_cast<uint32_t>(((y + g.last + 16) & ~static_cast<uintptr_t>(15)) - A);
        const uintptr_t ye = y + p.n;
        if (A >= y && A + nbytes <= ye) {               // warp-uniform: interior chunk
            const uint8_t *src = reinterpret_cast<const uint8_t *>(A);
            for (uint32_t o = 16 * lane; o < nbytes; o += 16 * 32) cp_async16(buf + o, src + o);
        } else {
            for (uint32_t o = 16 * lane; o < nbytes; o += 16 * 32) {
                const uintptr_t a = A + o;
                if (a >= y && a + 16 <= ye) {
                    cp_async16(buf + o, reinterpret_cast<const void *>(a));
                } else {
                    for (uint32_t b = 0; b < 16; ++b)
                        if (a + b >= y && a + b < ye)
                            asm volatile("st.shared.u8 [%0], %1;" ::"r"(buf + o + b),
                                         "r"(static_cast<uint32_t>(
                                             __ldg(reinterpret_cast<const uint8_t *>(a + b))))
                                         : "memory");
                }
            }
        }
    }
    cp_async_commit();   // one group per issue (possibly empty) keeps the count uniform
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
    // first steps of 32 queued survivors, on the chunk's stage (the queue only ever
    // holds survivors of the chunk being filtered: it is drained at the chunk's end)
    __device__ __forceinline__ void drain32(WarpQueueSink<Q, SH, GlobalText> &sink,
                                            const SmemText &txt, uint32_t lane) {
        __syncwarp();
        const uint32_t e = q1[n1 - 32 + lane];
        n1 -= 32;
        __syncwarp();
        if (lane == 0) *ctr = n1;
        __syncwarp();
        sink.steps_e_on(txt, true, e);
    }
    __device__ __forceinline__ void drain_all(WarpQueueSink<Q, SH, GlobalText> &sink,
                                              const SmemText &txt, uint32_t lane) {
        while (n1 >= 32) drain32(sink, txt, lane);
        if (n1) {
            __syncwarp();
            const bool act = lane < n1;
            const uint32_t e = act ? q1[lane] : 0u;
            n1 = 0;
            __syncwarp();
            if (lane == 0) *ctr = 0;
            __syncwarp();
            sink.steps_e_on(txt, act, e);
        }
    }
};

template <int Q, int SH>
__device__ __forceinline__ void stream_filter(const KParams &p, const SmemText &txt, const FTable &sF,
                                              uint32_t k0, uint32_t k1, uint32_t lane,
                                              StreamQueue<Q, SH> &qu,
                                              WarpQueueSink<Q, SH, GlobalText> &sink) {
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
            if (p.debug == 3) pm = 0;                   // phase A alone (measurement)
            const uint32_t c = __popc(pm);
            const uint32_t tot = __reduce_add_sync(HC_FULL, c);
            if (tot) {
                if (c) {
                    uint32_t slot = atomicAdd(qu.ctr, c);
#pragma unroll
                    for (int u = 0; u < kStreamUnroll; ++u)
                        if ((pm >> u) & 1u) qu.q1[slot++] = pos + u * step;
                }
                qu.n1 += tot;
            }
            k += 32 * kStreamUnroll;
            pos += kStreamUnroll * step;
        }
        if (qu.n1 < 32) break;
        qu.drain32(sink, txt, lane);
    }
    for (; k < k1; k += 32, pos += step) {          // ragged tail, one round at a time
        const bool in = k + lane < k1;
        const bool pass = in && sF.pass(qhash<Q, SH>(end8<Q>(txt, pos), p.mask));
        const uint32_t bm = __ballot_sync(HC_FULL, pass);
        if (bm) {
            if (pass) qu.q1[qu.n1 + __popc(bm & lanemask_lt())] = pos;
            qu.n1 += __popc(bm);
            __syncwarp();
            if (lane == 0) *qu.ctr = qu.n1;
            if (qu.n1 >= 32) qu.drain32(sink, txt, lane);
        }
    }
}

template <int Q, int SH, int NB>
__device__ __forceinline__ void stream_loop(const KParams &p, const FTable &sF,
                                            WarpQueueSink<Q, SH, GlobalText> &sink,
                                            StreamQueue<Q, SH> &qu, uint32_t bufs0,
                                            uint32_t gw, uint32_t total_warps, uint32_t lane) {
    const uint32_t y32 = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p.y));
#pragma unroll
    for (int b = 0; b < NB - 1; ++b) stream_issue(p, gw + b * total_warps, bufs0 + b * p.stage_bytes, lane);
    uint32_t b = 0;
    for (uint32_t c = gw; c < p.nchunks; c += total_warps) {
        // refill the buffer filtered last round with the chunk NB-1 ahead
        const uint32_t bn = b == 0 ? NB - 1 : b - 1;
        stream_issue(p, c + (NB - 1) * total_warps, bufs0 + bn * p.stage_bytes, lane);
        cp_async_wait<NB - 1>();   // chunk c's group is complete (this lane's copies)
        __syncwarp();              // ... and every lane's, visible to the warp
        const StreamChunk g = stream_chunk(p, c);
        const uint32_t buf = fence_value(bufs0 + b * p.stage_bytes);
        const SmemText txt{buf + ((y32 + g.first) & 15u) - g.first};
        if (p.debug != 1) {
            stream_filter<Q, SH>(p, txt, sF, g.k0, g.k1, lane, qu, sink);
            qu.drain_all(sink, txt, lane);
        }
        __syncwarp();              // every lane is done with buffer b before its refill
        b = b + 1 == NB ? 0 : b + 1;
    }
    cp_async_wait<0>();
}

// The same loop with each chunk moved by ONE 1-D TMA bulk copy (cp.async.bulk, issued
// by lane 0, completion on the buffer's mbarrier) instead of 16-byte cp.async per lane;
// the partial 16-byte words at the two ends of an unaligned text are stored by the
// lanes (first / last chunk only).
template <int Q, int SH, int NB>
__device__ __forceinline__ void stream_loop_tma(const KParams &p, const FTable &sF,
                                                WarpQueueSink<Q, SH, GlobalText> &sink,
                                                StreamQueue<Q, SH> &qu, uint32_t bufs0, uint64_t *bar,
                                                uint32_t gw, uint32_t total_warps, uint32_t lane) {
    const uint32_t y32 = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p.y));
    const uintptr_t y = reinterpret_cast<uintptr_t>(p.y), ye = y + p.n;
    if (lane == 0) {
        for (int b = 0; b < NB; ++b) mbar_init(&bar[b], 1);
        fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](uint32_t c, uint32_t b) {
        if (c >= p.nchunks) return;
        const StreamChunk g = stream_chunk(p, c);
        const uintptr_t A = (y + g.first) & ~static_cast<uintptr_t>(15);
        const uint32_t nbytes =
            static_cast<uint32_t>(((y + g.last + 16) & ~static_cast<uintptr_t>(15)) - A);
        const uint32_t buf = bufs0 + b * p.stage_bytes;
        const uintptr_t lo = max(A, (y + 15) & ~static_cast<uintptr_t>(15));
        const uintptr_t hi = min(A + nbytes, ye & ~static_cast<uintptr_t>(15));
        if (A < lo || A + nbytes > hi) {                 // edge chunk: bytes outside [lo, hi)
            for (uintptr_t a = A + lane; a < A + nbytes; a += 32)
                if ((a < lo || a >= hi) && a >= y && a < ye)
                    asm volatile("st.shared.u8 [%0], %1;" ::"r"(buf + static_cast<uint32_t>(a - A)),
                                 "r"(static_cast<uint32_t>(__ldg(reinterpret_cast<const uint8_t *>(a))))
                                 : "memory");
        }
        __syncwarp();
        if (lane == 0) {
            fence_proxy_async();                         // earlier generic reads of the buffer
            if (hi > lo) {
                mbar_arrive_expect_tx(&bar[b], static_cast<uint32_t>(hi - lo));
                bulk_g2s(buf + static_cast<uint32_t>(lo - A), reinterpret_cast<const void *>(lo),
                         static_cast<uint32_t>(hi - lo), &bar[b]);
            } else {
                mbar_arrive(&bar[b]);
            }
        }
    };
#pragma unroll
    for (int b = 0; b < NB - 1; ++b) issue(gw + b * total_warps, b);
    uint32_t b = 0, par = 0;   // par: bit b = phase parity of buffer b's next completion
    for (uint32_t c = gw; c < p.nchunks; c += total_warps) {
        const uint32_t bn = b == 0 ? NB - 1 : b - 1;
        issue(c + (NB - 1) * total_warps, bn);
        mbar_wait(&bar[b], (par >> b) & 1u);
        par ^= 1u << b;
        const StreamChunk g = stream_chunk(p, c);
        const uint32_t buf = fence_value(bufs0 + b * p.stage_bytes);
        const SmemText txt{buf + ((y32 + g.first) & 15u) - g.first};
        if (p.debug != 1) {
            stream_filter<Q, SH>(p, txt, sF, g.k0, g.k1, lane, qu, sink);
            qu.drain_all(sink, txt, lane);
        }
        __syncwarp();
        b = b + 1 == NB ? 0 : b + 1;
    }
}

template <int Q, int SH>
__global__ void __launch_bounds__(kStreamMaxThreads) stream_kernel(const KParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t NW = blockDim.x / 32;
    const StreamLayout L = stream_layout(p.alpha, p.m, NW, p.stage_bytes, p.stages);
    uint32_t *sFp = reinterpret_cast<uint32_t *>(smem + L.f_off);
    uint8_t *sx = smem + L.x_off;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) trace_cta(p, 0);
    pdl_launch_dependents();
    const uint32_t total_warps = gridDim.x * NW;
    const uint32_t gw = blockIdx.x * NW + warp;
    const uint32_t bufs0 = smem_u32(smem + L.buf_off) + warp * p.stages * p.stage_bytes;
    load_table(p, sFp, sx);
    if (tid == 0) s_params[0] = p;
    __syncthreads();
    const FTable sF{fence_value(smem_u32(sFp))};
    WarpOut wo{reinterpret_cast<uint32_t *>(smem + L.wbuf_off) + warp * kWarpBuf, 0u};
    const GlobalText gtxt{p.y};
    WarpQueueSink<Q, SH, GlobalText> sink{p, gtxt, sF, sx, nullptr,
                                          reinterpret_cast<uint32_t *>(smem + L.q2_off) + warp * kWarpBuf,
                                          0u, 0u, wo, lane};
    uint32_t *ctr = reinterpret_cast<uint32_t *>(smem + L.ctr_off) + warp;
    if (lane == 0) *ctr = 0;
    __syncwarp();
    StreamQueue<Q, SH> qu{reinterpret_cast<uint32_t *>(smem + L.q_off) + warp * kStreamQ1, ctr, 0u};
    if (p.tma_chunk) {
        uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L.ctr_off + round_up(NW * 4u, 8)) + warp * 4;
        if (p.stages == 3)
            stream_loop_tma<Q, SH, 3>(p, sF, sink, qu, bufs0, bar, gw, total_warps, lane);
        else
            stream_loop_tma<Q, SH, 2>(p, sF, sink, qu, bufs0, bar, gw, total_warps, lane);
    } else if (p.stages == 2)
        stream_loop<Q, SH, 2>(p, sF, sink, qu, bufs0, gw, total_warps, lane);
    else if (p.stages == 3)
        stream_loop<Q, SH, 3>(p, sF, sink, qu, bufs0, gw, total_warps, lane);
    else
        stream_loop<Q, SH, 4>(p, sF, sink, qu, bufs0, gw, total_warps, lane);
    sink.drain();
    wo.flush(p, lane);
    if (lane == 0) trace_cta(p, 1);
}

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
        const GlobalText gtxt{pp.y};
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
__global__ void __launch_bounds__(2 * kStreamMaxThreads) mstream_kernel(const KParams p, const MParams mp) {
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
        const GlobalText gtxt{p.y};
        for (uint32_t c = gw; c < p.nchunks; c += total_warps) {
            const uint32_t k0 = c * p.seg_per_chunk;
            mstream_filter<Q, SH, GlobalText>(p, gtxt, P, k0, min(k0 + p.seg_per_chunk, p.K), lane, mw,
                                              sx0, L.x_stride);
        }
    } else if (p.stages == 3)
        mstream_loop<Q, SH, 3>(p, P, mw, sx0, L.x_stride, bufs0, gw, total_warps, lane);
    else
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
        const GlobalText gtxt{pp.y};
        WarpOut wo{mw.wbuf_of(i), mw.state[2 * i + 1]};
        WarpQueueSink<Q, SH, GlobalText> sink{pp, gtxt, ft, sx0 + i * L.x_stride, nullptr,
                                              mw.q2_of(i), 0u, mw.state[2 * i], wo, lane, i};
        sink.drain();
        wo.flush(pp, lane);
    }
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
}

// ------------------------------------------------------------------ launchers
using KernFn = void (*)(const KParams);

// (q, s) -> kernel instantiation.  s = floor(alpha/q) <= 15/q; for q = 1 the hash
// is the byte itself and s plays no role.
template <template <int, int> class Pick>
static KernFn pick(uint32_t q, uint32_t s) {
#define HC_C(Q, SH) \
    if (q == Q && s == SH) return Pick<Q, SH>::fn();
    if (q == 1) return Pick<1, 0>::fn();
    HC_C(2, 0) HC_C(2, 1) HC_C(2, 2) HC_C(2, 3) HC_C(2, 4) HC_C(2, 5) HC_C(2, 6) HC_C(2, 7)
    HC_C(3, 0) HC_C(3, 1) HC_C(3, 2) HC_C(3, 3) HC_C(3, 4) HC_C(3, 5)
    HC_C(4, 0) HC_C(4, 1) HC_C(4, 2) HC_C(4, 3)
    HC_C(5, 0) HC_C(5, 1) HC_C(5, 2) HC_C(5, 3)
    HC_C(6, 0) HC_C(6, 1) HC_C(6, 2)
    HC_C(7, 0) HC_C(7, 1) HC_C(7, 2)
    HC_C(8, 0) HC_C(8, 1)
#undef HC_C
    return nullptr;
}
template <int Q, int SH>
struct PickStaged {
    static KernFn fn() { return staged_kernel<Q, SH>; }
};
template <int Q, int SH>
struct PickStream {
    static KernFn fn() { return stream_kernel<Q, SH>; }
};
template <int Q, int SH>
struct PickShc {
    static KernFn fn() { return shc_kernel<Q, SH>; }
};
template <int Q, int SH>
struct PickGather {
    static KernFn fn() { return gather_kernel<Q, SH>; }
};

struct KernCache {
    KernFn fn;
    int smem;
    int occ;
};

static cudaError_t launch_common(KernFn kern, const KParams &p, int threads, int smem,
                                 int work_units, int max_ctas, int ctas_per_sm, cudaStream_t st,
                                 LaunchInfo *li) {
    // per-thread caches of the driver queries (they cost more than a whole large-m
    // search): the dynamic shared-memory limit is raised once per kernel to the
    // device maximum (so any later smem size is allowed), occupancy per (kernel, smem)
    static thread_local KernFn attr_set[128];
    static thread_local int nattr = 0;
    static thread_local KernCache cache[256];
    static thread_local int ncache = 0;
    static thread_local int sms = 0, smem_max = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    }
    bool have_attr = false;
    for (int c = 0; c < nattr; ++c) have_attr |= attr_set[c] == kern;
    if (!have_attr) {
        cudaFuncAttributes fa;
        cudaError_t err = cudaFuncGetAttributes(&fa, kern);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_max - static_cast<int>(fa.sharedSizeBytes));
        if (err != cudaSuccess) {
            if (std::getenv("HC_DEBUG"))
                std::fprintf(stderr, "libhc: cudaFuncSetAttribute: %s\n", cudaGetErrorName(err));
            return err;
        }
        if (nattr < 128) attr_set[nattr++] = kern;
    }
    if (smem > smem_max) return cudaErrorInvalidValue;
    int occ = -1;
    for (int c = 0; c < ncache; ++c)
        if (cache[c].fn == kern && cache[c].smem == smem) occ = cache[c].occ;
    if (occ < 0) {
        cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        if (err != cudaSuccess) {
            if (std::getenv("HC_DEBUG"))
                std::fprintf(stderr, "libhc: occupancy(smem=%d): %s\n", smem, cudaGetErrorName(err));
            return err;
        }
        if (ncache < 256) cache[ncache++] = KernCache{kern, smem, occ};
    }
    if (occ < 1) return cudaErrorInvalidConfiguration;
    if (ctas_per_sm > 0 && occ > ctas_per_sm) occ = ctas_per_sm;
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

cudaError_t launch_staged(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li) {
    KernFn kern = pick<PickStaged>(p.q, p.s);
    if (!kern) return cudaErrorInvalidValue;
    const int smem = staged_smem_bytes(p.alpha, p.m, p.stage_bytes, p.stages, p.slot_bytes, p.nbox);
    return launch_common(kern, p, kStagedThreads, smem, static_cast<int>(p.ntiles), max_ctas,
                         ctas_per_sm, st, li);
}

cudaError_t launch_gather(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li) {
    KernFn kern = pick<PickGather>(p.q, p.s);
    if (!kern) return cudaErrorInvalidValue;
    const int smem = gather_smem_bytes(p.alpha, p.m);
    const int warps_needed = static_cast<int>(p.nchunks);
    const int ctas = (warps_needed + kGatherThreads / 32 - 1) / (kGatherThreads / 32);
    return launch_common(kern, p, kGatherThreads, smem, ctas, max_ctas, ctas_per_sm, st, li);
}

cudaError_t launch_stream(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                          LaunchInfo *li) {
    KernFn kern = pick<PickStream>(p.q, p.s);
    if (!kern) return cudaErrorInvalidValue;
    const uint32_t nw = p.block_warps;
    const int smem = stream_smem_bytes(p.alpha, p.m, p.stage_bytes, p.stages, nw);
    const int ctas = static_cast<int>((p.nchunks + nw - 1) / nw);
    return launch_common(kern, p, static_cast<int>(32 * nw), smem, ctas, max_ctas, ctas_per_sm, st, li);
}

cudaError_t launch_shc(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                       LaunchInfo *li) {
    KernFn kern = pick<PickShc>(p.q, p.s);
    if (!kern) return cudaErrorInvalidValue;
    const uint32_t nw = p.block_warps;
    const int smem = shc_smem_bytes(p.alpha, p.m, p.stage_bytes, p.slot_bytes, nw);
    const int ctas = static_cast<int>((p.nchunks + nw - 1) / nw);
    return launch_common(kern, p, static_cast<int>(32 * nw), smem, ctas, max_ctas, ctas_per_sm, st, li);
}

cudaError_t launch_mstream(const KParams &p, const MParams &mp, cudaStream_t st, int max_ctas,
                           int ctas_per_sm, LaunchInfo *li) {
    using MFn = void (*)(const KParams, const MParams);
    MFn kern = nullptr;
#define HC_M(Q, SH) \
    if (p.q == Q && p.s == SH) kern = mstream_kernel<Q, SH>;
    if (p.q == 1) kern = mstream_kernel<1, 0>;
    HC_M(2, 0) HC_M(2, 1) HC_M(2, 2) HC_M(2, 3) HC_M(2, 4) HC_M(2, 5) HC_M(2, 6) HC_M(2, 7)
    HC_M(3, 0) HC_M(3, 1) HC_M(3, 2) HC_M(3, 3) HC_M(3, 4) HC_M(3, 5)
    HC_M(4, 0) HC_M(4, 1) HC_M(4, 2) HC_M(4, 3)
    HC_M(5, 0) HC_M(5, 1) HC_M(5, 2) HC_M(5, 3)
    HC_M(6, 0) HC_M(6, 1) HC_M(6, 2)
    HC_M(7, 0) HC_M(7, 1) HC_M(7, 2)
    HC_M(8, 0) HC_M(8, 1)
#undef HC_M
    if (!kern) return cudaErrorInvalidValue;
    const uint32_t nw = p.block_warps;
    const int smem = mstream_smem_bytes(p.alpha, p.m, p.stage_bytes, nw, mp.npat, p.stages);
    static thread_local MFn attr_done[64];
    static thread_local int nattr = 0;
    bool have = false;
    for (int c = 0; c < nattr; ++c) have |= attr_done[c] == kern;
    if (!have) {
        int dev = 0, smax = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaFuncAttributes fa;
        cudaError_t err = cudaFuncGetAttributes(&fa, kern);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smax - static_cast<int>(fa.sharedSizeBytes));
        if (err != cudaSuccess) return err;
        if (nattr < 64) attr_done[nattr++] = kern;
    }
    static thread_local int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int occ = 0;
    cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, static_cast<int>(32 * nw), smem);
    if (err != cudaSuccess) return err;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    if (ctas_per_sm > 0 && occ > ctas_per_sm) occ = ctas_per_sm;
    long grid = static_cast<long>(sms) * occ;
    const long need = (p.nchunks + nw - 1) / nw;
    if (grid > need) grid = need;
    if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
    if (grid < 1) grid = 1;
    kern<<<static_cast<unsigned>(grid), 32 * nw, smem, st>>>(p, mp);
    if (li) {
        li->grid = static_cast<int>(grid);
        li->block = static_cast<int>(32 * nw);
        li->smem = smem;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------ ordering
__global__ void widen_kernel(const uint32_t *src, int64_t *dst, uint32_t k) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
        dst[i] = static_cast<int64_t>(src[i]);
}


// Runs right after the search kernel, one CTA: publishes the count to the host
// (mapped pinned word), resets the device counter for the next call, and when
// 1 <= count <= kSmallSort orders the positions (distinct keys) and writes the first
// min(count, max_out) as int64:
//   count <= kRankSort : rank counting (key i goes to #{j : key_j < key_i});
//   otherwise          : a bucket pass on the top 11 of the ceil(log2 n) bits
//                        (shared counters, scan, scatter), then each key's rank inside
//                        its bucket by counting; a bucket larger than kBucketMax
//                        (skewed positions) sends the whole set to a block radix sort.
constexpr uint32_t kRankSort = 256;
constexpr int kFinishThreads = 1024;
constexpr int kFinishItems = kSmallSort / kFinishThreads;
constexpr uint32_t kBucketBits = 11;
constexpr uint32_t kBuckets = 1u << kBucketBits;
constexpr uint32_t kBucketMax = 32;
using FinishSort = cub::BlockRadixSort<uint32_t, kFinishThreads, kFinishItems>;
__global__ void __launch_bounds__(kFinishThreads) finish_kernel(uint32_t *counter, const uint32_t *pos,
                                                                uint32_t cap, int64_t *dst,
                                                                uint32_t max_out, uint32_t nbits,
                                                                volatile uint32_t *host_count,
                                                                unsigned long long *trace) {
    __shared__ union {
        typename FinishSort::TempStorage sort;
        struct {
            uint32_t cnt[kBuckets];     // keys per bucket, then bucket starts
            uint32_t keys[kSmallSort];  // keys grouped by bucket
            uint32_t warp_sum[32];
            uint32_t maxcnt;
        } b;
    } sm;
    if (trace && threadIdx.x == 0) trace[0] = gtimer();
    pdl_wait();   // the search grid has completed and its writes are visible
    if (trace && threadIdx.x == 0) trace[1] = gtimer();
    const uint32_t count = *counter;
    __syncthreads();
    if (threadIdx.x == 0) {
        *host_count = count;
        counter[0] = 0;
        counter[1] = 0;   // staged path: dynamic tile counter
    }
    if (dst == nullptr || max_out == 0 || count == 0 || count > cap || count > kSmallSort) return;
    const uint32_t k = min(count, max_out);
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (count == 1) {
        if (t == 0) dst[0] = static_cast<int64_t>(pos[0]);
        return;
    }
    if (count <= kRankSort) {
        if (t < count) sm.b.keys[t] = pos[t];
        __syncthreads();
        if (t < count) {
            const uint32_t key = sm.b.keys[t];
            uint32_t r = 0;
            for (uint32_t i = 0; i < count; ++i) r += sm.b.keys[i] < key;
            if (r < k) dst[r] = static_cast<int64_t>(key);
        }
        return;
    }
    // bucket pass: key -> bucket key >> shift (< kBuckets since key < 2^nbits)
    const uint32_t shift = nbits > kBucketBits ? nbits - kBucketBits : 0u;
    for (uint32_t i = t; i < kBuckets; i += kFinishThreads) sm.b.cnt[i] = 0;
    if (t == 0) sm.b.maxcnt = 0;
    __syncthreads();
    uint32_t key[kFinishItems], slot[kFinishItems];
#pragma unroll
    for (int i = 0; i < kFinishItems; ++i) {
        const uint32_t g = t + i * kFinishThreads;
        key[i] = g < count ? pos[g] : 0u;
        slot[i] = g < count ? atomicAdd(&sm.b.cnt[key[i] >> shift], 1u) : 0u;
    }
    __syncthreads();
    // exclusive scan of the 2048 counters: 2 per thread, warp shuffles, warp totals
    const uint32_t c0 = sm.b.cnt[2 * t], c1 = sm.b.cnt[2 * t + 1];
    uint32_t incl = c0 + c1;
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(HC_FULL, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) sm.b.warp_sum[warp] = incl;
    const uint32_t mx = __reduce_max_sync(HC_FULL, max(c0, c1));
    if (lane == 0) atomicMax(&sm.b.maxcnt, mx);
    __syncthreads();
    if (warp == 0) {
        uint32_t w = sm.b.warp_sum[lane];
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(HC_FULL, w, o);
            if (lane >= o) w += v;
        }
        sm.b.warp_sum[lane] = w - sm.b.warp_sum[lane];   // exclusive warp offsets
    }
    __syncthreads();
    const uint32_t base = sm.b.warp_sum[warp] + incl - (c0 + c1);
    const bool skewed = sm.b.maxcnt > kBucketMax;
    __syncthreads();
    if (!skewed) {
        sm.b.cnt[2 * t] = base;              // bucket starts
        sm.b.cnt[2 * t + 1] = base + c0;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kFinishItems; ++i)
            if (t + i * kFinishThreads < count) sm.b.keys[sm.b.cnt[key[i] >> shift] + slot[i]] = key[i];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kFinishItems; ++i) {
            if (t + i * kFinishThreads >= count) continue;
            const uint32_t bk = key[i] >> shift;
            const uint32_t lo = sm.b.cnt[bk];
            const uint32_t hi = bk + 1 < kBuckets ? sm.b.cnt[bk + 1] : count;
            uint32_t r = lo;
            for (uint32_t j = lo; j < hi; ++j) r += sm.b.keys[j] < key[i];
            if (r < k) dst[r] = static_cast<int64_t>(key[i]);
        }
        return;
    }
    // skewed positions: block radix sort (blocked arrangement, all-ones pads)
    uint32_t keys[kFinishItems];
#pragma unroll
    for (int i = 0; i < kFinishItems; ++i) {
        const uint32_t g = t * kFinishItems + i;
        keys[i] = g < count ? pos[g] : 0xffffffffu;
    }
    // real keys are < 2^nbits, the all-ones pads have bit nbits set: sorting bits
    // [0, nbits] puts the pads last
    const uint32_t hb = nbits < 32 ? nbits + 1 : 32;
    FinishSort(sm.sort).SortBlockedToStriped(keys, 0, static_cast<int>(hb));
#pragma unroll
    for (int i = 0; i < kFinishItems; ++i) {
        const uint32_t r = t + i * kFinishThreads;  // striped: rank r
        if (r < k) dst[r] = static_cast<int64_t>(keys[i]);
    }
}

cudaError_t launch_finish(uint32_t *counter, const uint32_t *pos, uint32_t cap, int64_t *dst,
                          uint32_t max_out, uint32_t n_bound, uint32_t *host_count_dev,
                          cudaStream_t st, unsigned long long *trace) {
    uint32_t nbits = 1;
    while (nbits < 32 && (static_cast<uint64_t>(1) << nbits) <= n_bound) ++nbits;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(kFinishThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, finish_kernel, counter, pos, cap, dst, max_out, nbits,
                              host_count_dev, trace);
}

// count > kSmallSort: CUB radix sort on ceil(log2 n) bits, then widen the first k.
cudaError_t sort_large(const uint32_t *pos, uint32_t count, uint32_t n_bound, int64_t *dst,
                       uint32_t k, cudaStream_t st, int *launches) {
    int end_bit = 1;
    while (end_bit < 32 && (static_cast<uint64_t>(1) << end_bit) <= n_bound) ++end_bit;
    uint32_t *alt = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t err = cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, pos, alt,
                                                     static_cast<int>(count), 0, end_bit, st);
    if (err != cudaSuccess) return err;
    err = cudaMallocAsync(reinterpret_cast<void **>(&alt),
                          static_cast<size_t>(count) * 4 + tmp_bytes + 256, st);
    if (err != cudaSuccess) return err;
    void *tmp = reinterpret_cast<void *>(
        (reinterpret_cast<uintptr_t>(alt) + static_cast<size_t>(count) * 4 + 255) &
        ~static_cast<uintptr_t>(255));
    err = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, pos, alt, static_cast<int>(count), 0,
                                         end_bit, st);
    if (err == cudaSuccess) {
        const uint32_t blocks = min((k + 255) / 256, 148u * 8u);
        widen_kernel<<<blocks, 256, 0, st>>>(alt, dst, k);
        err = cudaGetLastError();
        if (launches) *launches += 1 + (end_bit + 7) / 8 + 1;  // histogram + onesweep passes + widen
    }
    cudaError_t e2 = cudaFreeAsync(alt, st);
    return err != cudaSuccess ? err : e2;
}

}  // namespace hc
