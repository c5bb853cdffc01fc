// hc_device.cuh — device code shared by the search kernels of libhc (sm_100a):
// the Hash Chain searching phase (Fig. 5 left) as data-parallel
// CUDA.  Each kernel lives in its own translation unit (hc_stream.cu, hc_gather.cu,
// hc_mstream.cu, hc_scan.cu, hc_shc.cu, hc_staged.cu); this header holds what they share.
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
//                paper's loop inside their segment as a flat state machine
//                (run_segments_impl), keeping the warp converged.  Long walks are
//                done by the whole warp (walk_warp), long verifications compare
//                1 KiB per warp round (verify_warp).
// F (2^alpha u32 words) and x live in shared memory on every path.
// Matches go to a per-warp shared buffer, flushed 32 at a time with one
// atomicAdd (ballot/popc ranks); the finish kernels order them (hc_finish.cu).
//
// HC_INSTRUMENT (compile-time, default 0): measurement-only branches (opts.debug
// modes, %globaltimer traces) exist only in the instrumented build
// (libhc_instr.so, tools/); the production library compiles them out.
#pragma once

#include <cstdio>
#include <cstdlib>

#include "hc_internal.h"

#ifndef HC_INSTRUMENT
#define HC_INSTRUMENT 0
#endif
#ifndef HC_BOUNDS
#define HC_BOUNDS 0      // 1: every text access bounds-checked (libhc_chk.so, tests only)
#endif
#ifndef HC_FEW_BUILDS
#define HC_FEW_BUILDS 0  // 1: only the (q, s) instantiations the bounds-check driver uses
#endif
#ifndef HC_LDG_MODE
#define HC_LDG_MODE 1   // global text words: 0 = ld.global.nc, 1 = + .L2::64B (default: measured
                        // 293 -> 167 MB DRAM read at C2 m = 128), 2 = + L1::no_allocate
#endif

namespace hc {

#define HC_FULL 0xffffffffu
constexpr uint32_t kWordBits = 32;       // w (R2)
constexpr uint32_t kLongWalk = 4;        // walks past this many links with as many left go warp-wide
constexpr uint32_t kCoopVerifyMin = 64;  // m above which verification is warp-wide
constexpr uint32_t kAbortWalks = 16;     // warp-wide walks in one phase-B batch: walk-heavy text
constexpr int kUnroll = 4;               // lattice rounds whose loads are issued together
constexpr int kWalkUnroll = 4;           // walk steps evaluated per phase-B iteration
constexpr uint32_t kSurvWarps = 2;       // staged: survivor/producer warps per CTA

// Launch parameters, copied to shared memory at kernel start so that the out-of-line
// phase-B routine can read them without a stack copy.
constexpr int kMaxPat = kMaxPatterns;   // patterns per multi-pattern launch (stream path)
static __shared__ KParams s_params[kMaxPat];
constexpr bool kInstrument = HC_INSTRUMENT != 0;   // measurement-only branches compiled in
constexpr uint32_t kRegion = 32;         // staged: survivor entries per filter warp per slot

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_inval(uint64_t *bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
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
__device__ __forceinline__ void chk_shared(uint32_t a, uint32_t bytes);   // HC_BOUNDS build
// 1-D TMA bulk copy global -> shared, completion signalled on `bar` (tx bytes).
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
#if HC_BOUNDS
    chk_shared(dst, 16);
    chk_shared(dst + bytes - 16, 16);
    if ((bytes & 15) || (reinterpret_cast<uintptr_t>(src) & 15)) __trap();
#endif
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
    if (kInstrument && p.trace && it < p.trace_tiles)
        p.trace[(static_cast<size_t>(blockIdx.x) * p.trace_tiles + it) * 4 + ev] = gtimer();
}
// CTA entry (ev 0) / exit (ev 1) stamps after the per-tile records (one thread)
__device__ __forceinline__ void trace_cta(const KParams &p, uint32_t ev) {
    if (kInstrument && p.trace)
        p.trace[static_cast<size_t>(gridDim.x) * p.trace_tiles * 4 + blockIdx.x * 2 + ev] = gtimer();
}
// debug 12 (instrumented build): latest time any warp passed point i of the search's
// critical path (point 0: earliest CTA entry, stored complemented), kept after the
// per-CTA records of the trace buffer
__device__ __forceinline__ void path_ts(const KParams &p, uint32_t i) {
    if (kInstrument && p.trace && p.debug == 12 && (threadIdx.x & 31) == 0) {
        unsigned long long *a =
            p.trace + static_cast<size_t>(gridDim.x) * (p.trace_tiles * 4 + 2) + 8 + i;
        const unsigned long long t = gtimer();
        atomicMax(a, i == 0 ? ~t : t);
    }
}
// debug 12: event counters next to the stamps (one lane per warp counts)
__device__ __forceinline__ void path_cnt(const KParams &p, uint32_t i, uint32_t lane) {
    if (kInstrument && p.trace && p.debug == 12 && lane == 0)
        atomicAdd(p.trace + static_cast<size_t>(gridDim.x) * (p.trace_tiles * 4 + 2) + 24 + i, 1ull);
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
// Bounds-checked build (HC_BOUNDS=1, libhc_chk.so; compute-sanitizer is closed on this GPU
// pool, so the memcheck is our own): an aligned global word must hold at least one byte of
// [y, y + n), a shared access must lie inside the CTA's dynamic shared memory, copies into
// shared memory must read inside the text.  A violation traps: the parity driver of
// tests/test_gpu_tools.py (every path, aligned and unaligned texts) then fails.  The checks
// cost ~50% of a search, so they are not part of the instrumented (timing) build.
__device__ __forceinline__ void chk_fail() {
#if HC_BOUNDS
    __trap();
#endif
}
#if HC_BOUNDS
extern __shared__ __align__(128) uint8_t hc_chk_dyn_smem[];   // the kernels' dynamic shared memory
#endif
__device__ __forceinline__ void chk_shared(uint32_t a, uint32_t bytes) {
#if HC_BOUNDS
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    const uint32_t lo = static_cast<uint32_t>(__cvta_generic_to_shared(hc_chk_dyn_smem));
    if (a < lo || a + bytes > lo + dyn || (a & (bytes - 1))) chk_fail();
#endif
}
__device__ __forceinline__ void chk_text_range(const uint8_t *y, uint32_t n, uintptr_t a, uint32_t bytes) {
#if HC_BOUNDS
    if (a < reinterpret_cast<uintptr_t>(y) || a + bytes > reinterpret_cast<uintptr_t>(y) + n) chk_fail();
#endif
}
struct GlobalText {
    const uint8_t *y;
#if HC_BOUNDS
    uint32_t n = 0;   // text length: accesses are checked when set
    __device__ __forceinline__ void chk(uintptr_t a, uint32_t bytes) const {
        const uintptr_t y0 = reinterpret_cast<uintptr_t>(y);
        if (n && (a + bytes <= y0 || a >= y0 + n || (a & (bytes - 1)))) chk_fail();
    }
#else
    __device__ __forceinline__ void chk(uintptr_t, uint32_t) const {}
#endif
    __device__ __forceinline__ uintptr_t addr(uint32_t p) const {
        return reinterpret_cast<uintptr_t>(y) + p;
    }
    __device__ __forceinline__ uint64_t word(uintptr_t aligned) const {
        chk(aligned, 8);
#if HC_LDG_MODE == 1
        uint64_t r;
        asm("ld.global.nc.L2::64B.u64 %0, [%1];" : "=l"(r) : "l"(aligned));
        return r;
#elif HC_LDG_MODE == 2
        uint64_t r;
        asm("ld.global.nc.L1::no_allocate.L2::64B.u64 %0, [%1];" : "=l"(r) : "l"(aligned));
        return r;
#else
        return __ldg(reinterpret_cast<const unsigned long long *>(aligned));
#endif
    }
    __device__ __forceinline__ uint32_t word32(uintptr_t aligned) const {
        chk(aligned, 4);
#if HC_LDG_MODE >= 1
        uint32_t r;
        asm("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(r) : "l"(aligned));
        return r;
#else
        return __ldg(reinterpret_cast<const unsigned int *>(aligned));
#endif
    }
    __device__ __forceinline__ uint32_t byte(uint32_t p) const {
        chk(reinterpret_cast<uintptr_t>(y) + p, 1);
        return __ldg(y + p);
    }
    __device__ __forceinline__ GlobalText shfl(uint32_t) const { return *this; }  // same in all lanes
    static constexpr bool kLoSafe = false;  // the word before may be outside y
};

// The search's text as seen by the survivors (bounds-checked in the instrumented build).
__device__ __forceinline__ GlobalText global_text(const KParams &p) {
#if HC_BOUNDS
    return GlobalText{p.y, p.n};
#else
    return GlobalText{p.y};
#endif
}

// Shared-memory loads by shared-space address.  Not volatile: callers make the
// address depend on a value produced after the mbarrier wait (see fence_value), so
// they cannot be hoisted above it.
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
    chk_shared(a, 8);
    uint64_t r;
    asm("ld.shared.u64 %0, [%1];" : "=l"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    chk_shared(a, 4);
    uint32_t r;
    asm("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    chk_shared(a, 1);
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
    __device__ __forceinline__ uint32_t word32(uint32_t aligned) const { return lds32(aligned); }
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
// The filter bitmap (2^alpha bits, bit v set iff F[v] != 0) in shared memory: the l.6
// test alone, 32x smaller than F, so it loads in one short round trip while F itself
// arrives by a TMA bulk copy behind it.
struct FBits {
    uint32_t base;
    __device__ __forceinline__ bool pass(uint32_t v) const {
        return (lds32(base + 4 * (v >> 5)) >> (v & 31)) & 1u;
    }
};

// Stream path, phase A: the filter bitmap replicated per lane in shared memory (word
// (v >> 5) of lane l's copy at word index (v >> 5) * 32 + l, i.e. in bank l; sh = 7), so the
// l.6 test of 32 random hash values never conflicts.  (The same lookups in F: ~5
// wavefronts per load on DNA, measured 6 us of a 64 us search at m = 16 and 13 us of 88 at
// m = 8.)  The replicas take 2^alpha words, as F does; where they do not fit the kernel
// keeps one copy (col the same in all lanes, sh = 2).  The survivors read F itself.
struct PassBits {
    uint32_t col;          // shared address of this lane's column (table + 4 * lane, or table)
    uint32_t sh;           // log2 of the byte stride between bitmap words: 7 or 2
    __device__ __forceinline__ bool pass(uint32_t v) const {
        return (lds32(col + ((v >> 5) << sh)) >> (v & 31)) & 1u;
    }
};
// builds the bitmap (replicated or not) from the global one (2^alpha bits, >= 4 words);
// whole CTA, one round trip: every warp loads up to 32 words and hands them round by shuffle
__device__ __forceinline__ void load_pass_bits(const KParams &p, uint32_t *tab) {
    const uint32_t nw = (1u << p.alpha) > 32 ? (1u << p.alpha) / 32 : 1u;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    if (!p.lane_bits) {
        for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x) tab[i] = __ldg(p.Fbits + i);
        return;
    }
    for (uint32_t base = warp * 32; base < nw; base += NW * 32) {
        const uint32_t v = base + lane < nw ? __ldg(p.Fbits + base + lane) : 0u;
        const uint32_t cnt = min(32u, nw - base);
        for (uint32_t k = 0; k < cnt; ++k) tab[(base + k) * 32 + lane] = __shfl_sync(HC_FULL, v, k);
    }
}

// The 8 text bytes y[p-7 .. p] as a little-endian u64 (byte 7 = y[p]).  Only the
// top Q bytes are meaningful.  Reads just the aligned 8-byte words holding y[p]
// and y[p-Q+1] (both inside the text).  On global text such a word can extend up to
// 7 bytes before y[0] or past y[n-1]: an aligned 8-byte word never crosses a page, so
// this cannot fault, but a checker that tracks exact allocation sizes (compute-
// sanitizer on a cudaMalloc of exactly n bytes) reports those bytes.  They never
// influence a result (only the Q bytes of the q-gram are hashed).
template <int Q, class T>
__device__ __forceinline__ uint64_t end8(const T &t, uint32_t p) {
    auto a = t.addr(p);
    using A = decltype(a);
    if constexpr (Q <= 4) {
        // q-grams of up to 4 bytes: the two aligned 4-byte words and one funnel shift (the
        // hash reads only the upper half of the result)
        const A a4 = a & ~static_cast<A>(3);
        const uint32_t off = static_cast<uint32_t>(a & 3);
        const uint32_t hi = t.word32(a4);
        uint32_t lo = 0;
        if constexpr (Q > 1) {
            if (T::kLoSafe || off + 1 < static_cast<uint32_t>(Q)) lo = t.word32(a4 - 4);
        }
        return static_cast<uint64_t>(__funnelshift_l(lo, hi, 24 - 8 * off)) << 32;
    }
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
            if (base + lane == 0) p.counter[4] = v;   // the first slot's position (epilogue)
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
        if (base + lane == 0) p.counter[4] = buf[0];  // the first slot's position (epilogue)
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
    if (kInstrument && p.debug == 5 && lane == 0) atomicAdd(p.counter + 7, 1u);
    // Walk-heavy text (allow_abort, gather path): Fig. 5's loop would re-hash most q-grams
    // many times over (the stress config C5: ~7 hashes per text byte).  A batch that needs
    // more than kAbortWalks warp-wide walks raises the give-up flag, and every later
    // batch returns as soon as it would start a warp-wide walk: the search finishes its
    // (cheap) lattice filter and first steps, and the host re-runs it on the scan path,
    // which hashes every q-gram once (hc_scan.cu).  Only batches with warp-wide walks (rare
    // on non-repetitive text) read the flag.
    uint32_t nwalks = 0, nit = 0;
    while (__any_sync(HC_FULL, active)) {
        if (kInstrument && p.debug == 5 && lane == 0) atomicAdd(p.counter + 6, 1u);
        path_cnt(p, 0, lane);
        path_ts(p, 9 + min(nit++, 6u));
        bool need_v = false, stepped = false;
        if (long_walks) {
            // walks that passed kLongWalk link tests and still have >= kLongWalk steps to
            // go (near-matches, true matches) finish warp-wide, one lane at a time
            uint32_t lm = __ballot_sync(HC_FULL, active && walk && wsteps >= kLongWalk &&
                                                     (j - i) >= kLongWalk * Q);
            if (p.allow_abort && lm) {
                volatile uint32_t *flag = p.counter + 3;
                if (nwalks == 0 && *flag) return wo.cnt;     // another batch gave up already
                if ((nwalks += __popc(lm)) > kAbortWalks) {
                    if (lane == 0) *flag = 1u;
                    return wo.cnt;
                }
            }
            while (lm) {
                const uint32_t L = __ffs(lm) - 1;
                lm &= lm - 1;
                uint32_t jL = __shfl_sync(HC_FULL, j, L);
                const uint32_t iL = __shfl_sync(HC_FULL, i, L);
                const uint32_t zL = __shfl_sync(HC_FULL, z, L);
                uint32_t vL = 0;
                bool broke = false;
                path_cnt(p, 1, lane);
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
                path_cnt(p, 2, lane);
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
// step (l.9-12) tests the link bit of v_1 = h(y[e-2q+1..e-q]) in F[v_0]; if it is clear
// the loop breaks and the next window ends at j = e - q + S (l.18).  If F[h(j)] == 0
// that window shifts by S again (l.6) to j + S >= a_k + S, out of the segment
// (R11), and the segment is finished.  Otherwise window j takes its own first walk step
// (l.7-12): if the link bit of h(j - q) is clear in F[h(j)] the loop breaks again and
// the next window ends at j - q + S = a_k - 2q + 2S, which is past the segment when
// S >= 2q: finished as well.  Otherwise the segment continues at `start` = e (first
// link set) or j.  Exact: these are the paper's steps in order, with the four hashes
// loaded in parallel (one memory round trip).  On DNA this finishes ~95% of the lattice
// survivors.
template <int Q, int SH, class T, class FT>
__device__ __forceinline__ bool first_steps_eval(const KParams &p, const T &txt, const FT &sF,
                                                 bool act, uint32_t e, uint32_t &start) {
    start = e;
    if (!act) return false;
    if (p.m < 2 * Q) return true;                        // no walk step to test (R7)
    const uint32_t j = e - Q + p.S;
    const bool jin = j < p.n;                            // else the break leaves the text
    const uint64_t W0 = end8<Q>(txt, e), W1 = end8<Q>(txt, e - Q);
    const uint64_t W2 = end8<Q>(txt, jin ? j : e), W3 = end8<Q>(txt, jin ? j - Q : e);
    const uint32_t v1 = qhash<Q, SH>(W1, p.mask);
    const uint32_t v3 = qhash<Q, SH>(W3, p.mask);
    const uint32_t z0 = sF[qhash<Q, SH>(W0, p.mask)];
    const uint32_t z2 = sF[qhash<Q, SH>(W2, p.mask)];
    if (((z0 >> (v1 & (kWordBits - 1))) & 1u) != 0u) {  // link set: walk on
        if constexpr (!T::kLoSafe) {
            // the walk will read back through the window (a true occurrence walks all of
            // it, then verifies it): start its lines on their way to L2 now, so that the
            // phase-B round trips of this segment hit L2 instead of DRAM
            if (p.m >= 64) {
                const uintptr_t lo = txt.addr(e + 1 - p.m) & ~static_cast<uintptr_t>(127);
                for (uintptr_t a = lo; a <= txt.addr(e); a += 128)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
            }
        }
        return true;
    }
    start = j;                                           // break at the first step
    if (!jin || z2 == 0u) return false;                  // window j shifts out (l.6, l.18)
    if (p.S >= 2 * Q && ((z2 >> (v3 & (kWordBits - 1))) & 1u) == 0u)
        return false;                                    // window j breaks at its first step
    return true;
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
    // (An out-of-line copy of the first steps shared by all call sites was measured: the
    // gather kernel at m >= 512 4-15% faster (smaller code, everything runs cold there), but
    // m = 64 and the stream kernel's filter loop 5-7% slower: a call inside the hot loop.)
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


__host__ __device__ inline uint32_t round_up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

__device__ __forceinline__ void load_x(const KParams &p, uint8_t *sx);
__device__ __forceinline__ void load_table(const KParams &p, uint32_t *sF, uint8_t *sx) {
    // F (2^alpha words) and x, with every thread's loads issued before its stores: one
    // L2 round trip for the whole table instead of one per loop trip
    const uint32_t nF = 1u << p.alpha;
    if (nF >= 4) {
        const uint4 *src = reinterpret_cast<const uint4 *>(p.F);
        uint4 *dst = reinterpret_cast<uint4 *>(sF);
        const uint32_t n4 = nF / 4;
        for (uint32_t w0 = threadIdx.x; w0 < n4; w0 += 8 * blockDim.x) {
            uint4 v[8];
#pragma unroll
            for (uint32_t r = 0; r < 8; ++r) {
                const uint32_t w = w0 + r * blockDim.x;
                if (w < n4) v[r] = __ldg(src + w);
            }
#pragma unroll
            for (uint32_t r = 0; r < 8; ++r) {
                const uint32_t w = w0 + r * blockDim.x;
                if (w < n4) dst[w] = v[r];
            }
        }
    } else {
        for (uint32_t w = threadIdx.x; w < nF; w += blockDim.x) sF[w] = __ldg(p.F + w);
    }
    load_x(p, sx);
}
__device__ __forceinline__ void load_x(const KParams &p, uint8_t *sx) {
    // x in 16-byte vectors (the device copy of x has >= 15 readable bytes past m), with
    // the bytes from m on zeroed up to m + 8 so that 8-byte compares of x never read
    // uninitialised shared memory
    const uint32_t n16 = (p.m + 8 + 15) / 16;
    for (uint32_t w = threadIdx.x; w < n16; w += blockDim.x) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (16 * w < p.m) v = __ldg(reinterpret_cast<const uint4 *>(p.x) + w);
        uint32_t *vw = reinterpret_cast<uint32_t *>(&v);
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
            const uint32_t b = 16 * w + 4 * j;
            if (b >= p.m) vw[j] = 0;
            else if (b + 4 > p.m) vw[j] &= (1u << (8 * (p.m - b))) - 1u;
        }
        reinterpret_cast<uint4 *>(sx)[w] = v;
    }
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

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    chk_shared(dst, 16);
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
    // steps (first_steps_eval reads the q-grams ending at a_k - q, a_k - q + S and
    // a_k - 2q + S, all inside this range)
    const uint32_t a0 = p.m - 1 + g.k0 * p.S;
    g.first = a0 + 1 >= 2 * p.q ? a0 + 1 - 2 * p.q : 0u;
    const uint32_t alast = p.m - 1 + (g.k1 - 1) * p.S;
    g.last = max(alast, min(alast + p.S - p.q, p.n - 1));
    return g;
}
// Issues chunk c's copies into the buffer at shared address `buf` (one warp).  The
// 16-byte words wholly inside y are copied with cp.async; the bytes of the partial
// words at the two ends of an unaligned text are stored directly (first/last chunk).
// Copies text bytes [first, last] into the buffer at shared address `buf` (one warp):
// the 16-byte words wholly inside y with cp.async, the bytes of the partial words at the
// two ends of an unaligned text directly.  Text byte t lands at buf + (y + t) % 16 +
// (t - first).  One commit group per call (possibly empty).
__device__ __forceinline__ void issue_range(const KParams &p, bool any, uint32_t first, uint32_t last,
                                            uint32_t buf, uint32_t lane) {
    if (any) {
        const uintptr_t y = reinterpret_cast<uintptr_t>(p.y);
        const uintptr_t A = (y + first) & ~static_cast<uintptr_t>(15);
        const uint32_t nbytes =
            static_cast<uint32_t>(((y + last + 16) & ~static_cast<uintptr_t>(15)) - A);
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
__device__ __forceinline__ void stream_issue(const KParams &p, uint32_t c, uint32_t buf,
                                             uint32_t lane) {
    StreamChunk g{0, 0, 0, 0};
    if (c < p.nchunks) g = stream_chunk(p, c);
    issue_range(p, c < p.nchunks, g.first, g.last, buf, lane);
}

// ------------------------------------------------------------------ fused epilogue
// Every search kernel ends here: the last CTA to finish publishes the
// occurrence count to the host (mapped pinned memory), resets the counter words for the
// next call, and orders up to epi_cap positions into the caller's int64 buffer in its
// own (now idle) shared memory.  One kernel launch per hc_search in the common case;
// the host orders only what the epilogue could not (hc_finish.cu).

// Orders `count` distinct positions pos[0..count) (2 <= count), all < 2^nbits, into
// dst[0..k) ascending, in shared memory `sm` (>= epi_bytes(count) bytes), by the whole
// block (any size).  Small sets by rank counting; larger ones by a bucket pass (power-of-two
// buckets, count/2 to count of them, at most 2048: bucket = position >> sh over the whole
// text) and rank counting inside each bucket.  When some bucket holds more than
// kEpiBucketMax keys (clustered positions) the pass is repeated once on the positions'
// offset from their minimum; false when that does not help either (the host then orders
// them; nothing is assumed of dst).  The code is kept SMALL (scalar loops, not unrolled):
// it runs once per search on one SM whose instruction cache has never seen it, and the
// vectorised version of round 2a spent most of its 12.7 us (4,144 positions) fetching
// instructions: each phase took 2-3 us however few keys a thread had.
#if HC_INSTRUMENT
static __device__ unsigned long long g_epi_ts[16];  // debug 10: block_order phase stamps
#define HC_EPI_TS(i) do { if (threadIdx.x == 0) { g_epi_ts[i] = gtimer(); g_epi_ts[8 + i] = clock64(); } } while (0)
#else
#define HC_EPI_TS(i) do { } while (0)
#endif
constexpr uint32_t kEpiRankMax = 256;
constexpr uint32_t kEpiBucketMax = 64;
static __device__ __noinline__ bool block_order(const uint32_t *pos, uint32_t count, int64_t *dst, uint32_t k,
                                                uint8_t *sm, uint32_t nbits) {
    const uint32_t T = blockDim.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t *tmp = reinterpret_cast<uint32_t *>(sm);            // 64 words
    uint32_t *ks = tmp + 64;                                     // keys, then the sorted keys
    const uint32_t cnt4 = (count + 3) & ~3u;
    // all keys to shared memory with 16-byte cp.async copies: one L2 round trip (the
    // scratch is 16-byte aligned and has >= 3 words of slack past any count)
#pragma unroll 1
    for (uint32_t i = 4 * t; i < count; i += 4 * T)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(ks + i)), "l"(pos + i)
                     : "memory");
    HC_EPI_TS(0);
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    HC_EPI_TS(1);
    if (count <= kEpiRankMax) {
        if (t < count) {
            const uint32_t key = ks[t];
            uint32_t r = 0;
#pragma unroll 1
            for (uint32_t j = 0; j < count; ++j) r += ks[j] < key;
            if (r < k) dst[r] = static_cast<int64_t>(key);
        }
        return true;
    }
    uint32_t NB = 32, lb = 5;
    while (NB < 2048 && 2 * NB < count) NB <<= 1, ++lb;          // count/2 <= NB < count
    uint32_t *c = ks + cnt4;                                     // NB bucket counters
    uint32_t *k2 = c + NB;                                       // keys grouped by bucket
    uint32_t lo = 0, sh = nbits > lb ? nbits - lb : 0u;          // bucket = (key - lo) >> sh < NB
    const uint32_t per = (NB + T - 1) / T;                       // counters per scanning thread
    const uint32_t b0 = min(t * per, NB), b1 = min(b0 + per, NB);
#pragma unroll 1
    for (uint32_t attempt = 0;; ++attempt) {
#pragma unroll 1
        for (uint32_t i = t; i < NB; i += T) c[i] = 0;
        __syncthreads();
#pragma unroll 1
        for (uint32_t i = t; i < count; i += T) atomicAdd(&c[(ks[i] - lo) >> sh], 1u);   // histogram
        __syncthreads();
        HC_EPI_TS(3);
        uint32_t loc = 0, big = 0;                               // exclusive scan of the counters
#pragma unroll 1
        for (uint32_t i = b0; i < b1; ++i) {
            const uint32_t v = c[i];
            big |= v > kEpiBucketMax;
            loc += v;
        }
        uint32_t incl = loc;
#pragma unroll 1
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(HC_FULL, incl, o);
            if (lane >= o) incl += x;
        }
        if (lane == 31) tmp[warp] = incl;
        if (!__syncthreads_or(big)) {
            uint32_t run = incl - loc;
#pragma unroll 1
            for (uint32_t w = 0; w < warp; ++w) run += tmp[w];
#pragma unroll 1
            for (uint32_t i = b0; i < b1; ++i) {
                const uint32_t v = c[i];
                c[i] = run;
                run += v;
            }
            break;
        }
        if (attempt) return false;
        // clustered positions: buckets over [min, max] instead of the whole text
        uint32_t mn = 0xffffffffu, mx = 0;
#pragma unroll 1
        for (uint32_t i = t; i < count; i += T) {
            mn = min(mn, ks[i]);
            mx = max(mx, ks[i]);
        }
        mn = __reduce_min_sync(HC_FULL, mn);
        mx = __reduce_max_sync(HC_FULL, mx);
        __syncthreads();                                         // tmp is free again
        if (lane == 0) {
            tmp[warp] = mn;
            tmp[32 + warp] = mx;
        }
        __syncthreads();
#pragma unroll 1
        for (uint32_t w = 0; w < (T >> 5); ++w) {
            mn = min(mn, tmp[w]);
            mx = max(mx, tmp[32 + w]);
        }
        lo = mn;
        sh = 0;
        while (((mx - lo) >> sh) >= NB) ++sh;
        __syncthreads();
    }
    __syncthreads();
    HC_EPI_TS(4);
#pragma unroll 1
    for (uint32_t i = t; i < count; i += T) {                    // scatter by bucket
        const uint32_t key = ks[i];
        k2[atomicAdd(&c[(key - lo) >> sh], 1u)] = key;
    }
    __syncthreads();                                             // c[b] = end of bucket b
    HC_EPI_TS(5);
#pragma unroll 1
    for (uint32_t i = t; i < count; i += T) {                    // rank inside the bucket
        const uint32_t key = k2[i];
        const uint32_t b = (key - lo) >> sh;
        const uint32_t b_lo = b ? c[b - 1] : 0u, b_hi = c[b];
        uint32_t r = b_lo;
#pragma unroll 1
        for (uint32_t j = b_lo; j < b_hi; ++j) r += k2[j] < key;
        ks[r] = key;                                             // sorted (ks is free now)
    }
    __syncthreads();
    const uint32_t kk = min(k, count);
#pragma unroll 1
    for (uint32_t i = t; i < kk; i += T) dst[i] = static_cast<int64_t>(ks[i]);   // coalesced
    HC_EPI_TS(6);
    return true;
}

// True in every thread of the last CTA of the grid to get here.  Every thread fences its
// own position stores and counter atomics before the CTA takes its ticket, and the last
// CTA fences again before reading what the others wrote.
__device__ __forceinline__ bool cta_is_last(uint32_t *ticket) {
    __shared__ uint32_t s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1 ? 1u : 0u;
    __syncthreads();
    const bool last = s_last != 0;
    if (last) __threadfence();
    return last;
}

// The last CTA's work for one search: publish, order when possible, reset the counters.
// `smem` is the CTA's dynamic shared memory (idle by now), `smem_bytes` its size.
// `count` and `pos0` (the position in slot 0 of the scratch, counter[4]) were read by the
// caller together with the give-up flag: one round trip after the ticket, not three.
__device__ __forceinline__ void publish_search(uint32_t *counter, const uint32_t *out, uint32_t cap,
                                               uint32_t *host_count, int64_t *dst, uint32_t k_out,
                                               uint32_t epi_cap, uint8_t *smem, bool fault,
                                               uint32_t nbits, uint32_t count, uint32_t pos0) {
    bool ordered = count == 0 || dst == nullptr || k_out == 0;
    if (!ordered && count <= cap && count <= epi_cap) {
        if (count == 1) {
            if (threadIdx.x == 0) dst[0] = static_cast<int64_t>(pos0);
            ordered = true;
        } else {
            unsigned long long t0 = 0;
            if (kInstrument && threadIdx.x == 0) t0 = gtimer();
            ordered = block_order(out, count, dst, k_out, smem, nbits);
            if (kInstrument && threadIdx.x == 0) {   // debug 10: ordering time, ns
                counter[6] = static_cast<uint32_t>(gtimer() - t0);
                counter[7] = count;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (kInstrument && fault && ordered && count > 0 && dst && k_out)
            dst[0] += 1;                           // fault-injection hook (tests only)
        counter[0] = 0;
        counter[1] = 0;
        host_count[1] = ordered ? 1u : 0u;
        host_count[0] = count;
    }
}

// Largest count the epilogue orders in `smem_bytes` of dynamic shared memory.
#ifndef HC_EPI_MAX
#define HC_EPI_MAX 8192
#endif
inline uint32_t epi_cap_for(int smem_bytes) {
    uint32_t c = smem_bytes > 544 ? (static_cast<uint32_t>(smem_bytes) - 544u) / 12u : 0u;
    c = c < kSmallSort ? c : kSmallSort;
    return c < HC_EPI_MAX ? c : HC_EPI_MAX;
}

// Single-pattern kernels: the epilogue of search p (call from every thread at the end).
__device__ __forceinline__ void search_epilogue(const KParams &p, uint8_t *smem) {
    const bool last_cta = cta_is_last(p.counter + 2);
    path_ts(p, 7);
    if (!last_cta) return;
    // count, give-up flag and the first position in ONE round trip (independent loads)
    uint32_t c0, c3, pos0;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(c0) : "l"(p.counter));
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(c3) : "l"(p.counter + 3));
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(pos0) : "l"(p.counter + 4));
    if (c3) {
        // the search gave up (walk-heavy text, see gather_kernel): the host re-runs it on
        // the scan path; nothing of this run is published but the verdict
        if (threadIdx.x == 0) {
            p.counter[0] = p.counter[1] = p.counter[2] = p.counter[3] = 0;
            p.host_count[1] = 2u;
            p.host_count[0] = 0u;
        }
        return;
    }
    publish_search(p.counter, p.out, p.cap, p.host_count, p.dst, p.k_out, p.epi_cap, smem,
                   p.debug == 9, p.nbits, c0, pos0);
    __syncthreads();
    if (threadIdx.x == 0) p.counter[2] = 0;
    path_ts(p, 8);
}

// ------------------------------------------------------------------ launch helpers
using KernFn = void (*)(const KParams);

// (q, s) -> kernel instantiation.  s = floor(alpha/q) <= 15/q; for q = 1 the hash
// is the byte itself and s plays no role.  31 builds (tests/test_gpu_parity.py
// test_every_kernel_build runs each of them).
template <template <int, int> class Pick>
static typename Pick<1, 0>::Fn pick(uint32_t q, uint32_t s) {
#define HC_C(Q, SH) \
    if (q == Q && s == SH) return Pick<Q, SH>::fn();
    if (q == 1) return Pick<1, 0>::fn();
#if HC_FEW_BUILDS
    HC_C(2, 4) HC_C(2, 5) HC_C(3, 3) HC_C(4, 3) HC_C(6, 2) HC_C(8, 1)
#else
    HC_C(2, 0) HC_C(2, 1) HC_C(2, 2) HC_C(2, 3) HC_C(2, 4) HC_C(2, 5) HC_C(2, 6) HC_C(2, 7)
    HC_C(3, 0) HC_C(3, 1) HC_C(3, 2) HC_C(3, 3) HC_C(3, 4) HC_C(3, 5)
    HC_C(4, 0) HC_C(4, 1) HC_C(4, 2) HC_C(4, 3)
    HC_C(5, 0) HC_C(5, 1) HC_C(5, 2) HC_C(5, 3)
    HC_C(6, 0) HC_C(6, 1) HC_C(6, 2)
    HC_C(7, 0) HC_C(7, 1) HC_C(7, 2)
    HC_C(8, 0) HC_C(8, 1)
#endif
#undef HC_C
    return nullptr;
}

// Persistent-grid launch of `kern` (hc_launch.cu): the grid is (SMs x resident CTAs),
// capped at `work_units` CTAs and at max_ctas / ctas_per_sm when > 0.  The dynamic
// shared-memory limit and the occupancy are cached per (device, kernel).
cudaError_t launch_kernel(const void *kern, void **args, int threads, int smem, long work_units,
                          int max_ctas, int ctas_per_sm, cudaStream_t st, LaunchInfo *li);

}  // namespace hc
