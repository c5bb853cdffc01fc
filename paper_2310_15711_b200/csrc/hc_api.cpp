// hc_api.cpp — host side of libhc: the C-ABI of include/hc.h.
//
//   hc_prepare     Preprocessing (Fig. 3) on the host + upload of F and x.
//   hc_search(_ex) validation, path choice, search kernel launch (hc_*.cu),
//                  count read-back, position ordering.
//
// The table build below is this library's own implementation of Fig. 3: it
// hashes every q-gram of x once (closed form of Eq. 3, reading R4), applies
// Eq. 1 to every adjacent non-overlapping pair (the pairs the chains of Fig. 3
// visit), then Eq. 2 with optimisation 1, and takes H_v
// as the hash of the first q-gram of the chain ending at m-1.  It
// shares no code with oracle/; tests check the two tables are identical.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <memory>
#include <vector>

#include "hc.h"
#include "hc_internal.h"

#ifndef HC_INSTRUMENT
#define HC_INSTRUMENT 0
#endif

struct hc_handle {
    std::vector<uint8_t> x;
    std::vector<uint32_t> F;
    uint32_t m = 0, q = 0, alpha = 0, s = 0, mask = 0, hv = 0;
    int device = 0;
    uint32_t *dF = nullptr;        // device image: F | filter bitmap | x (zero-padded)
    uint32_t *dFbits = nullptr;
    uint8_t *dx = nullptr;
    std::shared_ptr<void> block;   // hc_prepare_batch: device block shared by the batch
};

namespace {

thread_local int g_last_error = HC_OK;

int fail(int code) {
    g_last_error = code;
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    if (std::getenv("HC_DEBUG")) std::fprintf(stderr, "libhc: %s: %s (%s)\n", what, cudaGetErrorString(e), cudaGetErrorName(e));
    cudaGetLastError();  // clear sticky-free errors
    return fail(e == cudaErrorMemoryAllocation ? HC_ENOMEM : HC_ECUDA);
}

int check_params(const uint8_t *x, size_t m, int q, int alpha) {
    if (m == 0 || x == nullptr || q < 1) return HC_EINVAL;
    if (m > HC_MAX_PATTERN) return HC_ETOOLONG;
    if (static_cast<size_t>(q) > m) return HC_ETOOSHORT;
    if (q > 8) return HC_EINVAL;
    if (alpha < 1 || alpha > HC_MAX_ALPHA) return HC_EALPHA;
    return HC_OK;
}

// Fig. 3 Preprocessing result for x (see the file header for the construction).
void build_table(const uint8_t *x, uint32_t m, uint32_t q, uint32_t alpha, uint32_t *F,
                 uint32_t *s_out, uint32_t *hv_out) {
    const uint32_t s = alpha / q;                 // Eq. 4
    const uint32_t mask = (1u << alpha) - 1u;     // F'
    const uint32_t ng = m - q + 1;                // q-grams of x
    std::vector<uint32_t> h(ng);
    for (uint32_t i = 0; i < ng; ++i) {           // h of x[i .. i+q-1]: sum_k x[i+k] 2^(s k)
        uint32_t v = 0;
        for (uint32_t k = 0; k < q; ++k) v += static_cast<uint32_t>(x[i + k]) << (s * k);
        h[i] = v & mask;
    }
    std::fill(F, F + (1u << alpha), 0u);
    for (uint32_t i = 0; i + 2 * q <= m; ++i)     // Eq. 1: u1 = x[i..i+q-1], u2 = next q bytes
        F[h[i + q]] |= 1u << (h[i] & (HC_WORD_BITS - 1));
    const uint32_t nfirst = std::min(q, ng);      // Eq. 2 + optimisation 1
    for (uint32_t i = 0; i < nfirst; ++i)
        if (F[h[i]] == 0) F[h[i]] = 1;
    *s_out = s;
    *hv_out = h[m % q];                           // first q-gram of the chain ending at m-1
}

// Device image of a handle's table, one allocation: F (2^alpha words) | the filter bitmap
// (bit v set iff F[v] != 0: the l.6 test of Fig. 5 alone, 2^alpha bits, at least 16 B) |
// x followed by at least 24 zero bytes.  Each part starts 16-byte aligned and has a
// size that is a multiple of 16, so the kernels can move F and x with 1-D TMA bulk copies
// and 16-byte loads without reading past the image.
struct ImageLayout {
    size_t f_off, bits_off, x_off, bytes;
};
ImageLayout image_layout(uint32_t alpha, size_t m) {
    ImageLayout L;
    const size_t fbytes = (size_t(1) << alpha) * sizeof(uint32_t);
    L.f_off = 0;
    L.bits_off = (fbytes + 15) & ~size_t(15);
    L.x_off = L.bits_off + std::max<size_t>(16, ((size_t(1) << alpha) / 8 + 15) & ~size_t(15));
    L.bytes = L.x_off + ((m + 24 + 15) & ~size_t(15));
    return L;
}
void write_image(const hc_handle *h, uint8_t *dst) {   // dst: image_layout(...).bytes, zeroed
    const ImageLayout L = image_layout(h->alpha, h->m);
    std::memcpy(dst + L.f_off, h->F.data(), h->F.size() * sizeof(uint32_t));
    uint32_t *bits = reinterpret_cast<uint32_t *>(dst + L.bits_off);
    for (size_t v = 0; v < h->F.size(); ++v)
        if (h->F[v]) bits[v >> 5] |= 1u << (v & 31);
    std::memcpy(dst + L.x_off, h->x.data(), h->m);
}
void bind_image(hc_handle *h, uint8_t *base) {
    const ImageLayout L = image_layout(h->alpha, h->m);
    h->dF = reinterpret_cast<uint32_t *>(base + L.f_off);
    h->dFbits = reinterpret_cast<uint32_t *>(base + L.bits_off);
    h->dx = base + L.x_off;
}

// Per-host-thread, per-device scratch: [kCtr counter words | positions (cap u32)] plus
// two mapped pinned words the search kernel's epilogue writes (count, ordered flag).  hc_search returns only
// after all of its device work completed, so the next call on this thread (any
// stream) can reuse it.  A new buffer's counter is zeroed by cudaMemsetAsync on the
// stream that will use it (a plain cudaMemset runs on the legacy stream, which a
// non-blocking caller stream does not wait for), and every finish kernel resets it.
struct Scratch {
    int dev = -1;
    uint32_t *buf = nullptr;       // device
    size_t cap = 0;                // position capacity
    uint32_t *host_count = nullptr;      // pinned, mapped
    uint32_t *host_count_dev = nullptr;  // its device alias
};
thread_local Scratch g_scratch[8];

cudaError_t get_scratch(int dev, size_t cap, cudaStream_t st, Scratch **out) {
    if (dev < 0 || dev >= 8) return cudaErrorInvalidDevice;
    Scratch &sc = g_scratch[dev];
    if (!sc.host_count) {
        void *hp = nullptr;
        cudaError_t e = cudaHostAlloc(&hp, 64, cudaHostAllocMapped | cudaHostAllocPortable);
        if (e != cudaSuccess) return e;
        void *dp = nullptr;
        e = cudaHostGetDevicePointer(&dp, hp, 0);
        if (e != cudaSuccess) return e;
        sc.host_count = static_cast<uint32_t *>(hp);
        sc.host_count_dev = static_cast<uint32_t *>(dp);
    }
    if (!sc.buf || sc.cap < cap) {
        if (sc.buf) cudaFree(sc.buf);
        sc.buf = nullptr;
        const size_t want = std::max<size_t>(cap, sc.cap + sc.cap / 2);
        // + 4 words: the epilogue copies positions in 16-byte pieces
        cudaError_t e = cudaMalloc(&sc.buf, (hc::kCtr + want + 4) * sizeof(uint32_t));
        if (e != cudaSuccess) {
            sc.cap = 0;
            return e;
        }
        e = cudaMemsetAsync(sc.buf, 0, hc::kCtr * sizeof(uint32_t), st);
        if (e != cudaSuccess) return e;
        sc.cap = want;
    }
    sc.dev = dev;
    *out = &sc;
    return cudaSuccess;
}

std::once_flag g_pool_once[64];
void tune_pool(int dev) {
    if (dev < 0 || dev >= 64) return;
    std::call_once(g_pool_once[dev], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
}

// CUDA events of one timed call (time_kernel): ev0 .. ev1, and optionally a mid event.
struct Events {
    cudaEvent_t e0 = nullptr, em = nullptr, e1 = nullptr;
    Events(bool on, bool mid) {
        if (!on) return;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        if (mid) cudaEventCreate(&em);
    }
    ~Events() {
        if (e0) cudaEventDestroy(e0);
        if (em) cudaEventDestroy(em);
        if (e1) cudaEventDestroy(e1);
    }
    void record0(cudaStream_t st) { if (e0) cudaEventRecord(e0, st); }
    void record_mid(cudaStream_t st) { if (em) cudaEventRecord(em, st); }
    void record1(cudaStream_t st) { if (e1) cudaEventRecord(e1, st); }
    void elapsed(float *total, float *mid) {
        if (!e1 || cudaEventSynchronize(e1) != cudaSuccess) return;
        cudaEventElapsedTime(total, e0, e1);
        if (em) cudaEventElapsedTime(mid, e0, em);
    }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

int sm_count(int dev) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 1;
}

int max_smem_optin(int dev) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v > 0 ? v : 48 * 1024;
}
// dynamic shared memory a kernel may request: the opt-in maximum less the kernels'
// static shared memory (s_params and the finish / sort buffers stay below 2 KiB)
int smem_budget(int dev) { return max_smem_optin(dev) - 2048; }

// Default path choice: stream the whole text through per-warp shared
// buffers when the shift is small (the lattice is dense, every sector is read);
// gather otherwise.  Measured on C2 (B200): the stream path leads the staged (TMA
// ring) path at every m <= 64 and the gather path up to m = 32 (S = 27); gather leads
// from m = 128, and m = 64 is a tie.
constexpr uint32_t kStagedMaxShift = 32;
constexpr uint32_t kDefaultStageBytes = 24576;
constexpr uint32_t kDefaultStages = 2;
// dynamic shared memory per staged CTA for 3 CTAs per SM: 228 KB per SM, 1 KB
// reserved per CTA, 1.3 KB static
constexpr uint32_t kStagedSmem3 = 233472 / 3 - 1024 - 1280;
constexpr uint32_t kDefaultChunkBytes = 3072;   // stream path: text bytes per warp chunk
constexpr uint32_t kDefaultStreamBufs = 2;      // stream path: buffers per warp
constexpr uint32_t kDefaultStreamWarps = hc::kStreamFatThreads / 32;   // stream path: most warps per CTA (one CTA per SM)
constexpr uint32_t kDenseShift = 8;   // up to this shift 24 warps at 85 registers, above 20 warps at 96 (hc_stream.cu)
constexpr uint32_t kShcLaneBytes = 128;         // SHC path: text bytes per lane and chunk
// hc_search_batch: patterns of equal (m, q, alpha) with shifts up to this share one
// streamed pass over the text (multi-pattern stream kernel)
constexpr uint32_t kMultiMaxShift = 32;
// ... and from this shift up: below it the survivors dominate and separate searches on the
// library's streams are faster (C2 m = 8: 87 vs 116 us per pattern; C3/C4 m <= 8 as well)
constexpr uint32_t kMultiMinShift = 9;
// ... and with the gather access (the patterns share the lattice's DRAM sectors) up to
#ifndef HC_MULTI_GATHER_MAX_SHIFT
#define HC_MULTI_GATHER_MAX_SHIFT 256
#endif
constexpr uint32_t kMultiGatherMaxShift = HC_MULTI_GATHER_MAX_SHIFT;

cudaError_t launch_search(int path, const hc::KParams &p, cudaStream_t st, const hc_search_opts &o,
                          hc::LaunchInfo *li) {
    switch (path) {
    case HC_PATH_STAGED: return hc::launch_staged(p, st, o.max_ctas, o.ctas_per_sm, li);
    case HC_PATH_STREAM: return hc::launch_stream(p, st, o.max_ctas, o.ctas_per_sm, li);
    case HC_PATH_SHC: return hc::launch_shc(p, st, o.max_ctas, o.ctas_per_sm, li);
    case HC_PATH_SCAN: return hc::launch_scan(p, st, o.max_ctas, o.ctas_per_sm, li);
    default: return hc::launch_gather(p, st, o.max_ctas, o.ctas_per_sm, li);
    }
}

// Launch parameters and path of one search (hc_search_ex and hc_search_batch).
int setup_search(const hc_handle *h, const uint8_t *y_dev, uint32_t nn, const hc_search_opts &o,
                 hc::KParams &p, int &path) {
    const uint32_t m = h->m, q = h->q;
    const uint32_t S = m - q + 1;
    const uint32_t windows = nn - m + 1;
    const uint32_t K = (windows + S - 1) / S;
    p = hc::KParams{};
    p.y = y_dev;
    p.n = nn;
    p.F = h->dF;
    p.Fbits = h->dFbits;
    p.x = h->dx;
    p.m = m;
    p.q = q;
    p.s = h->s;
    p.mask = h->mask;
    p.hv = h->hv;
    p.S = S;
    p.alpha = h->alpha;
    p.K = K;
    p.debug = static_cast<uint32_t>(o.debug);
    p.tma_chunk = o.tma_chunk > 0 ? (static_cast<uint32_t>(o.tma_chunk) + 15) & ~15u : 0u;
    p.trace = o.trace;
    p.trace_tiles = o.trace_tiles > 0 ? static_cast<uint32_t>(o.trace_tiles) : 0u;

    path = o.path;
    if (path == HC_PATH_AUTO) {
        path = S <= kStagedMaxShift ? HC_PATH_STREAM : HC_PATH_GATHER;
        // the gather search may give up on walk-heavy text and be re-run on the scan path
        // (hc_gather.cu), when the scan path can take this pattern
#ifdef HC_NO_ABORT
        p.allow_abort = 0 &&
#else
        p.allow_abort = path == HC_PATH_GATHER &&
#endif
                        hc::scan_smem_bytes(p.alpha, m, q, 0) <= smem_budget(h->device);
    }
    if (path == HC_PATH_STAGED) {
        uint32_t stage = o.tile_bytes > 0 ? static_cast<uint32_t>(o.tile_bytes) : kDefaultStageBytes;
        // at least 32 segments (one per lane of a warp) per tile
        const uint32_t need = 32 * S + m + 48;
        if (stage < need) stage = need;
        stage = (stage + 15) & ~15u;
        // an even number (2..16): each of the 2 survivor warps owns every other
        // iteration, hence the tile chains of half the stages
        p.stages = o.stages > 0 ? std::min<uint32_t>(16u, static_cast<uint32_t>(o.stages) + 1u) & ~1u
                                : kDefaultStages;
        p.stage_bytes = stage;
        // segments whose bytes [k0*S, m-1+k1*S) fit with 16 B of misalignment slack at
        // each end: (k1-k0)*S + m - 1 + 32 <= stage
        p.seg_per_tile = (stage - 32 - (m - 1)) / S;
        p.ntiles = (K + p.seg_per_tile - 1) / p.seg_per_tile;
        // survivor boxes of the survivor warps: a segment's text (<= m + S - 1 bytes)
        // in whole 16-byte chunks, as many as fit next to the stages for 3 CTAs per SM
        p.slot_bytes = 16 * ((m + S + 29) / 16);
        {
            const uint32_t fixed = static_cast<uint32_t>(
                hc::staged_smem_bytes(p.alpha, m, p.stage_bytes, p.stages, p.slot_bytes, 0)) + 16;
            const uint32_t room = fixed < kStagedSmem3 ? kStagedSmem3 - fixed : 0u;
            p.nbox = std::min<uint32_t>(64u, room / (2 * (p.slot_bytes + 8)));
        }
        const int smem = hc::staged_smem_bytes(p.alpha, m, p.stage_bytes, p.stages, p.slot_bytes, p.nbox);
        if (smem > smem_budget(h->device)) {
            if (o.path == HC_PATH_STAGED) return HC_EINVAL;
            path = HC_PATH_GATHER;
        }
    }
    if (path == HC_PATH_STREAM) {
        const uint32_t target = o.tile_bytes > 0 ? static_cast<uint32_t>(o.tile_bytes) : kDefaultChunkBytes;
        // a multiple of 32 * kUnroll segments, so the filter runs full unrolled steps
        // (of 32 for large shifts)
        const uint32_t unit = S <= 32 ? 128u : 32u;
        p.seg_per_chunk = unit * std::max<uint32_t>(1u, (target / S + unit / 2) / unit);
        p.nchunks = (K + p.seg_per_chunk - 1) / p.seg_per_chunk;
        // chunk bytes [a_k0 - 2q + 1, a_k1 - q] plus 16-byte alignment slack
        p.stage_bytes = (p.seg_per_chunk * S + 2 * q + 32 + 15) & ~15u;
        p.stages = kDefaultStreamBufs;   // 2 buffers per warp (3 and 4 measured slower)
        p.tma_chunk = 1;   // chunks move by one 1-D TMA bulk copy each
        // One CTA per SM with up to 24 warps: F and the per-lane filter bitmaps (2^alpha words
        // each) are held once per SM instead of once per 8-warp CTA, which leaves room for
        // 24 warps' chunk buffers.  Fewer warps when the buffers do not fit; the filter bitmap
        // unreplicated (lane_bits = 0) when even 8 warps do not fit beside the replicas.
        p.lane_bits = 1;
        if (o.block_warps >= 1 && o.block_warps <= static_cast<int>(kDefaultStreamWarps)) {
            p.block_warps = static_cast<uint32_t>(o.block_warps);
            if (hc::stream_smem_bytes(p.alpha, m, p.stage_bytes, p.stages, p.block_warps, 1) >
                smem_budget(h->device))
                p.lane_bits = 0;
        } else {
            const uint32_t w0 = S <= kDenseShift ? kDefaultStreamWarps : hc::kStreamRegThreads / 32;
            p.block_warps = w0;
            while (p.block_warps > 8 &&
                   hc::stream_smem_bytes(p.alpha, m, p.stage_bytes, p.stages, p.block_warps, 1) >
                       smem_budget(h->device))
                p.block_warps -= 4;
            if (hc::stream_smem_bytes(p.alpha, m, p.stage_bytes, p.stages, p.block_warps, 1) >
                smem_budget(h->device)) {
                p.lane_bits = 0;
                p.block_warps = w0;
                while (p.block_warps > 8 &&
                       hc::stream_smem_bytes(p.alpha, m, p.stage_bytes, p.stages, p.block_warps, 0) >
                           smem_budget(h->device))
                    p.block_warps -= 4;
            }
        }
        // final drain on private boxes (hc_stream.cu): 16 bytes of slack + the segment's reach
        // m + S - 1 in whole 16-byte words, one box per lane in the warp's idle chunk buffers
        {
            const uint32_t slot = 16 + ((m + S - 1 + 30 + 15) & ~15u);
            p.slot_bytes = 32 * slot <= p.stages * p.stage_bytes && o.seg_per_lane >= 0 ? slot : 0u;
        }
        // shifts too long for per-warp buffers (S > ~200) take the gather path, which
        // reads only the q-grams it hashes anyway
        if (hc::stream_smem_bytes(p.alpha, m, p.stage_bytes, p.stages, p.block_warps, p.lane_bits) >
            smem_budget(h->device))
            path = HC_PATH_GATHER;
    }
    if (path == HC_PATH_SHC) {
        // each lane owns c consecutive segments (about kShcLaneBytes of text)
        // (measured on C2: 32 bytes per lane for shifts <= 16, 256 above: 1.2-1.6x faster
        // than a uniform 128)
        const uint32_t lane_target = o.tile_bytes > 0 ? static_cast<uint32_t>(o.tile_bytes) / 32
                                                      : (S <= 16 ? 32u : 2 * kShcLaneBytes);
        const uint32_t c = std::max<uint32_t>(1u, (lane_target + S / 2) / S);
        p.shc = 1;
        p.seg_per_chunk = 32 * c;
        p.nchunks = (K + p.seg_per_chunk - 1) / p.seg_per_chunk;
        p.stages = 2;
        // chunk bytes [a_k0 - m + 1, a_k1 - 1] plus alignment slack
        p.stage_bytes = (p.seg_per_chunk * S + m + 48 + 15) & ~15u;
        // box: the lane's bytes (c S + m - 1) in whole 16-byte words, then x (m) and the
        // 8-byte word reads around its end
        p.slot_bytes = (c * S + 2 * m + 40 + 15) & ~15u;
        uint32_t nw = o.block_warps >= 1 && o.block_warps <= 8 ? static_cast<uint32_t>(o.block_warps) : 8u;
        while (nw > 1 && hc::shc_smem_bytes(p.alpha, m, p.stage_bytes, p.slot_bytes, nw) >
                             smem_budget(h->device))
            --nw;
        if (hc::shc_smem_bytes(p.alpha, m, p.stage_bytes, p.slot_bytes, nw) > smem_budget(h->device))
            return HC_EINVAL;   // m too long for per-lane boxes
        p.block_warps = nw;
    }
    if (path == HC_PATH_SCAN) {
        // pieces of window ends staged with their (m-1)-byte halo (hc_scan.cu)
        p.nchunks = 0;
        if (hc::scan_smem_bytes(p.alpha, m, q, 0) > smem_budget(h->device))
            return HC_EINVAL;   // pattern too long for the staged pieces
    }
    if (path == HC_PATH_GATHER) {
        // lattice points per lane per chunk (1, 2 or 4; the chunk's loads go out together):
        // 4 while every resident warp (about 32 per SM) still gets a chunk, fewer for the
        // short lattices of large m, so that the latency-bound chains spread over all warps
        uint32_t spl = 4;
        if (o.seg_per_lane > 0) {
            spl = o.seg_per_lane >= 4 ? 4u : (o.seg_per_lane >= 2 ? 2u : 1u);
        } else {
            const uint64_t warps = static_cast<uint64_t>(sm_count(h->device)) * 32u;
            while (spl > 1 && K < warps * 32u * spl) spl /= 2;
        }
        p.seg_per_chunk = 32 * spl;
        p.nchunks = (K + p.seg_per_chunk - 1) / p.seg_per_chunk;
        if (hc::gather_smem_bytes(p.alpha, m) > smem_budget(h->device)) return HC_EINVAL;
    }

    return HC_OK;
}

// hc_search_batch resources, per host thread and device: kBatchStreams non-blocking
// streams, each with its own scratch (counter + positions), and a mapped pinned array
// the finish kernels write the patterns' counts into.
constexpr int kBatchStreams = 8;
struct BatchRes {
    cudaStream_t st[kBatchStreams] = {};
    cudaEvent_t ev[kBatchStreams + 1] = {};
    Scratch sc[kBatchStreams];
    uint32_t *hcounts = nullptr, *hcounts_dev = nullptr;
    size_t ncounts = 0;
};
thread_local BatchRes g_batch[8];

// Batch scratch of one pool stream: [kMaxPatterns counters of 16 B | positions], the
// positions of a multi-pattern launch's pattern g at offset g * (cap / npat).
constexpr size_t kCtrWords = hc::kCtr * hc::kMaxPatterns;
cudaError_t batch_scratch(Scratch &sc, size_t cap, cudaStream_t st) {
    if (!sc.buf || sc.cap < cap) {
        if (sc.buf) cudaFree(sc.buf);
        sc.buf = nullptr;
        cudaError_t e = cudaMalloc(&sc.buf, (kCtrWords + cap + 4) * sizeof(uint32_t));
        if (e != cudaSuccess) {
            sc.cap = 0;
            return e;
        }
        e = cudaMemsetAsync(sc.buf, 0, kCtrWords * sizeof(uint32_t), st);   // on the user stream
        if (e != cudaSuccess) return e;
        sc.cap = cap;
    }
    return cudaSuccess;
}

cudaError_t batch_res(int dev, size_t npat, BatchRes **out) {
    if (dev < 0 || dev >= 8) return cudaErrorInvalidDevice;
    BatchRes &r = g_batch[dev];
    if (!r.st[0]) {
        for (int i = 0; i < kBatchStreams; ++i) {
            cudaError_t e = cudaStreamCreateWithFlags(&r.st[i], cudaStreamNonBlocking);
            if (e != cudaSuccess) return e;
        }
        for (int i = 0; i <= kBatchStreams; ++i) {
            cudaError_t e = cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
    }
    if (r.ncounts < npat) {
        if (r.hcounts) cudaFreeHost(r.hcounts);
        r.hcounts = nullptr;
        r.ncounts = 0;
        void *hp = nullptr;
        const size_t want = std::max<size_t>(npat, 256);
        cudaError_t e = cudaHostAlloc(&hp, want * 8, cudaHostAllocMapped | cudaHostAllocPortable);
        if (e != cudaSuccess) return e;
        void *dp = nullptr;
        e = cudaHostGetDevicePointer(&dp, hp, 0);
        if (e != cudaSuccess) return e;
        r.hcounts = static_cast<uint32_t *>(hp);
        r.hcounts_dev = static_cast<uint32_t *>(dp);
        r.ncounts = want;
    }
    *out = &r;
    return cudaSuccess;
}

}  // namespace

extern "C" {

const char *hc_version(void) { return "hc-b200 0.1 (sm_100a)"; }

int hc_last_error(void) { return g_last_error; }

const char *hc_strerror(int code) {
    switch (code) {
        case HC_OK: return "ok";
        case HC_EINVAL: return "invalid argument";
        case HC_ETOOSHORT: return "pattern shorter than q (q > m)";
        case HC_EALPHA: return "alpha outside [1, 15]";
        case HC_ENOMEM: return "out of memory";
        case HC_ECUDA: return "CUDA runtime error";
        case HC_ETOOLONG: return "text or pattern too long";
        case HC_ENODEV: return "no usable CUDA device";
        default: return "unknown error";
    }
}

int hc_build_table(const uint8_t *x, size_t m, int q, int alpha, uint32_t *F_out, int *s_out,
                   uint32_t *hv_out) {
    const int rc = check_params(x, m, q, alpha);
    if (rc != HC_OK) return fail(rc);
    if (!F_out) return fail(HC_EINVAL);
    uint32_t s = 0, hv = 0;
    build_table(x, static_cast<uint32_t>(m), static_cast<uint32_t>(q), static_cast<uint32_t>(alpha),
                F_out, &s, &hv);
    if (s_out) *s_out = static_cast<int>(s);
    if (hv_out) *hv_out = hv;
    return HC_OK;
}

hc_handle *hc_prepare(const uint8_t *x, size_t m, int q, int alpha) {
    const int rc = check_params(x, m, q, alpha);
    if (rc != HC_OK) {
        fail(rc);
        return nullptr;
    }
    hc_handle *h = new (std::nothrow) hc_handle();
    if (!h) {
        fail(HC_ENOMEM);
        return nullptr;
    }
    h->m = static_cast<uint32_t>(m);
    h->q = static_cast<uint32_t>(q);
    h->alpha = static_cast<uint32_t>(alpha);
    h->mask = (1u << alpha) - 1u;
    h->x.assign(x, x + m);
    h->F.assign(1u << alpha, 0u);
    build_table(x, h->m, h->q, h->alpha, h->F.data(), &h->s, &h->hv);

    cudaError_t e = cudaGetDevice(&h->device);
    if (e != cudaSuccess) {
        delete h;
        cuda_fail(e, "cudaGetDevice");
        g_last_error = HC_ENODEV;
        return nullptr;
    }
    {
        const ImageLayout L = image_layout(h->alpha, h->m);
        std::vector<uint8_t> img(L.bytes, 0);
        write_image(h, img.data());
        void *base = nullptr;
        e = cudaMalloc(&base, L.bytes);
        if (e == cudaSuccess) {
            bind_image(h, static_cast<uint8_t *>(base));
            e = cudaMemcpy(base, img.data(), L.bytes, cudaMemcpyHostToDevice);
        }
    }
    if (e != cudaSuccess) {
        cuda_fail(e, "hc_prepare upload");
        hc_destroy(h);
        return nullptr;
    }
    g_last_error = HC_OK;
    return h;
}

// Device blocks of hc_prepare_batch are recycled (size classes of powers of two, per
// device) instead of cudaMalloc / cudaFree per batch: cudaFree synchronises the device
// and both calls showed multi-millisecond outliers in the end-to-end loop.
namespace {
std::mutex g_block_mu;
std::vector<std::pair<size_t, void *>> g_block_pool[8];
void *block_get(int dev, size_t bytes, size_t *cls) {
    size_t c = 4096;
    while (c < bytes) c <<= 1;
    *cls = c;
    {
        std::lock_guard<std::mutex> lk(g_block_mu);
        auto &pool = g_block_pool[dev & 7];
        for (size_t i = 0; i < pool.size(); ++i)
            if (pool[i].first == c) {
                void *p = pool[i].second;
                pool.erase(pool.begin() + static_cast<long>(i));
                return p;
            }
    }
    void *p = nullptr;
    return cudaMalloc(&p, c) == cudaSuccess ? p : nullptr;
}
void block_put(int dev, size_t cls, void *p) {
    std::lock_guard<std::mutex> lk(g_block_mu);
    auto &pool = g_block_pool[dev & 7];
    if (pool.size() < 64) pool.emplace_back(cls, p);
    else cudaFree(p);
}
}  // namespace

int hc_prepare_batch(const uint8_t *const *xs, const size_t *ms, size_t P, int q, int alpha,
                     hc_handle **hs_out) {
    if (P == 0) return HC_OK;
    if (!xs || !ms || !hs_out) return fail(HC_EINVAL);
    for (size_t i = 0; i < P; ++i) {
        const int rc = check_params(xs[i], ms[i], q, alpha);
        if (rc != HC_OK) return fail(rc);
    }
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        cuda_fail(e, "cudaGetDevice");
        return fail(HC_ENODEV);
    }
    // host tables (Fig. 3 per pattern), laid out as the device block: one image per pattern
    std::vector<size_t> off(P + 1, 0);
    for (size_t i = 0; i < P; ++i) off[i + 1] = off[i] + image_layout(static_cast<uint32_t>(alpha), ms[i]).bytes;
    std::vector<hc_handle *> hs(P, nullptr);
    std::vector<uint8_t> staging(off[P], 0);
    for (size_t i = 0; i < P; ++i) {
        hc_handle *h = new (std::nothrow) hc_handle();
        if (!h) {
            for (hc_handle *t : hs) delete t;
            return fail(HC_ENOMEM);
        }
        hs[i] = h;
        h->m = static_cast<uint32_t>(ms[i]);
        h->q = static_cast<uint32_t>(q);
        h->alpha = static_cast<uint32_t>(alpha);
        h->mask = (1u << alpha) - 1u;
        h->device = dev;
        h->x.assign(xs[i], xs[i] + ms[i]);
        h->F.assign(size_t(1) << alpha, 0u);
        build_table(xs[i], h->m, h->q, h->alpha, h->F.data(), &h->s, &h->hv);
        write_image(h, staging.data() + off[i]);
    }
    size_t cls = 0;
    void *blk = block_get(dev, off[P], &cls);
    e = blk ? cudaMemcpy(blk, staging.data(), off[P], cudaMemcpyHostToDevice) : cudaErrorMemoryAllocation;
    if (e != cudaSuccess) {
        if (blk) block_put(dev, cls, blk);
        for (hc_handle *t : hs) delete t;
        return cuda_fail(e, "hc_prepare_batch upload");
    }
    // the block goes back to the pool with the last handle (searches using it are
    // complete by then: the caller must not destroy a handle while a search on it is
    // in flight, as for hc_prepare handles)
    std::shared_ptr<void> block(blk, [dev, cls](void *p) { block_put(dev, cls, p); });
    for (size_t i = 0; i < P; ++i) {
        bind_image(hs[i], static_cast<uint8_t *>(blk) + off[i]);
        hs[i]->block = block;
        hs_out[i] = hs[i];
    }
    g_last_error = HC_OK;
    return HC_OK;
}

void hc_destroy(hc_handle *h) {
    if (!h) return;
    if (!h->block) {   // hc_prepare: own allocation (batch handles share h->block)
        if (h->dF) cudaFree(h->dF);
    }
    delete h;
}

int hc_table(const hc_handle *h, const uint32_t **F, int *alpha, int *s, int *w, uint32_t *h_v) {
    if (!h) return fail(HC_EINVAL);
    if (F) *F = h->F.data();
    if (alpha) *alpha = static_cast<int>(h->alpha);
    if (s) *s = static_cast<int>(h->s);
    if (w) *w = HC_WORD_BITS;
    if (h_v) *h_v = h->hv;
    return HC_OK;
}

int64_t hc_search_ex(const hc_handle *h, const uint8_t *y_dev, size_t n, int64_t *pos_out,
                     size_t max_out, cudaStream_t stream, const hc_search_opts *opts,
                     hc_search_stats *stats) {
    if (!h) return fail(HC_EINVAL);
    if (n > 0 && !y_dev) return fail(HC_EINVAL);
    if (n > HC_MAX_TEXT) return fail(HC_ETOOLONG);
    hc_search_opts o{};
    if (opts) o = *opts;
    if (!HC_INSTRUMENT && (o.debug != 0 || o.trace != nullptr))
        return fail(HC_EINVAL);   // measurement-only modes exist in libhc_instr.so only
    if (stats) *stats = hc_search_stats{};
    g_last_error = HC_OK;
    if (n < h->m) return 0;  // S:123, reading R9

    DeviceGuard guard(h->device);
    tune_pool(h->device);
    const bool want_pos = pos_out != nullptr && max_out > 0;
    const uint32_t m = h->m, q = h->q;
    const uint32_t S = m - q + 1;
    const uint32_t nn = static_cast<uint32_t>(n);
    const uint32_t windows = nn - m + 1;
    const uint32_t K = (windows + S - 1) / S;

    hc::KParams p{};
    int path = 0;
    {
        const int rc = setup_search(h, y_dev, nn, o, p, path);
        if (rc != HC_OK) return fail(rc);
    }

    // scratch: [counter | positions]
    size_t cap = 0;
    if (want_pos) cap = std::min<size_t>(std::max<size_t>(max_out, size_t(1) << 16), windows);
    const uint32_t k_out = want_pos ? static_cast<uint32_t>(std::min<size_t>(max_out, windows)) : 0;

    int launches = 0, reruns = 0;
    uint32_t count = 0;
    float kms = 0.f, sms = 0.f;
    hc::LaunchInfo li;
    // time_kernel: ev0 before the first search launch, ev1 after the call's last kernel
    // (re-recorded after a re-run or a host-launched ordering: the span then also holds
    // the count read-back gaps); time_kernel = 2 also keeps evS right after the first
    // search kernel (search + fused epilogue, one kernel).
    Events ev(o.time_kernel != 0, o.time_kernel >= 2);
    ev.record0(stream);
    for (int attempt = 0;; ++attempt) {
        Scratch *sc = nullptr;
        cudaError_t e = get_scratch(h->device, cap, stream, &sc);
        if (e != cudaSuccess) return cuda_fail(e, "scratch");
        p.counter = sc->buf;
        p.out = want_pos ? sc->buf + hc::kCtr : nullptr;
        p.cap = static_cast<uint32_t>(cap);
        p.host_count = sc->host_count_dev;
        p.dst = want_pos ? pos_out : nullptr;
        p.k_out = k_out;
        p.nbits = hc::bits_for(nn);
        sc->host_count[0] = 0xffffffffu;
        sc->host_count[1] = 0;
        // one kernel: search + fused epilogue (count publication, ordering when it can)
        e = launch_search(path, p, stream, o, &li);
        ++launches;
        if (attempt == 0) ev.record_mid(stream);
        ev.record1(stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) {
            // the counters may be left non-zero: force a fresh scratch next time
            cudaFree(sc->buf);
            sc->buf = nullptr;
            sc->cap = 0;
            return cuda_fail(e, "search kernel");
        }
        const volatile uint32_t *hcnt = sc->host_count;
        count = hcnt[0];
        if (hcnt[1] == 2u) {
            // walk-heavy text: the gather search gave up; the scan path hashes every
            // q-gram once (hc_scan.cu) and returns exactly the same result
            hc_search_opts os = o;
            os.path = HC_PATH_SCAN;
            const int rc = setup_search(h, y_dev, nn, os, p, path);
            if (rc != HC_OK) return fail(rc);
            ++reruns;
            continue;
        }
        const bool ordered = hcnt[1] != 0;
#if HC_INSTRUMENT
        if (o.debug == 10) {
            unsigned long long ts[16] = {};
            hc::read_epi_ts(ts);
            std::fprintf(stderr, "epilogue block_order phases (ns): load %llu hist %llu scan %llu "
                                 "scatter %llu rank+store %llu\n", ts[1] - ts[0], ts[3] - ts[1],
                         ts[4] - ts[3], ts[5] - ts[4], ts[6] - ts[5]);
        }
#endif
        if (HC_INSTRUMENT && (o.debug == 5 || o.debug == 10) && stats) {
            cudaMemcpy(stats->dbg, sc->buf + 6, 8, cudaMemcpyDeviceToHost);
            cudaMemset(sc->buf + 4, 0, 16);
        }
        if (want_pos && count > cap) {
            // position scratch overflowed: the count is exact, re-run with room for all
            cap = count;
            ++reruns;
            continue;
        }
        if (want_pos && count > 0 && !ordered) {
            // more positions than the epilogue's shared memory holds (or clustered): order
            // them on the device from the scratch (hc_finish.cu)
            const uint32_t k = static_cast<uint32_t>(std::min<size_t>(count, max_out));
            e = hc::order_positions(sc->buf + hc::kCtr, count, nn, pos_out, k, stream, &launches);
            ev.record1(stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
            if (e != cudaSuccess) return cuda_fail(e, "ordering");
        }
        break;
    }
    ev.elapsed(&kms, &sms);
    if (stats) {
        stats->path = path;
        stats->grid = li.grid;
        stats->block = li.block;
        stats->smem_bytes = li.smem;
        stats->tiles = path == HC_PATH_STAGED ? p.ntiles : p.nchunks;
        stats->launches = launches;
        stats->reruns = reruns;
        stats->kernel_ms = kms;
        stats->search_ms = sms;
    }
    return static_cast<int64_t>(count);
}

int hc_search_batch(const hc_handle *const *hs, size_t npat, const uint8_t *y_dev, size_t n,
                    int64_t *counts, int64_t *const *pos_out, const size_t *max_out,
                    cudaStream_t stream, const hc_search_opts *opts, hc_search_stats *stats) {
    if (npat == 0) return HC_OK;
    if (!hs || !counts || (n > 0 && !y_dev)) return fail(HC_EINVAL);
    if (n > HC_MAX_TEXT) return fail(HC_ETOOLONG);
    hc_search_opts o{};
    if (opts) o = *opts;
    o.debug = 0;
    o.trace = nullptr;
    if (stats) *stats = hc_search_stats{};
    g_last_error = HC_OK;
    const int dev = hs[0] ? hs[0]->device : -1;
    for (size_t i = 0; i < npat; ++i)
        if (!hs[i] || hs[i]->device != dev) return fail(HC_EINVAL);
    DeviceGuard guard(dev);
    tune_pool(dev);
    BatchRes *r = nullptr;
    cudaError_t e = batch_res(dev, npat, &r);
    if (e != cudaSuccess) return cuda_fail(e, "batch resources");
    const uint32_t nn = static_cast<uint32_t>(n);

    // the pool streams start after the caller's stream (y_dev is ready there)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (o.time_kernel) {
        cudaEventCreate(&ev0);
        cudaEventCreate(&ev1);
        cudaEventRecord(ev0, stream);
    }
    cudaEventRecord(r->ev[kBatchStreams], stream);
    for (int j = 0; j < kBatchStreams; ++j) cudaStreamWaitEvent(r->st[j], r->ev[kBatchStreams], 0);

    // One exit for every failure after this point: the caller's stream waits for the
    // pool streams (launches already queued keep writing r->hcounts and the scratch),
    // everything is synchronised, the events are destroyed, and the pool scratch is
    // dropped (its counters may be left non-zero).  Only then is the error returned.
    auto join_pool = [&]() {
        for (int j = 0; j < kBatchStreams; ++j) {
            cudaEventRecord(r->ev[j], r->st[j]);
            cudaStreamWaitEvent(stream, r->ev[j], 0);
        }
    };
    auto bail = [&](int code) -> int {
        join_pool();
        cudaStreamSynchronize(stream);
        cudaGetLastError();
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        for (int j = 0; j < kBatchStreams; ++j) {
            if (r->sc[j].buf) cudaFree(r->sc[j].buf);
            r->sc[j].buf = nullptr;
            r->sc[j].cap = 0;
        }
        return code;
    };

    std::vector<size_t> caps(npat, 0);
    int launches = 0;
    int nlaunch = 0;   // search launches so far (round-robin over the pool streams)
    auto same_shape = [&](const hc_handle *a, const hc_handle *b) {
        return a->m == b->m && a->q == b->q && a->alpha == b->alpha;
    };
    for (size_t i = 0; i < npat;) {
        const hc_handle *h = hs[i];
        r->hcounts[2 * i] = 0xffffffffu;
        r->hcounts[2 * i + 1] = 0;
        if (n < h->m) {
            r->hcounts[2 * i] = 0;
            r->hcounts[2 * i + 1] = 1;
            ++i;
            continue;
        }
        const size_t windows = n - h->m + 1;
        const uint32_t S = h->m - h->q + 1;
        // multi-pattern launch: the next patterns of the same (m, q, alpha)
        size_t g = 1;
        const bool stream_multi = S <= kMultiMaxShift;
        const int multi_path = stream_multi ? HC_PATH_STREAM : HC_PATH_GATHER;
        const bool multi_ok = (o.no_multi == 2 || (o.no_multi == 0 && S >= kMultiMinShift)) &&
                              S <= kMultiGatherMaxShift &&
                              (o.path == HC_PATH_AUTO || o.path == multi_path);
        if (multi_ok)
            while (i + g < npat && g < static_cast<size_t>(hc::kMaxPatterns) && hs[i + g] &&
                   n >= hs[i + g]->m && same_shape(h, hs[i + g]))
                ++g;
        const int j = nlaunch++ % kBatchStreams;
        Scratch &sc = r->sc[j];
        hc::KParams p{};
        int path = 0;
        if (g > 1) {
            // stream geometry; all g F tables in one CTA's shared memory: 16 warps per CTA
            // and 2 KiB chunks when more than two share it, else the stream defaults
            hc_search_opts og = o;
            og.path = multi_path;
            for (; g > 1; --g) {
                og.tile_bytes = stream_multi && o.tile_bytes == 0 && g > 2 ? 2048 : o.tile_bytes;
                const int rc = setup_search(h, y_dev, nn, og, p, path);
                if (rc != HC_OK) return fail(bail(rc));
                if (path != multi_path) continue;
                if (stream_multi) {
                    p.block_warps = o.block_warps > 0 ? std::min<uint32_t>(16u, static_cast<uint32_t>(o.block_warps))
                                                      : (g > 2 ? 16u : 8u);
                    p.stages = 2;   // multi-pattern kernel: 2 buffers per warp
                } else {   // gather access, no stage buffers
                    p.mgather = 1;
                    p.block_warps = o.block_warps > 0 ? std::min<uint32_t>(16u, static_cast<uint32_t>(o.block_warps))
                                                      : 8u;
                    p.stage_bytes = 0;
                    p.stages = 2;
                }
                if (hc::mstream_smem_bytes(p.alpha, p.m, p.stage_bytes, p.block_warps,
                                           static_cast<uint32_t>(g), p.stages) <=
                    smem_budget(dev))
                    break;
            }
        }
        if (g == 1) {
            const int rc = setup_search(h, y_dev, nn, o, p, path);
            if (rc != HC_OK) return fail(bail(rc));
        }
        // per-pattern position capacity
        size_t cap = 0;
        for (size_t t = 0; t < g; ++t) {
            const size_t mo = max_out ? max_out[i + t] : 0;
            if (pos_out && pos_out[i + t] && mo > 0)
                cap = std::max(cap, std::min<size_t>(std::max<size_t>(mo, size_t(1) << 16), windows));
        }
        const size_t stride = (cap + 3) & ~size_t(3);   // 16-byte aligned per-pattern regions
        e = batch_scratch(sc, std::max<size_t>(stride * g, 1), r->st[j]);
        if (e != cudaSuccess) return bail(cuda_fail(e, "batch scratch"));
        hc::LaunchInfo li;
        p.nbits = hc::bits_for(nn);
        if (g == 1) {
            const size_t mo = max_out ? max_out[i] : 0;
            const bool want_pos = pos_out && pos_out[i] && mo > 0;
            caps[i] = want_pos ? cap : 0;
            p.counter = sc.buf;
            p.out = want_pos ? sc.buf + kCtrWords : nullptr;
            p.cap = static_cast<uint32_t>(caps[i]);
            p.host_count = r->hcounts_dev + 2 * i;
            p.dst = want_pos ? pos_out[i] : nullptr;
            p.k_out = want_pos ? static_cast<uint32_t>(std::min<size_t>(mo, windows)) : 0u;
            r->hcounts[2 * i + 1] = 0;
            e = launch_search(path, p, r->st[j], o, &li);
        } else {
            hc::MParams mp{};
            mp.npat = static_cast<uint32_t>(g);
            for (size_t t = 0; t < g; ++t) {
                const hc_handle *ht = hs[i + t];
                const size_t mo = max_out ? max_out[i + t] : 0;
                const bool want_pos = pos_out && pos_out[i + t] && mo > 0;
                caps[i + t] = want_pos ? cap : 0;
                mp.F[t] = ht->dF;
                mp.x[t] = ht->dx;
                mp.hv[t] = ht->hv;
                mp.counter[t] = sc.buf + hc::kCtr * t;
                mp.out[t] = want_pos ? sc.buf + kCtrWords + t * stride : nullptr;
                mp.cap[t] = static_cast<uint32_t>(caps[i + t]);
                mp.host_count[t] = r->hcounts_dev + 2 * (i + t);
                mp.dst[t] = want_pos ? pos_out[i + t] : nullptr;
                mp.k_out[t] = want_pos ? static_cast<uint32_t>(std::min<size_t>(mo, windows)) : 0u;
                r->hcounts[2 * (i + t)] = 0xffffffffu;
                r->hcounts[2 * (i + t) + 1] = 0;
            }
            e = hc::launch_mstream(p, mp, r->st[j], o.max_ctas, o.ctas_per_sm, &li);
        }
        ++launches;
        if (e != cudaSuccess) return bail(cuda_fail(e, "batch launch"));
        i += g;
    }
    join_pool();
    e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return bail(cuda_fail(e, "batch execution"));
    // patterns whose positions did not fit the scratch, or that the epilogue could not
    // order (the pool scratch has been reused since), are run again on their own (their
    // counts are exact already); the device time of the batch
    // (stats->kernel_ms) runs to the end of these re-runs
    int reruns = 0;
    for (size_t i = 0; i < npat; ++i) {
        const uint32_t c = reinterpret_cast<volatile uint32_t *>(r->hcounts)[2 * i];
        const uint32_t flag = reinterpret_cast<volatile uint32_t *>(r->hcounts)[2 * i + 1];
        const bool ordered = flag == 1u;
        const bool gave_up = flag == 2u;   // walk-heavy text: the count is not known
        counts[i] = c;
        const size_t mo = max_out ? max_out[i] : 0;
        const bool want_pos = pos_out && pos_out[i] && mo > 0;
        if (gave_up || (want_pos && c > 0 && (c > caps[i] || !ordered))) {
            hc_search_opts orr = o;
            orr.time_kernel = 0;
            hc_search_stats rs{};
            const int64_t c2 = hc_search_ex(hs[i], y_dev, n, want_pos ? pos_out[i] : nullptr,
                                            want_pos ? mo : 0, stream, &orr, &rs);
            if (c2 < 0) return bail(static_cast<int>(c2));
            launches += rs.launches;
            counts[i] = c2;
            ++reruns;
        }
    }
    float kms = 0.f;
    if (o.time_kernel) {
        cudaEventRecord(ev1, stream);
        if (cudaEventSynchronize(ev1) == cudaSuccess) cudaEventElapsedTime(&kms, ev0, ev1);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
    }
    if (stats) {
        stats->launches = launches;
        stats->reruns = reruns;
        stats->kernel_ms = kms;
    }
    return HC_OK;
}

int64_t hc_search(const hc_handle *h, const uint8_t *y_dev, size_t n, int64_t *pos_out,
                  size_t max_out, cudaStream_t stream) {
    return hc_search_ex(h, y_dev, n, pos_out, max_out, stream, nullptr, nullptr);
}

int64_t hc_search_host(const hc_handle *h, const uint8_t *y_host, size_t n, int64_t *pos_out_host,
                       size_t max_out, cudaStream_t stream) {
    if (!h) return fail(HC_EINVAL);
    if (n > 0 && !y_host) return fail(HC_EINVAL);
    if (n > HC_MAX_TEXT) return fail(HC_ETOOLONG);
    g_last_error = HC_OK;
    if (n < h->m) return 0;
    DeviceGuard guard(h->device);
    tune_pool(h->device);
    const bool want_pos = pos_out_host != nullptr && max_out > 0;
    const size_t k_cap = want_pos ? std::min<size_t>(max_out, n - h->m + 1) : 0;
    uint8_t *dy = nullptr;
    int64_t *dpos = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&dy), n, stream);
    if (e == cudaSuccess && want_pos) e = cudaMallocAsync(reinterpret_cast<void **>(&dpos), k_cap * 8, stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dy, y_host, n, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) {
        if (dy) cudaFreeAsync(dy, stream);
        if (dpos) cudaFreeAsync(dpos, stream);
        return cuda_fail(e, "hc_search_host upload");
    }
    const int64_t cnt = hc_search_ex(h, dy, n, dpos, k_cap, stream, nullptr, nullptr);
    if (cnt > 0 && want_pos) {
        const size_t k = std::min<size_t>(static_cast<size_t>(cnt), k_cap);
        e = cudaMemcpyAsync(pos_out_host, dpos, k * 8, cudaMemcpyDeviceToHost, stream);
    }
    cudaFreeAsync(dy, stream);
    if (dpos) cudaFreeAsync(dpos, stream);
    cudaError_t e2 = cudaStreamSynchronize(stream);
    if (cnt < 0) return cnt;
    if (e != cudaSuccess) return cuda_fail(e, "hc_search_host read-back");
    if (e2 != cudaSuccess) return cuda_fail(e2, "hc_search_host sync");
    return cnt;
}

int hc_search_batch_host(const hc_handle *const *hs, size_t npat, const uint8_t *y_host, size_t n,
                         int64_t *counts, int64_t *const *pos_out_host, const size_t *max_out,
                         cudaStream_t stream, const hc_search_opts *opts, hc_search_stats *stats) {
    if (npat == 0) return HC_OK;
    if (!hs || !counts || (n > 0 && !y_host)) return fail(HC_EINVAL);
    if (n > HC_MAX_TEXT) return fail(HC_ETOOLONG);
    for (size_t i = 0; i < npat; ++i)
        if (!hs[i]) return fail(HC_EINVAL);
    g_last_error = HC_OK;
    DeviceGuard guard(hs[0]->device);
    tune_pool(hs[0]->device);
    // one device block: the text, then each pattern's position buffer (8-byte aligned)
    std::vector<size_t> off(npat + 1, 0);
    const size_t ybytes = (n + 15) & ~size_t(15);
    off[0] = ybytes;
    for (size_t i = 0; i < npat; ++i) {
        const bool want = pos_out_host && pos_out_host[i] && max_out && max_out[i] > 0 && n >= hs[i]->m;
        const size_t k = want ? std::min<size_t>(max_out[i], n - hs[i]->m + 1) : 0;
        off[i + 1] = off[i] + 8 * k;
    }
    uint8_t *blk = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&blk), std::max<size_t>(off[npat], 16), stream);
    if (e != cudaSuccess) return cuda_fail(e, "hc_search_batch_host alloc");
    if (n > 0) e = cudaMemcpyAsync(blk, y_host, n, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) {
        cudaFreeAsync(blk, stream);
        return cuda_fail(e, "hc_search_batch_host upload");
    }
    std::vector<int64_t *> dpos(npat, nullptr);
    std::vector<size_t> ks(npat, 0);
    for (size_t i = 0; i < npat; ++i) {
        ks[i] = (off[i + 1] - off[i]) / 8;
        if (ks[i]) dpos[i] = reinterpret_cast<int64_t *>(blk + off[i]);
    }
    int rc = hc_search_batch(hs, npat, blk, n, counts, dpos.data(), ks.data(), stream, opts, stats);
    if (rc == HC_OK) {
        for (size_t i = 0; i < npat && e == cudaSuccess; ++i) {
            const size_t k = std::min<size_t>(ks[i], counts[i] > 0 ? static_cast<size_t>(counts[i]) : 0);
            if (k) e = cudaMemcpyAsync(pos_out_host[i], dpos[i], 8 * k, cudaMemcpyDeviceToHost, stream);
        }
    }
    cudaFreeAsync(blk, stream);
    const cudaError_t e2 = cudaStreamSynchronize(stream);
    if (rc != HC_OK) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "hc_search_batch_host read-back");
    if (e2 != cudaSuccess) return cuda_fail(e2, "hc_search_batch_host sync");
    return HC_OK;
}

}  // extern "C"
