// hc_scan.cu — "hash every position, then filter" window scan (HC_PATH_SCAN; the SURVEY
// 8(a) design choice the north star names beside the sequential skip loop).
//
// The paper's loop (Fig. 5 left) re-hashes the same q-grams many times when
// most windows pass the filter and walk far: on walk-heavy texts (the stress config C5)
// every window end of a clean stretch walks its whole chain, ~7 hashes per text
// byte.  Here every q-gram of a staged piece of text is hashed ONCE and the three facts
// the loop asks of a position p become bits:
//   N(p) = [F[h(p)] != 0]                       filter test at window end p (l.5-6)
//   L(p) = bit lambda(h(p - q)) of F[h(p)]      link test of a walk step from p (l.11-12)
//   H(p) = [h(p) == H_v]                        the test after a completed walk (l.14)
// kept as bitmaps over the piece's positions (one ballot per 32 positions).  The walk
// of Fig. 5 from window end e tests L(e), L(e - q), ..., L(e - (T-1) q) (T = floor(m/q) - 1
// link tests) and, completed, H(e - T q): bits q apart.  So for every window end at once
//   V(e) = N(e) AND L(e) AND L(e - q) ... AND L(e - (T-1) q) AND H(e - T q)
// is a handful of shifted word ANDs (runs of T ones at stride q by doubling: shifts of
// k q bits), and the windows with V(e) are verified against x (l.16).
//
// Exactness (reading R16): every occurrence e satisfies V(e) -- its q-grams
// are x's, whose F words are non-zero and whose adjacent pairs are linked (Eq. 1-2,
// Fig. 3), and its chain ends at the q-gram whose hash is H_v -- and every
// window HC verifies satisfies V(e) too.  So {e : V(e) and y[e-m+1..e] == x} is exactly
// HC's output; windows HC would have skipped may be verified as well, never reported
// unless they match.  This is the filter-soundness invariant the oracle tests pin.
//
// Pieces of kScanPiece window ends per warp, staged with their (m-1)-byte halo by
// 16-byte cp.async copies, two buffers per warp.
#include "hc_device.cuh"

namespace hc {

constexpr uint32_t kScanWarps = 8;             // warps per CTA
constexpr uint32_t kScanPiece = 2048;          // window ends per warp piece
struct ScanLayout {
    uint32_t f_off, x_off, warp_off, warp_bytes, total;
    uint32_t buf_bytes, nw;                    // stage bytes; words per bitmap
};
__host__ __device__ inline ScanLayout scan_layout(uint32_t alpha, uint32_t m, uint32_t q) {
    ScanLayout L;
    L.f_off = 0;
    L.x_off = round_up((1u << alpha) * 4u, 16);
    L.warp_off = L.x_off + round_up(m + 8, 16);
    L.buf_bytes = round_up(kScanPiece + m + 48, 16);
    // positions [(a0 - m + q) & ~31, a1): < kScanPiece + m + 32, a multiple of 4 words
    L.nw = round_up((kScanPiece + m + 31) / 32 + 1, 4);
    // stage x 2 | N, L, H, R, A, V (nw words each) | match buffer
    L.warp_bytes = round_up(2 * L.buf_bytes + 6 * 4 * L.nw + kWarpBuf * 4u, 128);
    L.total = L.warp_off + kScanWarps * L.warp_bytes;
    (void)q;
    return L;
}
int scan_smem_bytes(uint32_t alpha, uint32_t m, uint32_t q, uint32_t) {
    return static_cast<int>(scan_layout(alpha, m, q).total);
}

// Word w of src shifted up by `a` bits across the word array (bit i of the result = bit
// i - a of src, 0 below).
__device__ __forceinline__ uint32_t shifted_word(const uint32_t *src, int32_t w, uint32_t a) {
    const int32_t ws = w - static_cast<int32_t>(a >> 5);
    const uint32_t b = a & 31u;
    const uint32_t hi = ws >= 0 ? src[ws] : 0u;
    const uint32_t lo = (b && ws >= 1) ? src[ws - 1] : 0u;
    return b ? (hi << b) | (lo >> (32 - b)) : hi;
}

template <int Q, int SH>
__global__ void __launch_bounds__(kScanWarps * 32) scan_kernel(const KParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const ScanLayout Lo = scan_layout(p.alpha, p.m, Q);
    uint32_t *sFp = reinterpret_cast<uint32_t *>(smem + Lo.f_off);
    uint8_t *sx = smem + Lo.x_off;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint8_t *wr = smem + Lo.warp_off + warp * Lo.warp_bytes;
    const uint32_t bufs0 = smem_u32(wr);
    const uint32_t QW = Lo.nw;                      // words of one bitmap
    uint32_t *Nb = reinterpret_cast<uint32_t *>(wr + 2 * Lo.buf_bytes);
    uint32_t *Lb = Nb + QW, *Hb = Lb + QW, *Rb = Hb + QW, *Ab = Rb + QW, *Vb = Ab + QW;
    uint32_t *wbuf = Vb + QW;
    const uint32_t total_warps = gridDim.x * kScanWarps;
    const uint32_t gw = blockIdx.x * kScanWarps + warp;
    const uint32_t npieces = (p.n - p.m + 1 + kScanPiece - 1) / kScanPiece;
    auto issue = [&](uint32_t c, uint32_t buf) {   // window ends [a0, a1): text [a0-m+1, a1-1]
        const uint32_t a0 = p.m - 1 + c * kScanPiece;
        const uint32_t a1 = c < npieces ? min(a0 + kScanPiece, p.n) : a0 + 1;
        issue_range(p, c < npieces, a0 + 1 - p.m, a1 - 1, buf, lane);
    };
    issue(gw, bufs0);                               // first piece's copy before the table
    load_table(p, sFp, sx);
    if (tid == 0) s_params[0] = p;
    __syncthreads();
    const FTable sF{fence_value(smem_u32(sFp))};
    WarpOut wo{wbuf, 0u};
    const uint32_t y32 = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p.y));
    const uint32_t T = p.m / Q - 1;                 // link tests of a complete walk
    uint32_t bsel = 0;
    for (uint32_t c = gw; c < npieces; c += total_warps) {
        issue(c + total_warps, bufs0 + (bsel ^ 1u) * Lo.buf_bytes);
        cp_async_wait<1>();
        __syncwarp();
        const uint32_t a0 = p.m - 1 + c * kScanPiece;
        const uint32_t a1 = min(a0 + kScanPiece, p.n);
        const uint32_t first = a0 + 1 - p.m;
        const uint32_t buf = fence_value(bufs0 + bsel * Lo.buf_bytes);
        const SmemText txt{buf + ((y32 + first) & 15u) - first};      // text t at base + t
        const uint32_t Ps = a0 + Q - p.m;          // first q-gram inside the piece
        const uint32_t base = Ps & ~31u;            // bit 0 of word 0 = position base
        const uint32_t nwu = (a1 - base + 31) / 32; // words in use (<= QW - 1)
        // 1. one hash per position: lane l takes position base + 32 w + l; h(p - q) is lane
        //    l - q's hash (lanes < q: the previous word's lanes 32 - q + l)
        uint32_t hlast = 0;
        for (uint32_t w0 = 0; w0 < QW; w0 += 4) {                  // 4 words in flight (ILP)
            uint32_t h[4], z[4];
            bool in[4];
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) {
                const uint32_t pos = base + 32 * (w0 + u) + lane;
                in[u] = w0 + u < nwu && pos >= Ps && pos < a1;
                h[u] = in[u] ? qhash<Q, SH>(end8<Q>(txt, pos), p.mask) : 0u;
            }
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) z[u] = in[u] ? sF[h[u]] : 0u;
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) {
                const uint32_t pos = base + 32 * (w0 + u) + lane;
                const uint32_t up = __shfl_up_sync(HC_FULL, h[u], Q);
                const uint32_t wrap = __shfl_sync(HC_FULL, u ? h[u - 1] : hlast, (lane + 32 - Q) & 31);
                const uint32_t hp = lane >= Q ? up : wrap;                // h(pos - q)
                const bool lbit = in[u] && pos >= Ps + Q && ((z[u] >> (hp & (kWordBits - 1))) & 1u);
                const uint32_t nm = __ballot_sync(HC_FULL, z[u] != 0u);
                const uint32_t lm = __ballot_sync(HC_FULL, lbit);
                const uint32_t hm = __ballot_sync(HC_FULL, in[u] && h[u] == p.hv);
                if (lane == 0) {
                    Nb[w0 + u] = nm;
                    Lb[w0 + u] = lm;
                    Hb[w0 + u] = hm;
                }
            }
            hlast = h[3];
        }
        __syncwarp();
        // 2. V = N & (runs of T ones of L at stride q, ending at the bit) & (H << T q).
        //    Runs by doubling: R_1 = L, R_2k = R_k & (R_k << k q); A accumulates R_s for the
        //    binary digits of T (A_{s+k} = A_s & (R_k << s q)).
        {
            uint32_t s = 0, k = 1, t = T;
            for (uint32_t i = lane; i < QW; i += 32) Rb[i] = Lb[i];
            __syncwarp();
            while (t) {
                if (t & 1u) {
                    for (uint32_t i = lane; i < QW; i += 32) {
                        const uint32_t rs = shifted_word(Rb, static_cast<int32_t>(i), s * Q);
                        Ab[i] = s ? Ab[i] & rs : rs;
                    }
                    s += k;
                    __syncwarp();
                }
                t >>= 1;
                if (t) {                                // R_2k = R_k & (R_k << k q), via V
                    for (uint32_t i = lane; i < QW; i += 32)
                        Vb[i] = Rb[i] & shifted_word(Rb, static_cast<int32_t>(i), k * Q);
                    __syncwarp();
                    for (uint32_t i = lane; i < QW; i += 32) Rb[i] = Vb[i];
                    __syncwarp();
                    k <<= 1;
                }
            }
            for (uint32_t i = lane; i < QW; i += 32) {
                const uint32_t hs = shifted_word(Hb, static_cast<int32_t>(i), T * Q);
                Vb[i] = Nb[i] & (T ? Ab[i] : 0xffffffffu) & hs;
            }
            __syncwarp();
        }
        // 3. verify every window end e in [a0, a1) with V(e) (l.16-17, index per R1)
        for (uint32_t i0 = 0; i0 < QW; i0 += 32) {
            const uint32_t i = i0 + lane;
            uint32_t bits = i < QW ? Vb[i] : 0u;
            while (__any_sync(HC_FULL, bits != 0u)) {
                bool found = false;
                uint32_t start = 0;
                if (bits) {
                    const uint32_t b = __ffs(bits) - 1;
                    bits &= bits - 1;
                    const uint32_t e = base + 32 * i + b;
                    if (e >= a0 && e < a1) {
                        start = e + 1 - p.m;
                        found = verify(txt, sx, start, p.m);
                    }
                }
                wo.push(found, start, p, lane);
            }
        }
        __syncwarp();
        bsel ^= 1u;
    }
    cp_async_wait<0>();
    wo.flush(p, lane);
    search_epilogue(p, smem);
}

template <int Q, int SH>
struct PickScan {
    using Fn = KernFn;
    static KernFn fn() { return scan_kernel<Q, SH>; }
};

cudaError_t launch_scan(const KParams &p, cudaStream_t st, int max_ctas, int ctas_per_sm,
                        LaunchInfo *li) {
    KernFn kern = pick<PickScan>(p.q, p.s);
    if (!kern) return cudaErrorInvalidValue;
    const int smem = scan_smem_bytes(p.alpha, p.m, p.q, 0);
    const long pieces = (static_cast<long>(p.n) - p.m + 1 + kScanPiece - 1) / kScanPiece;
    const long ctas = (pieces + kScanWarps - 1) / kScanWarps;
    KParams a = p;
    a.epi_cap = epi_cap_for(smem);
    void *args[] = {&a};
    return launch_kernel(reinterpret_cast<const void *>(kern), args, kScanWarps * 32, smem, ctas,
                         max_ctas, ctas_per_sm, st, li);
}

}  // namespace hc
