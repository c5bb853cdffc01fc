// hc_inst.cu — kernel instantiations for one q-gram length, compiled once per q
// (-DHC_Q=1..8) so that the 8 units build in parallel.  Each unit exports the
// staged and gather kernels for every shift s = floor(alpha/q) <= 15/q and lattice
// word size WD (8 always, 4 when q <= 4, 1 = general unaligned lattice).
#include "hc_internal.h"
#include "hc_device.cuh"

#ifndef HC_Q
#error "compile with -DHC_Q=<1..8>"
#endif

namespace hc {

namespace {
constexpr int kQ = HC_Q;
constexpr int kMaxSh = kQ == 1 ? 0 : 15 / kQ;

template <int SH>
KernFn pick_staged(uint32_t wd) {
    if constexpr (SH > kMaxSh) {
        return nullptr;
    } else {
        if (wd == 8) return staged_kernel<kQ, SH, 8>;
        if constexpr (kQ <= 4) {
            if (wd == 4) return staged_kernel<kQ, SH, 4>;
        }
        if (wd == 1) return staged_kernel<kQ, SH, 1>;
        return nullptr;
    }
}
template <int SH>
KernFn pick_gather(uint32_t wd) {
    if constexpr (SH > kMaxSh) {
        return nullptr;
    } else {
        if (wd == 8) return gather_kernel<kQ, SH, 8>;
        if constexpr (kQ <= 4) {
            if (wd == 4) return gather_kernel<kQ, SH, 4>;
        }
        if (wd == 1) return gather_kernel<kQ, SH, 1>;
        return nullptr;
    }
}
template <bool STAGED, int SH = 0>
KernFn pick(uint32_t sh, uint32_t wd) {
    if constexpr (SH > 7) {
        return nullptr;
    } else {
        if (sh == SH) return STAGED ? pick_staged<SH>(wd) : pick_gather<SH>(wd);
        return pick<STAGED, SH + 1>(sh, wd);
    }
}
}  // namespace

#define HC_CAT2(a, b) a##b
#define HC_CAT(a, b) HC_CAT2(a, b)
KernFn HC_CAT(staged_kernel_q, HC_Q)(uint32_t s, uint32_t wd) {
    return pick<true>(kQ == 1 ? 0u : s, wd);
}
KernFn HC_CAT(gather_kernel_q, HC_Q)(uint32_t s, uint32_t wd) {
    return pick<false>(kQ == 1 ? 0u : s, wd);
}

}  // namespace hc
