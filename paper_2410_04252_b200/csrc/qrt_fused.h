// libqrt — QR fused into the next gate pass ("reorder on load").
//
// A QR (reference perform_qr, dist_sim.cpp:203-240) permutes the index bits
// of the whole distributed state.  Instead of a separate exchange kernel, the
// first gate pass after the QR gathers its tile straight from the source
// PEs' live buffers (local HBM or a peer's over NVLink 5, CUDA IPC mappings)
// and writes its result into this PE's spare buffer: the exchange overlaps
// the pass's math and the intermediate HBM round trip of the exchange
// disappears.  Ranks meet at one barrier before such a pass (every source
// buffer is complete) and before any later write into a buffer a peer may
// still read.
#pragma once

#include <cstdint>

#include "qrt_internal.h"

namespace qrt {

struct FusedSource {
    const amp_t* src[kMaxLocalPEs];  // every PE's live buffer, by global PE index
    amp_t* dst[kMaxLocalPEs];        // this process's PEs' spare buffers, by local PE index
    int src_of[64];                  // destination position t <- source position src_of[t]
    int n, nl, pe_begin;
};

// Shared-memory tables of one CTA: source index of tile element e is
//   S = cta ^ hi[e >> c] ^ lo[0][el & 63] ^ lo[1][(el >> 6) & 63],  el = e & (2^c - 1)
// (the position permutation is linear over XOR on disjoint bits).
inline constexpr int kFusedSmemWords = 2 * 64 + 1;  // + (1 << (T - c)) for hi

__device__ __forceinline__ std::uint64_t fused_perm(const FusedSource& f, std::uint64_t x) {
    std::uint64_t s = 0;
    while (x) {
        const int t = __ffsll(static_cast<long long>(x)) - 1;
        s |= 1ull << f.src_of[t];
        x &= x - 1;
    }
    return s;
}

// Fills hi[nt], lo[128], cta (smem words) for the CTA whose destination tile
// has CTA offset `base` on global PE `pe_dst`; tab[h] = destination offsets of
// the tile's high bits.  Ends with __syncthreads().
__device__ __forceinline__ void fused_tables(const FusedSource& f, const std::uint64_t* tab, int nt, std::uint64_t base,
                                             int pe_dst, std::uint64_t* words) {
    std::uint64_t* hi = words + kFusedSmemWords;
    for (int h = threadIdx.x; h < nt; h += blockDim.x) hi[h] = fused_perm(f, tab[h]);
    for (int i = threadIdx.x; i < 128; i += blockDim.x) {
        const std::uint64_t l = static_cast<std::uint64_t>(i & 63) << (6 * (i >> 6));
        words[i] = fused_perm(f, l);
    }
    if (threadIdx.x == 0)
        words[128] = fused_perm(f, (static_cast<std::uint64_t>(pe_dst) << f.nl) | base);
    __syncthreads();
}

__device__ __forceinline__ const amp_t* fused_src(const FusedSource& f, const std::uint64_t* words, int e, int cmask,
                                                  int c) {
    const std::uint64_t* hi = words + kFusedSmemWords;
    const int el = e & cmask;
    const std::uint64_t S = words[128] ^ hi[e >> c] ^ words[el & 63] ^ words[64 + ((el >> 6) & 63)];
    QRT_DCHECK((S >> f.nl) < (1ull << (f.n - f.nl)) && f.src[S >> f.nl] != nullptr);
    return f.src[S >> f.nl] + (S & ((1ull << f.nl) - 1));
}

}  // namespace qrt
