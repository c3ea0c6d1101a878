// libqrt — register-coset EVC passes (reference local_pauli_expectation +
// expectation, dist_sim.cpp:84-97 and :289-298).  Shared by the host planner
// (qrt_pauli.cu) and the kernel (qrt_coset.cu).
//
// A pass loads a 2^12-amplitude tile (positions B) into shared memory once.
// Its flip-mask groups are covered by *cosets*: five tile bits Q; every
// thread of the 128-thread CTA then holds the 32 amplitudes of one coset of
// Q in registers and evaluates every group whose flip mask x lies in Q from
// registers alone: for the 16 canonical pairs (r, r^x) of the coset
//   sum_t F_t s_t(i) comp_t(conj(v[i^x]) v[i])
//     = sigma(thread) * sum_rho C[rho] * comp(conj(a[r^x]) a[r]),
// where the 16-entry table C folds every term's sign over the register bits
// and sigma = (-1)^{popc(W & mf) + popc(pe & gz)} is the sign over the bits
// outside Q, common to the group's terms (the host splits a group when it is
// not).  For Jordan-Wigner words (Re(w) only, real coefficients) a pair costs
// three fp64 instructions, and one shared-memory read of a coset (16 B per
// amplitude) serves up to C(5,4)+C(5,2) = 15 groups.
#pragma once

#include <cstdint>

#include "qrt_internal.h"

namespace qrt {

inline constexpr int kCosetBits = 5;                                  // 32 amplitudes per thread
inline constexpr int kCosetThreads = 1 << (kTileBits - kCosetBits);   // 128
inline constexpr int kCosetMaxSets = 40;
inline constexpr int kCosetMaxGroups = 320;
inline constexpr int kCosetMaxTab = 2048;  // doubles in the launch parameters

// CosetGroup::mf also carries gz shifted to this bit (W < 2^n_local <= 2^40
// never reaches it), so W | pe << kCosetPeShift folds both sign masks into one.
inline constexpr int kCosetPeShift = 40;

struct CosetGroup {
    std::uint64_t mf;  // sign bits outside Q, as bits of the thread word W (| gz << kCosetPeShift)
    std::uint64_t gz;  // sign bits over the PE index
    std::int16_t tab;  // first double of the group's table(s) in CosetParams::tabs
    std::int8_t xq;    // flip mask over the coset's register bits (nonzero)
    std::int8_t mode;  // 0: Re(w) only with real coefficients (16 doubles), 1: general (64 doubles),
                       // 2: Im(w) only with real coefficients (16 doubles; single-bit masks only)
};

struct CosetSet {
    std::int8_t S[kCosetBits];                // tile bit of register bit q
    std::int8_t tb[kTileBits - kCosetBits];   // tile bit of thread-index bit i
    std::int16_t g_begin, g_count;
    std::uint32_t present;  // bit x: some fast group has mask x
    std::uint8_t xbeg[32];  // fast groups sorted by mask: [xbeg[x-1], xbeg[x]) have mask x
    std::uint8_t one_cnt[kCosetBits];  // then single-bit-mask groups: one_cnt[k] with mask 1 << k; generic after them
    std::uint8_t one_re[kCosetBits];   // ... of which the first one_re[k] are mode 0 and the next one_im[k] mode 2
    std::uint8_t one_im[kCosetBits];
    // host-precomputed per set (coset_set_tables): the thread's tile index is
    // eb_lo[t & 15] | eb_hi[t >> 4], and swq[q] the swizzled offset of register bit q
    std::uint16_t eb_lo[16];
    std::uint16_t eb_hi[8];
    std::int16_t swq[kCosetBits];
    // >= 0: every present fast mask has exactly one group, whose table sits at
    // tab1 + 16 * popc(present & (2^x - 1)) (no per-group metadata on the table
    // path, QRT_EVC_SINGLE); -1 otherwise
    std::int16_t tab1;
    // >= 0 for every register bit k: the set has no fast groups and exactly one
    // single-bit group of mask 1 << k for each k with onetab[k] >= 0, whose
    // table starts at onetab[k] (mode in onemode bits 2k..2k+1); the group's
    // index is g_begin + popc(onemask below k).  onemask == 0: not this form.
    std::int16_t onetab[kCosetBits];
    std::uint8_t onemask;
    std::uint16_t onemode;
};

// Shared-memory swizzle of tile element e (GF(2)-linear): the host twin of the
// kernels' swz(), used to precompute CosetSet::swq.
inline constexpr int coset_swz(int e) {
    return e ^ (((e >> 3) ^ (e >> 6) ^ (e >> 9) ^ (e >> 12)) & 7);
}

inline void coset_set_tables(CosetSet& S) {
    for (int v = 0; v < 16; ++v) {
        int e = 0;
        for (int i = 0; i < 4; ++i) e |= ((v >> i) & 1) << S.tb[i];
        S.eb_lo[v] = static_cast<std::uint16_t>(e);
    }
    for (int v = 0; v < 8; ++v) {
        int e = 0;
        for (int i = 0; i < 3; ++i) e |= ((v >> i) & 1) << S.tb[4 + i];
        S.eb_hi[v] = static_cast<std::uint16_t>(e);
    }
    for (int q = 0; q < kCosetBits; ++q) S.swq[q] = static_cast<std::int16_t>(coset_swz(1 << S.S[q]));
}

// W = tile index (bits 0..11) | outer index of the CTA (bit 12 + i <-> outer axis i).
struct CosetParams {
    const amp_t* ptrs[kMaxLocalPEs];
    int c;
    int n_outer;
    int n_sets;
    int pe_begin;
    int tiles_per_pe;
    int d_begin, d_count;  // I/Z words of this pass (global term array), Walsh-Hadamard path
    int n_tab;             // doubles of tabs in use (staged in shared memory)
    int set_tables;        // 1: per-set thread-index / swizzle tables from the host (QRT_EVC_SET_TABLES)
    int present_guard;     // 1: skip a set's weight-2/4 mask tests when it has none (QRT_EVC_PRESENT_GUARD)
    int single;            // 1: take the tab1 path of sets with one group per fast mask (QRT_EVC_SINGLE)
    int fill_mode;         // 1: pipelined tile fill with warp-reduced base + unrolled linear-swizzle addressing (QRT_EVC_FILL)
    const double* gtabs;   // device copy of tabs[0, n_tab) (coalesced staging)
    // Tile / outer axes as index vectors: element (outer b, tile e) sits at
    //   XOR_i b_i outer_vec[i]  ^  XOR_{i >= c} e_i tile_vec[i]  ^  (e & (2^c - 1)).
    // Ordinary passes use unit vectors (axes = positions); *linear* passes
    // (wide flip masks) use a GF(2) basis whose tile axes are the flip masks
    // themselves, so every batched group flips a single tile bit.
    std::uint64_t tile_vec[kTileBits];
    std::uint64_t outer_vec[64];
    CosetSet sets[kCosetMaxSets];
    CosetGroup groups[kCosetMaxGroups];
    double tabs[kCosetMaxTab];
};

// I/Z word of the Walsh-Hadamard path (same layout as the tiled EVC kernel's).
struct CosetDiagTerm {
    std::uint64_t m;   // full sign mask (local positions)
    std::uint64_t gz;  // PE-index sign mask
    double2 f;         // coefficient
    int m_tile;        // sign mask bits inside the tile, tile-bit indices
    int pad;
};

void launch_coset_pass(CosetParams& P, const CosetDiagTerm* dterms, int pe_count, double* red,
                       cudaStream_t stream, int device);

}  // namespace qrt
