// libqrt — register-coset EVC pass kernel (see qrt_coset.h).
//
// Reference semantics: per PE, partial[pe] += sum_t coeff_t * pe_sign_t *
// local_pauli_expectation(sub[pe], mask_t)  (dist_sim.cpp:84-97, 289-295),
// evaluated pair-wise over the canonical half of each flip-mask group.
// One CTA = one 2^12-amplitude tile = 128 threads x 32-amplitude cosets.

#include <algorithm>
#include <cstdlib>

#include "qrt_coset.h"

namespace qrt {

namespace {

using u64 = std::uint64_t;

__device__ __forceinline__ int swz(int e) {
    const int x = e >> 3;
    return e ^ ((x ^ (x >> 3) ^ (x >> 6) ^ (x >> 9)) & 7);
}

__device__ __forceinline__ int insert_zero(int v, int bit) {
    return ((v >> bit) << (bit + 1)) | (v & ((1 << bit) - 1));
}

__host__ __device__ constexpr int top_bit(int v) { return v >= 16 ? 4 : v >= 8 ? 3 : v >= 4 ? 2 : v >= 2 ? 1 : 0; }
__host__ __device__ constexpr int ins0(int v, int bit) { return ((v >> bit) << (bit + 1)) | (v & ((1 << bit) - 1)); }

// sum_rho T[rho] * Re(conj(a[r^XQ]) a[r]) over the 16 canonical pairs
// (r, r^XQ) of the coset, r without the top bit of XQ (register indices are
// compile-time: one code body per mask).
// QRT_EVC_EARLY_TABLES: issue the group's 8 table loads (LDS.128) before the
// pair products, pinned by volatile asm, so their latency overlaps the DMUL /
// DFMA work instead of stalling the accumulation chains (the compiler places
// them after the products to save registers).  Kept on while the table
// address came from a per-group record (JW -0.4%); with the table path
// (CosetSet::tab1) the compiler's own placement is faster: 30q JW EVC
// 767 -> 749 ms (same-box A/B, profiles/r2/evcvar), so it is off.
#ifndef QRT_EVC_EARLY_TABLES
#define QRT_EVC_EARLY_TABLES 0
#endif

#ifndef QRT_EVC_PE_FOLD
#define QRT_EVC_PE_FOLD 1
#endif
#ifndef QRT_EVC_BYTE_GATHER
#define QRT_EVC_BYTE_GATHER 1
#endif
#ifndef QRT_EVC_THREAD_ACC
#define QRT_EVC_THREAD_ACC 0
#endif
#ifndef QRT_EVC_FMA_SIGN
#define QRT_EVC_FMA_SIGN 1
#endif
#ifndef QRT_EVC_EB_PREFETCH
#define QRT_EVC_EB_PREFETCH 1
#endif
#ifndef QRT_EVC_UNIFORM_PRESENT
#define QRT_EVC_UNIFORM_PRESENT 1
#endif

__device__ __forceinline__ double2 lds_f64x2(const double2* p) {
    double2 v;
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}

// (-1)^{popc(W & mf) + popc(pe & gz)} as a double: one POPC of the folded
// mask, the parity lands in the sign bit (fma(sign, r, acc) == acc +- r exactly).
__device__ __forceinline__ double group_sign(std::uint64_t W, std::uint64_t pe, const CosetGroup& G) {
#if QRT_EVC_PE_FOLD
    const std::uint64_t m = (W | (pe << kCosetPeShift)) & G.mf;  // gz rides in mf above bit 40
#else
    const std::uint64_t m = (W & G.mf) ^ (pe & G.gz);
#endif
    const unsigned x = static_cast<unsigned>(m) ^ static_cast<unsigned>(m >> 32);
    return __hiloint2double(static_cast<int>(0x3ff00000u | (static_cast<unsigned>(__popc(x)) << 31)), 0);
}

#ifndef QRT_EVC_ACCS
#define QRT_EVC_ACCS 4  // independent accumulator chains per group (2 / 8: see DESIGN §8)
#endif

template <int XQ>
__device__ __forceinline__ double coset_group(const double2 (&a)[32], const double2* __restrict__ T2) {
    constexpr int H = top_bit(XQ);
#if QRT_EVC_ACCS != 4
    constexpr int NA = QRT_EVC_ACCS;
    double accn[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) accn[i] = 0.0;
#pragma unroll
    for (int h = 0; h < 8; ++h) {
        const double2 t = lds_f64x2(T2 + h);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int rho = 2 * h + u;
            const int r = ins0(rho, H);
            const int s = r ^ XQ;
            const double2 A = a[s], B = a[r];
            accn[rho % NA] = fma(u ? t.y : t.x, fma(A.x, B.x, A.y * B.y), accn[rho % NA]);
        }
    }
#pragma unroll
    for (int w = NA / 2; w > 0; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) accn[i] += accn[i + w];
    return accn[0];
#else
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#if QRT_EVC_EARLY_TABLES
    double2 tt[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) tt[h] = lds_f64x2(T2 + h);
#endif
#pragma unroll
    for (int h = 0; h < 8; ++h) {
#if QRT_EVC_EARLY_TABLES
        const double2 t = tt[h];
#else
        const double2 t = T2[h];  // table entries 2h, 2h+1 (shared-memory broadcast)
#endif
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int rho = 2 * h + u;
            const int r = ins0(rho, H);
            const int s = r ^ XQ;
            const double2 A = a[s], B = a[r];
            acc[rho & 3] = fma(u ? t.y : t.x, fma(A.x, B.x, A.y * B.y), acc[rho & 3]);
        }
    }
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
#endif
}

// Single-bit register mask XQ (linear passes), any table mode: the 16 pairs
// (r, r^XQ) from registers; mode 0 tables weight Re(w) only, mode 1 tables
// (64 doubles) map (Re w, Im w) to the complex accumulator.
template <int XQ>
__device__ __forceinline__ double2 coset_one(const double2 (&a)[32], const double* __restrict__ T, int mode) {
    constexpr int H = top_bit(XQ);
    const double2* __restrict__ T2 = reinterpret_cast<const double2*>(T);  // tables are 16-byte aligned
    double2 acc = make_double2(0.0, 0.0);
    if (mode != 1) {  // one real table over Re(w) (mode 0) or Im(w) (mode 2)
        const bool im = mode == 2;
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int h = 0; h < 8; ++h) {
            const double2 t = T2[h];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int rho = 2 * h + u, r = ins0(rho, H), s = r ^ XQ;
                const double2 A = a[s], B = a[r];
                const double w = im ? fma(A.x, B.y, -A.y * B.x) : fma(A.x, B.x, A.y * B.y);
                s4[rho & 3] = fma(u ? t.y : t.x, w, s4[rho & 3]);
            }
        }
        acc.x = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    } else {
#pragma unroll
        for (int h = 0; h < 8; ++h) {
            const double2 t0 = T2[h], t1 = T2[8 + h], t2 = T2[16 + h], t3 = T2[24 + h];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int rho = 2 * h + u, r = ins0(rho, H), s = r ^ XQ;
                const double2 A = a[s], B = a[r];
                const double re = fma(A.x, B.x, A.y * B.y), im = fma(A.x, B.y, -A.y * B.x);
                acc.x = fma(u ? t0.y : t0.x, re, fma(u ? t2.y : t2.x, im, acc.x));
                acc.y = fma(u ? t1.y : t1.x, re, fma(u ? t3.y : t3.x, im, acc.y));
            }
        }
    }
    return acc;
}

// sum_rho T[rho] * Im(conj(a[r^XQ]) a[r]) (Im(w)-only groups, real coefficients).
template <int XQ>
__device__ __forceinline__ double coset_group_im(const double2 (&a)[32], const double2* __restrict__ T2) {
    constexpr int H = top_bit(XQ);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int h = 0; h < 8; ++h) {
        const double2 t = T2[h];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int rho = 2 * h + u;
            const int r = ins0(rho, H);
            const int s = r ^ XQ;
            const double2 A = a[s], B = a[r];
            acc[rho & 3] = fma(u ? t.y : t.x, fma(A.x, B.y, -A.y * B.x), acc[rho & 3]);
        }
    }
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// The single-bit groups of mask 1 << K: one_re[K] Re(w)-only, then one_im[K]
// Im(w)-only (both real, 16-entry tables), then general ones (64 entries).
template <int K>
__device__ __forceinline__ void coset_ones(const double2 (&a)[32], const CosetParams& P, const CosetSet& S,
                                           const double* __restrict__ tabs, int& g, std::uint64_t W, std::uint64_t pe,
                                           double2& acc) {
    const int n = S.one_cnt[K], nre = S.one_re[K], nim = S.one_im[K];
    const double2* __restrict__ t2 = reinterpret_cast<const double2*>(tabs);
    for (int i = 0; i < nre; ++i, ++g) {
        const CosetGroup& G = P.groups[g];
        const double r = coset_group<1 << K>(a, t2 + (G.tab >> 1));
        const int odd = (__popcll(W & G.mf) + __popcll(pe & G.gz)) & 1;
        acc.x += odd ? -r : r;
    }
    for (int i = 0; i < nim; ++i, ++g) {
        const CosetGroup& G = P.groups[g];
        const double r = coset_group_im<1 << K>(a, t2 + (G.tab >> 1));
        const int odd = (__popcll(W & G.mf) + __popcll(pe & G.gz)) & 1;
        acc.x += odd ? -r : r;
    }
    for (int i = nre + nim; i < n; ++i, ++g) {
        const CosetGroup& G = P.groups[g];
        const double2 r = coset_one<1 << K>(a, tabs + G.tab, 1);
        const int odd = (__popcll(W & G.mf) + __popcll(pe & G.gz)) & 1;
        acc.x += odd ? -r.x : r.x;
        acc.y += odd ? -r.y : r.y;
    }
}

// The single single-bit group of mask 1 << K (CosetSet::onemask form): table
// offset and mode come with the set, so the table loads wait on nothing.
template <int K>
__device__ __forceinline__ void coset_one1(const double2 (&a)[32], const CosetParams& P, const CosetSet& S,
                                           const double* __restrict__ tabs, unsigned onemask, unsigned onemode,
                                           std::uint64_t W, std::uint64_t pe, double2& acc) {
    if (!((onemask >> K) & 1u)) return;
    const int mode = (onemode >> (2 * K)) & 3;
    const double* T = tabs + S.onetab[K];
    const CosetGroup& G = P.groups[S.g_begin + __popc(onemask & ((1u << K) - 1u))];
#if QRT_EVC_FMA_SIGN
    const double sg = group_sign(W, pe, G);
    if (mode != 1) {
        const double2* T2 = reinterpret_cast<const double2*>(T);
        const double r = mode == 0 ? coset_group<1 << K>(a, T2) : coset_group_im<1 << K>(a, T2);
        acc.x = fma(sg, r, acc.x);
    } else {
        const double2 r = coset_one<1 << K>(a, T, 1);
        acc.x = fma(sg, r.x, acc.x);
        acc.y = fma(sg, r.y, acc.y);
    }
#else
    const int odd = (__popcll(W & G.mf) + __popcll(pe & G.gz)) & 1;
    if (mode != 1) {
        const double2* T2 = reinterpret_cast<const double2*>(T);
        const double r = mode == 0 ? coset_group<1 << K>(a, T2) : coset_group_im<1 << K>(a, T2);
        acc.x += odd ? -r : r;
    } else {
        const double2 r = coset_one<1 << K>(a, T, 1);
        acc.x += odd ? -r.x : r.x;
        acc.y += odd ? -r.y : r.y;
    }
#endif
}

// Any flip mask / table mode, pairs read from the shared-memory tile
// (groups outside the Jordan-Wigner fast set: odd weights, Im(w) terms,
// complex coefficients).
__device__ __noinline__ double2 coset_generic(const double2* __restrict__ tile, int sb, const int* swq, int xq,
                                              int mode, const double* __restrict__ T) {
    const int H = 31 - __clz(xq);
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int rho = 0; rho < 16; ++rho) {
        const int r = insert_zero(rho, H), s = r ^ xq;
        int orr = sb, os = sb;
        for (int q = 0; q < kCosetBits; ++q) {
            if ((r >> q) & 1) orr ^= swq[q];
            if ((s >> q) & 1) os ^= swq[q];
        }
        const double2 A = tile[os], B = tile[orr];
        const double re = fma(A.x, B.x, A.y * B.y);
        if (mode == 0) {
            acc.x = fma(T[rho], re, acc.x);
        } else {
            const double im = fma(A.x, B.y, -A.y * B.x);
            acc.x = fma(T[rho], re, fma(T[32 + rho], im, acc.x));
            acc.y = fma(T[16 + rho], re, fma(T[48 + rho], im, acc.y));
        }
    }
    return acc;
}

// The fast groups of a coset set (Re(w) only, real coefficients, flip
// masks of weight 2 or 4) are sorted by mask: [xbeg[x-1], xbeg[x]) have mask
// x.  The 15 masks are walked in a fixed unrolled order (one code body per
// mask, no switch), so the coset stays in registers.
template <int XQ>
__device__ __forceinline__ void coset_fast(const double2 (&a)[32], const CosetParams& P, const CosetSet& S,
                                           const double2* __restrict__ tabs, unsigned present, std::uint64_t W,
                                           std::uint64_t pe, double2& acc) {
    if (!((present >> XQ) & 1u)) return;
    const int g0 = S.g_begin + S.xbeg[XQ - 1], g1 = S.g_begin + S.xbeg[XQ];
    for (int g = g0; g < g1; ++g) {
        const CosetGroup& G = P.groups[g];
        const double r = coset_group<XQ>(a, tabs + (G.tab >> 1));
        const int odd = (__popcll(W & G.mf) + __popcll(pe & G.gz)) & 1;
        acc.x += odd ? -r : r;
    }
}

#if QRT_EVC_THREAD_ACC
// Table path with the group sign moved onto the table entries (an integer XOR
// of their sign bits) and the products accumulated into four per-thread
// chains that run across groups and sets: no per-group tree or sign tail.
template <int XQ>
__device__ __forceinline__ void coset_fast1t(const double2 (&a)[32], const CosetParams& P, const CosetSet& S,
                                             const double2* __restrict__ tabs, unsigned present, int tab1,
                                             std::uint64_t W, std::uint64_t pe, double (&acc4)[4]) {
    if (!((present >> XQ) & 1u)) return;
    constexpr int H = top_bit(XQ);
    const int i = __popc(present & ((1u << XQ) - 1u));
    const CosetGroup& G = P.groups[S.g_begin + i];
    const std::uint64_t m = (W & G.mf) ^ (pe & G.gz);
    const int sb = static_cast<int>(static_cast<unsigned>(__popc(static_cast<unsigned>(m) ^
                                                                 static_cast<unsigned>(m >> 32))) << 31);
    const double2* __restrict__ T2 = tabs + (tab1 >> 1) + 8 * i;
#pragma unroll
    for (int h = 0; h < 8; ++h) {
        const double2 t = T2[h];
        const double tx = __hiloint2double(__double2hiint(t.x) ^ sb, __double2loint(t.x));
        const double ty = __hiloint2double(__double2hiint(t.y) ^ sb, __double2loint(t.y));
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int rho = 2 * h + u;
            const int r = ins0(rho, H);
            const int s = r ^ XQ;
            const double2 A = a[s], B = a[r];
            acc4[rho & 3] = fma(u ? ty : tx, fma(A.x, B.x, A.y * B.y), acc4[rho & 3]);
        }
    }
}
#endif

// One group per present mask (CosetSet::tab1 >= 0): the group's rank among
// the set's fast groups is popc(present below XQ), so its table address needs
// no per-group metadata load (only the sign masks are read, off the chain).
template <int XQ>
__device__ __forceinline__ void coset_fast1(const double2 (&a)[32], const CosetParams& P, const CosetSet& S,
                                            const double2* __restrict__ tabs, unsigned present, int tab1,
                                            std::uint64_t W, std::uint64_t pe, double2& acc) {
    if (!((present >> XQ) & 1u)) return;
    const int i = __popc(present & ((1u << XQ) - 1u));
    const double r = coset_group<XQ>(a, tabs + (tab1 >> 1) + 8 * i);
    const CosetGroup& G = P.groups[S.g_begin + i];
#if QRT_EVC_FMA_SIGN
    acc.x = fma(group_sign(W, pe, G), r, acc.x);
#else
    const int odd = (__popcll(W & G.mf) + __popcll(pe & G.gz)) & 1;
    acc.x += odd ? -r : r;
#endif
}

__device__ __forceinline__ double2 block_sum(double2 v, double2* scratch) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_down_sync(0xffffffffu, v.x, o);
        v.y += __shfl_down_sync(0xffffffffu, v.y, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double2 r = make_double2(0.0, 0.0);
    if (threadIdx.x == 0)
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            r.x += scratch[w].x;
            r.y += scratch[w].y;
        }
    return r;
}

// Every coset set of the pass over one tile (128 threads; t = thread index
// within them): load the thread's 32-amplitude coset into registers, then
// the fast (weight-2/4), single-bit and generic groups of the set.
template <bool GENERIC, bool ONES>
__device__ __forceinline__ void coset_tile_sets(const CosetParams& P, const double2* __restrict__ tile,
                                                const double2* __restrict__ stab, int t, u64 wout, u64 pe,
                                                double2& acc) {
#if QRT_EVC_THREAD_ACC
    double acc4[4] = {0.0, 0.0, 0.0, 0.0};
#endif
#if QRT_EVC_EB_PREFETCH
    // the thread-index tables are per-thread-indexed constant loads (serialised
    // over distinct addresses): fetch the next set's while this one computes
    int eb_lo = 0, eb_hi = 0;
    if (P.set_tables && P.n_sets > 0) {
        eb_lo = P.sets[0].eb_lo[t & 15];
        eb_hi = P.sets[0].eb_hi[t >> 4];
    }
#endif
    for (int s = 0; s < P.n_sets; ++s) {
        const CosetSet& S = P.sets[s];
        int ebase, swq[kCosetBits];
        if (P.set_tables) {  // host tables (coset_set_tables)
#if QRT_EVC_EB_PREFETCH
            ebase = eb_lo | eb_hi;
#else
            ebase = S.eb_lo[t & 15] | S.eb_hi[t >> 4];
#endif
#pragma unroll
            for (int q = 0; q < kCosetBits; ++q) swq[q] = S.swq[q];
        } else {
            ebase = 0;
#pragma unroll
            for (int i = 0; i < kTileBits - kCosetBits; ++i) ebase |= ((t >> i) & 1) << S.tb[i];
#pragma unroll
            for (int q = 0; q < kCosetBits; ++q) swq[q] = swz(1 << S.S[q]);
        }
        const int sb = swz(ebase);
        double2 a[32];
#if QRT_EVC_BYTE_GATHER
        {
            // byte offsets from the dynamic shared-memory base, XOR-composed (swz is
            // GF(2)-linear, x16 distributes over XOR, and the tile's own offset is a
            // multiple of 64 KiB): one LOP3 per amplitude, the base an immediate
            extern __shared__ __align__(16) unsigned char smem_raw[];
            const unsigned toff = static_cast<unsigned>(reinterpret_cast<const unsigned char*>(tile) - smem_raw);
            unsigned qb[kCosetBits];
#pragma unroll
            for (int q = 0; q < kCosetBits; ++q) qb[q] = static_cast<unsigned>(swq[q]) << 4;
            const unsigned sbb = toff | (static_cast<unsigned>(sb) << 4);
#pragma unroll
            for (int r = 0; r < 32; ++r) {
                unsigned o = sbb;
#pragma unroll
                for (int q = 0; q < kCosetBits; ++q)
                    if ((r >> q) & 1) o ^= qb[q];
                a[r] = *reinterpret_cast<const double2*>(smem_raw + o);
            }
        }
#else
        {
#pragma unroll
            for (int r = 0; r < 32; ++r) {
                int o = sb;
#pragma unroll
                for (int q = 0; q < kCosetBits; ++q)
                    if ((r >> q) & 1) o ^= swq[q];
                a[r] = tile[o];
            }
        }
#endif
        const u64 W = static_cast<u64>(ebase) | wout;
#if QRT_EVC_EB_PREFETCH
        if (P.set_tables && s + 1 < P.n_sets) {
            eb_lo = P.sets[s + 1].eb_lo[t & 15];
            eb_hi = P.sets[s + 1].eb_hi[t >> 4];
        }
#endif
        const unsigned present = S.present;
        const int tab1 = S.tab1;
        if (P.single && tab1 >= 0) {
#if QRT_EVC_UNIFORM_PRESENT
            // warp-uniform by construction; REDUX puts it in a uniform register so the
            // 15 mask blocks branch without convergence barriers (JW passes 803 -> 782 ms
            // at 30q; on every set it cost GF(2)-linear passes 1.5%)
            const unsigned present = __reduce_or_sync(0xffffffffu, S.present);
#endif
#if QRT_EVC_THREAD_ACC
            coset_fast1t<3>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<5>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<6>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<9>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<10>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<12>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<15>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<17>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<18>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<20>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<23>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<24>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<27>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<29>(a, P, S, stab, present, tab1, W, pe, acc4);
            coset_fast1t<30>(a, P, S, stab, present, tab1, W, pe, acc4);
#else
            coset_fast1<3>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<5>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<6>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<9>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<10>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<12>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<15>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<17>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<18>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<20>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<23>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<24>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<27>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<29>(a, P, S, stab, present, tab1, W, pe, acc);
            coset_fast1<30>(a, P, S, stab, present, tab1, W, pe, acc);
#endif
        } else if (present || !P.present_guard) {  // linear-pass sets have no weight-2/4 groups: skip the 15 mask tests
        coset_fast<3>(a, P, S, stab, present, W, pe, acc);
        coset_fast<5>(a, P, S, stab, present, W, pe, acc);
        coset_fast<6>(a, P, S, stab, present, W, pe, acc);
        coset_fast<9>(a, P, S, stab, present, W, pe, acc);
        coset_fast<10>(a, P, S, stab, present, W, pe, acc);
        coset_fast<12>(a, P, S, stab, present, W, pe, acc);
        coset_fast<15>(a, P, S, stab, present, W, pe, acc);
        coset_fast<17>(a, P, S, stab, present, W, pe, acc);
        coset_fast<18>(a, P, S, stab, present, W, pe, acc);
        coset_fast<20>(a, P, S, stab, present, W, pe, acc);
        coset_fast<23>(a, P, S, stab, present, W, pe, acc);
        coset_fast<24>(a, P, S, stab, present, W, pe, acc);
        coset_fast<27>(a, P, S, stab, present, W, pe, acc);
        coset_fast<29>(a, P, S, stab, present, W, pe, acc);
        coset_fast<30>(a, P, S, stab, present, W, pe, acc);
        }
        int g1 = S.g_begin + S.xbeg[31];
        const unsigned onemask = S.onemask;
        if (ONES && P.single && onemask) {
            const double* __restrict__ dt = reinterpret_cast<const double*>(stab);
            const unsigned onemode = S.onemode;
            coset_one1<0>(a, P, S, dt, onemask, onemode, W, pe, acc);
            coset_one1<1>(a, P, S, dt, onemask, onemode, W, pe, acc);
            coset_one1<2>(a, P, S, dt, onemask, onemode, W, pe, acc);
            coset_one1<3>(a, P, S, dt, onemask, onemode, W, pe, acc);
            coset_one1<4>(a, P, S, dt, onemask, onemode, W, pe, acc);
            continue;  // the set holds nothing else
        }
        if (ONES) {
            const double* __restrict__ dt = reinterpret_cast<const double*>(stab);
            coset_ones<0>(a, P, S, dt, g1, W, pe, acc);
            coset_ones<1>(a, P, S, dt, g1, W, pe, acc);
            coset_ones<2>(a, P, S, dt, g1, W, pe, acc);
            coset_ones<3>(a, P, S, dt, g1, W, pe, acc);
            coset_ones<4>(a, P, S, dt, g1, W, pe, acc);
        }
        if (GENERIC)
        for (int g = g1; g < S.g_begin + S.g_count; ++g) {
            const CosetGroup& G = P.groups[g];
            const double2 r = coset_generic(tile, sb, swq, G.xq, G.mode, P.tabs + G.tab);
            const int odd = (__popcll(W & G.mf) + __popcll(pe & G.gz)) & 1;
            acc.x += odd ? -r.x : r.x;
            acc.y += odd ? -r.y : r.y;
        }
    }
#if QRT_EVC_THREAD_ACC
    acc.x += (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
#endif
}

template <int MINB, bool GENERIC, bool ONES>
__global__ void __launch_bounds__(kCosetThreads, MINB)
    coset_pass_kernel(const __grid_constant__ CosetParams P, const CosetDiagTerm* __restrict__ dterms,
                      double* __restrict__ red) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double2 scratch[kCosetThreads / 32];
    constexpr int E = 1 << kTileBits;
    const int c = P.c, t = threadIdx.x;
    double2* tile = reinterpret_cast<double2*>(smem_raw);
    u64* tabo = reinterpret_cast<u64*>(tile + E);
    double2* stab = reinterpret_cast<double2*>(tabo + ((1 << (kTileBits - c)) | 1) + 1);  // 16-B aligned tables
    double* Wsh = reinterpret_cast<double*>(stab + (P.n_tab >> 1));
    for (int i = t; i < (P.n_tab >> 1); i += kCosetThreads) {
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&stab[i]));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(P.gtabs + 2 * i));
    }

    const u64 b = static_cast<u64>(blockIdx.x);  // bit i <-> outer axis i
    u64 base = 0;
    for (int i = 0; i < P.n_outer; ++i)
        if ((b >> i) & 1ull) base ^= P.outer_vec[i];
    for (int h = t; h < (1 << (kTileBits - c)); h += kCosetThreads) {
        u64 o = 0;
        for (int i = c; i < kTileBits; ++i)
            if ((h >> (i - c)) & 1) o ^= P.tile_vec[i];
        tabo[h] = o;
    }
    __syncthreads();
    const amp_t* __restrict__ v = P.ptrs[blockIdx.y];
    const u64 pe = static_cast<u64>(P.pe_begin) + blockIdx.y;
    const int cmask = (1 << c) - 1;
    for (int e = t; e < E; e += kCosetThreads) {
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&tile[swz(e)]));
        QRT_DCHECK((base ^ tabo[e >> c] ^ (e & cmask)) < (static_cast<u64>(P.tiles_per_pe) << kTileBits));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(&v[base ^ tabo[e >> c] ^ (e & cmask)]));
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();

    double2 acc = make_double2(0.0, 0.0);
    if (P.d_count > 0) {  // I/Z words: Walsh-Hadamard transform of |v|^2 over the tile
        for (int e = t; e < E; e += kCosetThreads) {
            const double2 a = tile[swz(e)];
            Wsh[e] = fma(a.x, a.x, a.y * a.y);
        }
        __syncthreads();
        for (int s = 0; s < kTileBits; ++s) {
            for (int i = t; i < (E >> 1); i += kCosetThreads) {
                const int i0 = insert_zero(i, s), i1 = i0 | (1 << s);
                const double x = Wsh[i0], y = Wsh[i1];
                Wsh[i0] = x + y;
                Wsh[i1] = x - y;
            }
            __syncthreads();
        }
        for (int k = t; k < P.d_count; k += kCosetThreads) {
            const CosetDiagTerm tm = dterms[P.d_begin + k];
            const int odd = (__popcll(base & tm.m) + __popcll(pe & tm.gz)) & 1;
            const double val = odd ? -Wsh[tm.m_tile] : Wsh[tm.m_tile];
            acc.x = fma(tm.f.x, val, acc.x);
            acc.y = fma(tm.f.y, val, acc.y);
        }
    }

    coset_tile_sets<GENERIC, ONES>(P, tile, stab, t, b << kTileBits, pe, acc);
    const double2 tot = block_sum(acc, scratch);
    if (t == 0) {
        double* slot = red + 2 * (static_cast<std::size_t>(blockIdx.y) * gridDim.x + blockIdx.x);
        slot[0] += tot.x;
        slot[1] += tot.y;
    }
}


__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n)); }

__device__ __forceinline__ void mbar_wait(unsigned addr, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity));
}

// Fill barriers of the three-buffer pipelines.  Tile k lives in buffer k % 3
// and its fill completes barrier (k % 3) + 3 * ((k / 3) & 1): each barrier then
// serves every sixth tile, all consumed by the same team.  A parity wait only
// distinguishes a barrier's current phase from the one before it; with one
// barrier per buffer, a team that finished two tiles before the fill of tile
// k - 3 (its own previous buffer use, issued by itself) completed saw that
// phase's parity, took it for tile k's and read a half-filled buffer (a rare
// wrong energy on few-group linear passes: 24 qubits, 2,000 uniform words).
// With six barriers the phase before the awaited one is always the same
// team's previous use of that barrier (complete), and the phase after it is
// only issued once this team has released the buffer.
__device__ __forceinline__ int fill_bar(int k) { return (k % 3) + 3 * ((k / 3) & 1); }
__device__ __forceinline__ unsigned fill_parity(int k) { return static_cast<unsigned>((k / 6) & 1); }

// Persistent, software-pipelined variant for passes without I/Z words: one
// 256-thread CTA per SM holds three tile buffers; two teams of 128 threads
// evaluate alternate tiles (team = tile index & 1) while the third buffer
// fills.  Tile k lives in buffer k % 3 and is loaded by the other team right
// after that team finished tile k - 3 in the same buffer; completion travels
// through one mbarrier per buffer (cp.async.mbarrier.arrive.noinc, 128
// arrivals per fill), so a team never waits for HBM while the other computes.
template <bool GENERIC, bool ONES>
__global__ void __launch_bounds__(2 * kCosetThreads, 1)
    coset_pipe_kernel(const __grid_constant__ CosetParams P, double* __restrict__ red) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double2 scratch[2 * kCosetThreads / 32];
    __shared__ __align__(8) unsigned long long full[6];
    constexpr int E = 1 << kTileBits;
    const int c = P.c;
    const int team = threadIdx.x >> 7, tid = threadIdx.x & (kCosetThreads - 1);
    // one or two compute teams: with one, two of the three buffers are always
    // filling (128 KiB in flight per SM) — for passes whose tiles compute
    // faster than they load (GF(2)-linear passes: scattered 64-byte runs)
    const int nteams = static_cast<int>(blockDim.x) / kCosetThreads;
    double2* bufs = reinterpret_cast<double2*>(smem_raw);  // 3 x E
    u64* tabo = reinterpret_cast<u64*>(bufs + 3 * E);
    double2* stab = reinterpret_cast<double2*>(tabo + ((1 << (kTileBits - c)) | 1) + 1);
    for (int i = threadIdx.x; i < (P.n_tab >> 1); i += blockDim.x) {
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&stab[i]));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(P.gtabs + 2 * i));
    }
    for (int h = threadIdx.x; h < (1 << (kTileBits - c)); h += blockDim.x) {
        u64 o = 0;
        for (int i = c; i < kTileBits; ++i)
            if ((h >> (i - c)) & 1) o ^= P.tile_vec[i];
        tabo[h] = o;
    }
    if (threadIdx.x < 6) {
        const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&full[threadIdx.x]));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(kCosetThreads));
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();

    const int tiles = P.tiles_per_pe;
    const int stride = static_cast<int>(gridDim.x);
    const int ntile = (tiles - static_cast<int>(blockIdx.x) + stride - 1) / stride;  // this CTA's tiles
    const amp_t* __restrict__ v = P.ptrs[blockIdx.y];
    const u64 pe = static_cast<u64>(P.pe_begin) + blockIdx.y;
    const int cmask = (1 << c) - 1;
    auto tile_of = [&](int k) { return static_cast<u64>(blockIdx.x) + static_cast<u64>(k) * stride; };
    auto issue = [&](int k) {  // this team's 128 threads fill buffer k % 3 with tile k
        const u64 b = tile_of(k);
        // base = XOR of the outer axes of b's set bits: lane i takes axes i, i+32, ...
        // and the warp XOR-reduces (every thread walking all axes cost ~7% of the
        // instructions of a GF(2)-linear pass)
        u64 base = 0;
        if (P.fill_mode) {
            for (int i = tid & 31; i < P.n_outer; i += 32)
                if ((b >> i) & 1ull) base ^= P.outer_vec[i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) base ^= __shfl_xor_sync(0xffffffffu, base, o);
        } else {
            for (int i = 0; i < P.n_outer; ++i)
                if ((b >> i) & 1ull) base ^= P.outer_vec[i];
        }
        double2* tile = bufs + (k % 3) * E;
        if (c <= 7 && P.fill_mode) {
            // e = tid + 128 i: the swizzle is GF(2)-linear, so swz(e) = swz(tid) ^ swz(128 i)
            // (a constant per unrolled i), and e >> c / e & cmask split the same way (the
            // per-element addressing was ~30% of a linear pass's instructions)
            const unsigned sa0 = static_cast<unsigned>(__cvta_generic_to_shared(tile));
            const int tsw = swz(tid), th = tid >> c;
            const u64 bl = base ^ static_cast<u64>(tid & cmask);
#pragma unroll
            for (int i = 0; i < E / kCosetThreads; ++i) {
                const unsigned sa = sa0 + 16u * static_cast<unsigned>(tsw ^ swz(i * kCosetThreads));
                QRT_DCHECK((bl ^ tabo[th + (i << (7 - c))]) < (static_cast<u64>(P.tiles_per_pe) << kTileBits));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa),
                             "l"(v + (bl ^ tabo[th + (i << (7 - c))])));
            }
        } else {
            for (int e = tid; e < E; e += kCosetThreads) {
                const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&tile[swz(e)]));
                QRT_DCHECK((base ^ tabo[e >> c] ^ (e & cmask)) < (static_cast<u64>(P.tiles_per_pe) << kTileBits));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa),
                             "l"(&v[base ^ tabo[e >> c] ^ (e & cmask)]));
            }
        }
        const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&full[fill_bar(k)]));
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(a));
    };
    // tile k is issued by the team that computed tile k - 3: (k - 3) mod nteams
    for (int k = 0; k < 3 && k < ntile; ++k)
        if ((k + 3 * nteams - 3) % nteams == team) issue(k);

    double2 acc = make_double2(0.0, 0.0);
    for (int k = team; k < ntile; k += nteams) {
        const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&full[fill_bar(k)]));
        mbar_wait(a, fill_parity(k));
        QRT_DCHECK(k % nteams == team && k < ntile);
#ifdef QRT_CHECKS
        {  // the awaited buffer really holds tile k (the state is read-only during EVC)
            const u64 bk = tile_of(k);
            u64 base = 0;
            for (int i = 0; i < P.n_outer; ++i)
                if ((bk >> i) & 1ull) base ^= P.outer_vec[i];
            for (int e = tid; e < E; e += 16 * kCosetThreads) {
                const double2 want = v[base ^ tabo[e >> c] ^ (e & cmask)];
                const double2 got = bufs[(k % 3) * E + swz(e)];
                QRT_DCHECK(got.x == want.x && got.y == want.y);
            }
        }
#endif
        coset_tile_sets<GENERIC, ONES>(P, bufs + (k % 3) * E, stab, tid, tile_of(k) << kTileBits, pe, acc);
        named_bar(1 + team, kCosetThreads);  // the team is done reading buffer k % 3
        if (k + 3 < ntile) issue(k + 3);
    }
    asm volatile("cp.async.wait_all;\n" ::);
    const double2 tot = block_sum(acc, scratch);
    if (threadIdx.x == 0) {
        // per-PE slots are tiles_per_pe apart (reduce_slots_kernel); this grid is narrower
        double* slot = red + 2 * (static_cast<std::size_t>(blockIdx.y) * P.tiles_per_pe + blockIdx.x);
        slot[0] += tot.x;
        slot[1] += tot.y;
    }
}

// ---------------------------------------------------------------------------
// Split cosets (Jordan-Wigner fast groups only).  A lane pair shares one
// 32-amplitude coset: the even lane holds the 32 real parts, the odd lane the
// 32 imaginary parts (64 registers instead of 128), because
//   sum_rho T[rho] Re(conj(a_s) a_r) = sum_rho T[rho] re_s re_r + sum_rho T[rho] im_s im_r
// splits into two independent per-lane sums that the final reduction adds
// anyway.  Each lane spends 2 fp64 instructions per pair (DMUL + DFMA, 4/3 of
// the fused form) but the register footprint halves, so twice the warps stay
// resident to hide the LDS / DFMA latencies that bound the 128-thread form;
// adjacent lanes read the two halves of one 16-byte amplitude, so a warp's
// coset loads stay conflict-free.

template <int XQ>
__device__ __forceinline__ double coset_group_split(const double (&a)[32], const double2* __restrict__ T2) {
    constexpr int H = top_bit(XQ);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int h = 0; h < 8; ++h) {
        const double2 t = T2[h];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int rho = 2 * h + u;
            const int r = ins0(rho, H);
            const int s = r ^ XQ;
            acc[rho & 3] = fma(u ? t.y : t.x, a[s] * a[r], acc[rho & 3]);
        }
    }
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

template <int XQ>
__device__ __forceinline__ void coset_fast_split(const double (&a)[32], const CosetParams& P, const CosetSet& S,
                                                 const double2* __restrict__ tabs, unsigned present, std::uint64_t W,
                                                 std::uint64_t pe, double& acc) {
    if (!((present >> XQ) & 1u)) return;
    const int g0 = S.g_begin + S.xbeg[XQ - 1], g1 = S.g_begin + S.xbeg[XQ];
    for (int g = g0; g < g1; ++g) {
        const CosetGroup& G = P.groups[g];
        const double r = coset_group_split<XQ>(a, tabs + (G.tab >> 1));
        const int odd = (__popcll(W & G.mf) + __popcll(pe & G.gz)) & 1;
        acc += odd ? -r : r;
    }
}

// t2 = lane index within the 256-thread team: coset t2 >> 1, part t2 & 1.
__device__ __forceinline__ void coset_tile_sets_split(const CosetParams& P, const double2* __restrict__ tile,
                                                      const double2* __restrict__ stab, int t2, u64 wout, u64 pe,
                                                      double& acc) {
    const int t = t2 >> 1, part = t2 & 1;
    const double* __restrict__ tiled = reinterpret_cast<const double*>(tile) + part;
    for (int s = 0; s < P.n_sets; ++s) {
        const CosetSet& S = P.sets[s];
        int ebase = 0;
#pragma unroll
        for (int i = 0; i < kTileBits - kCosetBits; ++i) ebase |= ((t >> i) & 1) << S.tb[i];
        int swq[kCosetBits];
#pragma unroll
        for (int q = 0; q < kCosetBits; ++q) swq[q] = swz(1 << S.S[q]);
        const int sb = swz(ebase);
        double a[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) {
            int o = sb;
#pragma unroll
            for (int q = 0; q < kCosetBits; ++q)
                if ((r >> q) & 1) o ^= swq[q];
            a[r] = tiled[2 * o];
        }
        const u64 W = static_cast<u64>(ebase) | wout;
        const unsigned present = S.present;
        coset_fast_split<3>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<5>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<6>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<9>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<10>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<12>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<15>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<17>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<18>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<20>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<23>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<24>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<27>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<29>(a, P, S, stab, present, W, pe, acc);
        coset_fast_split<30>(a, P, S, stab, present, W, pe, acc);
    }
}

constexpr int kSplitTeam = 2 * kCosetThreads;  // 256 lanes per tile

// coset_pipe_kernel with split cosets: two teams of 256 threads (16 warps per
// SM at <= 128 registers), three tile buffers, mbarrier-tracked cp.async fills.
__global__ void __launch_bounds__(2 * kSplitTeam, 1)
    coset_pipe_split_kernel(const __grid_constant__ CosetParams P, double* __restrict__ red) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double2 scratch[2 * kSplitTeam / 32];
    __shared__ __align__(8) unsigned long long full[6];
    constexpr int E = 1 << kTileBits;
    const int c = P.c;
    const int team = threadIdx.x / kSplitTeam, tid = threadIdx.x % kSplitTeam;
    double2* bufs = reinterpret_cast<double2*>(smem_raw);  // 3 x E
    u64* tabo = reinterpret_cast<u64*>(bufs + 3 * E);
    double2* stab = reinterpret_cast<double2*>(tabo + ((1 << (kTileBits - c)) | 1) + 1);
    for (int i = threadIdx.x; i < (P.n_tab >> 1); i += blockDim.x) {
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&stab[i]));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(P.gtabs + 2 * i));
    }
    for (int h = threadIdx.x; h < (1 << (kTileBits - c)); h += blockDim.x) {
        u64 o = 0;
        for (int i = c; i < kTileBits; ++i)
            if ((h >> (i - c)) & 1) o ^= P.tile_vec[i];
        tabo[h] = o;
    }
    if (threadIdx.x < 6) {
        const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&full[threadIdx.x]));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(kSplitTeam));
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();

    const int tiles = P.tiles_per_pe;
    const int stride = static_cast<int>(gridDim.x);
    const int ntile = (tiles - static_cast<int>(blockIdx.x) + stride - 1) / stride;
    const amp_t* __restrict__ v = P.ptrs[blockIdx.y];
    const u64 pe = static_cast<u64>(P.pe_begin) + blockIdx.y;
    const int cmask = (1 << c) - 1;
    auto tile_of = [&](int k) { return static_cast<u64>(blockIdx.x) + static_cast<u64>(k) * stride; };
    auto issue = [&](int k) {
        const u64 b = tile_of(k);
        u64 base = 0;
        for (int i = 0; i < P.n_outer; ++i)
            if ((b >> i) & 1ull) base ^= P.outer_vec[i];
        double2* tile = bufs + (k % 3) * E;
        for (int e = tid; e < E; e += kSplitTeam) {
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&tile[swz(e)]));
            QRT_DCHECK((base ^ tabo[e >> c] ^ (e & cmask)) < (static_cast<u64>(P.tiles_per_pe) << kTileBits));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa),
                         "l"(&v[base ^ tabo[e >> c] ^ (e & cmask)]));
        }
        const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&full[fill_bar(k)]));
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(a));
    };
    for (int k = 0; k < 3 && k < ntile; ++k)
        if (((k + 1) & 1) == team) issue(k);

    double acc = 0.0;
    for (int k = team; k < ntile; k += 2) {
        const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&full[fill_bar(k)]));
        mbar_wait(a, fill_parity(k));
        coset_tile_sets_split(P, bufs + (k % 3) * E, stab, tid, tile_of(k) << kTileBits, pe, acc);
        named_bar(1 + team, kSplitTeam);
        if (k + 3 < ntile) issue(k + 3);
    }
    asm volatile("cp.async.wait_all;\n" ::);
    const double2 tot = block_sum(make_double2(acc, 0.0), scratch);
    if (threadIdx.x == 0) {
        // per-PE slots are tiles_per_pe apart (reduce_slots_kernel); this grid is narrower
        double* slot = red + 2 * (static_cast<std::size_t>(blockIdx.y) * P.tiles_per_pe + blockIdx.x);
        slot[0] += tot.x;
        slot[1] += tot.y;
    }
}

}  // namespace

constexpr int kPipeSmemMax = 225 * 1024;  // dynamic shared memory of the pipelined kernels (+ ~1 KiB static)

void launch_coset_pass(CosetParams& P, const CosetDiagTerm* dterms, int pe_count, double* red,
                       cudaStream_t stream, int device) {
    static const int set_tables = [] {
        const char* e = std::getenv("QRT_EVC_SET_TABLES");
        return e ? std::atoi(e) : 1;
    }();
    P.set_tables = set_tables;
    static const int fill_mode = [] {  // measured: JW 962 -> 979 ms, uniform 2139 -> 2134 ms with 1
        const char* e = std::getenv("QRT_EVC_FILL");
        return e ? std::atoi(e) : 0;
    }();
    P.fill_mode = fill_mode;
    static const int present_guard = [] {
        const char* e = std::getenv("QRT_EVC_PRESENT_GUARD");
        return e ? std::atoi(e) : 1;
    }();
    P.present_guard = present_guard;
    static const int single = [] {
        const char* e = std::getenv("QRT_EVC_SINGLE");
        return e ? std::atoi(e) : 1;
    }();
    P.single = single;
    // Launches holding only Jordan-Wigner-type groups take the fast-only
    // kernel (218 registers, 2 CTAs/SM; QRT_COSET_OCC=3 squeezes it to 3 CTAs/SM
    // with spills, measured slower); any generic group needs the
    // shared-memory fallback body.
    static const int occ = [] {
        const char* e = std::getenv("QRT_COSET_OCC");
        return (e && std::atoi(e) == 3) ? 3 : 2;
    }();
    bool generic = false, any_ones = false;
    for (int i = 0; i < P.n_sets; ++i) {
        int ones = 0;
        for (int k = 0; k < kCosetBits; ++k) ones += P.sets[i].one_cnt[k];
        generic = generic || P.sets[i].xbeg[31] + ones < P.sets[i].g_count;
        any_ones = any_ones || ones > 0;
    }
    static bool attr_done[64] = {};
    if (!attr_done[device]) {
        QRT_CUDA(cudaFuncSetAttribute(coset_pass_kernel<2, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
        QRT_CUDA(cudaFuncSetAttribute(coset_pass_kernel<2, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
        QRT_CUDA(cudaFuncSetAttribute(coset_pass_kernel<2, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
        QRT_CUDA(cudaFuncSetAttribute(coset_pass_kernel<3, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
        attr_done[device] = true;
    }
    static const bool pipe = [] {
        const char* e = std::getenv("QRT_EVC_PIPE");
        return e ? std::atoi(e) != 0 : true;
    }();
    const std::size_t pipe_smem = 3 * (std::size_t{1} << kTileBits) * sizeof(double2) +
                                  ((std::size_t{1} << (kTileBits - P.c)) + 2) * sizeof(std::uint64_t) +
                                  static_cast<std::size_t>(P.n_tab) * sizeof(double);
    // (three tile buffers + the tile-offset table + the coefficient tables must fit
    // next to the static shared memory; a pass that does not takes the one-buffer kernel)
    if (pipe && P.d_count == 0 && occ == 2 && pipe_smem <= static_cast<std::size_t>(kPipeSmemMax)) {  // persistent pipeline
        static int nsm[64] = {};
        static bool pattr[64] = {};
        if (!nsm[device]) QRT_CUDA(cudaDeviceGetAttribute(&nsm[device], cudaDevAttrMultiProcessorCount, device));
        if (!pattr[device]) {
            QRT_CUDA(cudaFuncSetAttribute(coset_pipe_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPipeSmemMax));
            QRT_CUDA(cudaFuncSetAttribute(coset_pipe_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPipeSmemMax));
            QRT_CUDA(cudaFuncSetAttribute(coset_pipe_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPipeSmemMax));
            pattr[device] = true;
        }
        const std::size_t psmem = 3 * (std::size_t{1} << kTileBits) * sizeof(double2) +
                                  ((std::size_t{1} << (kTileBits - P.c)) + 2) * sizeof(std::uint64_t) +
                                  static_cast<std::size_t>(P.n_tab) * sizeof(double);
        dim3 pgrid(static_cast<unsigned>(std::min(nsm[device], P.tiles_per_pe)), static_cast<unsigned>(pe_count));
        static const bool split = [] {
            // measured slower (30q JW EVC 0.917 -> 1.144 s): the per-group
            // overhead (tables, signs, loop control) is duplicated per lane pair
            const char* e = std::getenv("QRT_EVC_SPLIT");
            return e ? std::atoi(e) != 0 : false;
        }();
        if (split && !generic && !any_ones) {  // Jordan-Wigner fast groups only: split cosets
            static bool sattr[64] = {};
            if (!sattr[device]) {
                QRT_CUDA(cudaFuncSetAttribute(coset_pipe_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              kPipeSmemMax));
                sattr[device] = true;
            }
            coset_pipe_split_kernel<<<pgrid, 2 * kSplitTeam, psmem, stream>>>(P, red);
            QRT_CUDA(cudaGetLastError());
            return;
        }
        // QRT_EVC_TEAMS: 2 (default) or 1 compute teams per SM for every pass,
        // or 0: one team on GF(2)-linear passes (single-bit groups), two otherwise
        static const int teams_knob = [] {
            const char* e = std::getenv("QRT_EVC_TEAMS");
            return e ? std::atoi(e) : 2;
        }();
        const int teams = teams_knob == 1 ? 1 : (teams_knob == 0 && any_ones) ? 1 : 2;
        const int pthreads = teams * kCosetThreads;
        if (generic)
            coset_pipe_kernel<true, true><<<pgrid, pthreads, psmem, stream>>>(P, red);
        else if (any_ones)
            coset_pipe_kernel<false, true><<<pgrid, pthreads, psmem, stream>>>(P, red);
        else
            coset_pipe_kernel<false, false><<<pgrid, pthreads, psmem, stream>>>(P, red);
        QRT_CUDA(cudaGetLastError());
        return;
    }
    const std::size_t smem = (std::size_t{1} << kTileBits) * sizeof(double2) +
                             ((std::size_t{1} << (kTileBits - P.c)) + 2) * sizeof(std::uint64_t) +
                             static_cast<std::size_t>(P.n_tab) * sizeof(double) +
                             (P.d_count > 0 ? (std::size_t{1} << kTileBits) * sizeof(double) : 0);
    dim3 grid(static_cast<unsigned>(P.tiles_per_pe), static_cast<unsigned>(pe_count));
    // single-bit-mask groups (linear passes) get their own instantiations so
    // the Jordan-Wigner fast kernel keeps its register allocation
    if (generic)
        coset_pass_kernel<2, true, true><<<grid, kCosetThreads, smem, stream>>>(P, dterms, red);
    else if (any_ones)
        coset_pass_kernel<2, false, true><<<grid, kCosetThreads, smem, stream>>>(P, dterms, red);
    else if (occ == 2)
        coset_pass_kernel<2, false, false><<<grid, kCosetThreads, smem, stream>>>(P, dterms, red);
    else
        coset_pass_kernel<3, false, false><<<grid, kCosetThreads, smem, stream>>>(P, dterms, red);
    QRT_CUDA(cudaGetLastError());
}

}  // namespace qrt
