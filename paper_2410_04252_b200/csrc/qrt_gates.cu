// libqrt — QSU gate runs (reference apply_gate_narrow, dist_sim.cpp:163-201).
//
// A call carries a sequence of narrow gates.  The host planner cuts it into
// *passes*: each pass picks a set B of kTileBits local positions (always
// containing the kCoalBits lowest positions, so every HBM access is a
// contiguous run of 2^kCoalBits amplitudes) and takes, in order, every gate
// whose targets lie in B (diagonal gates may target any position) without
// overtaking a deferred gate on a shared qubit — the reference's own tile
// construction (qsu_scheduler.cpp:37-60), re-applied at SM level.
//
// One pass = one kernel = one HBM round trip: each CTA loads the 2^12
// amplitudes that agree on all positions outside B into shared memory
// (XOR-swizzled against bank conflicts), applies the pass's gates in order
// with fp64 FMAs (dense matrices read from the launch parameters through the
// uniform constant path, diagonals from shared memory), and
// writes the tile back.  Algorithmic traffic per pass = 32 B x 2^(n-g);
// flops per dense k-qubit gate = 8 x 2^k x 2^(n-g).

#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <array>
#include <iterator>
#include <deque>
#include <memory>
#include <mutex>

#include "qrt_fused.h"
#include "qrt_light.h"

namespace qrt {

namespace {

constexpr int kDense = 0, kDiag = 1;
constexpr int kMaxDiagK = 8;
constexpr int kBigK = 16;  // cap for the out-of-place generic kernel

struct PePtrs {
    amp_t* p[kMaxLocalPEs];
};

struct GateOp {
    int kind;
    int k;
    int smat;          // diagonal gates: offset of the diagonal in the pass's smem stage
    int pmat;          // dense k<=4 gates: offset of the matrix in the launch parameters
    int gmat;          // offset into the call's matrix pool in global memory (double2 units)
    int bfrag;         // k=3,4 dense gates: offset of the DMMA B fragments (doubles), -1 if unused
    int tb[kMaxDiagK]; // tile-bit index of targets[j] (-1: outside the tile, diagonal only)
    int pos[kMaxDiagK];// physical position of targets[j]
};

struct PassHdr {
    int T;               // tile bits
    int c;               // leading tile bits that are exactly positions 0..c-1
    int n_ops;
    int op_begin;
    int mat_begin;       // first double2 of this pass's staged matrices in the pool
    int mat_count;
    int frag_begin;      // first double of this pass's DMMA B fragments in the fragment pool
    int frag_count;
    int n_outer;
    int gauss;           // DMMA gates use the 3-product (Gauss) complex form, see dense_gauss
    int tile_pos[kTileBits];
    int outer_pos[64];
};

// Dense k<=4 matrices travel inside the launch parameters (constant bank):
// every thread of a warp reads the same entry at the same time, so the loads
// go through the uniform/constant path instead of shared memory, whose
// register write-back was the bottleneck (ncu: lsu_writeback 80%, fp64 32%).
constexpr int kParamMats = 1664;  // double2 entries, 26 KiB (all params <= 32 KiB)
constexpr int kMaxPassOps = 40;   // op descriptors per pass, also in the parameters
constexpr int kDiagStage = 1024; // diagonal entries staged in smem per pass
constexpr int kFragStage = 6144; // DMMA B-fragment doubles staged in smem per pass (48 KiB)

struct PassParams {
    PePtrs ptrs;
    PassHdr hdr;
    GateOp ops[kMaxPassOps];
    double2 mats[kParamMats];
};

__device__ __forceinline__ int swz(int e) {
    int x = e >> 3;
    return e ^ ((x ^ (x >> 3) ^ (x >> 6) ^ (x >> 9)) & 7);
}

__device__ __forceinline__ void cfma(double2& acc, const double2 u, const double2 a) {
    acc.x = fma(u.x, a.x, acc.x);
    acc.x = fma(-u.y, a.y, acc.x);
    acc.y = fma(u.x, a.y, acc.y);
    acc.y = fma(u.y, a.x, acc.y);
}

__device__ __forceinline__ int insert_zero(int v, int bit) {
    return ((v >> bit) << (bit + 1)) | (v & ((1 << bit) - 1));
}

// Dense k <= 4: one thread owns a whole group of 2^K amplitudes in registers.
template <int K>
__device__ __forceinline__ void dense_small(double2* __restrict__ tile, const PassParams& P, int moff,
                                            const GateOp& op, int E) {
    constexpr int D = 1 << K;
    int tb[K], sb[K];
    int offm[D];
#pragma unroll
    for (int j = 0; j < K; ++j) sb[j] = tb[j] = op.tb[j];
    // ascending tile bits for zero insertion
#pragma unroll
    for (int a = 1; a < K; ++a)
#pragma unroll
        for (int b = K - 1; b >= a; --b)
            if (sb[b - 1] > sb[b]) {
                int t = sb[b];
                sb[b] = sb[b - 1];
                sb[b - 1] = t;
            }
#pragma unroll
    for (int m = 0; m < D; ++m) {
        int o = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) o |= ((m >> j) & 1) << tb[j];
        offm[m] = o;
    }
    const int groups = E >> K;
    for (int g = threadIdx.x; g < groups; g += blockDim.x) {
        int base = g;
#pragma unroll
        for (int j = 0; j < K; ++j) base = insert_zero(base, sb[j]);
        double2 a[D];
#pragma unroll
        for (int m = 0; m < D; ++m) a[m] = tile[swz(base | offm[m])];
        // rows in pairs: two independent accumulators per thread, row
        // offsets recomputed (keeps the unrolled matrix loads from hoisting)
#pragma unroll 1
        for (int r = 0; r < D; r += 2) {
            double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
            const int row = moff + r * D;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                cfma(acc0, P.mats[row + c], a[c]);
                cfma(acc1, P.mats[row + D + c], a[c]);
            }
            int o0 = 0, o1 = 0;
#pragma unroll
            for (int j = 0; j < K; ++j) {
                o0 |= ((r >> j) & 1) << tb[j];
                o1 |= (((r + 1) >> j) & 1) << tb[j];
            }
            tile[swz(base | o0)] = acc0;
            tile[swz(base | o1)] = acc1;
        }
    }
}

// 16-byte global -> shared copy that bypasses registers (LDGSTS), so every
// thread keeps all of its tile loads in flight at once.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// D = A B + C with a separate accumulator input.
__device__ __forceinline__ void dmma_8x8x4_c(double& d0, double& d1, double a, double b, double c0, double c1) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
                 : "=d"(d0), "=d"(d1)
                 : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// Dense k = 3, 4 on the FP64 tensor path (DMMA, m8n8k4): for 8 groups at a
// time, OUT[8 x 2D] = IN[8 x 2D] * M^T where M is the 2D x 2D real form of U
// ([[Re, -Im], [Im, Re]] blocks) — the interleaved (re, im) amplitude layout
// is already the real vector.  B fragments (M^T) stay in registers for the
// whole gate; each lane loads one double of A per k-block and stores one
// complex output per n-block.  Fragment layout (PTX m8n8k4.f64):
//   A: row = lane>>2, col = lane&3;  B: row = lane&3, col = lane>>2;
//   C: row = lane>>2, cols 2*(lane&3) + {0,1}.
template <int K>
__device__ __forceinline__ void dense_dmma(double2* __restrict__ tile, const double* __restrict__ frag,
                                           const GateOp& op, int E) {
    constexpr int D = 1 << K, R = 2 * D, NB = R / 8, KB = R / 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    int tb[K], sb[K];
#pragma unroll
    for (int j = 0; j < K; ++j) sb[j] = tb[j] = op.tb[j];
#pragma unroll
    for (int a = 1; a < K; ++a)
#pragma unroll
        for (int q = K - 1; q >= a; --q)
            if (sb[q - 1] > sb[q]) {
                const int t = sb[q];
                sb[q] = sb[q - 1];
                sb[q - 1] = t;
            }
    auto spread = [&](int m) {
        int o = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) o |= ((m >> j) & 1) << tb[j];
        return o;
    };
    // swz is linear over GF(2), so swz(base | off) = swz(base) ^ swz(off)
    // for disjoint bit sets: precompute the swizzled per-lane offsets once.
    int sa[KB], sc[NB];
#pragma unroll
    for (int kb = 0; kb < KB; ++kb) sa[kb] = swz(spread(2 * kb + ((lane & 3) >> 1)));
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) sc[nb] = swz(spread(4 * nb + (lane & 3)));
    const int comp = lane & 1;
    double* __restrict__ tiled = reinterpret_cast<double*>(tile);
    const double* __restrict__ fl = frag + lane;
    const int blocks = (E >> K) >> 3;
    auto row_base = [&](int rb) {
        int base = rb * 8 + (lane >> 2);
#pragma unroll
        for (int j = 0; j < K; ++j) base = insert_zero(base, sb[j]);
        return swz(base);
    };
    // two row-blocks per iteration: 2*NB independent accumulator chains
    for (int rb = warp; rb < blocks; rb += 2 * nwarps) {
        const int rb1 = rb + nwarps;
        const bool two = rb1 < blocks;
        const int s0 = row_base(rb), s1 = two ? row_base(rb1) : s0;
        double a0[KB], a1[KB];
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
            a0[kb] = tiled[2 * (s0 ^ sa[kb]) + comp];
            a1[kb] = tiled[2 * (s1 ^ sa[kb]) + comp];
        }
        double c0[NB][2], c1[NB][2];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) c0[nb][0] = c0[nb][1] = c1[nb][0] = c1[nb][1] = 0.0;
#pragma unroll
        for (int kb = 0; kb < KB; ++kb)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                const double b = fl[(nb * KB + kb) * 32];
                dmma_8x8x4(c0[nb][0], c0[nb][1], a0[kb], b);
                dmma_8x8x4(c1[nb][0], c1[nb][1], a1[kb], b);
            }
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) tile[s0 ^ sc[nb]] = make_double2(c0[nb][0], c0[nb][1]);
        if (two) {
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) tile[s1 ^ sc[nb]] = make_double2(c1[nb][0], c1[nb][1]);
        }
    }
}

// Dense k = 3, 4 on DMMA with the 3-multiplication complex product (Gauss):
// for U = X + iY and amplitudes a = p + iq,
//   k1 = X (p + q),  Re = k1 + (-(X + Y)) q,  Im = k1 + (Y - X) p,
// i.e. three real D x D products instead of the one 2D x 2D real form
// (24 instead of 32 DMMA.8x8x4 per 8 groups at k = 4); the Re / Im chains
// start from k1 as their accumulator input, so the only DADD left is p + q
// (one per amplitude; DMMA and DADD share the fp64 datapath, measured:
// tools/microbench_fp64.cu).  A fragments: lane holds amplitude
// c = 4 kb + (lane & 3) of group lane >> 2 (one 16-byte load gives p and q);
// C fragments: output amplitudes 8 nb + 2 (lane & 3) + {0, 1}.  B fragment
// slot ((t * NB + nb) * KB + kb) * 32 + lane holds M_t[n][k] with
// k = 4 kb + (lane & 3), n = 8 nb + (lane >> 2), M_0 = X, M_1 = Y - X, M_2 = -(X + Y).
// HOIST: the gate's 3 D^2/32 B fragments per lane are loaded into registers
// once (needs the 168-register budget) instead of from L1 every row-block pair.
template <int K, bool HOIST = false>
__device__ __forceinline__ void dense_gauss(double2* __restrict__ tile, const double* __restrict__ frag,
                                            const GateOp& op, int E) {
    constexpr int D = 1 << K, NB = D / 8, KB = D / 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    int tb[K], sb[K];
#pragma unroll
    for (int j = 0; j < K; ++j) sb[j] = tb[j] = op.tb[j];
#pragma unroll
    for (int a = 1; a < K; ++a)
#pragma unroll
        for (int q = K - 1; q >= a; --q)
            if (sb[q - 1] > sb[q]) {
                const int t = sb[q];
                sb[q] = sb[q - 1];
                sb[q - 1] = t;
            }
    auto spread = [&](int m) {
        int o = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) o |= ((m >> j) & 1) << tb[j];
        return o;
    };
    int sa[KB], sc[NB][2];
#pragma unroll
    for (int kb = 0; kb < KB; ++kb) sa[kb] = swz(spread(4 * kb + (lane & 3)));
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
        sc[nb][0] = swz(spread(8 * nb + 2 * (lane & 3)));
        sc[nb][1] = swz(spread(8 * nb + 2 * (lane & 3) + 1));
    }
    const double* __restrict__ fl = frag + lane;
    double bf[HOIST ? 3 * NB * KB : 1];
    if (HOIST) {
#pragma unroll
        for (int f = 0; f < 3 * NB * KB; ++f) bf[f] = fl[f * 32];
    }
    auto B = [&](int f) { return HOIST ? bf[HOIST ? f : 0] : fl[f * 32]; };
    const int blocks = (E >> K) >> 3;
    auto row_base = [&](int rb) {
        int base = rb * 8 + (lane >> 2);
#pragma unroll
        for (int j = 0; j < K; ++j) base = insert_zero(base, sb[j]);
        return swz(base);
    };
    for (int rb = warp; rb < blocks; rb += 2 * nwarps) {
        const int rb1 = rb + nwarps;
        const bool two = rb1 < blocks;
        const int s0 = row_base(rb), s1 = two ? row_base(rb1) : s0;
        // k1 = X (p + q) first; Re and Im chains then start from k1 as the
        // DMMA accumulator input, so the output needs no DADDs.
        double2 x0[KB], x1[KB];
        double k0[NB][2], k1[NB][2];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) k0[nb][0] = k0[nb][1] = k1[nb][0] = k1[nb][1] = 0.0;
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
            x0[kb] = tile[s0 ^ sa[kb]];
            x1[kb] = tile[s1 ^ sa[kb]];
            const double a0 = x0[kb].x + x0[kb].y, a1 = x1[kb].x + x1[kb].y;
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                const double b = B(nb * KB + kb);
                dmma_8x8x4(k0[nb][0], k0[nb][1], a0, b);
                dmma_8x8x4(k1[nb][0], k1[nb][1], a1, b);
            }
        }
        double re0[NB][2], im0[NB][2], re1[NB][2], im1[NB][2];
#pragma unroll
        for (int kb = 0; kb < KB; ++kb)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                const double bi = B((NB + nb) * KB + kb), br = B((2 * NB + nb) * KB + kb);
                if (kb == 0) {
                    dmma_8x8x4_c(re0[nb][0], re0[nb][1], x0[0].y, br, k0[nb][0], k0[nb][1]);
                    dmma_8x8x4_c(re1[nb][0], re1[nb][1], x1[0].y, br, k1[nb][0], k1[nb][1]);
                    dmma_8x8x4_c(im0[nb][0], im0[nb][1], x0[0].x, bi, k0[nb][0], k0[nb][1]);
                    dmma_8x8x4_c(im1[nb][0], im1[nb][1], x1[0].x, bi, k1[nb][0], k1[nb][1]);
                } else {
                    dmma_8x8x4(re0[nb][0], re0[nb][1], x0[kb].y, br);
                    dmma_8x8x4(re1[nb][0], re1[nb][1], x1[kb].y, br);
                    dmma_8x8x4(im0[nb][0], im0[nb][1], x0[kb].x, bi);
                    dmma_8x8x4(im1[nb][0], im1[nb][1], x1[kb].x, bi);
                }
            }
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
            for (int j = 0; j < 2; ++j) tile[s0 ^ sc[nb][j]] = make_double2(re0[nb][j], im0[nb][j]);
        if (two) {
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
#pragma unroll
                for (int j = 0; j < 2; ++j) tile[s1 ^ sc[nb][j]] = make_double2(re1[nb][j], im1[nb][j]);
        }
    }
}

// Dense 5 <= k <= 7: one warp per group, lanes split the rows.
__device__ __forceinline__ void dense_wide(double2* __restrict__ tile, const double2* __restrict__ u,
                                           const GateOp& op, int E) {
    const int K = op.k, D = 1 << K, per = D >> 5;
    // zero-insertion in ascending bit order: repeatedly pick the smallest
    // target bit above the previous one
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int groups = E >> K;
    for (int g = warp; g < groups; g += nwarps) {
        int base = g, prev = -1;
        for (int j = 0; j < K; ++j) {
            int low = 64;
            for (int q = 0; q < K; ++q) {
                const int b = op.tb[q];
                if (b > prev && b < low) low = b;
            }
            base = insert_zero(base, low);
            prev = low;
        }
        double2 acc[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = make_double2(0.0, 0.0);
        for (int c = 0; c < D; ++c) {
            int oc = 0;
            for (int j = 0; j < K; ++j) oc |= ((c >> j) & 1) << op.tb[j];
            const double2 x = tile[swz(base | oc)];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < per) cfma(acc[j], u[(lane + 32 * j) * D + c], x);
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (j >= per) continue;
            const int r = lane + 32 * j;
            int orow = 0;
            for (int b = 0; b < K; ++b) orow |= ((r >> b) & 1) << op.tb[b];
            tile[swz(base | orow)] = acc[j];
        }
        __syncwarp();
    }
}

__device__ __forceinline__ void diagonal(double2* __restrict__ tile, const double2* __restrict__ d,
                                         const GateOp& op, int E, std::uint64_t base) {
    const int k = op.k;
    int fixed = 0, inmask = 0;
    int tb[kMaxDiagK];
#pragma unroll
    for (int j = 0; j < kMaxDiagK; ++j) {
        tb[j] = j < k ? op.tb[j] : -1;
        if (j < k && tb[j] < 0) fixed |= static_cast<int>((base >> op.pos[j]) & 1ull) << j;
        if (tb[j] >= 0) inmask |= 1 << j;
    }
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        int m = fixed;
#pragma unroll
        for (int j = 0; j < kMaxDiagK; ++j)
            if ((inmask >> j) & 1) m |= ((e >> tb[j]) & 1) << j;
        const double2 w = d[m];
        const int s = swz(e);
        const double2 a = tile[s];
        double2 r;
        r.x = fma(w.x, a.x, -w.y * a.y);
        r.y = fma(w.x, a.y, w.y * a.x);
        tile[s] = r;
    }
}

// One CTA per tile; several CTAs per SM so one CTA's load / store phase
// overlaps another's fp64 math.  The pass's DMMA B fragments are read
// through L1 (they are shared by every CTA of the pass).
// FUSED: gather the tile through a pending QR (qrt_fused.h).  MINB: CTAs per
// SM the register budget is cut for (3: <= 168 registers, 4: <= 128).
template <bool FUSED, int MINB>
__global__ void __launch_bounds__(128, MINB)
    gate_pass_kernel(const __grid_constant__ PassParams P, const double2* __restrict__ pool,
                     const double* __restrict__ frags, int tiles_per_pe, const FusedSource* __restrict__ fs_arg) {
    const FusedSource* __restrict__ fs = FUSED ? fs_arg : nullptr;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const PassHdr& hdr = P.hdr;
    const int T = hdr.T, E = 1 << T, c = hdr.c;
    double2* tile = reinterpret_cast<double2*>(smem_raw);
    double2* smat = tile + E;
    std::uint64_t* tab = reinterpret_cast<std::uint64_t*>(smat + hdr.mat_count);
    const int nt = 1 << (T - c);
    const int t = blockIdx.x;
    std::uint64_t base = 0;
    {
        const std::uint64_t b = static_cast<std::uint64_t>(t % tiles_per_pe);
        for (int i = 0; i < hdr.n_outer; ++i) base |= ((b >> i) & 1ull) << hdr.outer_pos[i];
    }
    for (int h = threadIdx.x; h < nt; h += blockDim.x) {
        std::uint64_t o = 0;
        for (int i = c; i < T; ++i) o |= static_cast<std::uint64_t>((h >> (i - c)) & 1) << hdr.tile_pos[i];
        tab[h] = o;
    }
    for (int i = threadIdx.x; i < hdr.mat_count; i += blockDim.x) smat[i] = pool[hdr.mat_begin + i];
    __syncthreads();

    amp_t* __restrict__ v = P.ptrs.p[t / tiles_per_pe];
    const int cmask = (1 << c) - 1;
    if (fs) {  // fused QR: gather the tile from the source PEs, write to the spare buffer
        std::uint64_t* words = tab + nt;
        fused_tables(*fs, tab, nt, base, fs->pe_begin + t / tiles_per_pe, words);
        for (int e = threadIdx.x; e < E; e += blockDim.x) cp_async16(&tile[swz(e)], fused_src(*fs, words, e, cmask, c));
        v = fs->dst[t / tiles_per_pe];
    } else if (T == kTileBits && blockDim.x == 128 && c <= 7) {
        // e = tid + 128 i: the swizzle is GF(2)-linear (swz(e) = swz(tid) ^ swz(128 i), a
        // constant per unrolled i) and e >> c, e & cmask split the same way, so each
        // load is one shared-memory table read and two ORs
        const int tsw = swz(threadIdx.x), th = threadIdx.x >> c;
        const amp_t* __restrict__ vb = v + (base | (threadIdx.x & cmask));
#pragma unroll
        for (int i = 0; i < (1 << kTileBits) / 128; ++i) {
            QRT_DCHECK((base | tab[th + (i << (7 - c))] | (threadIdx.x & cmask)) <
                       (static_cast<std::uint64_t>(tiles_per_pe) << T));
            cp_async16(&tile[tsw ^ swz(i * 128)], vb + tab[th + (i << (7 - c))]);
        }
    } else {
        for (int e = threadIdx.x; e < E; e += blockDim.x) {
            QRT_DCHECK((base | tab[e >> c] | (e & cmask)) < (static_cast<std::uint64_t>(tiles_per_pe) << T));
            cp_async16(&tile[swz(e)], &v[base | tab[e >> c] | (e & cmask)]);
        }
    }
    cp_async_wait_all();
    __syncthreads();

    const double* __restrict__ pf = frags + hdr.frag_begin;
    for (int o = 0; o < hdr.n_ops; ++o) {
        const GateOp& op = P.ops[o];
        const int kind = op.kind, k = op.k;
        if (kind == kDiag) {
            diagonal(tile, smat + op.smat, op, E, base);
        } else {
            const int pm = op.pmat;
            switch (k) {
                case 1: dense_small<1>(tile, P, pm, op, E); break;
                case 2: dense_small<2>(tile, P, pm, op, E); break;
                case 3:
                    if (op.bfrag >= 0 && hdr.gauss == 2 && MINB == 3)
                        dense_gauss<3, true>(tile, pf + op.bfrag, op, E);
                    else if (op.bfrag >= 0 && hdr.gauss)
                        dense_gauss<3>(tile, pf + op.bfrag, op, E);
                    else if (op.bfrag >= 0)
                        dense_dmma<3>(tile, pf + op.bfrag, op, E);
                    else
                        dense_small<3>(tile, P, pm, op, E);
                    break;
                case 4:
                    if (op.bfrag >= 0 && hdr.gauss == 2 && MINB == 3)
                        dense_gauss<4, true>(tile, pf + op.bfrag, op, E);
                    else if (op.bfrag >= 0 && hdr.gauss)
                        dense_gauss<4>(tile, pf + op.bfrag, op, E);
                    else if (op.bfrag >= 0)
                        dense_dmma<4>(tile, pf + op.bfrag, op, E);
                    else
                        dense_small<4>(tile, P, pm, op, E);
                    break;
                default: dense_wide(tile, pool + op.gmat, op, E); break;
            }
        }
        __syncthreads();
    }
    if (T == kTileBits && blockDim.x == 128 && c <= 7) {  // as the load
        const int tsw = swz(threadIdx.x), th = threadIdx.x >> c;
        amp_t* __restrict__ vb = v + (base | (threadIdx.x & cmask));
#pragma unroll
        for (int i = 0; i < (1 << kTileBits) / 128; ++i) __stcs(vb + tab[th + (i << (7 - c))], tile[tsw ^ swz(i * 128)]);
        return;
    }
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        QRT_DCHECK((base | tab[e >> c] | (e & cmask)) < (static_cast<std::uint64_t>(tiles_per_pe) << T));
        __stcs(&v[base | tab[e >> c] | (e & cmask)], tile[swz(e)]);
    }
}

// Out-of-place generic gate for very wide payloads: out[i] = sum_c U[row(i)][c] in[...].
__global__ void wide_gate_kernel(const amp_t* __restrict__ in, amp_t* __restrict__ out, std::uint64_t amps,
                                 const double2* __restrict__ u, int k, int diag, const int* __restrict__ posv) {
    int pos[kBigK];
    std::uint64_t tmask = 0;
    for (int j = 0; j < k; ++j) {
        pos[j] = posv[j];
        tmask |= 1ull << pos[j];
    }
    const int D = 1 << k;
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < amps;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        int row = 0;
        for (int j = 0; j < k; ++j) row |= static_cast<int>((i >> pos[j]) & 1ull) << j;
        double2 acc = make_double2(0.0, 0.0);
        if (diag) {
            cfma(acc, u[row], in[i]);
        } else {
            const std::uint64_t cleared = i & ~tmask;
            for (int cidx = 0; cidx < D; ++cidx) {
                std::uint64_t src = cleared;
                for (int j = 0; j < k; ++j) src |= static_cast<std::uint64_t>((cidx >> j) & 1) << pos[j];
                cfma(acc, u[static_cast<std::size_t>(row) * D + cidx], in[src]);
            }
        }
        out[i] = acc;
    }
}

// In-place generic gate for 8 <= k <= kWideInPlaceK dense qubits: one CTA per
// group of 2^k amplitudes at a time (grid-stride), the group staged in shared
// memory; each warp owns output rows and reduces sum_c U[r][c] x[c] across
// its lanes (U row-major, read coalesced from L2).  Groups are disjoint, so
// the update is exact in place: no spare buffer (single-buffer states, e.g.
// 34 qubits on 2 GPUs) and no copy-back.
constexpr int kWideInPlaceK = 12;

__global__ void __launch_bounds__(256) wide_group_kernel(amp_t* __restrict__ v, std::uint64_t amps,
                                                         const double2* __restrict__ u, int k,
                                                         const int* __restrict__ posv) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* x = reinterpret_cast<double2*>(smem_raw);
    int pos[kBigK];
    std::uint64_t tmask = 0;
    for (int j = 0; j < k; ++j) {
        pos[j] = posv[j];
        tmask |= 1ull << pos[j];
    }
    // the other positions, ascending: group index bits -> offset bits
    int rest[64];
    int nrest = 0;
    for (int b = 0; (1ull << b) < amps; ++b)
        if (!((tmask >> b) & 1ull)) rest[nrest++] = b;
    const int D = 1 << k;
    const std::uint64_t groups = amps >> k;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (std::uint64_t g = blockIdx.x; g < groups; g += gridDim.x) {
        std::uint64_t base = 0;
        for (int i = 0; i < nrest; ++i) base |= ((g >> i) & 1ull) << rest[i];
        for (int c = threadIdx.x; c < D; c += blockDim.x) {
            std::uint64_t o = base;
            for (int j = 0; j < k; ++j) o |= static_cast<std::uint64_t>((c >> j) & 1) << pos[j];
            QRT_DCHECK(o < amps);
            x[c] = v[o];
        }
        __syncthreads();
        for (int r = warp; r < D; r += nwarps) {
            double2 acc = make_double2(0.0, 0.0);
            const double2* __restrict__ ur = u + static_cast<std::size_t>(r) * D;
            for (int c = lane; c < D; c += 32) cfma(acc, ur[c], x[c]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
                acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
            }
            if (lane == 0) {
                std::uint64_t o = base;
                for (int j = 0; j < k; ++j) o |= static_cast<std::uint64_t>((r >> j) & 1) << pos[j];
                v[o] = acc;  // row r's input x[r] is in shared memory; its HBM slot is free to overwrite
            }
        }
        __syncthreads();
    }
}

// In-place diagonal gate of any width (elementwise).
__global__ void wide_diag_kernel(amp_t* __restrict__ v, std::uint64_t amps, const double2* __restrict__ d, int k,
                                 const int* __restrict__ posv) {
    int pos[kBigK];
    for (int j = 0; j < k; ++j) pos[j] = posv[j];
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < amps;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        int row = 0;
        for (int j = 0; j < k; ++j) row |= static_cast<int>((i >> pos[j]) & 1ull) << j;
        const double2 a = v[i], w = d[row];
        v[i] = make_double2(fma(w.x, a.x, -w.y * a.y), fma(w.x, a.y, w.y * a.x));
    }
}

// CTA size of the gate pass kernel: 128 (3 CTAs / SM, the launch bound) or 64;
// QRT_GATE_THREADS overrides for experiments.
int gate_threads() {
    static int v = [] {
        const char* e = std::getenv("QRT_GATE_THREADS");
        const int t = e ? std::atoi(e) : 128;
        return t == 64 ? 64 : 128;
    }();
    return v;
}

// Register budget of the gate pass kernel: the 3-CTA launch bound (<= 168
// registers: room for the hoisted Gauss fragments, measured fastest);
// QRT_GATE_REGS=128 selects the 4-CTA bound (fragments re-read from L1).
int gate_minb() {
    static const int v = [] {
        const char* e = std::getenv("QRT_GATE_REGS");
        return e && std::atoi(e) == 128 ? 4 : 3;
    }();
    return v;
}

// Low positions every shared-memory gate pass starts from (its HBM runs are
// at least 2^c amplitudes); QRT_GATE_COAL overrides (0..4).
int gate_coal_bits() {
    static const int v = [] {
        const char* e = std::getenv("QRT_GATE_COAL");
        return e ? std::max(0, std::min(kCoalBits, std::atoi(e))) : kCoalBits;
    }();
    return v;
}

int sm_count(qrt_state* st) {
    static int cached[64] = {};
    if (!cached[st->device]) {
        int v = 0;
        QRT_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, st->device));
        cached[st->device] = v;
    }
    return cached[st->device];
}

struct HostOp {
    int kind, k;
    int pos[kBigK];
    std::uint64_t mask;
    const double* m;      // interleaved complex payload (caller's mats or a fused product)
    int mat_len;          // double2 entries
    bool sign = false;    // diagonal with every entry exactly +1 or -1
    bool realcol = false; // dense 1-qubit gate whose first column is real (phase-folded)
    std::uint64_t neg = 0;  // sign gates: entries that are -1
};

bool light_op(const HostOp& h) {
    if (h.kind == kDense) return h.k <= 2;
    return h.sign ? h.k <= kLightMaxDiagK : h.k <= 2;
}

// Light-pass stage count cap (QRT_LIGHT_STAGES overrides for experiments).
int light_max_stages() {
    static int v = [] {
        const char* e = std::getenv("QRT_LIGHT_STAGES");
        const int s = e ? std::atoi(e) : 4;
        return std::max(1, std::min(s, kLightMaxStages));
    }();
    return v;
}

bool env_on(const char* name, bool dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) != 0 : dflt;
}

// Merge the +-1 diagonal ops of one light stage (ops[begin, end)): every
// thread-uniform sign op (kLSignU) commutes with all register work of the
// stage, so they are pooled into as few ops as their fixed sources allow
// (<= 6 W bits each) and placed first; consecutive slot-mask ops (kLSignS)
// with <= 2 fixed sources together are combined.  Returns the new end.
int merge_sign_ops(LightOp* ops, int begin, int end) {
    auto bit_of = [](const LightOp& op, const std::vector<int>& F, int f) {
        int fo = 0;  // the op's own fixed value from the merged value f
        for (int i = 0; i < op.nsrc; ++i) {
            const int at = static_cast<int>(std::find(F.begin(), F.end(), op.src[i]) - F.begin());
            fo |= ((f >> at) & 1) << i;
        }
        return fo;
    };
    auto union_src = [](const std::vector<int>& F, const LightOp& op) {
        std::vector<int> u = F;
        for (int i = 0; i < op.nsrc; ++i)
            if (std::find(u.begin(), u.end(), op.src[i]) == u.end()) u.push_back(op.src[i]);
        return u;
    };
    auto finish = [](LightOp& m, const std::vector<int>& F) {
        m.nsrc = static_cast<std::int8_t>(F.size());
        for (std::size_t i = 0; i < F.size(); ++i) m.src[i] = static_cast<std::int8_t>(F[i]);
    };
    std::vector<LightOp> uni, rest;
    for (int o = begin; o < end; ++o) (ops[o].kind == kLSignU ? uni : rest).push_back(ops[o]);
    std::vector<LightOp> out;
    // pooled uniform signs
    for (std::size_t i = 0; i < uni.size();) {
        std::vector<int> F;
        std::size_t j = i;
        while (j < uni.size() && union_src(F, uni[j]).size() <= 6) F = union_src(F, uni[j++]);
        LightOp m = uni[i];
        m.tab = 0;
        for (int f = 0; f < (1 << F.size()); ++f) {
            std::uint64_t b = 0;
            for (std::size_t q = i; q < j; ++q) b ^= (uni[q].tab >> bit_of(uni[q], F, f)) & 1ull;
            m.tab |= b << f;
        }
        finish(m, F);
        out.push_back(m);
        i = j;
    }
    // consecutive slot-mask signs
    for (std::size_t i = 0; i < rest.size();) {
        if (rest[i].kind != kLSignS) {
            out.push_back(rest[i++]);
            continue;
        }
        std::vector<int> F;
        std::size_t j = i;
        while (j < rest.size() && rest[j].kind == kLSignS && union_src(F, rest[j]).size() <= 2)
            F = union_src(F, rest[j++]);
        LightOp m = rest[i];
        m.tab = 0;
        for (int f = 0; f < (1 << F.size()); ++f) {
            std::uint64_t mask = 0;
            for (std::size_t q = i; q < j; ++q) mask ^= (rest[q].tab >> (16 * bit_of(rest[q], F, f))) & 0xffffull;
            m.tab |= mask << (16 * f);
        }
        finish(m, F);
        out.push_back(m);
        i = j;
    }
    for (std::size_t i = 0; i < out.size(); ++i) ops[begin + static_cast<int>(i)] = out[i];
    return begin + static_cast<int>(out.size());
}

// Stage plan of one light pass (see qrt_light.h): runs of the pass's ops,
// each with four register positions S; dense targets lie in S, diagonal
// gates anywhere; an op never overtakes a deferred op on a shared position.
struct LightStagePlan {
    std::uint64_t S = 0;
    std::vector<int> ops;
};

// DMMA B-fragment layout of M^T for a dense k-qubit gate, M = the 2D x 2D
// real form of U ([[Re, -Im], [Im, Re]] blocks): for fragment slot
// ((nb * KB + kb) * 32 + lane), the interleaved payload index and the sign.
// PTX m8n8k4.f64 B fragment: row k = lane & 3, column n = lane >> 2.
std::vector<std::pair<int, double>> frag_map(int k) {
    const int D = 1 << k, R = 2 * D, NB = R / 8, KB = R / 4;
    std::vector<std::pair<int, double>> m;
    for (int nb = 0; nb < NB; ++nb)
        for (int kb = 0; kb < KB; ++kb)
            for (int lane = 0; lane < 32; ++lane) {
                const int kk = 4 * kb + (lane & 3), nn = 8 * nb + (lane >> 2);
                const int r = nn >> 1, i = nn & 1, c = kk >> 1, j = kk & 1;
                const int at = 2 * (r * D + c);
                if (i == j)
                    m.emplace_back(at, 1.0);  // Re
                else
                    m.emplace_back(at + 1, i == 0 ? -1.0 : 1.0);  // -Im / +Im
            }
    return m;
}

// Gauss form (see dense_gauss): slot ((t * NB + nb) * KB + kb) * 32 + lane
// holds M_t[n][k], k = 4 kb + (lane & 3), n = 8 nb + (lane >> 2), with
// M_0 = Re U, M_1 = Im U - Re U, M_2 = -(Re U + Im U).
void gauss_frags(int k, const double* m, double* dst) {
    const int D = 1 << k, NB = D / 8, KB = D / 4;
    for (int t = 0; t < 3; ++t)
        for (int nb = 0; nb < NB; ++nb)
            for (int kb = 0; kb < KB; ++kb)
                for (int lane = 0; lane < 32; ++lane) {
                    const int kk = 4 * kb + (lane & 3), nn = 8 * nb + (lane >> 2);
                    const double x = m[2 * (nn * D + kk)], y = m[2 * (nn * D + kk) + 1];
                    *dst++ = t == 0 ? x : t == 1 ? y - x : -(x + y);
                }
}

// DMMA gates in the Gauss form (dense_gauss; QRT_GAUSS=0: the 2D x 2D real
// form, dense_dmma).
int gauss_mode() {
    static const int v = [] {
        const char* e = std::getenv("QRT_GAUSS");
        return e ? std::atoi(e) : 2;
    }();
    return v;
}

// Per-thread storage recycled between calls for the DMMA fragment pool.
std::vector<double>& frag_storage() {
    static thread_local std::vector<double> v;
    return v;
}

// One HBM pass of a gate plan (structure only; payloads are packed later).
struct GatePass {
    bool wide = false;
    bool light = false;
    int T = 0, c = 0;
    std::vector<int> tile_pos;
    std::vector<int> ops;
    std::vector<LightStagePlan> stages;
};

int plan_light_stages(const std::vector<HostOp>& opsv, const std::vector<int>& taken, std::uint64_t B, int m_max,
                      std::vector<LightStagePlan>* out, std::vector<int>* leftover) {
    std::vector<int> rem = taken, keep;
    int applied = 0, stages = 0;
    auto stage_take = [&](std::uint64_t S, LightStagePlan* sp, std::vector<int>* kp) {
        std::uint64_t blocked = 0;
        int n = 0;
        for (int id : rem) {
            const HostOp& h = opsv[static_cast<std::size_t>(id)];
            if ((h.mask & blocked) || (h.kind == kDense && (h.mask & ~S))) {
                blocked |= h.mask;
                if (kp) kp->push_back(id);
                continue;
            }
            ++n;
            if (sp) sp->ops.push_back(id);
        }
        return n;
    };
    while (!rem.empty() && stages < m_max) {
        std::uint64_t best_S = 0;
        int best = -1;
        int seeds = 0;
        const std::size_t m = rem.size();
        for (std::size_t sd = 0; sd < m && seeds < 8; ++sd) {
            if (opsv[static_cast<std::size_t>(rem[sd])].kind != kDense) continue;
            ++seeds;
            std::uint64_t S = 0, blocked = 0;
            for (std::size_t q = 0; q < m; ++q) {
                const HostOp& h = opsv[static_cast<std::size_t>(rem[(sd + q) % m])];
                if (h.kind != kDense) {
                    if (h.mask & blocked) blocked |= h.mask;
                    continue;
                }
                if ((h.mask & blocked) || __builtin_popcountll(S | h.mask) > kLightRegBits) {
                    blocked |= h.mask;
                    continue;
                }
                S |= h.mask;
                if (__builtin_popcountll(S) == kLightRegBits) break;
            }
            const int got = stage_take(S, nullptr, nullptr);
            if (got > best) {
                best = got;
                best_S = S;
            }
        }
        // fill to four register positions from the top of B (keeps the
        // coalescing positions out of S where possible: direct HBM access)
        for (int p = 63; p >= 0 && __builtin_popcountll(best_S) < kLightRegBits; --p)
            if ((B >> p & 1ull) && !(best_S >> p & 1ull)) best_S |= 1ull << p;
        LightStagePlan sp;
        sp.S = best_S;
        keep.clear();
        applied += stage_take(best_S, &sp, &keep);
        rem.swap(keep);
        if (out) out->push_back(std::move(sp));
        ++stages;
    }
    if (leftover) *leftover = rem;
    return applied;
}


constexpr int kLightMarker = 1 << 20;  // PassHdr::T of a light pass: marker + index into GatePlan::light

// The device program of one qrt_apply_gates call, built on the host.
struct GatePlan {
    std::vector<GateOp> dev_ops;
    std::vector<PassHdr> hdrs;  // one per pass (T >= kLightMarker: light pass, T < 0: wide gate)
    std::vector<double2> pool;
    std::vector<std::vector<double2>> pmats;
    std::vector<double> frags;
    std::vector<int> wide_pos;
    std::vector<std::unique_ptr<LightParams>> light;
    double flops_per_amp = 0.0;  // reference-equivalent flops of the gates as given
    int fused = 0;               // 1-qubit gates folded into a neighbour
};

GatePlan plan_gates(int nl, int n_gates, const int* arity, const int* pos, const double* mats, const unsigned* flags) {
    GatePlan plan;
    auto T0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!std::getenv("QRT_DEBUG_PLAN")) return;
        auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "  %s %.3f ms\n", what, std::chrono::duration<double, std::milli>(t - T0).count());
        T0 = t;
    };
    const double amps_all = 1.0;  // flops are accumulated per amplitude
    // ---- decode and validate -------------------------------------------------
    std::vector<HostOp> opsv(static_cast<std::size_t>(n_gates));
    std::size_t pcur = 0, mcur = 0;
    double& call_flops = plan.flops_per_amp;
    for (int i = 0; i < n_gates; ++i) {
        HostOp& h = opsv[static_cast<std::size_t>(i)];
        h.k = arity[i];
        if (h.k < 1 || h.k > nl) fail(QRT_ERR_ACCESS_VIOLATION, "gate arity out of range for the local region");
        if (h.k > kBigK) fail(QRT_ERR_INVALID, "gate arity above the supported maximum of 16");
        h.kind = (flags && (flags[i] & QRT_GATE_DIAGONAL)) ? kDiag : kDense;
        h.mask = 0;
        for (int j = 0; j < h.k; ++j) {
            const int p = pos[pcur++];
            if (p < 0 || p >= nl) fail(QRT_ERR_ACCESS_VIOLATION, "gate targets a global position; reorder first");
            if (h.mask >> p & 1ull) fail(QRT_ERR_INVALID, "duplicate target position");
            h.mask |= 1ull << p;
            h.pos[j] = p;
        }
        h.m = mats + mcur;
        h.mat_len = h.kind == kDiag ? (1 << h.k) : (1 << (2 * h.k));
        mcur += static_cast<std::size_t>(2 * h.mat_len);
        call_flops += 8.0 * (h.kind == kDiag ? 1.0 : static_cast<double>(1 << h.k)) * amps_all;
    }

    // ---- fuse runs of single-qubit gates on one position -------------------------
    // U_j U_i for consecutive 1-qubit gates i < j on the same position (no gate
    // on that position in between; gates elsewhere commute exactly).  The
    // product is formed in fp64 on the host, so amplitudes differ from the
    // gate-by-gate order only by rounding (<= 1e-15 here).
    std::vector<std::array<double, 8>> fused;
    fused.reserve(static_cast<std::size_t>(n_gates));
    std::vector<char> dead(static_cast<std::size_t>(n_gates), 0);
    if (env_on("QRT_FUSE_1Q", true)) {
        std::vector<int> nxt(static_cast<std::size_t>(n_gates), -1), last(64, -1);
        for (int i = n_gates - 1; i >= 0; --i) {
            const HostOp& h = opsv[static_cast<std::size_t>(i)];
            if (h.k == 1) nxt[static_cast<std::size_t>(i)] = last[static_cast<std::size_t>(h.pos[0])];
            for (int j = 0; j < h.k; ++j) last[static_cast<std::size_t>(h.pos[j])] = i;
        }
        for (int i = 0; i < n_gates; ++i) {
            const int j = nxt[static_cast<std::size_t>(i)];
            if (j < 0) continue;
            HostOp& a = opsv[static_cast<std::size_t>(i)];
            HostOp& b = opsv[static_cast<std::size_t>(j)];
            if (b.k != 1) continue;
            std::array<double, 8> r{};
            auto ent = [](const HostOp& h, int row, int col, double& re, double& im) {
                if (h.kind == kDiag) {
                    re = row == col ? h.m[2 * row] : 0.0;
                    im = row == col ? h.m[2 * row + 1] : 0.0;
                } else {
                    re = h.m[2 * (2 * row + col)];
                    im = h.m[2 * (2 * row + col) + 1];
                }
            };
            if (a.kind == kDiag && b.kind == kDiag) {
                for (int d = 0; d < 2; ++d) {
                    const double ar = a.m[2 * d], ai = a.m[2 * d + 1], br = b.m[2 * d], bi = b.m[2 * d + 1];
                    r[static_cast<std::size_t>(2 * d)] = br * ar - bi * ai;
                    r[static_cast<std::size_t>(2 * d + 1)] = br * ai + bi * ar;
                }
                b.mat_len = 2;
            } else {
                for (int row = 0; row < 2; ++row)
                    for (int col = 0; col < 2; ++col) {
                        double sr = 0.0, si = 0.0;
                        for (int q = 0; q < 2; ++q) {
                            double br, bi, ar, ai;
                            ent(b, row, q, br, bi);
                            ent(a, q, col, ar, ai);
                            sr += br * ar - bi * ai;
                            si += br * ai + bi * ar;
                        }
                        r[static_cast<std::size_t>(2 * (2 * row + col))] = sr;
                        r[static_cast<std::size_t>(2 * (2 * row + col) + 1)] = si;
                    }
                b.kind = kDense;
                b.mat_len = 4;
            }
            fused.push_back(r);
            b.m = fused.back().data();
            dead[static_cast<std::size_t>(i)] = 1;
            ++plan.fused;
        }
    }
    for (HostOp& h : opsv) {
        if (h.kind != kDiag) continue;
        h.sign = true;
        h.neg = 0;
        for (int e = 0; e < h.mat_len; ++e) {
            const double re = h.m[2 * e], im = h.m[2 * e + 1];
            if (im != 0.0 || (re != 1.0 && re != -1.0)) h.sign = false;
            if (re == -1.0 && h.k <= kLightMaxDiagK) h.neg |= 1ull << e;
        }
    }

    // ---- fold row phases of 1-qubit gates forward ----------------------------------
    // U = diag(e^{i a}, e^{i b}) V with V's first column real (a = arg u00,
    // b = arg u10): V costs 6 instead of 8 fp64 operations per amplitude.  The
    // phase diagonal commutes with every diagonal gate and with gates on other
    // positions, so it is multiplied into the columns of the next dense gate
    // on the same position; the last dense gate on a position keeps its full
    // matrix.  The call's final state is unchanged (up to rounding).
    std::deque<std::vector<double>> owned;
    if (env_on("QRT_PHASE_FOLD", true)) {
        // factor a 1-qubit gate only if the next dense gate on its position
        // exists and is narrow (k <= 4), so absorbing the phases stays cheap
        std::vector<char> next_dense(static_cast<std::size_t>(n_gates), 0);
        {
            std::vector<int> next_k(64, 0);  // arity of the nearest later dense gate per position
            for (int i = n_gates - 1; i >= 0; --i) {
                const HostOp& h = opsv[static_cast<std::size_t>(i)];
                if (dead[static_cast<std::size_t>(i)] || h.kind != kDense) continue;
                if (h.k == 1) {
                    const int nk = next_k[static_cast<std::size_t>(h.pos[0])];
                    next_dense[static_cast<std::size_t>(i)] = nk >= 1 && nk <= 4;
                }
                for (int j = 0; j < h.k; ++j) next_k[static_cast<std::size_t>(h.pos[j])] = h.k;
            }
        }
        std::vector<std::array<double, 4>> pend(64, {1.0, 0.0, 1.0, 0.0});  // (d0, d1) per position
        std::vector<char> has(64, 0);
        for (int i = 0; i < n_gates; ++i) {
            HostOp& h = opsv[static_cast<std::size_t>(i)];
            if (dead[static_cast<std::size_t>(i)] || h.kind != kDense) continue;
            bool touched = false;
            for (int j = 0; j < h.k; ++j) touched = touched || has[static_cast<std::size_t>(h.pos[j])];
            const bool factor = h.k == 1 && next_dense[static_cast<std::size_t>(i)];
            if (!touched && !factor) continue;
            const int D = 1 << h.k;
            owned.emplace_back(h.m, h.m + 2 * D * D);
            std::vector<double>& M = owned.back();
            // absorb pending column phases of the targets
            for (int j = 0; j < h.k; ++j) {
                const std::size_t pj = static_cast<std::size_t>(h.pos[j]);
                if (!has[pj]) continue;
                for (int r = 0; r < D; ++r)
                    for (int c = 0; c < D; ++c) {
                        const int bit = (c >> j) & 1;
                        const double dr = pend[pj][2 * bit], di = pend[pj][2 * bit + 1];
                        double& xr = M[static_cast<std::size_t>(2 * (r * D + c))];
                        double& xi = M[static_cast<std::size_t>(2 * (r * D + c) + 1)];
                        const double nr = xr * dr - xi * di, ni = xr * di + xi * dr;
                        xr = nr;
                        xi = ni;
                    }
                has[pj] = 0;
            }
            if (factor) {  // row phases out, first column real
                const std::size_t pj = static_cast<std::size_t>(h.pos[0]);
                for (int r = 0; r < 2; ++r) {
                    const double ar = M[static_cast<std::size_t>(4 * r)], ai = M[static_cast<std::size_t>(4 * r + 1)];
                    const double mag = std::hypot(ar, ai);
                    const double cr = mag > 0.0 ? ar / mag : 1.0, ci = mag > 0.0 ? ai / mag : 0.0;  // e^{i arg}
                    for (int c = 0; c < 2; ++c) {  // row r times e^{-i arg}
                        double& xr = M[static_cast<std::size_t>(2 * (2 * r + c))];
                        double& xi = M[static_cast<std::size_t>(2 * (2 * r + c) + 1)];
                        const double nr = xr * cr + xi * ci, ni = xi * cr - xr * ci;
                        xr = nr;
                        xi = ni;
                    }
                    M[static_cast<std::size_t>(4 * r)] = mag;
                    M[static_cast<std::size_t>(4 * r + 1)] = 0.0;
                    pend[pj][2 * r] = cr;
                    pend[pj][2 * r + 1] = ci;
                }
                has[pj] = 1;
                h.realcol = true;
            }
            h.m = M.data();
        }
    }

    lap("decode+fuse");
    // ---- plan passes -----------------------------------------------------------
    // The decomposition depends only on the gate structure (arity, positions,
    // kinds after fusion, sign classification), not on payload values: a VQE
    // loop re-applies the same circuit with new angles every iteration, so it
    // is cached by that structure and only the payloads are re-packed below.
    using Pass = GatePass;
    std::vector<std::uint64_t> skey;
    skey.reserve(4 + 4 * static_cast<std::size_t>(n_gates));
    skey.push_back(static_cast<std::uint64_t>(nl));
    skey.push_back(static_cast<std::uint64_t>(n_gates));
    skey.push_back((nl >= kTileBits && env_on("QRT_LIGHT", true) ? 1u : 0u) | (static_cast<unsigned>(light_max_stages()) << 1));
    for (int i = 0; i < n_gates; ++i) {
        const HostOp& h = opsv[static_cast<std::size_t>(i)];
        std::uint64_t w = static_cast<std::uint64_t>(h.k) | (static_cast<std::uint64_t>(h.kind) << 8) |
                          (static_cast<std::uint64_t>(dead[static_cast<std::size_t>(i)]) << 9) |
                          (static_cast<std::uint64_t>(h.sign) << 10) | (static_cast<std::uint64_t>(h.mat_len) << 16);
        skey.push_back(w);
        skey.push_back(h.mask);
        skey.push_back(h.sign ? h.neg : 0);
        std::uint64_t order = 0;
        for (int j = 0; j < h.k && j < 10; ++j) order |= static_cast<std::uint64_t>(h.pos[j]) << (6 * j);
        skey.push_back(order);
    }
    static std::mutex plan_mu;
    static std::deque<std::pair<std::vector<std::uint64_t>, std::shared_ptr<const std::vector<GatePass>>>> plan_cache;
    std::shared_ptr<const std::vector<GatePass>> cached;
    if (env_on("QRT_PLAN_CACHE", true)) {
        std::lock_guard<std::mutex> lock(plan_mu);
        for (auto& e : plan_cache)
            if (e.first == skey) cached = e.second;
    }
    std::vector<Pass> passes;
    if (cached) passes = *cached;
    std::vector<int> remaining;
    remaining.reserve(static_cast<std::size_t>(n_gates));
    for (int i = 0; i < n_gates; ++i)
        if (!dead[static_cast<std::size_t>(i)]) remaining.push_back(i);
    auto is_wide = [&](const HostOp& h) {
        return h.kind == kDiag ? h.k > kMaxDiagK : h.k > kMaxTileGateK;
    };
    const bool whole = nl <= kTileBits;
    const bool light_ok = nl >= kTileBits && env_on("QRT_LIGHT", true);
    const int m_max = light_max_stages();
    // The take phase for tile positions B: in order, every gate whose targets
    // are inside B (diagonals anywhere) unless it follows a deferred gate on a
    // shared qubit or the per-pass staging budgets are exhausted.  The first
    // gate taken fixes the pass kind: a light pass (register-resident,
    // qrt_light.cu) takes only 1-/2-qubit and diagonal gates.
    auto take = [&](std::uint64_t B, Pass* ps, std::vector<int>* keep) -> int {
        std::uint64_t blocked = 0;
        int param_used = 0, diag_used = 0, frag_used = 0, n = 0;
        int mode = -1;  // -1 undecided, 0 heavy, 1 light
        bool closed = false, wide = false;
        for (int id : remaining) {
            const HostOp& h = opsv[static_cast<std::size_t>(id)];
            if (closed || (h.mask & blocked)) {
                blocked |= h.mask;
                if (keep) keep->push_back(id);
                continue;
            }
            if (is_wide(h)) {
                if (n == 0) {  // runs alone, out of place
                    wide = closed = true;
                    ++n;
                    if (ps) ps->ops.push_back(id);
                } else {
                    blocked |= h.mask;
                    if (keep) keep->push_back(id);
                }
                continue;
            }
            const bool fits = h.kind == kDiag || (h.mask & ~B) == 0;
            if (fits && mode < 0) mode = (light_ok && light_op(h)) ? 1 : 0;
            bool ok = fits;
            if (ok && mode == 1) {
                const int in_mats = h.kind == kDense ? h.mat_len : (h.sign ? 0 : h.mat_len);
                ok = light_op(h) && n < kLightMaxOps && param_used + in_mats <= kLightMaxMats;
                if (ok) param_used += in_mats;
            } else if (ok) {
                const int T_here = whole ? nl : kTileBits;
                const bool dmma = h.kind == kDense && (h.k == 3 || h.k == 4) && T_here >= h.k + 3;
                const int in_params = (h.kind == kDense && h.k <= 4 && !dmma) ? h.mat_len : 0;
                const int in_smem = h.kind == kDiag ? h.mat_len : 0;
                const int in_frag = dmma ? (gauss_mode() ? 3 : 4) * h.mat_len : 0;  // (2D)^2 real entries
                ok = param_used + in_params <= kParamMats && diag_used + in_smem <= kDiagStage &&
                     frag_used + in_frag <= kFragStage && n < kMaxPassOps;
                if (ok) {
                    param_used += in_params;
                    diag_used += in_smem;
                    frag_used += in_frag;
                }
            }
            if (ok) {
                ++n;
                if (ps) ps->ops.push_back(id);
            } else {
                blocked |= h.mask;
                if (keep) keep->push_back(id);
            }
        }
        if (ps) {
            ps->wide = wide;
            ps->light = mode == 1 && !wide;
        }
        return n;
    };
    // Gates a pass over B actually applies: light passes are cut to the
    // stage budget.
    auto evaluate = [&](std::uint64_t B, Pass* ps, std::vector<int>* keep) -> int {
        Pass tmp;
        std::vector<int> k1;
        Pass* pp = ps ? ps : &tmp;
        std::vector<int>* kp = keep ? keep : &k1;
        const int got = take(B, pp, kp);
        if (!pp->light) return got;
        std::vector<int> left;
        std::vector<LightStagePlan>* sp = ps ? &ps->stages : nullptr;
        const int applied = plan_light_stages(opsv, pp->ops, B, m_max, sp, &left);
        if (ps) {
            if (!left.empty()) {  // unapplied ops go back, original order
                std::vector<int> merged;
                merged.reserve(kp->size() + left.size());
                std::merge(kp->begin(), kp->end(), left.begin(), left.end(), std::back_inserter(merged));
                kp->swap(merged);
                std::vector<int> app;
                for (const auto& s : ps->stages) app.insert(app.end(), s.ops.begin(), s.ops.end());
                ps->ops = app;
            }
        }
        return applied;
    };
    // Candidate tile positions seeded from one of the first remaining gates:
    // grow B from the coalescing bits by the targets of gates in order
    // (rotated to start at the seed), skipping gates that are blocked or
    // would overflow the tile.  The candidate that applies most gates wins
    // (ties: the earliest seed).  Seeding from several gates lets a pass
    // follow the light cone of the circuit instead of the first layer only.
    constexpr int kSeeds = 16;
    auto candidate = [&](std::size_t seed) {
        std::uint64_t B = (1ull << gate_coal_bits()) - 1, blocked = 0;
        const std::size_t m = remaining.size();
        for (std::size_t q = 0; q < m; ++q) {
            const HostOp& h = opsv[static_cast<std::size_t>(remaining[(seed + q) % m])];
            if (h.kind == kDiag) {
                if (h.mask & blocked) blocked |= h.mask;
                continue;
            }
            if ((h.mask & blocked) || is_wide(h) || __builtin_popcountll(B | h.mask) > kTileBits) {
                blocked |= h.mask;
                continue;
            }
            B |= h.mask;
            if (__builtin_popcountll(B) == kTileBits) break;
        }
        for (int p = 0; p < nl && __builtin_popcountll(B) < kTileBits; ++p) B |= 1ull << p;
        return B;
    };
    if (cached) remaining.clear();
    while (!remaining.empty()) {
        std::uint64_t B = 0;
        if (whole) {
            B = (nl >= 64) ? ~0ull : ((1ull << nl) - 1);
        } else {
            int best = -1;
            const std::size_t seeds = std::min<std::size_t>(kSeeds, remaining.size());
            for (std::size_t sd = 0; sd < seeds; ++sd) {
                const std::uint64_t cand = candidate(sd);
                const int got = evaluate(cand, nullptr, nullptr);
                if (got > best) {
                    best = got;
                    B = cand;
                }
            }
        }
        Pass ps;
        std::vector<int> keep;
        keep.reserve(remaining.size());
        evaluate(B, &ps, &keep);
        if (ps.ops.empty()) fail(QRT_ERR_INVALID, "gate planner made no progress");
        if (!ps.wide) {
            for (int p = 0; p < nl; ++p)
                if (B >> p & 1ull) ps.tile_pos.push_back(p);
            ps.T = static_cast<int>(ps.tile_pos.size());
            ps.c = 0;
            while (ps.c < ps.T && ps.tile_pos[static_cast<std::size_t>(ps.c)] == ps.c) ++ps.c;
        }
        passes.push_back(std::move(ps));
        remaining.swap(keep);
    }
    if (!cached && env_on("QRT_PLAN_CACHE", true)) {
        std::lock_guard<std::mutex> lock(plan_mu);
        plan_cache.emplace_back(std::move(skey), std::make_shared<const std::vector<GatePass>>(passes));
        if (plan_cache.size() > 512) plan_cache.pop_front();
    }

    lap("plan");
    // ---- pack descriptors + matrices into one upload ------------------------------
    std::vector<GateOp>& dev_ops = plan.dev_ops;
    std::vector<PassHdr>& hdrs = plan.hdrs;
    std::vector<double2>& pool = plan.pool;
    std::vector<std::vector<double2>>& pmats = plan.pmats;
    pmats.resize(passes.size());
    std::vector<double>& frags = plan.frags;
    {
        // reuse the previous call's storage (no page faults on ~14 MB of
        // fragments per call) and size it exactly
        frags.swap(frag_storage());
        frags.clear();
        std::size_t need = 0;
        for (const auto& ps : passes)
            if (!ps.light && !ps.wide)
                for (int id : ps.ops) {
                    const HostOp& o = opsv[static_cast<std::size_t>(id)];
                    if (o.kind == kDense && (o.k == 3 || o.k == 4) && ps.T >= o.k + 3)
                        need += (gauss_mode() ? 3u : 4u) * o.mat_len;
                }
        frags.reserve(need);
    }
    std::vector<int>& wide_pos = plan.wide_pos;  // for wide passes: positions (kBigK per pass)
    std::vector<std::unique_ptr<LightParams>>& light = plan.light;
    auto build_light = [&](const std::vector<int>& tile_pos, int c, const std::vector<LightStagePlan>& stages) {
        auto L = std::make_unique<LightParams>();
        std::memset(L.get(), 0, sizeof(LightParams));
        int tb_of[64];
        for (int p = 0; p < 64; ++p) tb_of[p] = -1;
        std::uint64_t inB = 0;
        for (int i = 0; i < kTileBits; ++i) {
            L->tile_pos[i] = static_cast<std::int8_t>(tile_pos[static_cast<std::size_t>(i)]);
            tb_of[tile_pos[static_cast<std::size_t>(i)]] = i;
            inB |= 1ull << tile_pos[static_cast<std::size_t>(i)];
        }
        int no = 0;
        for (int p = 0; p < nl; ++p)
            if (!(inB >> p & 1ull)) L->outer_pos[no++] = static_cast<std::int8_t>(p);
        L->n_outer = no;
        L->c = c;
        L->tiles_per_pe = 1 << (nl - kTileBits);
        L->n_stages = static_cast<int>(stages.size());
        int n_ops = 0, n_mats = 0;
        const int lowmask = (1 << kCoalBits) - 1;
        for (std::size_t s = 0; s < stages.size(); ++s) {
            LightStage& S = L->st[s];
            int sbits = 0, q = 0;
            int reg_of[kTileBits];
            for (int i = 0; i < kTileBits; ++i) reg_of[i] = 4;
            for (int i = 0; i < kTileBits; ++i)
                if (stages[s].S >> tile_pos[static_cast<std::size_t>(i)] & 1ull) {
                    S.S[q] = static_cast<std::int8_t>(i);
                    reg_of[i] = q++;
                    sbits |= 1 << i;
                }
            // thread bits: the remaining tile bits ascending, except that the
            // three lowest lanes get distinct residues mod 3 (conflict-free
            // 16-byte shared-memory phases under swz) when S took a low bit
            std::vector<int> rest;
            for (int i = 0; i < kTileBits; ++i)
                if (!(sbits >> i & 1)) rest.push_back(i);
            if (sbits & lowmask) {
                std::vector<int> lead;
                for (int res = 0; res < 3; ++res)
                    for (std::size_t u = 0; u < rest.size(); ++u)
                        if (rest[u] % 3 == res) {
                            lead.push_back(rest[u]);
                            rest.erase(rest.begin() + static_cast<std::ptrdiff_t>(u));
                            break;
                        }
                rest.insert(rest.begin(), lead.begin(), lead.end());
            }
            for (int i = 0; i < kTileBits - kLightRegBits; ++i)
                S.tb[i] = static_cast<std::int8_t>(rest[static_cast<std::size_t>(i)]);
            if (s == 0) L->direct_in = (sbits & lowmask) == 0;
            if (s + 1 == stages.size()) L->direct_out = (sbits & lowmask) == 0;
            S.op_begin = static_cast<std::int16_t>(n_ops);
            // W bit of a position: tile bit, or 12 + index among the outer positions
            auto wbit = [&](int p) {
                if (tb_of[p] >= 0) return tb_of[p];
                for (int i = 0; i < no; ++i)
                    if (L->outer_pos[i] == p) return kTileBits + i;
                fail(QRT_ERR_INVALID, "light pass: diagonal target not in the local region");
            };
            int pend_bits = 0;  // register bits the pending slot signs depend on
            for (int id : stages[s].ops) {
                const HostOp& o = opsv[static_cast<std::size_t>(id)];
                LightOp& lo = L->ops[n_ops++];
                lo.k = static_cast<std::int8_t>(o.k);
                auto put_mat = [&](int len, auto&& entry) {
                    lo.mat = static_cast<std::int16_t>(n_mats);
                    for (int e = 0; e < len; ++e) L->mats[n_mats++] = entry(e);
                };
                if (o.kind == kDense) {
                    const int qa = reg_of[tb_of[o.pos[0]]];
                    int touched = 1 << qa;
                    if (o.k == 1) {
                        lo.kind = kL1;
                        lo.realcol = o.realcol ? 1 : 0;
                        lo.q0 = static_cast<std::int8_t>(qa);
                        put_mat(4, [&](int e) { return make_double2(o.m[2 * e], o.m[2 * e + 1]); });
                    } else {
                        const int qb = reg_of[tb_of[o.pos[1]]];
                        touched |= 1 << qb;
                        lo.kind = kL2;
                        const bool swap = qa > qb;
                        lo.q0 = static_cast<std::int8_t>(swap ? qb : qa);
                        lo.q1 = static_cast<std::int8_t>(swap ? qa : qb);
                        auto sw = [&](int x) { return swap ? (((x & 1) << 1) | (x >> 1)) : x; };
                        put_mat(16, [&](int e) {
                            const int r = sw(e >> 2), cc = sw(e & 3);
                            const int at = 4 * r + cc;
                            return make_double2(o.m[2 * at], o.m[2 * at + 1]);
                        });
                    }
                    // pending slot signs commute with this gate unless they
                    // depend on one of its register bits
                    if (pend_bits & touched) {
                        lo.flush = 1;
                        pend_bits = 0;
                    }
                    continue;
                }
                // diagonal: register targets and fixed (W-bit) sources
                int nsrc = 0, regmask = 0;
                for (int j = 0; j < kLightMaxDiagK; ++j) {
                    lo.rq[j] = 4;
                    lo.src[j] = 0;
                    lo.fj[j] = 0;
                }
                for (int j = 0; j < o.k; ++j) {
                    const int tb = tb_of[o.pos[j]];
                    if (tb >= 0 && reg_of[tb] < 4) {
                        lo.rq[j] = static_cast<std::int8_t>(reg_of[tb]);
                        regmask |= 1 << reg_of[tb];
                    } else {
                        lo.src[nsrc] = static_cast<std::int8_t>(wbit(o.pos[j]));
                        lo.fj[nsrc] = static_cast<std::int8_t>(j);
                        ++nsrc;
                    }
                }
                lo.nsrc = static_cast<std::int8_t>(nsrc);
                auto entry_index = [&](int f, int r) {
                    int m = 0;
                    for (int i = 0; i < nsrc; ++i) m |= ((f >> i) & 1) << lo.fj[i];
                    for (int j = 0; j < o.k; ++j)
                        if (lo.rq[j] < 4) m |= ((r >> lo.rq[j]) & 1) << j;
                    return m;
                };
                if (!o.sign) {  // phase diagonal (k <= 2): commutes with pending signs
                    lo.kind = kLDiag;
                    put_mat(o.mat_len, [&](int e) { return make_double2(o.m[2 * e], o.m[2 * e + 1]); });
                } else if (regmask == 0) {
                    lo.kind = kLSignU;
                    lo.tab = 0;
                    for (int f = 0; f < (1 << nsrc); ++f)
                        if ((o.neg >> entry_index(f, 0)) & 1ull) lo.tab |= 1ull << f;
                } else if (nsrc <= 2) {
                    lo.kind = kLSignS;
                    lo.tab = 0;
                    for (int f = 0; f < (1 << nsrc); ++f)
                        for (int r = 0; r < 16; ++r)
                            if ((o.neg >> entry_index(f, r)) & 1ull) lo.tab |= 1ull << (16 * f + r);
                    pend_bits |= regmask;
                } else {
                    lo.kind = kLSignG;
                    lo.tab = o.neg;
                    pend_bits |= regmask;
                }
            }
            if (env_on("QRT_MERGE_SIGNS", true)) n_ops = merge_sign_ops(L->ops, S.op_begin, n_ops);
            for (int o = S.op_begin; o < n_ops; ++o) {
                LightOp& lo = L->ops[o];
                int code = kCodeDiag;
                if (lo.kind == kL1) code = lo.realcol ? kCodeReal1 + lo.q0 : lo.q0;
                else if (lo.kind == kL2) {
                    static const int pair_code[4][4] = {{-1, 4, 5, 6}, {-1, -1, 7, 8}, {-1, -1, -1, 9}, {-1, -1, -1, -1}};
                    code = pair_code[lo.q0][lo.q1];
                } else if (lo.kind == kLSignU) code = kCodeSignU;
                else if (lo.kind == kLSignS) code = kCodeSignS;
                else if (lo.kind == kLSignG) code = kCodeSignG;
                lo.code = static_cast<std::int8_t>(code | (lo.flush ? kCodeFlush : 0));
                if (const char* dbg = std::getenv("QRT_DEBUG_PLAN"); dbg && std::atoi(dbg) >= 2)
                    std::fprintf(stderr, "light op code %d flush %d\n", code, lo.flush ? 1 : 0);
            }
            S.op_count = static_cast<std::int16_t>(n_ops - S.op_begin);
        }
        if (n_ops > kLightMaxOps || n_mats > kLightMaxMats) fail(QRT_ERR_INVALID, "light pass over budget");
        return L;
    };
    for (std::size_t pidx = 0; pidx < passes.size(); ++pidx) {
        Pass& ps = passes[pidx];
        PassHdr h{};
        if (ps.light) {
            h.T = kLightMarker + static_cast<int>(light.size());
            light.push_back(build_light(ps.tile_pos, ps.c, ps.stages));
            hdrs.push_back(h);
            continue;
        }
        if (ps.wide) {
            const HostOp& o = opsv[static_cast<std::size_t>(ps.ops[0])];
            h.n_ops = 1;
            h.op_begin = static_cast<int>(dev_ops.size());
            h.mat_begin = static_cast<int>(pool.size());
            h.mat_count = o.mat_len;
            GateOp g{};
            g.kind = o.kind;
            g.k = o.k;
            g.smat = -1;
            g.gmat = h.mat_begin;
            dev_ops.push_back(g);
            for (int e = 0; e < o.mat_len; ++e)
                pool.push_back(make_double2(o.m[2 * static_cast<std::size_t>(e)],
                                            o.m[2 * static_cast<std::size_t>(e) + 1]));
            h.T = -static_cast<int>(wide_pos.size()) - 1;  // marks a wide pass; index into wide_pos
            for (int j = 0; j < kBigK; ++j) wide_pos.push_back(j < o.k ? o.pos[j] : 0);
            hdrs.push_back(h);
            continue;
        }
        h.T = ps.T;
        h.c = ps.c;
        h.n_ops = static_cast<int>(ps.ops.size());
        h.op_begin = static_cast<int>(dev_ops.size());
        h.mat_begin = static_cast<int>(pool.size());
        for (int i = 0; i < ps.T; ++i) h.tile_pos[i] = ps.tile_pos[static_cast<std::size_t>(i)];
        int no = 0;
        std::uint64_t inB = 0;
        for (int p : ps.tile_pos) inB |= 1ull << p;
        for (int p = 0; p < nl; ++p)
            if (!(inB >> p & 1ull)) h.outer_pos[no++] = p;
        h.n_outer = no;
        int tb_of[64];
        for (int p = 0; p < 64; ++p) tb_of[p] = -1;
        for (int i = 0; i < ps.T; ++i) tb_of[ps.tile_pos[static_cast<std::size_t>(i)]] = i;
        // diagonals staged contiguously in the pool (copied to smem per CTA),
        // dense k<=4 matrices into the launch parameters, k=5..7 from global
        auto put = [&](std::vector<double2>& dst, const HostOp& o) {
            for (int e = 0; e < o.mat_len; ++e)
                dst.push_back(make_double2(o.m[2 * static_cast<std::size_t>(e)],
                                           o.m[2 * static_cast<std::size_t>(e) + 1]));
        };
        int staged = 0;
        h.frag_begin = static_cast<int>(frags.size());
        h.gauss = gauss_mode();
        std::vector<std::pair<int, int>> late;  // (op index in dev_ops, host op)
        for (int id : ps.ops) {
            const HostOp& o = opsv[static_cast<std::size_t>(id)];
            GateOp g{};
            g.kind = o.kind;
            g.k = o.k;
            g.smat = g.pmat = g.bfrag = -1;
            for (int j = 0; j < o.k; ++j) {
                g.tb[j] = tb_of[o.pos[j]];
                g.pos[j] = o.pos[j];
            }
            if (o.kind == kDiag) {
                g.smat = staged;
                g.gmat = h.mat_begin + staged;
                put(pool, o);
                staged += o.mat_len;
            } else if ((o.k == 3 || o.k == 4) && ps.T >= o.k + 3) {
                // DMMA B fragments of M^T, M = real form of U (see dense_dmma)
                const int D = 1 << o.k, R = 2 * D;
                g.bfrag = static_cast<int>(frags.size()) - h.frag_begin;
                // fragment slot -> (interleaved source index, sign), built once per k
                static const std::vector<std::pair<int, double>> map3 = frag_map(3), map4 = frag_map(4);
                const auto& fm = o.k == 3 ? map3 : map4;
                const std::size_t at = frags.size();
                if (h.gauss) {
                    frags.resize(at + 3u * static_cast<std::size_t>(D) * D);
                    gauss_frags(o.k, o.m, frags.data() + at);
                } else {
                    frags.resize(at + static_cast<std::size_t>(R) * R);
                    double* dst = frags.data() + at;
                    for (std::size_t e = 0; e < fm.size(); ++e) dst[e] = fm[e].second * o.m[fm[e].first];
                }
            } else if (o.k <= 4) {
                g.pmat = static_cast<int>(pmats[pidx].size());
                put(pmats[pidx], o);
            } else {
                late.emplace_back(static_cast<int>(dev_ops.size()), id);
            }
            dev_ops.push_back(g);
        }
        h.mat_count = staged;
        h.frag_count = static_cast<int>(frags.size()) - h.frag_begin;
        for (auto [di, id] : late) {
            dev_ops[static_cast<std::size_t>(di)].gmat = static_cast<int>(pool.size());
            put(pool, opsv[static_cast<std::size_t>(id)]);
        }
        hdrs.push_back(h);
    }
    lap("pack");
    return plan;
}

}  // namespace

void apply_gates(qrt_state* st, int n_gates, const int* arity, const int* pos, const double* mats,
                 const unsigned* flags) {
    GatePlan plan = plan_gates(st->nl, n_gates, arity, pos, mats, flags);
    const double amps_all = static_cast<double>(st->amps) * st->pe_count;
    const double call_flops = plan.flops_per_amp * amps_all;
    const auto& dev_ops = plan.dev_ops;
    const auto& hdrs = plan.hdrs;
    const auto& pool = plan.pool;
    const auto& pmats = plan.pmats;
    const auto& frags = plan.frags;
    const auto& wide_pos = plan.wide_pos;
    auto& light = plan.light;
    struct GiveBack {
        std::vector<double>& f;
        ~GiveBack() { frag_storage().swap(f); }
    } give_back{plan.frags};
    // A pending QR is executed by the first pass (qrt_fused.h) unless that
    // pass is an out-of-place wide gate.
    bool fuse_first = false;
    FusedSource fsrc{};
    // A light (register-resident) pass computes too little per tile to hide a
    // pull over whole 2^31-amplitude peer buffers: past 2^30 per PE its QR runs
    // in place first (34q HEA with 2 PEs on each of 4 GPUs: gates 3.24 s fused
    // vs ~2.1 s), while DMMA gate passes keep pulling up to fused_qr_max_log2().
    static const int light_fuse_max = [] {
        const char* e = std::getenv("QRT_FUSED_LIGHT_MAX_LOG2");
        return e ? std::atoi(e) : 30;
    }();
    if (st->qr_pending) {
        const bool light_first = !hdrs.empty() && hdrs[0].T >= kLightMarker;
        if (!hdrs.empty() && hdrs[0].T >= 0 && !(light_first && st->nl > light_fuse_max)) {
            fuse_first = true;
            ensure_alt(st);
            for (int pe = 0; pe < st->p; ++pe) fsrc.src[pe] = st->peer[st->cur][static_cast<std::size_t>(pe)];
            for (int i = 0; i < st->pe_count; ++i) fsrc.dst[i] = st->bufs[st->cur ^ 1][static_cast<std::size_t>(i)];
            for (int s2 = 0; s2 < st->n; ++s2) fsrc.src_of[st->qr_dest[static_cast<std::size_t>(s2)]] = s2;
            fsrc.n = st->n;
            fsrc.nl = st->nl;
            fsrc.pe_begin = st->pe_begin;
        } else {
            flush_reorder(st);
        }
    }
    const std::size_t ops_bytes = dev_ops.size() * sizeof(GateOp);
    const std::size_t pool_off = (ops_bytes + 255) & ~std::size_t{255};
    const std::size_t pool_bytes = pool.size() * sizeof(double2);
    const std::size_t wpos_off = (pool_off + pool_bytes + 255) & ~std::size_t{255};
    const std::size_t frag_off = (wpos_off + wide_pos.size() * sizeof(int) + 255) & ~std::size_t{255};
    const std::size_t fs_off = (frag_off + frags.size() * sizeof(double) + 255) & ~std::size_t{255};
    const std::size_t total = fs_off + sizeof(FusedSource) + 16;
    char* host = static_cast<char*>(ensure_pinned(st, total));
    QRT_CUDA(cudaStreamSynchronize(st->stream));  // pinned buffer may still feed a previous copy
    std::memcpy(host, dev_ops.data(), ops_bytes);
    std::memcpy(host + pool_off, pool.data(), pool_bytes);
    std::memcpy(host + wpos_off, wide_pos.data(), wide_pos.size() * sizeof(int));
    std::memcpy(host + frag_off, frags.data(), frags.size() * sizeof(double));
    std::memcpy(host + fs_off, &fsrc, sizeof(FusedSource));
    char* dev = static_cast<char*>(ensure_ops(st, total));
    QRT_CUDA(cudaMemcpyAsync(dev, host, total, cudaMemcpyHostToDevice, st->stream));
    const GateOp* d_ops = reinterpret_cast<const GateOp*>(dev);
    const double2* d_pool = reinterpret_cast<const double2*>(dev + pool_off);
    const int* d_wpos = reinterpret_cast<const int*>(dev + wpos_off);
    const double* d_frags = reinterpret_cast<const double*>(dev + frag_off);
    const FusedSource* d_fs = reinterpret_cast<const FusedSource*>(dev + fs_off);

    static bool attr_done[64] = {};
    if (!attr_done[st->device]) {
        QRT_CUDA(cudaFuncSetAttribute(gate_pass_kernel<false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        QRT_CUDA(cudaFuncSetAttribute(gate_pass_kernel<true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        QRT_CUDA(cudaFuncSetAttribute(gate_pass_kernel<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        QRT_CUDA(cudaFuncSetAttribute(gate_pass_kernel<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_done[st->device] = true;
    }

    static thread_local PassParams params;  // 29 KiB: keep off the stack
    ProfileScope prof(st, QRT_K_GATES);
    st->stats[QRT_K_GATES].flops += call_flops;
    for (std::size_t pi = 0; pi < hdrs.size(); ++pi) {
        const PassHdr& h = hdrs[pi];
        const bool fused = fuse_first && pi == 0;
        if (fused) barrier_on_stream(st);  // every source buffer complete on every rank
        if (h.T >= kLightMarker) {
            LightParams& L = *light[static_cast<std::size_t>(h.T - kLightMarker)];
            for (int i = 0; i < st->pe_count; ++i) L.ptrs[i] = st->live(i);
            launch_light_pass(L, L.tiles_per_pe * st->pe_count, st->stream, st->device, fused ? d_fs : nullptr);
            if (fused) {
                st->cur ^= 1;
                st->qr_pending = false;
                st->spare_busy = st->comm && st->comm->world > 1;
            }
            st->stats[QRT_K_GATES].launches++;
            st->stats[QRT_K_GATES].bytes += 32.0 * amps_all;
            continue;
        }
        if (h.T < 0 && (dev_ops[static_cast<std::size_t>(h.op_begin)].kind == kDiag ||
                        dev_ops[static_cast<std::size_t>(h.op_begin)].k <= kWideInPlaceK)) {  // wide, in place
            const GateOp& g = dev_ops[static_cast<std::size_t>(h.op_begin)];
            const int widx = -h.T - 1;
            static bool wattr[64] = {};
            if (!wattr[st->device]) {
                QRT_CUDA(cudaFuncSetAttribute(wide_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (1 << kWideInPlaceK) * static_cast<int>(sizeof(double2))));
                wattr[st->device] = true;
            }
            for (int i = 0; i < st->pe_count; ++i) {
                amp_t* live = st->live(i);
                if (g.kind == kDiag)
                    wide_diag_kernel<<<st->sm_count * 8, 256, 0, st->stream>>>(live, st->amps, d_pool + g.gmat, g.k,
                                                                              d_wpos + widx);
                else
                    wide_group_kernel<<<st->sm_count * 4, 256, (std::size_t{1} << g.k) * sizeof(double2), st->stream>>>(
                        live, st->amps, d_pool + g.gmat, g.k, d_wpos + widx);
                QRT_CUDA(cudaGetLastError());
            }
            st->stats[QRT_K_GATES].launches += static_cast<std::uint64_t>(st->pe_count);
            st->stats[QRT_K_GATES].bytes += 32.0 * amps_all;
            continue;
        }
        if (h.T < 0) {  // wider than kWideInPlaceK: out of place into the alternate buffer, then copied back
            if (st->inplace) fail(QRT_ERR_OOM, "dense gate wider than 12 qubits needs a second state buffer");
            ensure_alt(st);
            if (st->spare_busy) {  // peers may still pull our old live buffer (now the spare)
                barrier_on_stream(st);
                st->spare_busy = false;
            }
            const GateOp& g = dev_ops[static_cast<std::size_t>(h.op_begin)];
            const int widx = -h.T - 1;
            for (int i = 0; i < st->pe_count; ++i) {
                amp_t* src = st->bufs[st->cur][static_cast<std::size_t>(i)];
                amp_t* dst = st->bufs[st->cur ^ 1][static_cast<std::size_t>(i)];
                wide_gate_kernel<<<st->sm_count * 8, 256, 0, st->stream>>>(src, dst, st->amps, d_pool + g.gmat, g.k,
                                                                  g.kind == kDiag, d_wpos + widx);
                QRT_CUDA(cudaGetLastError());
                QRT_CUDA(cudaMemcpyAsync(src, dst, st->amps * sizeof(amp_t), cudaMemcpyDeviceToDevice, st->stream));
            }
            st->stats[QRT_K_GATES].launches += static_cast<std::uint64_t>(st->pe_count);
            st->stats[QRT_K_GATES].bytes += 64.0 * amps_all;
            continue;
        }
        for (int i = 0; i < st->pe_count; ++i) params.ptrs.p[i] = st->live(i);
        params.hdr = h;
        std::copy(dev_ops.begin() + h.op_begin, dev_ops.begin() + h.op_begin + h.n_ops, params.ops);
        std::copy(pmats[pi].begin(), pmats[pi].end(), params.mats);
        const int tiles = 1 << (st->nl - h.T);
        const int total_tiles = tiles * st->pe_count;
        const std::size_t nt = static_cast<std::size_t>(1) << (h.T - h.c);
        const std::size_t smem = (static_cast<std::size_t>(1) << h.T) * sizeof(double2) +
                                 static_cast<std::size_t>(h.mat_count) * sizeof(double2) +
                                 (nt + (fused ? kFusedSmemWords + nt : 0)) * sizeof(std::uint64_t);
        auto kern = fused ? (gate_minb() == 4 ? gate_pass_kernel<true, 4> : gate_pass_kernel<true, 3>)
                          : (gate_minb() == 4 ? gate_pass_kernel<false, 4> : gate_pass_kernel<false, 3>);
        kern<<<total_tiles, gate_threads(), smem, st->stream>>>(params, d_pool, d_frags, tiles, fused ? d_fs : nullptr);
        QRT_CUDA(cudaGetLastError());
        if (fused) {
            st->cur ^= 1;
            st->qr_pending = false;
            st->spare_busy = st->comm && st->comm->world > 1;
        }
        st->stats[QRT_K_GATES].launches++;
        st->stats[QRT_K_GATES].bytes += 32.0 * amps_all;
    }
}

void gate_plan_info(int nl, int n_gates, const int* arity, const int* pos, const double* mats, const unsigned* flags,
                    int* passes, int* light_passes, int* light_stages, int* fused) {
    if (nl < 1 || nl > 62) fail(QRT_ERR_INVALID, "n_local out of range");
    GatePlan plan = plan_gates(nl, n_gates, arity, pos, mats, flags);
    int lp = 0, ls = 0;
    for (const auto& L : plan.light) {
        ++lp;
        ls += L->n_stages;
    }
    if (passes) *passes = static_cast<int>(plan.hdrs.size());
    if (light_passes) *light_passes = lp;
    if (light_stages) *light_stages = ls;
    if (fused) *fused = plan.fused;
}

}  // namespace qrt
