// libqrt — expectation value computation for one EVC plan tile
// (reference local_pauli_expectation + expectation, dist_sim.cpp:84-97 and
// :289-298) and the state norm (:115-120).
//
// Terms are batched by their X|Y flip mask x.  For x != 0 the pair (i, i^x)
// contributes  s_t(i) [w + (-1)^{#Y} conj(w)],  w = conj(v[i^x]) v[i],
// s_t(i) = (-1)^{popc(i & (z|y))}, so only the canonical half of the pairs is
// visited and only Re(w) or Im(w) is needed: the X/Y flip and the Z/Y phase
// are applied in registers.  Within a group the sign masks differ in only a
// few bits D (for Jordan-Wigner words: the Y letters), so
//   sum_t F_t s_t(i) val_t(i) = (-1)^{popc(i & m0)} (C_re[k] Re w + C_im[k] Im w),
//   k = the bits of i at D,
// with a 2^|D|-entry coefficient table built once per group per CTA: the
// per-pair cost no longer grows with the number of terms.  Terms with x = 0
// (I/Z words) are read off a Walsh-Hadamard transform of |v|^2 over the
// tile, O(1) per term per CTA.
//
// A pass loads a 2^12-amplitude tile (positions B chosen so the flip masks of
// many groups lie inside B) into shared memory once (cp.async) and evaluates
// every group it covers.  Per-CTA partial sums are reduced in a fixed order
// (warp shuffle -> block -> deterministic tree per PE), so results are
// run-to-run identical.  Algorithmic traffic per pass = 16 B x 2^(n-g) read.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <queue>
#include <unordered_map>
#include <unordered_set>
#include <deque>
#include <memory>
#include <mutex>

#include "qrt_coset.h"

namespace qrt {

namespace {

constexpr int kMaxDiffBits = 5;  // coefficient table of <= 32 entries per group

struct PePtrsP {
    const amp_t* p[kMaxLocalPEs];
};

struct PTerm {
    std::uint64_t m;   // sign mask bits outside the tile (outer parity per CTA); full mask for I/Z words
    std::uint64_t gz;  // PE-index sign mask
    double2 f;         // folded coefficient (x2 and i^#Y for flip terms)
    int dk;            // sign-mask difference to the group's m0, in table-index bits
    int comp;          // 0: Re(w), 1: Im(w)
    int m_tile;        // I/Z words: sign mask in tile-bit indices
    int pad;
};

struct PGroup {
    int xy_tile;  // flip mask in tile-bit indices
    int hbit;     // canonical bit (top bit of xy_tile)
    int t_begin, t_count;
    int m0_tile;  // common sign mask (first term), tile-bit indices
    int nd;       // |D|
    int dpos[kMaxDiffBits];
    int need;     // bit 0: some term reads Re(w), bit 1: some term reads Im(w)
    int real;     // every coefficient of the group is real (imaginary part exactly 0)
};

struct PPass {
    int T, c, n_outer;
    int tile_pos[kTileBits];
    int outer_pos[64];
    int g_begin, g_count;
    int d_begin, d_count;
    int pe_begin;
};

__device__ __forceinline__ int insert_zero(int v, int bit) {
    return ((v >> bit) << (bit + 1)) | (v & ((1 << bit) - 1));
}
__device__ __forceinline__ double flip_if(double v, int odd) { return odd ? -v : v; }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
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

// The pair loop of one group; NEED selects Re(w) / Im(w) / both at compile time.
template <int NEED>
__device__ __forceinline__ double2 group_pairs(const double2* __restrict__ tile, const PGroup& G,
                                               const double4* __restrict__ tbl, int half, int lane) {
    double2 acc = make_double2(0.0, 0.0);
    const int X = G.xy_tile, h = G.hbit, m0 = G.m0_tile, nd = G.nd;
    int dpos[kMaxDiffBits];
#pragma unroll
    for (int i = 0; i < kMaxDiffBits; ++i) dpos[i] = G.dpos[i];
    for (int idx = lane; idx < half; idx += 32) {
        const int e = insert_zero(idx, h);
        const double2 a = tile[e ^ X];
        const double2 b = tile[e];
        int k = 0;
#pragma unroll
        for (int i = 0; i < kMaxDiffBits; ++i)
            if (i < nd) k |= ((e >> dpos[i]) & 1) << i;
        const double4 cf = tbl[k];  // (C_re.x, C_re.y, C_im.x, C_im.y)
        const int odd = __popc(e & m0) & 1;
        if (NEED & 1) {
            const double re = flip_if(fma(a.x, b.x, a.y * b.y), odd);
            acc.x = fma(cf.x, re, acc.x);
            acc.y = fma(cf.y, re, acc.y);
        }
        if (NEED & 2) {
            const double im = flip_if(fma(a.x, b.y, -a.y * b.x), odd);
            acc.x = fma(cf.z, im, acc.x);
            acc.y = fma(cf.w, im, acc.y);
        }
    }
    return acc;
}

// Fast path when the canonical bit h >= 5: the low five tile bits of the
// canonical element are the lane id, everything else depends only on the
// (warp-uniform) iteration index, so signs, table index bits and addresses
// split into a per-lane constant and a uniform part computed once per step.
template <int NEED, int ND, bool REAL>
__device__ __forceinline__ double2 group_pairs_lane(const double2* __restrict__ tile, const PGroup& G,
                                                    const double4* __restrict__ tbl, int half, int lane) {
    double acx[4] = {0.0, 0.0, 0.0, 0.0}, acy[4] = {0.0, 0.0, 0.0, 0.0};
    const int X = G.xy_tile, h = G.hbit, m0 = G.m0_tile;
    const int E = half << 1;
    // table-index bits split into lane bits (tile bits < 5) and uniform bits
    int lane_k = 0, DH = 0;
#pragma unroll
    for (int i = 0; i < ND; ++i) {
        const int b = G.dpos[i];
        if (b < 5)
            lane_k |= ((lane >> b) & 1) << i;
        else
            DH |= 1 << b;
    }
    const int lane_par = __popc(lane & m0) & 1;
    const double2* __restrict__ tb = tile + lane;
    const double2* __restrict__ ta = tile + (lane ^ (X & 31));
    const int Xhi = X & ~31;
    const int free = ((E - 1) & ~31) & ~(1 << h) & ~DH;  // enumerated uniformly
    int s = 0;
    do {  // each pattern of the uniform table-index bits
        int k = lane_k;
#pragma unroll
        for (int i = 0; i < ND; ++i) {
            const int b = G.dpos[i];
            if (b >= 5) k |= ((s >> b) & 1) << i;
        }
        const double4 cf = tbl[k];
        // all uniform parts with that pattern (ascending submasks of `free`),
        // four at a time into independent accumulators
        auto pair_val = [&](int ehi, double& re_out, double& im_out) {
            const int odd = lane_par ^ (__popc(ehi & m0) & 1);
            const double2 b = tb[ehi];
            const double2 a = ta[ehi ^ Xhi];
            if (NEED & 1) re_out = flip_if(fma(a.x, b.x, a.y * b.y), odd);
            if (NEED & 2) im_out = flip_if(fma(a.x, b.y, -a.y * b.x), odd);
        };
        int f = 0;
        if (__popc(free) >= 2) {
            do {
                const int f1 = (f - free) & free, f2 = (f1 - free) & free, f3 = (f2 - free) & free;
                double r[4] = {0.0, 0.0, 0.0, 0.0}, q[4] = {0.0, 0.0, 0.0, 0.0};
                pair_val(s | f, r[0], q[0]);
                pair_val(s | f1, r[1], q[1]);
                pair_val(s | f2, r[2], q[2]);
                pair_val(s | f3, r[3], q[3]);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (NEED & 1) {
                        acx[u] = fma(cf.x, r[u], acx[u]);
                        if (!REAL) acy[u] = fma(cf.y, r[u], acy[u]);
                    }
                    if (NEED & 2) {
                        acx[u] = fma(cf.z, q[u], acx[u]);
                        if (!REAL) acy[u] = fma(cf.w, q[u], acy[u]);
                    }
                }
                f = (f3 - free) & free;
            } while (f != 0);
        } else {
            do {
                double r = 0.0, q = 0.0;
                pair_val(s | f, r, q);
                if (NEED & 1) {
                    acx[0] = fma(cf.x, r, acx[0]);
                    if (!REAL) acy[0] = fma(cf.y, r, acy[0]);
                }
                if (NEED & 2) {
                    acx[0] = fma(cf.z, q, acx[0]);
                    if (!REAL) acy[0] = fma(cf.w, q, acy[0]);
                }
                f = (f - free) & free;
            } while (f != 0);
        }
        s = (s - DH) & DH;
    } while (s != 0);
    return make_double2((acx[0] + acx[1]) + (acx[2] + acx[3]), (acy[0] + acy[1]) + (acy[2] + acy[3]));
}

template <int NEED, bool REAL>
__device__ __forceinline__ double2 group_pairs_nd(const double2* __restrict__ tile, const PGroup& G,
                                                  const double4* __restrict__ tbl, int half, int lane) {
    switch (G.nd) {
        case 0: return group_pairs_lane<NEED, 0, REAL>(tile, G, tbl, half, lane);
        case 1: return group_pairs_lane<NEED, 1, REAL>(tile, G, tbl, half, lane);
        case 2: return group_pairs_lane<NEED, 2, REAL>(tile, G, tbl, half, lane);
        case 3: return group_pairs_lane<NEED, 3, REAL>(tile, G, tbl, half, lane);
        case 4: return group_pairs_lane<NEED, 4, REAL>(tile, G, tbl, half, lane);
        default: return group_pairs<NEED>(tile, G, tbl, half, lane);
    }
}

__global__ void __launch_bounds__(kThreads, 2)
    pauli_pass_kernel(PePtrsP ptrs, const PPass P, const PGroup* __restrict__ groups, const PTerm* __restrict__ terms,
                      double* __restrict__ red) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double2 scratch[kThreads / 32];
    __shared__ double4 tables[kThreads / 32][1 << kMaxDiffBits];
    const int T = P.T, E = 1 << T, c = P.c;
    double2* tile = reinterpret_cast<double2*>(smem_raw);
    std::uint64_t* tab = reinterpret_cast<std::uint64_t*>(tile + E);
    double* W = reinterpret_cast<double*>(tab + (1 << (T - c)));

    std::uint64_t base = 0;
    for (int i = 0; i < P.n_outer; ++i) base |= ((static_cast<std::uint64_t>(blockIdx.x) >> i) & 1ull) << P.outer_pos[i];
    for (int h = threadIdx.x; h < (1 << (T - c)); h += blockDim.x) {
        std::uint64_t o = 0;
        for (int i = c; i < T; ++i) o |= static_cast<std::uint64_t>((h >> (i - c)) & 1) << P.tile_pos[i];
        tab[h] = o;
    }
    __syncthreads();
    const amp_t* __restrict__ v = ptrs.p[blockIdx.y];
    const std::uint64_t pe = static_cast<std::uint64_t>(P.pe_begin) + blockIdx.y;
    const int cmask = (1 << c) - 1;
    for (int e = threadIdx.x; e < E; e += blockDim.x) cp_async16(&tile[e], &v[base | tab[e >> c] | (e & cmask)]);
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();

    double2 acc = make_double2(0.0, 0.0);
    if (P.d_count > 0) {  // I/Z words: WHT of |v|^2 over the tile
        for (int e = threadIdx.x; e < E; e += blockDim.x) {
            const double2 a = tile[e];
            W[e] = fma(a.x, a.x, a.y * a.y);
        }
        __syncthreads();
        for (int s = 0; s < T; ++s) {
            for (int i = threadIdx.x; i < (E >> 1); i += blockDim.x) {
                const int i0 = insert_zero(i, s), i1 = i0 | (1 << s);
                const double a = W[i0], b = W[i1];
                W[i0] = a + b;
                W[i1] = a - b;
            }
            __syncthreads();
        }
        for (int t = threadIdx.x; t < P.d_count; t += blockDim.x) {
            const PTerm tm = terms[P.d_begin + t];
            const int odd = (__popcll(base & tm.m) + __popcll(pe & tm.gz)) & 1;
            const double val = flip_if(W[tm.m_tile], odd);
            acc.x = fma(tm.f.x, val, acc.x);
            acc.y = fma(tm.f.y, val, acc.y);
        }
    }

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int half = E >> 1;
    double4* tbl = tables[warp];
    for (int gi = warp; gi < P.g_count; gi += nwarps) {
        const PGroup G = groups[P.g_begin + gi];
        // coefficient table: entry k = sum_t F_t (-1)^{outer_t + pe_t + popc(k & dk_t)}
        if (lane < (1 << G.nd)) {
            double4 e4 = make_double4(0.0, 0.0, 0.0, 0.0);
            for (int t = 0; t < G.t_count; ++t) {
                const PTerm tm = terms[G.t_begin + t];
                const int odd = (__popcll(base & tm.m) + __popcll(pe & tm.gz) + __popc(lane & tm.dk)) & 1;
                const double fx = flip_if(tm.f.x, odd), fy = flip_if(tm.f.y, odd);
                if (tm.comp) {
                    e4.z += fx;
                    e4.w += fy;
                } else {
                    e4.x += fx;
                    e4.y += fy;
                }
            }
            tbl[lane] = e4;
        }
        __syncwarp();
        double2 g;
        if (G.hbit < 5 || half < 32) {
            switch (G.need) {
                case 1: g = group_pairs<1>(tile, G, tbl, half, lane); break;
                case 2: g = group_pairs<2>(tile, G, tbl, half, lane); break;
                default: g = group_pairs<3>(tile, G, tbl, half, lane); break;
            }
        } else if (G.real) {
            switch (G.need) {
                case 1: g = group_pairs_nd<1, true>(tile, G, tbl, half, lane); break;
                case 2: g = group_pairs_nd<2, true>(tile, G, tbl, half, lane); break;
                default: g = group_pairs_nd<3, true>(tile, G, tbl, half, lane); break;
            }
        } else {
            switch (G.need) {
                case 1: g = group_pairs_nd<1, false>(tile, G, tbl, half, lane); break;
                case 2: g = group_pairs_nd<2, false>(tile, G, tbl, half, lane); break;
                default: g = group_pairs_nd<3, false>(tile, G, tbl, half, lane); break;
            }
        }
        acc.x += g.x;
        acc.y += g.y;
        __syncwarp();
    }
    const double2 tot = block_sum(acc, scratch);
    if (threadIdx.x == 0) {
        double* slot = red + 2 * (static_cast<std::size_t>(blockIdx.y) * gridDim.x + blockIdx.x);
        slot[0] += tot.x;
        slot[1] += tot.y;
    }
}

// Flip masks too wide for a shared-memory tile: the canonical pairs are read
// straight from HBM (both partners), one group per grid-stride sweep.  Used
// for generic Pauli words (e.g. uniformly random strings); Jordan-Wigner
// words always take the tiled kernel above.
struct WGroup {
    std::uint64_t x;      // flip mask, local positions
    int hbit;             // canonical bit
    int t_begin, t_count;
};

__global__ void __launch_bounds__(256) pauli_wide_kernel(PePtrsP ptrs, int nl, int pe_begin, const WGroup* __restrict__ groups,
                                                         int n_groups, const PTerm* __restrict__ terms,
                                                         double* __restrict__ red) {
    __shared__ double2 scratch[8];
    const amp_t* __restrict__ v = ptrs.p[blockIdx.y];
    const std::uint64_t pe = static_cast<std::uint64_t>(pe_begin) + blockIdx.y;
    const std::uint64_t half = 1ull << (nl - 1);
    double2 acc = make_double2(0.0, 0.0);
    for (int gi = 0; gi < n_groups; ++gi) {
        const WGroup G = groups[gi];
        for (std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; idx < half;
             idx += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
            const std::uint64_t e = ((idx >> G.hbit) << (G.hbit + 1)) | (idx & ((1ull << G.hbit) - 1));
            const double2 a = v[e ^ G.x];
            const double2 b = v[e];
            const double re = fma(a.x, b.x, a.y * b.y);
            const double im = fma(a.x, b.y, -a.y * b.x);
            for (int t = 0; t < G.t_count; ++t) {
                const PTerm tm = terms[G.t_begin + t];
                const int odd = (__popcll(e & tm.m) + __popcll(pe & tm.gz)) & 1;
                const double val = flip_if(tm.comp ? im : re, odd);
                acc.x = fma(tm.f.x, val, acc.x);
                acc.y = fma(tm.f.y, val, acc.y);
            }
        }
    }
    const double2 tot = block_sum(acc, scratch);
    if (threadIdx.x == 0) {
        double* slot = red + 2 * (static_cast<std::size_t>(blockIdx.y) * gridDim.x + blockIdx.x);
        slot[0] += tot.x;
        slot[1] += tot.y;
    }
}

// Deterministic per-PE reduction of `count` slots of (re, im).
__global__ void __launch_bounds__(256) reduce_slots_kernel(const double* __restrict__ red, int count, double* out) {
    __shared__ double2 scratch[8];
    const double* r = red + 2 * static_cast<std::size_t>(blockIdx.x) * count;
    double2 acc = make_double2(0.0, 0.0);
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        acc.x += r[2 * i];
        acc.y += r[2 * i + 1];
    }
    const double2 tot = block_sum(acc, scratch);
    if (threadIdx.x == 0) {
        out[2 * blockIdx.x] = tot.x;
        out[2 * blockIdx.x + 1] = tot.y;
    }
}

__global__ void __launch_bounds__(256) norm_kernel(const amp_t* __restrict__ v, std::uint64_t amps, double* red) {
    __shared__ double2 scratch[8];
    double2 acc = make_double2(0.0, 0.0);
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < amps;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        const double2 a = __ldcs(&v[i]);
        acc.x = fma(a.x, a.x, fma(a.y, a.y, acc.x));
    }
    const double2 tot = block_sum(acc, scratch);
    if (threadIdx.x == 0) {
        red[2 * blockIdx.x] = tot.x;
        red[2 * blockIdx.x + 1] = 0.0;
    }
}

int popc(std::uint64_t v) { return __builtin_popcountll(v); }

// Gathers `local` (2 doubles per owned PE) into `all` (2 doubles per PE).
// `d_local` sits in the reduction buffer, which callers size with 2·p
// further doubles behind it: the all-gather lands there, so no
// per-call stream-ordered allocation sits between the EVC kernels.
void gather_partials(qrt_state* st, const double* d_local, double* all) {
    const std::size_t per = 2 * static_cast<std::size_t>(st->pe_count);
    if (st->comm && st->comm->world > 1) {
        double* buf = const_cast<double*>(d_local) + per;
        QRT_NCCL(ncclAllGather(d_local, buf, per, ncclDouble, st->comm->nccl, st->stream));
        QRT_CUDA(cudaMemcpyAsync(all, buf, 2 * static_cast<std::size_t>(st->p) * sizeof(double), cudaMemcpyDeviceToHost,
                                 st->stream));
        QRT_CUDA(cudaStreamSynchronize(st->stream));
    } else {
        QRT_CUDA(cudaMemcpyAsync(all + 2 * static_cast<std::size_t>(st->pe_begin), d_local, per * sizeof(double),
                                 cudaMemcpyDeviceToHost, st->stream));
        QRT_CUDA(cudaStreamSynchronize(st->stream));
    }
}

int compress_bits(std::uint64_t m, const int* tile_pos, int T) {
    int r = 0;
    for (int i = 0; i < T; ++i) r |= static_cast<int>((m >> tile_pos[i]) & 1ull) << i;
    return r;
}

}  // namespace

struct PauliPlanHost {
    int T = 0;
    std::vector<PGroup> dgroups;
    std::vector<PTerm> dterms;
    std::vector<PPass> hdrs;  // tiled passes (shared-memory pair loop)
    std::vector<WGroup> wgroups;
    std::vector<std::unique_ptr<CosetParams>> cosets;  // register-coset passes
    std::vector<CosetDiagTerm> cdterms;
    int coset_sets = 0;
    int linear_passes = 0;  // coset launches on GF(2)-linear tiles (wide flip masks)
};

namespace {

bool coset_enabled() {
    const char* e = std::getenv("QRT_EVC_COSET");
    return e ? std::atoi(e) != 0 : true;
}

// Builds the register-coset launches of one tile pass (positions B; flip-mask
// groups `gidx` into `flips`, each with its terms; `diag` I/Z terms if any).
// Groups are covered greedily by 5-bit register sets Q; within a set each
// group is split by the sign bits its terms have outside Q (so that one
// thread sign serves all of them) and folded into a 16-entry table.
// sm[t]: the sign mask (Z|Y) of term t in the pass's coordinates; y only
// supplies Y counts.  cols (nullptr: unit vectors) maps each coordinate axis
// p to its index vector (linear passes, see CosetParams::tile_vec).
void build_coset_pass(PauliPlanHost& plan, int nl, int pe_begin, std::uint64_t B,
                      const std::vector<std::pair<std::uint64_t, std::vector<int>>>& flips, const std::vector<int>& gidx,
                      const std::vector<int>& diag, const std::uint64_t* y, const std::uint64_t* sm,
                      const std::uint64_t* gz, const double* coeffs, const std::vector<std::uint64_t>* qsets,
                      const std::uint64_t* cols = nullptr) {
    int tile_pos[kTileBits], outer_pos[64], tb_of[64], ob_of[64];
    int ti = 0, no = 0;
    for (int p = 0; p < 64; ++p) tb_of[p] = ob_of[p] = -1;
    for (int p = 0; p < nl; ++p) {
        if (B >> p & 1ull) {
            tb_of[p] = ti;
            tile_pos[ti++] = p;
        } else {
            ob_of[p] = no;
            outer_pos[no++] = p;
        }
    }
    int c = 0;  // leading tile axes that are the unit positions 0..c-1 (addressed directly)
    while (c < kTileBits && tile_pos[c] == c && (!cols || cols[c] == (1ull << c))) ++c;
    auto to_tile = [&](std::uint64_t m) {
        int r = 0;
        for (int i = 0; i < kTileBits; ++i) r |= static_cast<int>((m >> tile_pos[i]) & 1ull) << i;
        return r;
    };
    auto fresh = [&]() {
        auto P = std::make_unique<CosetParams>();
        std::memset(P.get(), 0, sizeof(CosetParams));
        P->c = c;
        P->n_outer = no;
        P->pe_begin = pe_begin;
        P->tiles_per_pe = 1 << (nl - kTileBits);
        for (int i = 0; i < kTileBits; ++i) P->tile_vec[i] = cols ? cols[tile_pos[i]] : 1ull << tile_pos[i];
        for (int i = 0; i < no; ++i) P->outer_vec[i] = cols ? cols[outer_pos[i]] : 1ull << outer_pos[i];
        return P;
    };
    auto P = fresh();
    int n_groups = 0, n_tab = 0;
    if (!diag.empty()) {
        P->d_begin = static_cast<int>(plan.cdterms.size());
        P->d_count = static_cast<int>(diag.size());
        for (int t : diag) {
            CosetDiagTerm tm{};
            tm.m = sm[t];
            tm.gz = gz[t];
            tm.f = make_double2(coeffs[2 * t], coeffs[2 * t + 1]);
            tm.m_tile = to_tile(tm.m & B);
            plan.cdterms.push_back(tm);
        }
    }
    // tile-bit flip masks of the groups
    std::vector<int> left = gidx;
    std::vector<int> xt(flips.size(), 0);
    for (int g : gidx) xt[static_cast<std::size_t>(g)] = to_tile(flips[static_cast<std::size_t>(g)].first);
    std::stable_sort(left.begin(), left.end(), [&](int a, int b) {
        return __builtin_popcount(static_cast<unsigned>(xt[static_cast<std::size_t>(a)])) >
               __builtin_popcount(static_cast<unsigned>(xt[static_cast<std::size_t>(b)]));
    });
    std::size_t next_fixed = 0;
    while (!left.empty()) {
        // ---- choose Q: 5 tile bits covering most remaining groups (or the
        // next set of the global cover, padded to 5 tile bits)
        int bestQ = 0, best = -1;
        if (qsets && next_fixed < qsets->size()) {
            bestQ = to_tile((*qsets)[next_fixed++]);
            for (int b = kTileBits - 1; b >= 0 && __builtin_popcount(static_cast<unsigned>(bestQ)) < kCosetBits; --b)
                bestQ |= 1 << b;
            best = 0;
        }
        const std::size_t seeds = best >= 0 ? 0 : std::min<std::size_t>(12, left.size());
        for (std::size_t sd = 0; sd < seeds; ++sd) {
            const int x = xt[static_cast<std::size_t>(left[sd])];
            const int need = kCosetBits - __builtin_popcount(static_cast<unsigned>(x));
            std::vector<int> free;
            for (int b = 0; b < kTileBits; ++b)
                if (!(x >> b & 1)) free.push_back(b);
            // all ways to add `need` bits (<= C(11,4) = 330)
            std::vector<int> pick(static_cast<std::size_t>(need));
            for (int i = 0; i < need; ++i) pick[static_cast<std::size_t>(i)] = i;
            const int F = static_cast<int>(free.size());
            while (true) {
                int Q = x;
                for (int i = 0; i < need; ++i) Q |= 1 << free[static_cast<std::size_t>(pick[static_cast<std::size_t>(i)])];
                int cnt = 0;
                for (int g : left) cnt += (xt[static_cast<std::size_t>(g)] & ~Q) == 0;
                if (cnt > best) {
                    best = cnt;
                    bestQ = Q;
                }
                int i = need - 1;
                while (i >= 0 && pick[static_cast<std::size_t>(i)] == F - need + i) --i;
                if (i < 0) break;
                ++pick[static_cast<std::size_t>(i)];
                for (int j = i + 1; j < need; ++j) pick[static_cast<std::size_t>(j)] = pick[static_cast<std::size_t>(j - 1)] + 1;
            }
        }
        std::vector<int> in, keep;
        for (int g : left) ((xt[static_cast<std::size_t>(g)] & ~bestQ) == 0 ? in : keep).push_back(g);
        left.swap(keep);
        if (in.empty()) continue;
        // ---- the set: register bits, thread bits (conflict-free lanes)
        CosetSet S{};
        int reg_of[kTileBits];
        {
            int q = 0;
            for (int i = 0; i < kTileBits; ++i) {
                reg_of[i] = -1;
                if (bestQ >> i & 1) {
                    S.S[q] = static_cast<std::int8_t>(i);
                    reg_of[i] = q++;
                }
            }
            std::vector<int> rest, lead;
            for (int i = 0; i < kTileBits; ++i)
                if (!(bestQ >> i & 1)) rest.push_back(i);
            for (int res = 0; res < 3; ++res)
                for (std::size_t u = 0; u < rest.size(); ++u)
                    if (rest[u] % 3 == res) {
                        lead.push_back(rest[u]);
                        rest.erase(rest.begin() + static_cast<std::ptrdiff_t>(u));
                        break;
                    }
            rest.insert(rest.begin(), lead.begin(), lead.end());
            for (int i = 0; i < kTileBits - kCosetBits; ++i) S.tb[i] = static_cast<std::int8_t>(rest[static_cast<std::size_t>(i)]);
            coset_set_tables(S);
        }
        auto to_reg = [&](int tilemask) {
            int r = 0;
            for (int i = 0; i < kTileBits; ++i)
                if ((tilemask >> i & 1) && reg_of[i] >= 0) r |= 1 << reg_of[i];
            return r;
        };
        // W-bit mask of sign bits outside Q
        auto to_w = [&](std::uint64_t m) {
            std::uint64_t w = 0;
            for (int p = 0; p < nl; ++p) {
                if (!(m >> p & 1ull)) continue;
                if (tb_of[p] >= 0) {
                    if (!(bestQ >> tb_of[p] & 1)) w |= 1ull << tb_of[p];
                } else {
                    w |= 1ull << (kTileBits + ob_of[p]);
                }
            }
            return w;
        };
        // ---- groups of the set, sorted by register flip mask, split by outside signs
        struct Sub {
            int xq;
            std::uint64_t mf, gz;
            std::vector<int> terms;
        };
        std::vector<Sub> subs;
        for (int g : in) {
            const int xq = to_reg(xt[static_cast<std::size_t>(g)]);
            for (int t : flips[static_cast<std::size_t>(g)].second) {
                const std::uint64_t m = sm[t];
                const std::uint64_t mf = to_w(m);
                auto it = std::find_if(subs.begin(), subs.end(), [&](const Sub& u) {
                    return u.xq == xq && u.mf == mf && u.gz == gz[t];
                });
                if (it == subs.end()) {
                    subs.push_back(Sub{xq, mf, gz[t], {}});
                    it = subs.end() - 1;
                }
                it->terms.push_back(t);
            }
        }
        // fast subgroups (Re(w) only, real coefficients, weight-2/4 masks)
        // first, sorted by mask; the generic ones after them
        auto fast_of = [&](const Sub& u) {
            const int w = __builtin_popcount(static_cast<unsigned>(u.xq));
            if (w != 2 && w != 4) return false;
            for (int t : u.terms)
                if ((__builtin_popcountll(y[t]) & 1) || coeffs[2 * t + 1] != 0.0) return false;
            return true;
        };
        // then the single-bit masks (linear passes; any table mode, evaluated
        // from the register coset), sorted by mask; the generic ones last
        auto re_real_of = [&](const Sub& u) {
            for (int t : u.terms)
                if ((__builtin_popcountll(y[t]) & 1) || coeffs[2 * t + 1] != 0.0) return false;
            return true;
        };
        auto im_real_of = [&](const Sub& u) {  // Im(w) only (odd Y counts), real coefficients
            for (int t : u.terms)
                if (!(__builtin_popcountll(y[t]) & 1) || coeffs[2 * t + 1] != 0.0) return false;
            return true;
        };
        auto one_of = [&](const Sub& u) { return !fast_of(u) && __builtin_popcount(static_cast<unsigned>(u.xq)) == 1; };
        auto cls = [&](const Sub& u) { return fast_of(u) ? 0 : one_of(u) ? 1 : 2; };
        // single-bit groups of one mask: Re(w)-only real (mode 0) first, then
        // Im(w)-only real (mode 2), then general, so the kernel walks each
        // run with a fixed body
        auto one_mode = [&](const Sub& u) { return re_real_of(u) ? 0 : im_real_of(u) ? 1 : 2; };
        std::stable_sort(subs.begin(), subs.end(), [&](const Sub& a, const Sub& b) {
            const int ca = cls(a), cb = cls(b);
            if (ca != cb) return ca < cb;
            if (ca == 1 && a.xq == b.xq) return one_mode(a) < one_mode(b);
            return ca < 2 && a.xq < b.xq;
        });
        // emit in chunks that fit the launch parameters (a set whose
        // subgroups overflow one launch is repeated with the same Q)
        std::size_t at = 0;
        while (at < subs.size()) {
            auto room = [&](std::size_t from) {
                std::size_t end = from;
                int g = n_groups, tb = n_tab;
                while (end < subs.size() && end - from < 255) {
                    const int need =
                        (re_real_of(subs[end]) || (one_of(subs[end]) && im_real_of(subs[end]))) ? 16 : 64;
                    if (g + 1 > kCosetMaxGroups || tb + need > kCosetMaxTab) break;
                    ++g;
                    tb += need;
                    ++end;
                }
                return end;
            };
            std::size_t end = room(at);
            if (end == at || P->n_sets >= kCosetMaxSets) {
                plan.cosets.push_back(std::move(P));
                P = fresh();
                n_groups = n_tab = 0;
                end = room(at);
                if (end == at) fail(QRT_ERR_INVALID, "EVC coset group exceeds the launch budget");
            }
            CosetSet Sc = S;
            Sc.g_begin = static_cast<std::int16_t>(n_groups);
            Sc.g_count = static_cast<std::int16_t>(end - at);
            for (int xq = 0; xq < 32; ++xq) {
                int cnt = 0;
                for (std::size_t q = at; q < end; ++q) cnt += fast_of(subs[q]) && subs[q].xq <= xq;
                Sc.xbeg[xq] = static_cast<std::uint8_t>(cnt);  // fast subgroups with mask <= xq
            }
            Sc.present = 0;
            for (std::size_t q = at; q < end; ++q)
                if (fast_of(subs[q])) Sc.present |= 1u << subs[q].xq;
            for (int k = 0; k < kCosetBits; ++k) {
                int cnt = 0;
                for (std::size_t q = at; q < end; ++q) cnt += one_of(subs[q]) && subs[q].xq == (1 << k);
                Sc.one_cnt[k] = static_cast<std::uint8_t>(cnt);  // single-bit subgroups, after the fast ones
                int nre = 0, nim = 0;
                for (std::size_t q = at; q < end; ++q)
                    if (one_of(subs[q]) && subs[q].xq == (1 << k)) {
                        nre += one_mode(subs[q]) == 0;
                        nim += one_mode(subs[q]) == 1;
                    }
                Sc.one_re[k] = static_cast<std::uint8_t>(nre);
                Sc.one_im[k] = static_cast<std::uint8_t>(nim);
            }
            for (std::size_t q = at; q < end; ++q) {
                const Sub& u = subs[q];
                CosetGroup& G = P->groups[n_groups++];
                G.xq = static_cast<std::int8_t>(u.xq);
                if (nl > kCosetPeShift || (u.gz >> (64 - kCosetPeShift)) != 0)
                    fail(QRT_ERR_INVALID, "EVC sign masks exceed the folded layout");
                G.mf = u.mf | (u.gz << kCosetPeShift);
                G.gz = u.gz;
                G.tab = static_cast<std::int16_t>(n_tab);
                const bool re_real = re_real_of(u);
                const bool im_real = !re_real && one_of(u) && im_real_of(u);
                G.mode = re_real ? 0 : im_real ? 2 : 1;
                const int H = 31 - __builtin_clz(static_cast<unsigned>(u.xq));
                double* T = P->tabs + n_tab;
                const int tl = G.mode == 1 ? 64 : 16;
                n_tab += tl;
                for (int e = 0; e < tl; ++e) T[e] = 0.0;
                for (int t : u.terms) {
                    const int ycnt = __builtin_popcountll(y[t]);
                    const double sgn = ((ycnt & 3) == 1 || (ycnt & 3) == 2) ? -2.0 : 2.0;
                    const double fx = sgn * coeffs[2 * t], fy = sgn * coeffs[2 * t + 1];
                    const int mq = to_reg(to_tile((sm[t]) & B));
                    for (int rho = 0; rho < 16; ++rho) {
                        const int r = ((rho >> H) << (H + 1)) | (rho & ((1 << H) - 1));
                        const double sg = (__builtin_popcount(static_cast<unsigned>(r & mq)) & 1) ? -1.0 : 1.0;
                        if (re_real || im_real) {  // mode 0 weights Re(w), mode 2 Im(w), into the real part
                            T[rho] += sg * fx;
                        } else if (ycnt & 1) {
                            T[32 + rho] += sg * fx;
                            T[48 + rho] += sg * fy;
                        } else {
                            T[rho] += sg * fx;
                            T[16 + rho] += sg * fy;
                        }
                    }
                }
            }
            {  // one group per present fast mask: tables contiguous in mask order (fast groups first)
                int nfast = 0;
                for (std::size_t q = at; q < end; ++q) nfast += fast_of(subs[q]);
                Sc.tab1 = (nfast > 0 && nfast == __builtin_popcount(Sc.present))
                              ? P->groups[Sc.g_begin].tab
                              : static_cast<std::int16_t>(-1);
            }
            {  // linear-pass sets: at most one single-bit group per register bit and nothing else
                Sc.onemask = 0;
                Sc.onemode = 0;
                for (int k = 0; k < kCosetBits; ++k) Sc.onetab[k] = -1;
                bool ok = Sc.present == 0;
                for (int k = 0; k < kCosetBits; ++k) ok = ok && Sc.one_cnt[k] <= 1;
                int ng = 0;
                for (int k = 0; k < kCosetBits; ++k) ng += Sc.one_cnt[k];
                ok = ok && ng == Sc.g_count && ng > 0;
                if (ok) {
                    int g = Sc.g_begin;
                    for (int k = 0; k < kCosetBits; ++k)
                        if (Sc.one_cnt[k]) {
                            const CosetGroup& G = P->groups[g++];
                            Sc.onemask |= static_cast<std::uint8_t>(1u << k);
                            Sc.onetab[k] = G.tab;
                            Sc.onemode |= static_cast<std::uint16_t>((G.mode & 3) << (2 * k));
                        }
                }
            }
            P->sets[P->n_sets++] = Sc;
            P->n_tab = n_tab;
            ++plan.coset_sets;
            at = end;
        }
    }
    plan.cosets.push_back(std::move(P));
}

}  // namespace

namespace {

// Greedy cover of flip masks (weight <= 5) by sets of <= 5 positions, lazy
// evaluation: a candidate's score is the number of still-uncovered masks
// among its subsets.  Candidates: each mask united with an overlapping mask
// (weight <= 5) or, for weight-4 masks, with one neighbouring position.
// Returns the sets in pick order and, per set, the masks it took.
std::vector<std::pair<std::uint64_t, std::vector<std::uint64_t>>> cover_masks(const std::vector<std::uint64_t>& masks) {
    std::unordered_set<std::uint64_t> unc(masks.begin(), masks.end());
    auto score = [&](std::uint64_t Q) {
        int n = 0;
        for (std::uint64_t sub = Q; sub; sub = (sub - 1) & Q) n += unc.count(sub) ? 1 : 0;
        return n;
    };
    // neighbour positions of every mask: positions of overlapping masks
    std::unordered_map<int, std::vector<std::uint64_t>> by_bit;
    for (std::uint64_t m : masks)
        for (std::uint64_t r = m; r; r &= r - 1) by_bit[__builtin_ctzll(r)].push_back(m);
    std::unordered_set<std::uint64_t> cand;
    for (std::uint64_t g : masks) {
        cand.insert(g);
        std::uint64_t nb = 0;
        for (std::uint64_t r = g; r; r &= r - 1)
            for (std::uint64_t h : by_bit[__builtin_ctzll(r)]) {
                if (__builtin_popcountll(g | h) <= kCosetBits) cand.insert(g | h);
                nb |= h;
            }
        if (__builtin_popcountll(g) == kCosetBits - 1)
            for (std::uint64_t r = nb & ~g; r; r &= r - 1) cand.insert(g | (r & (~r + 1)));
    }
    std::priority_queue<std::pair<int, std::uint64_t>> heap;
    for (std::uint64_t Q : cand) heap.emplace(score(Q), Q);
    std::vector<std::pair<std::uint64_t, std::vector<std::uint64_t>>> out;
    while (!unc.empty() && !heap.empty()) {
        auto [sc, Q] = heap.top();
        heap.pop();
        const int now = score(Q);
        if (now == 0) continue;
        if (now < sc && !heap.empty() && now < heap.top().first) {
            heap.emplace(now, Q);
            continue;
        }
        std::vector<std::uint64_t> took;
        for (std::uint64_t sub = Q; sub; sub = (sub - 1) & Q)
            if (unc.erase(sub)) took.push_back(sub);
        out.emplace_back(Q, std::move(took));
    }
    for (std::uint64_t m : unc) out.emplace_back(m, std::vector<std::uint64_t>{m});  // not reached in practice
    return out;
}

}  // namespace

// Host planning of one EVC tile: flip-mask groups, tile passes, coefficient
// folding, and the wide (full-vector) groups.  No device access.
PauliPlanHost build_pauli_plan(int nl, int pe_begin, int n_terms, const std::uint64_t* x, const std::uint64_t* y,
                               const std::uint64_t* z, const std::uint64_t* gz, const double* coeffs) {
    const std::uint64_t local_mask = nl >= 64 ? ~0ull : ((1ull << nl) - 1);
    PauliPlanHost plan;
    auto& dgroups = plan.dgroups;
    auto& dterms = plan.dterms;
    auto& hdrs = plan.hdrs;
    auto& wgroups = plan.wgroups;
    // ---- group by flip mask -------------------------------------------------
    std::map<std::uint64_t, std::vector<int>> by_xy;
    for (int t = 0; t < n_terms; ++t) by_xy[x[t] | y[t]].push_back(t);
    const int T = std::min(kTileBits, nl);
    const int coal = std::min(kCoalBits, nl);
    const std::uint64_t coal_mask = (1ull << coal) - 1;
    std::vector<std::uint64_t> zy(static_cast<std::size_t>(n_terms));
    for (int t = 0; t < n_terms; ++t) zy[static_cast<std::size_t>(t)] = z[t] | y[t];
    std::vector<int> diag;
    std::vector<std::pair<std::uint64_t, std::vector<int>>> flips, wide;
    // wide flip masks (and, on linear passes, any mask too heavy for a
    // register coset) go to linear passes (GF(2) tile axes = the masks)
    // unless QRT_EVC_LINEAR=0
    const bool linear = coset_enabled() && nl >= kTileBits && T == kTileBits && [] {
        const char* e = std::getenv("QRT_EVC_LINEAR");
        return e ? std::atoi(e) != 0 : true;
    }();
    for (auto& kv : by_xy) {
        if (kv.first == 0)
            diag = kv.second;
        else if (popc(kv.first | coal_mask) > T || (linear && popc(kv.first) > kCosetBits))
            wide.emplace_back(kv.first, kv.second);
        else
            flips.emplace_back(kv.first, kv.second);
    }

    // ---- passes: tile positions covering many flip masks --------------------
    struct Pass {
        std::uint64_t B;
        std::vector<int> groups;  // indices into flips
        bool has_diag;
        std::vector<std::uint64_t> qsets;  // register sets of the global cover (coset passes)
    };
    std::vector<Pass> passes;
    bool global_cover = coset_enabled() && nl >= kTileBits && T == kTileBits && !flips.empty() &&
                        (wide.empty() || linear);
    {
        const char* e = std::getenv("QRT_EVC_GLOBAL_COVER");
        if (e && std::atoi(e) == 0) global_cover = false;
    }
    for (const auto& f : flips) global_cover = global_cover && popc(f.first) <= kCosetBits;
    if (global_cover) {
        // cover every flip mask by <= 5-position register sets, then pack the
        // sets into tile passes (B holds the coalescing positions + 8 more)
        std::vector<std::uint64_t> masks;
        std::unordered_map<std::uint64_t, int> idx;
        for (std::size_t i = 0; i < flips.size(); ++i) {
            masks.push_back(flips[i].first);
            idx[flips[i].first] = static_cast<int>(i);
        }
        auto sets = cover_masks(masks);
        std::vector<std::size_t> rem(sets.size());
        for (std::size_t i = 0; i < sets.size(); ++i) rem[i] = i;
        const std::uint64_t coal_bits = (1ull << coal) - 1;
        auto fill = [&](std::uint64_t b) {
            for (int p = 0; p < nl && popc(b) < T; ++p) b |= 1ull << p;
            return b;
        };
        bool first = true;
        while (!rem.empty()) {
            auto count = [&](std::uint64_t b) {
                int n = 0;
                for (std::size_t i : rem) n += (sets[i].first & ~b) == 0;
                return n;
            };
            std::uint64_t B = 0;
            int best = -1;
            for (std::size_t sd = 0; sd < std::min<std::size_t>(16, rem.size()); ++sd) {
                std::uint64_t b = coal_bits;
                for (std::size_t q = 0; q < rem.size(); ++q) {
                    const std::uint64_t m = sets[rem[(sd + q) % rem.size()]].first;
                    if (popc(b | m) <= T) b |= m;
                    if (popc(b) == T) break;
                }
                b = fill(b);
                const int got = count(b);
                if (got > best) {
                    best = got;
                    B = b;
                }
            }
            for (int w = coal; w + (T - coal) <= nl; ++w) {
                const std::uint64_t b = coal_bits | (((1ull << (T - coal)) - 1) << w);
                const int got = count(b);
                if (got > best) {
                    best = got;
                    B = b;
                }
            }
            Pass ps{B, {}, first && !diag.empty(), {}};
            first = false;
            std::vector<std::size_t> keep;
            for (std::size_t i : rem) {
                if (sets[i].first & ~B) {
                    keep.push_back(i);
                    continue;
                }
                ps.qsets.push_back(sets[i].first);
                for (std::uint64_t m : sets[i].second) ps.groups.push_back(idx[m]);
            }
            if (ps.qsets.empty()) fail(QRT_ERR_INVALID, "EVC set packing made no progress");
            passes.push_back(std::move(ps));
            rem.swap(keep);
        }
    }
    std::vector<int> left(global_cover ? 0 : flips.size());
    for (std::size_t i = 0; i < left.size(); ++i) left[i] = static_cast<int>(i);
    std::stable_sort(left.begin(), left.end(), [&](int a, int b) {
        return popc(flips[static_cast<std::size_t>(a)].first) > popc(flips[static_cast<std::size_t>(b)].first);
    });
    bool diag_done = diag.empty() || global_cover;
    while (!left.empty() || !diag_done) {
        std::uint64_t B = (1ull << coal) - 1;
        if (T == nl) {
            B = local_mask;
        } else {
            // candidates: greedy unions of flip masks seeded at each of the
            // first remaining groups, and windows of consecutive positions
            // above the coalescing bits (Jordan-Wigner masks are local in
            // qubit order); the one holding most remaining groups wins
            auto covered = [&](std::uint64_t b) {
                int n = 0;
                for (int gi : left) n += (flips[static_cast<std::size_t>(gi)].first & ~b) == 0;
                return n;
            };
            auto fill = [&](std::uint64_t b) {
                for (int p = 0; p < nl && popc(b) < T; ++p) b |= 1ull << p;
                return b;
            };
            int best = -1;
            const std::size_t seeds = std::min<std::size_t>(16, left.size());
            for (std::size_t sd = 0; sd < std::max<std::size_t>(seeds, 1); ++sd) {
                std::uint64_t b = (1ull << coal) - 1;
                for (std::size_t q = 0; q < left.size(); ++q) {
                    const std::uint64_t m = flips[static_cast<std::size_t>(left[(sd + q) % left.size()])].first;
                    if (popc(b | m) <= T) b |= m;
                    if (popc(b) == T) break;
                }
                b = fill(b);
                const int got = covered(b);
                if (got > best) {
                    best = got;
                    B = b;
                }
            }
            for (int w = coal; w + (T - coal) <= nl; ++w) {
                const std::uint64_t b = ((1ull << coal) - 1) | (((1ull << (T - coal)) - 1) << w);
                const int got = covered(b);
                if (got > best) {
                    best = got;
                    B = b;
                }
            }
        }
        Pass ps{B, {}, !diag_done};
        diag_done = true;
        std::vector<int> keep;
        for (int gi : left)
            ((flips[static_cast<std::size_t>(gi)].first & ~B) == 0 ? ps.groups : keep).push_back(gi);
        if (ps.groups.empty() && !ps.has_diag) fail(QRT_ERR_INVALID, "EVC planner made no progress");
        passes.push_back(std::move(ps));
        left.swap(keep);
    }

    // ---- device descriptors ---------------------------------------------------
    const bool coset_ok = coset_enabled() && nl >= kTileBits && T == kTileBits;
    for (const Pass& ps : passes) {
        bool coset = coset_ok;
        for (int gi : ps.groups)
            if (popc(flips[static_cast<std::size_t>(gi)].first) > kCosetBits) coset = false;
        if (coset) {
            build_coset_pass(plan, nl, pe_begin, ps.B, flips, ps.groups, ps.has_diag ? diag : std::vector<int>{}, y,
                             zy.data(), gz, coeffs, ps.qsets.empty() ? nullptr : &ps.qsets);
            continue;
        }
        PPass h{};
        h.T = T;
        h.pe_begin = pe_begin;
        int ti = 0, no = 0;
        for (int p = 0; p < nl; ++p) {
            if (ps.B >> p & 1ull)
                h.tile_pos[ti++] = p;
            else
                h.outer_pos[no++] = p;
        }
        h.n_outer = no;
        h.c = 0;
        while (h.c < T && h.tile_pos[h.c] == h.c) ++h.c;
        h.d_begin = static_cast<int>(dterms.size());
        h.d_count = 0;
        if (ps.has_diag) {
            for (int t : diag) {
                PTerm tm{};
                tm.m = z[t] | y[t];
                tm.gz = gz[t];
                tm.f = make_double2(coeffs[2 * t], coeffs[2 * t + 1]);
                tm.m_tile = compress_bits(tm.m & ps.B, h.tile_pos, T);
                dterms.push_back(tm);
            }
            h.d_count = static_cast<int>(diag.size());
        }
        h.g_begin = static_cast<int>(dgroups.size());
        for (int gi : ps.groups) {
            const auto& [xy, members] = flips[static_cast<std::size_t>(gi)];
            // chunks whose sign masks differ from the first in <= kMaxDiffBits tile bits
            std::size_t at = 0;
            while (at < members.size()) {
                const int t0 = members[at];
                const int xt = compress_bits(xy, h.tile_pos, T);
                // the canonical bit (top bit of the flip mask) is 0 in every visited
                // element, so sign-mask bits there never matter: drop them
                const int hmask = 1 << (31 - __builtin_clz(static_cast<unsigned>(xt)));
                const int m0 = compress_bits((z[t0] | y[t0]) & ps.B, h.tile_pos, T) & ~hmask;
                int D = 0;
                std::size_t end = at;
                while (end < members.size()) {
                    const int t = members[end];
                    const int d = (compress_bits((z[t] | y[t]) & ps.B, h.tile_pos, T) & ~hmask) ^ m0;
                    if (popc(static_cast<std::uint64_t>(D | d)) > kMaxDiffBits) break;
                    D |= d;
                    ++end;
                }
                PGroup G{};
                G.xy_tile = compress_bits(xy, h.tile_pos, T);
                G.hbit = 31 - __builtin_clz(static_cast<unsigned>(G.xy_tile));
                G.m0_tile = m0;
                G.nd = 0;
                for (int b = 0; b < T; ++b)
                    if (D >> b & 1) G.dpos[G.nd++] = b;
                G.t_begin = static_cast<int>(dterms.size());
                G.t_count = static_cast<int>(end - at);
                G.need = 0;
                G.real = 1;
                for (std::size_t q = at; q < end; ++q) {
                    const int t = members[q];
                    const int ycnt = popc(y[t]);
                    const double sgn = ((ycnt & 3) == 1 || (ycnt & 3) == 2) ? -2.0 : 2.0;
                    PTerm tm{};
                    tm.m = (z[t] | y[t]) & ~ps.B;  // outer parity: bits outside the tile only
                    tm.gz = gz[t];
                    tm.f = make_double2(sgn * coeffs[2 * t], sgn * coeffs[2 * t + 1]);
                    const int d = (compress_bits((z[t] | y[t]) & ps.B, h.tile_pos, T) & ~hmask) ^ m0;
                    int dk = 0;
                    for (int i = 0; i < G.nd; ++i) dk |= ((d >> G.dpos[i]) & 1) << i;
                    tm.dk = dk;
                    tm.comp = ycnt & 1;
                    G.need |= tm.comp ? 2 : 1;
                    if (coeffs[2 * t + 1] != 0.0) G.real = 0;
                    dterms.push_back(tm);
                }
                dgroups.push_back(G);
                at = end;
            }
        }
        h.g_count = static_cast<int>(dgroups.size()) - h.g_begin;
        hdrs.push_back(h);
    }
    // wide flip masks, linear passes: batches of up to T - coal groups whose
    // masks are independent above the coalescing bits.  In the pass's
    // coordinates i' (i = A^-1 i', column p of A^-1 = cols[p]) the k-th mask
    // is the unit vector of its pivot position piv_k (cols[piv_k] = the mask),
    // the other axes stay unit vectors, and a sign mask m becomes
    // m'_p = parity(cols[p] & m).  One HBM read of the state then serves the
    // whole batch instead of one read per group.
    if (linear && !wide.empty()) {
        std::vector<std::size_t> pending(wide.size());
        for (std::size_t i = 0; i < wide.size(); ++i) pending[i] = i;
        // unit low positions of a linear tile: 2 (64-byte runs; 10 groups per
        // pass, measured faster than 4 positions / 256-byte runs with 8 groups:
        // the passes are compute-bound).  QRT_EVC_LINEAR_COAL overrides (0..4:
        // every unit axis given up is one more group per HBM read).
        const int lcoal = [&] {
            const char* e = std::getenv("QRT_EVC_LINEAR_COAL");
            return std::max(0, std::min(coal, e ? std::atoi(e) : 2));
        }();
        const std::uint64_t coal_m = (1ull << lcoal) - 1;
        std::vector<std::uint64_t> smL(static_cast<std::size_t>(n_terms), 0);
        while (!pending.empty()) {
            std::vector<std::uint64_t> basis;
            std::vector<int> piv;
            std::vector<std::size_t> batch, rest;
            for (std::size_t w : pending) {
                if (static_cast<int>(batch.size()) == T - lcoal) {
                    rest.push_back(w);
                    continue;
                }
                std::uint64_t v = wide[w].first & ~coal_m;
                for (std::size_t k = 0; k < basis.size(); ++k)
                    if (v >> piv[k] & 1ull) v ^= basis[k];
                if (!v) {
                    rest.push_back(w);
                    continue;
                }
                basis.push_back(v);
                piv.push_back(63 - __builtin_clzll(v));
                batch.push_back(w);
            }
            std::uint64_t cols[64];
            for (int p = 0; p < 64; ++p) cols[p] = 1ull << p;
            std::uint64_t B = coal_m;
            for (std::size_t k = 0; k < batch.size(); ++k) {
                cols[piv[k]] = wide[batch[k]].first;
                B |= 1ull << piv[k];
            }
            for (int p = lcoal; p < nl && popc(B) < T; ++p) B |= 1ull << p;
            std::vector<std::pair<std::uint64_t, std::vector<int>>> fl;
            std::vector<int> gi;
            for (std::size_t k = 0; k < batch.size(); ++k) {
                fl.emplace_back(1ull << piv[k], wide[batch[k]].second);
                gi.push_back(static_cast<int>(k));
                for (int t : wide[batch[k]].second) {
                    std::uint64_t m = 0;
                    for (int p = 0; p < nl; ++p)
                        m |= static_cast<std::uint64_t>(popc(cols[p] & zy[static_cast<std::size_t>(t)]) & 1) << p;
                    smL[static_cast<std::size_t>(t)] = m;
                }
            }
            build_coset_pass(plan, nl, pe_begin, B, fl, gi, std::vector<int>{}, y, smL.data(), gz, coeffs, nullptr,
                             cols);
            ++plan.linear_passes;
            pending.swap(rest);
        }
        wide.clear();
    }
    // wide flip masks: full-vector sweeps (terms keep their full sign masks)
    for (const auto& [xy, members] : wide) {
        WGroup W{};
        W.x = xy;
        W.hbit = 63 - __builtin_clzll(xy);
        W.t_begin = static_cast<int>(dterms.size());
        W.t_count = static_cast<int>(members.size());
        for (int t : members) {
            const int ycnt = popc(y[t]);
            const double sgn = ((ycnt & 3) == 1 || (ycnt & 3) == 2) ? -2.0 : 2.0;
            PTerm tm{};
            tm.m = z[t] | y[t];
            tm.gz = gz[t];
            tm.f = make_double2(sgn * coeffs[2 * t], sgn * coeffs[2 * t + 1]);
            tm.comp = ycnt & 1;
            dterms.push_back(tm);
        }
        wgroups.push_back(W);
    }
    plan.T = T;
    return plan;
}

void pauli_expectation(qrt_state* st, int n_terms, const std::uint64_t* x, const std::uint64_t* y,
                       const std::uint64_t* z, const std::uint64_t* gz, const double* coeffs, double* partial) {
    const int nl = st->nl;
    const std::uint64_t local_mask = nl >= 64 ? ~0ull : ((1ull << nl) - 1);
    const std::uint64_t pe_mask = (st->p == 1) ? 0ull : static_cast<std::uint64_t>(st->p - 1);
    for (int t = 0; t < n_terms; ++t) {
        if ((x[t] | y[t] | z[t]) & ~local_mask) fail(QRT_ERR_INVALID, "term mask outside the local positions");
        if ((x[t] & y[t]) || (x[t] & z[t]) || (y[t] & z[t])) fail(QRT_ERR_INVALID, "overlapping X/Y/Z masks");
        if (gz[t] & ~pe_mask) fail(QRT_ERR_INVALID, "global Z mask outside the PE index");
    }
    for (int i = 0; i < 2 * st->p; ++i) partial[i] = 0.0;
    if (n_terms == 0) return;

    // A VQE loop evaluates the same Hamiltonian under the same layout every
    // iteration: plans are cached by their exact inputs.
    static std::mutex cache_mu;
    static std::deque<std::pair<std::vector<std::uint64_t>, std::shared_ptr<const PauliPlanHost>>> cache;
    std::vector<std::uint64_t> key;
    key.reserve(3 + 6 * static_cast<std::size_t>(n_terms));
    key.push_back(static_cast<std::uint64_t>(nl));
    key.push_back(static_cast<std::uint64_t>(st->pe_begin));
    key.push_back(static_cast<std::uint64_t>(n_terms));
    for (int t = 0; t < n_terms; ++t) {
        std::uint64_t cr, ci;
        std::memcpy(&cr, coeffs + 2 * t, 8);
        std::memcpy(&ci, coeffs + 2 * t + 1, 8);
        key.insert(key.end(), {x[t], y[t], z[t], gz[t], cr, ci});
    }
    // The lock covers the lookup / insertion only: the cached plan is immutable
    // (per-launch pointers are patched into a thread-local copy of each pass's
    // parameters below), so concurrent states never serialise on it.
    std::shared_ptr<const PauliPlanHost> plan_ptr;
    {
        std::lock_guard<std::mutex> lock(cache_mu);
        for (auto& e : cache)
            if (e.first == key) plan_ptr = e.second;
    }
    if (!plan_ptr) {
        auto built = std::make_shared<const PauliPlanHost>(build_pauli_plan(nl, st->pe_begin, n_terms, x, y, z, gz, coeffs));
        std::lock_guard<std::mutex> lock(cache_mu);
        cache.emplace_back(std::move(key), built);
        // one entry per EVC plan tile of the Hamiltonian (uniform 10k words: 26-60 tiles)
        if (cache.size() > 96) cache.pop_front();
        plan_ptr = std::move(built);
    }
    const PauliPlanHost& plan = *plan_ptr;
    const int T = plan.T;
    auto& dgroups = plan.dgroups;
    auto& dterms = plan.dterms;
    auto& hdrs = plan.hdrs;
    auto& wgroups = plan.wgroups;
    const std::size_t gbytes = dgroups.size() * sizeof(PGroup);
    const std::size_t toff = (gbytes + 255) & ~std::size_t{255};
    const std::size_t woff = (toff + dterms.size() * sizeof(PTerm) + 255) & ~std::size_t{255};
    const std::size_t coff = (woff + wgroups.size() * sizeof(WGroup) + 255) & ~std::size_t{255};
    const std::size_t goff = (coff + plan.cdterms.size() * sizeof(CosetDiagTerm) + 255) & ~std::size_t{255};
    std::vector<std::size_t> tab_off;
    std::size_t gend = goff;
    for (const auto& cp : plan.cosets) {
        tab_off.push_back(gend);
        gend = (gend + static_cast<std::size_t>(cp->n_tab) * sizeof(double) + 255) & ~std::size_t{255};
    }
    const std::size_t total = gend + 16;
    char* host = static_cast<char*>(ensure_pinned(st, total));
    QRT_CUDA(cudaStreamSynchronize(st->stream));
    std::memcpy(host, dgroups.data(), gbytes);
    std::memcpy(host + toff, dterms.data(), dterms.size() * sizeof(PTerm));
    std::memcpy(host + woff, wgroups.data(), wgroups.size() * sizeof(WGroup));
    std::memcpy(host + coff, plan.cdterms.data(), plan.cdterms.size() * sizeof(CosetDiagTerm));
    for (std::size_t i = 0; i < plan.cosets.size(); ++i)
        std::memcpy(host + tab_off[i], plan.cosets[i]->tabs, static_cast<std::size_t>(plan.cosets[i]->n_tab) * sizeof(double));
    char* dev = static_cast<char*>(ensure_ops(st, total));
    QRT_CUDA(cudaMemcpyAsync(dev, host, total, cudaMemcpyHostToDevice, st->stream));

    const int ctas = 1 << (nl - T);
    const std::size_t slots = static_cast<std::size_t>(ctas) * static_cast<std::size_t>(st->pe_count);
    double* red = ensure_red(st, 2 * slots + 2 * static_cast<std::size_t>(st->pe_count) + 2 * static_cast<std::size_t>(st->p));
    double* out = red + 2 * slots;
    QRT_CUDA(cudaMemsetAsync(red, 0, 2 * slots * sizeof(double), st->stream));

    static bool attr_done[64] = {};
    if (!attr_done[st->device]) {
        QRT_CUDA(cudaFuncSetAttribute(pauli_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_done[st->device] = true;
    }
    PePtrsP ptrs{};
    for (int i = 0; i < st->pe_count; ++i) ptrs.p[i] = st->live(i);
    {
        ProfileScope prof(st, QRT_K_PAULI);
        static thread_local std::unique_ptr<CosetParams> scratch_params;  // ~27 KiB: off the stack
        if (!scratch_params) scratch_params = std::make_unique<CosetParams>();
        for (std::size_t ci = 0; ci < plan.cosets.size(); ++ci) {
            CosetParams& cp = *scratch_params;
            cp = *plan.cosets[ci];
            cp.gtabs = reinterpret_cast<const double*>(dev + tab_off[ci]);
            for (int i = 0; i < st->pe_count; ++i) cp.ptrs[i] = st->live(i);
            launch_coset_pass(cp, reinterpret_cast<const CosetDiagTerm*>(dev + coff), st->pe_count, red, st->stream,
                              st->device);
            st->stats[QRT_K_PAULI].launches++;
            st->stats[QRT_K_PAULI].bytes += 16.0 * static_cast<double>(st->amps) * st->pe_count;
        }
        for (const PPass& h : hdrs) {
            const std::size_t smem = (std::size_t{1} << T) * sizeof(double2) +
                                     (std::size_t{1} << (T - h.c)) * sizeof(std::uint64_t) +
                                     (h.d_count > 0 ? (std::size_t{1} << T) * sizeof(double) : 0);
            dim3 grid(static_cast<unsigned>(ctas), static_cast<unsigned>(st->pe_count));
            pauli_pass_kernel<<<grid, kThreads, smem, st->stream>>>(
                ptrs, h, reinterpret_cast<const PGroup*>(dev), reinterpret_cast<const PTerm*>(dev + toff), red);
            QRT_CUDA(cudaGetLastError());
            st->stats[QRT_K_PAULI].launches++;
            st->stats[QRT_K_PAULI].bytes += 16.0 * static_cast<double>(st->amps) * st->pe_count;
        }
        if (!wgroups.empty()) {
            dim3 grid(static_cast<unsigned>(ctas), static_cast<unsigned>(st->pe_count));
            pauli_wide_kernel<<<grid, 256, 0, st->stream>>>(ptrs, nl, st->pe_begin,
                                                            reinterpret_cast<const WGroup*>(dev + woff),
                                                            static_cast<int>(wgroups.size()),
                                                            reinterpret_cast<const PTerm*>(dev + toff), red);
            QRT_CUDA(cudaGetLastError());
            st->stats[QRT_K_PAULI].launches++;
            // algorithmic bytes of the launch: one read of the state (all of its
            // groups are evaluated in one launch; per-group re-reads hit L2 — round 1
            // charged a sweep per group, which reported an HBM fraction of 1.15)
            st->stats[QRT_K_PAULI].bytes += 16.0 * static_cast<double>(st->amps) * st->pe_count;
        }
        reduce_slots_kernel<<<st->pe_count, 256, 0, st->stream>>>(red, ctas, out);
        QRT_CUDA(cudaGetLastError());
        st->stats[QRT_K_MISC].launches++;
    }
    // algorithmic flops: one complex MAC per amplitude per term (reference loop)
    st->stats[QRT_K_PAULI].flops += 8.0 * static_cast<double>(st->amps) * st->pe_count * n_terms;
    gather_partials(st, out, partial);
}

void pauli_plan_info(int nl, int n_terms, const std::uint64_t* x, const std::uint64_t* y, const std::uint64_t* z,
                     const std::uint64_t* gz, const double* coeffs, int* passes, int* groups, int* wide_groups,
                     double* seconds) {
    const auto t0 = std::chrono::steady_clock::now();
    PauliPlanHost plan = build_pauli_plan(nl, 0, n_terms, x, y, z, gz, coeffs);
    const auto t1 = std::chrono::steady_clock::now();
    if (std::getenv("QRT_DEBUG_PLAN"))
        std::fprintf(stderr, "evc plan: %zu tiled passes, %zu coset launches (%d linear), %d coset sets, %zu wide groups\n",
                     plan.hdrs.size(), plan.cosets.size(), plan.linear_passes, plan.coset_sets, plan.wgroups.size());
    if (passes) *passes = static_cast<int>(plan.hdrs.size() + plan.cosets.size());
    int coset_groups = 0;
    for (const auto& cp : plan.cosets)
        for (int si = 0; si < cp->n_sets; ++si) coset_groups += cp->sets[si].g_count;
    if (std::getenv("QRT_DEBUG_PLAN")) {
        int fast = 0, distinct = 0, sets = 0, hist[8] = {};
        for (const auto& cp : plan.cosets)
            for (int si = 0; si < cp->n_sets; ++si) {
                const CosetSet& S = cp->sets[si];
                ++sets;
                for (int xq = 1; xq < 32; ++xq) {
                    const int n = S.xbeg[xq] - S.xbeg[xq - 1];
                    if (n > 0) {
                        fast += n;
                        ++distinct;
                        ++hist[n < 7 ? n : 7];
                    }
                }
            }
        int dpasses = 0, dwords = 0;
        for (const auto& cp : plan.cosets)
            if (cp->d_count > 0) {
                ++dpasses;
                dwords += cp->d_count;
            }
        int tab1_sets = 0, one_sets = 0;
        for (const auto& cp : plan.cosets)
            for (int si = 0; si < cp->n_sets; ++si) {
                tab1_sets += cp->sets[si].tab1 >= 0;
                one_sets += cp->sets[si].onemask != 0;
            }
        std::fprintf(stderr, "evc cosets: table-path sets %d fast / %d single-bit\n", tab1_sets, one_sets);
        std::fprintf(stderr, "evc cosets: %d I/Z words in %d passes; %d sets, %d fast groups over %d (set, mask) pairs; "
                     "per-pair counts 1..7+:", dwords, dpasses, sets, fast, distinct);
        for (int i = 1; i < 8; ++i) std::fprintf(stderr, " %d", hist[i]);
        std::fprintf(stderr, "\n");
    }
    if (groups) *groups = static_cast<int>(plan.dgroups.size()) + coset_groups;
    if (wide_groups) *wide_groups = static_cast<int>(plan.wgroups.size());
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
}

double norm(qrt_state* st) {
    const int blocks = st->sm_count * 4;
    const std::size_t slots = static_cast<std::size_t>(blocks) * static_cast<std::size_t>(st->pe_count);
    double* red = ensure_red(st, 2 * slots + 2 * static_cast<std::size_t>(st->pe_count) + 2 * static_cast<std::size_t>(st->p));
    double* out = red + 2 * slots;
    for (int i = 0; i < st->pe_count; ++i) {
        norm_kernel<<<blocks, 256, 0, st->stream>>>(st->live(i), st->amps, red + 2 * static_cast<std::size_t>(i) * blocks);
        QRT_CUDA(cudaGetLastError());
    }
    reduce_slots_kernel<<<st->pe_count, 256, 0, st->stream>>>(red, blocks, out);
    QRT_CUDA(cudaGetLastError());
    st->stats[QRT_K_MISC].launches += static_cast<std::uint64_t>(st->pe_count) + 1;
    std::vector<double> all(2 * static_cast<std::size_t>(st->p), 0.0);
    gather_partials(st, out, all.data());
    double s = 0.0;
    for (int pe = 0; pe < st->p; ++pe) s += all[2 * static_cast<std::size_t>(pe)];
    return std::sqrt(s);
}

}  // namespace qrt
