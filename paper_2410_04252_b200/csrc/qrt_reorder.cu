// libqrt — qubit reordering (reference perform_qr, dist_sim.cpp:203-240).
//
// The reference builds a full second copy and walks all 2^n indices on one
// thread.  Here every PE *pushes* its amplitudes straight into the spare
// buffer of the destination PE — a local HBM store for the 2^-k of the data
// that stays, a peer store over NVLink 5 (CUDA IPC mapping) for the rest — in
// one kernel with no pack/unpack staging.  Ranks then meet at one NCCL
// all-reduce on the same stream (device-side barrier) and flip buffers.
//
// The kernel enumerates *destination* order: chunk bits of the destination
// offset are contiguous, so every warp writes 512 contiguous bytes to one
// peer; the host picks the physical placement of arriving qubits (see
// host/src/device_state.cpp) so the source side reads runs of >= 2^4
// amplitudes as well.  Relocated-amplitude accounting is exact (union-find
// over position pairs), equal to qr_data_volume(k, n) for k local<->global
// pairs (layout.cpp:91-94).
//
// The index mapping (`QrMap`) is shared by the kernel and the host-side plan
// query qrt_reorder_plan, which the CPU multi-process tests use to emulate
// the exchange exactly.

#include <cstdlib>
#include <numeric>

#include "qrt_internal.h"

namespace qrt {

namespace {

// Bit-mapping tables of one reorder, in destination-enumeration order:
//   u = (chunk, cls, e):  e = low C destination-local bits, chunk = the
//   remaining destination-local bits, cls = the destination PE bits fed by
//   source-local bits.
struct QrMap {
    int pe_begin;
    int C;     // chunk bits (destination-contiguous)
    int k;     // destination PE bits fed by source-local bits
    int n_hi;  // destination-local bits above the chunk
    int g;     // global bits
    int nl;
    std::uint64_t tab_src[2][64];  // e (two 6-bit halves) -> source / destination offset bits
    std::uint64_t tab_dst[2][64];
    int hi_src_pos[64];
    int hi_dst_pos[64];
    int cls_src_pos[8];
    int cls_dst_pe_bit[8];
    int j_dst_pos[8];  // source PE bit b -> destination position (local < nl, else nl + PE bit)
};

struct Bases {
    std::uint64_t src, dst;
    int pe;
};

__host__ __device__ inline Bases qr_bases(const QrMap& a, int src_pe, std::uint64_t chunk, int cls) {
    Bases b{0, 0, 0};
    for (int i = 0; i < a.n_hi; ++i) {
        const std::uint64_t bit = (chunk >> i) & 1ull;
        b.src |= bit << a.hi_src_pos[i];
        b.dst |= bit << a.hi_dst_pos[i];
    }
    for (int i = 0; i < a.g; ++i) {
        const int bit = (src_pe >> i) & 1;
        const int t = a.j_dst_pos[i];
        if (t < a.nl)
            b.dst |= static_cast<std::uint64_t>(bit) << t;
        else
            b.pe |= bit << (t - a.nl);
    }
    for (int i = 0; i < a.k; ++i) {
        const int bit = (cls >> i) & 1;
        b.src |= static_cast<std::uint64_t>(bit) << a.cls_src_pos[i];
        b.pe |= bit << a.cls_dst_pe_bit[i];
    }
    return b;
}

__host__ __device__ inline std::uint64_t qr_src_e(const QrMap& a, int e) {
    return a.tab_src[0][e & 63] | a.tab_src[1][(e >> 6) & 63];
}
__host__ __device__ inline std::uint64_t qr_dst_e(const QrMap& a, int e) {
    return a.tab_dst[0][e & 63] | a.tab_dst[1][(e >> 6) & 63];
}

struct QrArgs {
    amp_t* dst[kMaxLocalPEs];  // spare buffer of every PE (p <= 64)
    const amp_t* src[kMaxLocalPEs];
    QrMap m;
};

__global__ void __launch_bounds__(256) reorder_kernel(const __grid_constant__ QrArgs a) {
    const int lpe = blockIdx.y;
    const int j = a.m.pe_begin + lpe;
    const std::uint64_t chunk = blockIdx.x;
    const amp_t* __restrict__ src = a.src[lpe];
    const int E = 1 << a.m.C;
    const int ncls = 1 << a.m.k;
    for (int cls = 0; cls < ncls; ++cls) {
        const Bases b = qr_bases(a.m, j, chunk, cls);
        amp_t* __restrict__ dst = a.dst[b.pe];
        QRT_DCHECK(b.pe >= 0 && b.pe < (1 << a.m.g) && dst != nullptr);
        for (int e = threadIdx.x; e < E; e += blockDim.x) {
            QRT_DCHECK((b.dst | qr_dst_e(a.m, e)) < (1ull << a.m.nl) && (b.src | qr_src_e(a.m, e)) < (1ull << a.m.nl));
            dst[b.dst | qr_dst_e(a.m, e)] = __ldcs(&src[b.src | qr_src_e(a.m, e)]);
        }
    }
    __threadfence_system();  // peer stores visible before the stream-ordered barrier
}

int find(std::vector<int>& parent, int x) {
    while (parent[static_cast<std::size_t>(x)] != x)
        x = parent[static_cast<std::size_t>(x)] = parent[static_cast<std::size_t>(parent[static_cast<std::size_t>(x)])];
    return x;
}

// Validates `dest`, computes the exact relocation count and the mapping tables.
std::uint64_t build_map(int n, int nl, int pe_begin, const int* dest, QrMap& a, bool& identity) {
    const int g = n - nl;
    std::vector<int> src_of(static_cast<std::size_t>(n), -1);
    for (int s = 0; s < n; ++s) {
        if (dest[s] < 0 || dest[s] >= n || src_of[static_cast<std::size_t>(dest[s])] != -1)
            fail(QRT_ERR_INVALID, "reorder map is not a permutation of positions");
        src_of[static_cast<std::size_t>(dest[s])] = s;
    }
    // relocated = 2^n - #{i : PE(perm(i)) == PE(i)}; the equality constraints
    // bit_{src(t)} == bit_t (t global) join positions into components.
    std::vector<int> parent(static_cast<std::size_t>(n));
    std::iota(parent.begin(), parent.end(), 0);
    for (int t = nl; t < n; ++t) {
        int x = find(parent, t), y = find(parent, src_of[static_cast<std::size_t>(t)]);
        if (x != y) parent[static_cast<std::size_t>(x)] = y;
    }
    int comps = 0;
    for (int x = 0; x < n; ++x) comps += find(parent, x) == x ? 1 : 0;
    const std::uint64_t relocated = (n >= 64 ? 0 : (1ull << n)) - (1ull << comps);

    identity = true;
    for (int s = 0; s < n; ++s) identity = identity && dest[s] == s;

    // destination free positions: local F_L (ascending) and global F_G
    std::vector<int> fl, fg;
    for (int t = 0; t < n; ++t) {
        const int s = src_of[static_cast<std::size_t>(t)];
        if (s >= nl) continue;  // fed by a source PE bit
        (t < nl ? fl : fg).push_back(t);
    }
    const int k = static_cast<int>(fg.size());
    if (k > 8) fail(QRT_ERR_CONFIG, "reorder moves more than 8 local bits to global positions");
    a = QrMap{};
    a.pe_begin = pe_begin;
    a.nl = nl;
    a.g = g;
    a.k = k;
    const int nfl = static_cast<int>(fl.size());  // == nl - k
    a.C = std::min(12, nfl);
    a.n_hi = nfl - a.C;
    for (int h = 0; h < 2; ++h)
        for (int e = 0; e < 64; ++e) {
            std::uint64_t s = 0, d = 0;
            for (int b = 0; b < 6; ++b) {
                const int bit = h * 6 + b;
                if (bit >= a.C || !((e >> b) & 1)) continue;
                d |= 1ull << fl[static_cast<std::size_t>(bit)];
                s |= 1ull << src_of[static_cast<std::size_t>(fl[static_cast<std::size_t>(bit)])];
            }
            a.tab_src[h][e] = s;
            a.tab_dst[h][e] = d;
        }
    for (int i = 0; i < a.n_hi; ++i) {
        const int t = fl[static_cast<std::size_t>(a.C + i)];
        a.hi_dst_pos[i] = t;
        a.hi_src_pos[i] = src_of[static_cast<std::size_t>(t)];
    }
    for (int i = 0; i < k; ++i) {
        a.cls_dst_pe_bit[i] = fg[static_cast<std::size_t>(i)] - nl;
        a.cls_src_pos[i] = src_of[static_cast<std::size_t>(fg[static_cast<std::size_t>(i)])];
    }
    for (int b = 0; b < g; ++b) a.j_dst_pos[b] = dest[nl + b];
    return relocated;
}

// ---------------------------------------------------------------------------
// In-place QR (SURVEY.md §7 "in-place QR mandatory" at 34 qubits / p = 2,
// where two 128 GiB sub-vectors per GPU do not fit in 180 GB).  The reference
// builds a full second copy (dist_sim.cpp:224-233); here the position
// permutation `dest` is split into
//   rho   a permutation of local positions (staying qubits that move, and
//         the departing qubit's move to the slot its arriving partner takes),
//         applied as at most two involutions = passes of disjoint local
//         bit-transpositions (a 2-cycle is one pass), and
//   cross k transpositions (local slot d_i <-> PE bit b_i): a pairwise
//         symmetric exchange — PE j's slot class s swaps with PE s's slot
//         class j at the same offsets otherwise.
// Every element pair is read and written by exactly one thread (the pair's
// two PEs split the classes on one free position f), so both passes run in
// place with no staging buffer at all: the exchange reads the partner's
// amplitude over NVLink and stores this PE's amplitude into the partner's
// slot, so each direction of the link carries the same bytes as the push
// exchange, and the 2^-k of the data that stays is never touched.

struct Deposit {
    int E = 0;                      // low enumeration bits (table lookup)
    int n_hi = 0;                   // enumeration bits above E
    int hi_pos[64] = {};
    std::uint64_t tab[2][32] = {};  // e (two 5-bit halves) -> offset bits
};

void make_deposit(const std::vector<int>& rest, Deposit& d) {
    d = Deposit{};
    d.E = std::min(10, static_cast<int>(rest.size()));
    d.n_hi = static_cast<int>(rest.size()) - d.E;
    for (int h = 0; h < 2; ++h)
        for (int e = 0; e < 32; ++e) {
            std::uint64_t v = 0;
            for (int b = 0; b < 5; ++b) {
                const int bit = h * 5 + b;
                if (bit < d.E && ((e >> b) & 1)) v |= 1ull << rest[static_cast<std::size_t>(bit)];
            }
            d.tab[h][e] = v;
        }
    for (int i = 0; i < d.n_hi; ++i) d.hi_pos[i] = rest[static_cast<std::size_t>(d.E + i)];
}

__device__ __forceinline__ std::uint64_t dep_hi(const Deposit& d, std::uint64_t chunk) {
    std::uint64_t v = 0;
    for (int i = 0; i < d.n_hi; ++i) v |= ((chunk >> i) & 1ull) << d.hi_pos[i];
    return v;
}
__device__ __forceinline__ std::uint64_t dep_lo(const Deposit& d, int e) {
    return d.tab[0][e & 31] | d.tab[1][(e >> 5) & 31];
}

struct XchgArgs {
    amp_t* pe_ptr[kMaxLocalPEs];  // live buffer of every PE (IPC peer table)
    int pe_begin;
    int k;
    int d_pos[8];   // local slot of transposition i
    int pe_bit[8];  // PE-index bit of transposition i
    int f;          // free local position splitting each class pair between its two PEs (-1: none)
    int nl, p;      // local positions, PEs (QRT_CHECKS bounds)
    Deposit dep;    // the remaining local positions
};

constexpr int kXchgUnroll = 4;

__global__ void __launch_bounds__(256) exchange_kernel(const __grid_constant__ XchgArgs a) {
    const int j = a.pe_begin + static_cast<int>(blockIdx.y);
    int jc = 0;
    for (int i = 0; i < a.k; ++i) jc |= ((j >> a.pe_bit[i]) & 1) << i;
    const std::uint64_t chunks = 1ull << a.dep.n_hi;
    const std::uint64_t work = static_cast<std::uint64_t>((1 << a.k) - 1) * chunks;
    const int E = 1 << a.dep.E;
    amp_t* __restrict__ mine = a.pe_ptr[j];
    for (std::uint64_t w = blockIdx.x; w < work; w += gridDim.x) {
        const int ci = static_cast<int>(w / chunks);
        const std::uint64_t chunk = w % chunks;
        // XOR schedule: at step ci every PE j works with the PE whose class
        // bits are jc ^ (ci + 1), a perfect matching, so all GPUs exchange
        // pairwise at once instead of converging on one partner (an in-cast
        // that held k = 2 on 4 GPUs at 440 GB/s); never jc, which stays
        const int s = jc ^ (ci + 1);
        int sp = j;
        std::uint64_t ob = 0, pb = 0;
        for (int i = 0; i < a.k; ++i) {
            const int sb = (s >> i) & 1, jb = (jc >> i) & 1;
            sp = (sp & ~(1 << a.pe_bit[i])) | (sb << a.pe_bit[i]);
            ob |= static_cast<std::uint64_t>(sb) << a.d_pos[i];
            pb |= static_cast<std::uint64_t>(jb) << a.d_pos[i];
        }
        if (a.f >= 0) {
            const std::uint64_t hb = j < sp ? 0ull : 1ull;
            ob |= hb << a.f;
            pb |= hb << a.f;
        } else if (j > sp) {
            continue;  // no free position: the lower PE of the pair does it all
        }
        const std::uint64_t hi = dep_hi(a.dep, chunk);
        ob |= hi;
        pb |= hi;
        amp_t* __restrict__ peer = a.pe_ptr[sp];
        QRT_DCHECK(sp >= 0 && sp < a.p && sp != j && peer != nullptr);
        for (int e0 = threadIdx.x; e0 < E; e0 += kXchgUnroll * blockDim.x) {
            amp_t x[kXchgUnroll], y[kXchgUnroll];
            std::uint64_t lo[kXchgUnroll];
#pragma unroll
            for (int u = 0; u < kXchgUnroll; ++u) {
                const int e = e0 + u * static_cast<int>(blockDim.x);
                lo[u] = e < E ? dep_lo(a.dep, e) : 0;
                if (e < E) {
                    QRT_DCHECK((ob | lo[u]) < (1ull << a.nl) && (pb | lo[u]) < (1ull << a.nl) && ob != pb);
                    x[u] = __ldcs(&mine[ob | lo[u]]);
                    y[u] = __ldcs(&peer[pb | lo[u]]);
                }
            }
#pragma unroll
            for (int u = 0; u < kXchgUnroll; ++u) {
                const int e = e0 + u * static_cast<int>(blockDim.x);
                if (e < E) {
                    __stcs(&mine[ob | lo[u]], y[u]);
                    __stcs(&peer[pb | lo[u]], x[u]);
                }
            }
        }
    }
    __threadfence_system();  // peer stores visible before the stream-ordered barrier
}

struct LocalSwapArgs {
    amp_t* ptr[kMaxLocalPEs];  // this process's live buffers
    int m;                     // disjoint transpositions (a_i <-> c_i), a_i < c_i
    int a_pos[8];
    int c_pos[8];
    int nl;                    // local positions (QRT_CHECKS bounds)
    Deposit dep;               // the other local positions
};

// One involution of local positions, in place: the element with pattern v on
// the pair bits swaps with the pattern where each pair's two bits are
// exchanged; the lower offset of the two does the swap (block-uniform test).
__global__ void __launch_bounds__(256) local_swap_kernel(const __grid_constant__ LocalSwapArgs a) {
    amp_t* __restrict__ v = a.ptr[blockIdx.y];
    const std::uint64_t chunks = 1ull << a.dep.n_hi;
    const std::uint64_t work = (1ull << (2 * a.m)) * chunks;
    const int E = 1 << a.dep.E;
    for (std::uint64_t w = blockIdx.x; w < work; w += gridDim.x) {
        const int pat = static_cast<int>(w / chunks);
        const std::uint64_t chunk = w % chunks;
        std::uint64_t ob = 0, pb = 0;
        for (int i = 0; i < a.m; ++i) {
            const std::uint64_t ba = (pat >> (2 * i)) & 1, bc = (pat >> (2 * i + 1)) & 1;
            ob |= (ba << a.a_pos[i]) | (bc << a.c_pos[i]);
            pb |= (bc << a.a_pos[i]) | (ba << a.c_pos[i]);
        }
        if (pb <= ob) continue;  // fixed (equal) or handled from the partner's pattern
        const std::uint64_t hi = dep_hi(a.dep, chunk);
        ob |= hi;
        pb |= hi;
        for (int e0 = threadIdx.x; e0 < E; e0 += kXchgUnroll * blockDim.x) {
            amp_t x[kXchgUnroll], y[kXchgUnroll];
            std::uint64_t lo[kXchgUnroll];
#pragma unroll
            for (int u = 0; u < kXchgUnroll; ++u) {
                const int e = e0 + u * static_cast<int>(blockDim.x);
                lo[u] = e < E ? dep_lo(a.dep, e) : 0;
                if (e < E) {
                    QRT_DCHECK((pb | lo[u]) < (1ull << a.nl) && (ob | lo[u]) < (pb | lo[u]));
                    x[u] = __ldcs(&v[ob | lo[u]]);
                    y[u] = __ldcs(&v[pb | lo[u]]);
                }
            }
#pragma unroll
            for (int u = 0; u < kXchgUnroll; ++u) {
                const int e = e0 + u * static_cast<int>(blockDim.x);
                if (e < E) {
                    __stcs(&v[ob | lo[u]], y[u]);
                    __stcs(&v[pb | lo[u]], x[u]);
                }
            }
        }
    }
}

// Dense variant for transpositions touching a low position (< 5, i.e. inside a
// 32-byte sector or a short run): each thread owns all 4^M pattern elements
// of its rest index, loads them all and stores them permuted, so every sector
// is read and written whole once (the sparse kernel above moved half the
// elements of every sector and measured 59 GB of DRAM traffic for a 17 GB
// move, 30 qubits on 4 PEs).
template <int M>
__global__ void __launch_bounds__(256) local_swap_dense_kernel(const __grid_constant__ LocalSwapArgs a) {
    constexpr int NP = 1 << (2 * M);
    amp_t* __restrict__ v = a.ptr[blockIdx.y];
    std::uint64_t off[NP];
#pragma unroll
    for (int pat = 0; pat < NP; ++pat) {
        std::uint64_t o = 0;
#pragma unroll
        for (int i = 0; i < M; ++i)
            o |= (static_cast<std::uint64_t>((pat >> (2 * i)) & 1) << a.a_pos[i]) |
                 (static_cast<std::uint64_t>((pat >> (2 * i + 1)) & 1) << a.c_pos[i]);
        off[pat] = o;
    }
    const std::uint64_t chunks = 1ull << a.dep.n_hi;
    const int E = 1 << a.dep.E;
    for (std::uint64_t w = blockIdx.x; w < chunks; w += gridDim.x) {
        const std::uint64_t hi = dep_hi(a.dep, w);
        for (int e = threadIdx.x; e < E; e += blockDim.x) {
            const std::uint64_t base = hi | dep_lo(a.dep, e);
            QRT_DCHECK((base | off[NP - 1]) < (1ull << a.nl));
            amp_t x[NP];
#pragma unroll
            for (int pat = 0; pat < NP; ++pat) x[pat] = __ldcs(&v[base | off[pat]]);
#pragma unroll
            for (int pat = 0; pat < NP; ++pat) {
                int src = 0;  // the element at pattern `pat` receives the one with each pair's bits exchanged
#pragma unroll
                for (int i = 0; i < M; ++i)
                    src |= (((pat >> (2 * i)) & 1) << (2 * i + 1)) | (((pat >> (2 * i + 1)) & 1) << (2 * i));
                __stcs(&v[base | off[pat]], x[src]);
            }
        }
    }
}

// dest (position permutation) -> two passes of local transpositions + the
// cross transpositions.  Requires every global position to be fed by itself
// or by a local position (true for every flat / one-box QR event,
// layout.cpp:96-161); anything else is rejected.
struct InplacePlan {
    std::vector<std::pair<int, int>> local[2];
    std::vector<std::pair<int, int>> cross;  // (local slot, PE bit)
};

// True when every global position is fed by itself or by a local position
// (every flat / one-box QR event; hierarchical routing may move a global
// qubit between the intra and inter regions, which only the push kernel does).
bool inplace_decomposable(int n, int nl, const int* dest) {
    std::vector<int> src_of(static_cast<std::size_t>(n), -1);
    for (int s = 0; s < n; ++s) src_of[static_cast<std::size_t>(dest[s])] = s;
    for (int t = nl; t < n; ++t) {
        const int s = src_of[static_cast<std::size_t>(t)];
        if (s >= nl && s != t) return false;
    }
    return true;
}

InplacePlan plan_inplace(int n, int nl, const int* dest) {
    std::vector<int> src_of(static_cast<std::size_t>(n), -1);
    for (int s = 0; s < n; ++s) src_of[static_cast<std::size_t>(dest[s])] = s;
    InplacePlan P;
    std::vector<int> rho(static_cast<std::size_t>(nl), -1);
    for (int x = 0; x < nl; ++x) {
        const int t = dest[x];
        if (t < nl) {
            rho[static_cast<std::size_t>(x)] = t;  // staying qubit
        } else {
            const int d = dest[t];  // the arriving qubit's slot
            if (d >= nl) fail(QRT_ERR_CONFIG, "in-place reorder: global position moves to another global position");
            rho[static_cast<std::size_t>(x)] = d;
            P.cross.emplace_back(d, t - nl);
        }
    }
    for (int t = nl; t < n; ++t) {
        const int s = src_of[static_cast<std::size_t>(t)];
        if (s >= nl && s != t) fail(QRT_ERR_CONFIG, "in-place reorder: global position moves to another global position");
    }
    // rho = tau2 o tau1 per cycle (x_0 -> x_1 -> ... -> x_{c-1}):
    // tau1(x_i) = x_{-i}, tau2(x_i) = x_{1-i} (indices mod c).
    std::vector<char> seen(static_cast<std::size_t>(nl), 0);
    for (int x0 = 0; x0 < nl; ++x0) {
        if (seen[static_cast<std::size_t>(x0)]) continue;
        std::vector<int> cyc;
        for (int x = x0; !seen[static_cast<std::size_t>(x)]; x = rho[static_cast<std::size_t>(x)]) {
            seen[static_cast<std::size_t>(x)] = 1;
            cyc.push_back(x);
        }
        const int c = static_cast<int>(cyc.size());
        if (c < 2) continue;
        for (int pass = 0; pass < 2; ++pass)
            for (int i = 0; i < c; ++i) {
                const int jdx = ((pass == 0 ? -i : 1 - i) % c + c) % c;
                if (i < jdx) {
                    const int a = cyc[static_cast<std::size_t>(i)], b = cyc[static_cast<std::size_t>(jdx)];
                    P.local[pass].emplace_back(std::min(a, b), std::max(a, b));
                }
            }
    }
    if (P.local[0].empty()) std::swap(P.local[0], P.local[1]);
    return P;
}

void launch_local_pairs(qrt_state* st, const std::vector<std::pair<int, int>>& pairs, bool dense) {
    for (std::size_t base = 0; base < pairs.size(); base += (dense ? 2 : 8)) {
        LocalSwapArgs a{};
        a.m = static_cast<int>(std::min<std::size_t>(dense ? 2 : 8, pairs.size() - base));
        std::vector<char> used(static_cast<std::size_t>(st->nl), 0);
        for (int i = 0; i < a.m; ++i) {
            a.a_pos[i] = pairs[base + static_cast<std::size_t>(i)].first;
            a.c_pos[i] = pairs[base + static_cast<std::size_t>(i)].second;
            used[static_cast<std::size_t>(a.a_pos[i])] = used[static_cast<std::size_t>(a.c_pos[i])] = 1;
        }
        std::vector<int> rest;
        for (int x = 0; x < st->nl; ++x)
            if (!used[static_cast<std::size_t>(x)]) rest.push_back(x);
        make_deposit(rest, a.dep);
        a.nl = st->nl;
        for (int i = 0; i < st->pe_count; ++i) a.ptr[i] = st->live(i);
        const std::uint64_t work = dense ? (1ull << a.dep.n_hi) : ((1ull << (2 * a.m)) << a.dep.n_hi);
        const unsigned gx = static_cast<unsigned>(std::min<std::uint64_t>(work, static_cast<std::uint64_t>(st->sm_count) * 8));
        const dim3 grid(gx, static_cast<unsigned>(st->pe_count));
        if (!dense)
            local_swap_kernel<<<grid, 256, 0, st->stream>>>(a);
        else if (a.m == 1)
            local_swap_dense_kernel<1><<<grid, 256, 0, st->stream>>>(a);
        else
            local_swap_dense_kernel<2><<<grid, 256, 0, st->stream>>>(a);
        QRT_CUDA(cudaGetLastError());
        st->stats[QRT_K_QR].launches++;
    }
}

// Disjoint transpositions commute: pairs touching a low position (a run
// shorter than 2^5 amplitudes) take the dense kernel, two per pass; the rest
// move only their half of the elements in one sparse pass.
void launch_local_swaps(qrt_state* st, const std::vector<std::pair<int, int>>& pairs) {
    std::vector<std::pair<int, int>> low, high;
    for (const auto& pr : pairs) (std::min(pr.first, pr.second) < 5 ? low : high).push_back(pr);
    if (!low.empty()) launch_local_pairs(st, low, true);
    if (!high.empty()) launch_local_pairs(st, high, false);
}

void execute_inplace(qrt_state* st, const int* dest, std::uint64_t relocated) {
    if (st->p > kMaxLocalPEs) fail(QRT_ERR_CONFIG, "too many PEs for the in-place reorder kernel");
    const InplacePlan P = plan_inplace(st->n, st->nl, dest);
    ProfileScope prof(st, QRT_K_QR);
    for (int pass = 0; pass < 2; ++pass)
        if (!P.local[pass].empty()) launch_local_swaps(st, P.local[pass]);
    if (P.cross.empty()) return;
    if (P.cross.size() > 8) fail(QRT_ERR_CONFIG, "reorder moves more than 8 local bits to global positions");
    XchgArgs a{};
    a.pe_begin = st->pe_begin;
    a.k = static_cast<int>(P.cross.size());
    std::vector<char> used(static_cast<std::size_t>(st->nl), 0);
    for (int i = 0; i < a.k; ++i) {
        a.d_pos[i] = P.cross[static_cast<std::size_t>(i)].first;
        a.pe_bit[i] = P.cross[static_cast<std::size_t>(i)].second;
        used[static_cast<std::size_t>(a.d_pos[i])] = 1;
    }
    a.f = -1;
    for (int x = st->nl - 1; x >= 0; --x)
        if (!used[static_cast<std::size_t>(x)]) {
            a.f = x;
            used[static_cast<std::size_t>(x)] = 1;
            break;
        }
    std::vector<int> rest;
    for (int x = 0; x < st->nl; ++x)
        if (!used[static_cast<std::size_t>(x)]) rest.push_back(x);
    make_deposit(rest, a.dep);
    a.nl = st->nl;
    a.p = st->p;
    for (int pe = 0; pe < st->p; ++pe) a.pe_ptr[pe] = st->peer[st->cur][static_cast<std::size_t>(pe)];
    barrier_on_stream(st);  // every peer is done with the buffers touched here
    {
        ProfileScope xfer(st, QRT_K_QR_XFER, true);
        const std::uint64_t work = static_cast<std::uint64_t>((1 << a.k) - 1) << a.dep.n_hi;
        const unsigned gx =
            static_cast<unsigned>(std::min<std::uint64_t>(work, static_cast<std::uint64_t>(st->sm_count) * 8));
        exchange_kernel<<<dim3(gx, static_cast<unsigned>(st->pe_count)), 256, 0, st->stream>>>(a);
        QRT_CUDA(cudaGetLastError());
    }
    barrier_on_stream(st);  // every peer's stores into this PE have landed
    st->stats[QRT_K_QR].launches++;
    st->stats[QRT_K_QR_XFER].launches++;
    st->stats[QRT_K_QR_XFER].bytes += 16.0 * static_cast<double>(relocated) * st->pe_count / st->p;
    st->stats[QRT_K_QR].bytes += 16.0 * static_cast<double>(relocated) * st->pe_count / st->p;
}

}  // namespace


// Largest log2(amplitudes per PE) the fused (pull) QR is used for: at 2^31
// (32q on 2 GPUs, 34q on 8) it beats the in-place exchange (16.28 vs 16.73 s,
// profiles/r2/n2b); at 2^32 it lost even to the push exchange in round 1.
int fused_qr_max_log2() {
    static const int v = [] {
        const char* e = std::getenv("QRT_FUSED_QR_MAX_LOG2");
        return e ? std::atoi(e) : 31;
    }();
    return v;
}

bool fused_qr_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("QRT_FUSED_QR");
        return e ? std::atoi(e) != 0 : true;
    }();
    return on;
}

namespace {

// The push exchange: every PE stores its amplitudes into the spare buffer of
// the destination PE, then all ranks meet and flip buffers.
void execute_reorder(qrt_state* st, const int* dest) {
    QrArgs a{};
    bool identity = false;
    const std::uint64_t relocated = build_map(st->n, st->nl, st->pe_begin, dest, a.m, identity);
    if (identity) return;
    if (st->p > kMaxLocalPEs) fail(QRT_ERR_CONFIG, "too many PEs for the reorder kernel");
    ensure_alt(st);
    const int nxt = st->cur ^ 1;
    for (int pe = 0; pe < st->p; ++pe) a.dst[pe] = st->peer[nxt][static_cast<std::size_t>(pe)];
    for (int i = 0; i < st->pe_count; ++i) a.src[i] = st->live(i);
    {
        ProfileScope prof(st, QRT_K_QR);
        barrier_on_stream(st);  // no peer still reads the buffers written here (fused passes)
        {
            ProfileScope xfer(st, QRT_K_QR_XFER, true);
            dim3 grid(static_cast<unsigned>(1ull << a.m.n_hi), static_cast<unsigned>(st->pe_count));
            reorder_kernel<<<grid, 256, 0, st->stream>>>(a);
            QRT_CUDA(cudaGetLastError());
        }
        barrier_on_stream(st);
    }
    st->stats[QRT_K_QR].launches++;
    st->stats[QRT_K_QR_XFER].launches++;
    st->stats[QRT_K_QR_XFER].bytes += 16.0 * static_cast<double>(relocated) * st->pe_count / st->p;
    // bytes that cross to another PE (each way), counted for this process's PEs
    st->stats[QRT_K_QR].bytes += 16.0 * static_cast<double>(relocated) * st->pe_count / st->p;
    st->cur = nxt;
}

// An executed (not fused) QR: the in-place pairwise swap whenever the map
// allows it — it moves only the (1 - 2^-k) that changes PE and measured 679
// vs 531 GB/s per direction for the push kernel (2 x B200, 2^30 amplitudes
// per PE, profiles/r2_ncu_qr_nvlink.json) — else the push exchange into the spare
// buffer.  QRT_QR_PUSH=1 forces the push kernel on two-buffer states.
void execute_qr(qrt_state* st, const int* dest) {
    static const bool force_push = [] {
        const char* e = std::getenv("QRT_QR_PUSH");
        return e && std::atoi(e) != 0;
    }();
    const bool decomposable = inplace_decomposable(st->n, st->nl, dest);
    if (!st->inplace && (force_push || !decomposable)) {
        execute_reorder(st, dest);
        return;
    }
    if (!decomposable) fail(QRT_ERR_CONFIG, "in-place reorder: global position moves to another global position");
    QrMap m{};
    bool identity = false;
    const std::uint64_t relocated = build_map(st->n, st->nl, st->pe_begin, dest, m, identity);
    if (!identity) execute_inplace(st, dest, relocated);
}

}  // namespace

std::uint64_t reorder(qrt_state* st, const int* dest) {
    QrMap m{};
    bool identity = false;
    const std::uint64_t relocated = build_map(st->n, st->nl, st->pe_begin, dest, m, identity);
    if (identity) return 0;
    flush_reorder(st);
    if (st->inplace) {
        execute_qr(st, dest);
        return relocated;
    }
    // Pulling a tile's sources over NVLink scatters each CTA's reads over the
    // whole peer buffer; past 2^31 amplitudes (32 GiB) per PE the translation
    // misses outweigh the saved exchange (34-qubit HEA on 4 GPUs: 0.31 s
    // slower than even the push exchange), so larger states run in place.
    if (fused_qr_enabled() && st->p > 1 && st->nl <= fused_qr_max_log2()) {
        st->qr_pending = true;  // the next gate pass gathers through it
        st->qr_dest.assign(dest, dest + st->n);
        return relocated;
    }
    execute_qr(st, dest);
    return relocated;
}

void flush_reorder(qrt_state* st) {
    if (!st->qr_pending) return;
    st->qr_pending = false;
    execute_qr(st, st->qr_dest.data());
}

void reorder_inplace_plan(int n, int p, const int* dest, int* pairs0, int* n0, int* pairs1, int* n1, int* cross,
                          int* k) {
    if (p < 1 || (p & (p - 1))) fail(QRT_ERR_CONFIG, "p must be a power of two");
    const int nl = n - __builtin_ctz(static_cast<unsigned>(p));
    QrMap m{};
    bool identity = false;
    (void)build_map(n, nl, 0, dest, m, identity);  // validates the permutation
    const InplacePlan P = plan_inplace(n, nl, dest);
    auto put = [](const std::vector<std::pair<int, int>>& v, int* out, int* cnt) {
        *cnt = static_cast<int>(v.size());
        for (std::size_t i = 0; i < v.size(); ++i) {
            out[2 * i] = v[i].first;
            out[2 * i + 1] = v[i].second;
        }
    };
    put(P.local[0], pairs0, n0);
    put(P.local[1], pairs1, n1);
    put(P.cross, cross, k);
}

// Single-process NVLink microbenchmark of the QR exchange kernels (one PE per
// GPU, CUDA peer access instead of IPC): the k highest local positions swap
// with k PE bits on n_gpus GPUs at once, push (reorder_kernel into a second
// buffer) or in place (exchange_kernel).  One process drives every GPU, so
// ncu can attach and read the NVLink counters (never wrap a multi-rank run).
void qr_bench(int n_gpus, int nl, int k, int inplace, int iters, double* ms_out, double* gbs_out) {
    if (n_gpus < 2 || n_gpus > 8 || (n_gpus & (n_gpus - 1))) fail(QRT_ERR_CONFIG, "n_gpus must be 2, 4 or 8");
    const int g = __builtin_ctz(static_cast<unsigned>(n_gpus));
    if (k < 1 || k > g) fail(QRT_ERR_CONFIG, "k must be in [1, log2 n_gpus]");
    if (nl < kTileBits || nl > 33) fail(QRT_ERR_CONFIG, "n_local must be in [12, 33]");
    if (iters < 1) fail(QRT_ERR_CONFIG, "iters must be >= 1");
    int ndev = 0;
    QRT_CUDA(cudaGetDeviceCount(&ndev));
    if (ndev < n_gpus) fail(QRT_ERR_NO_DEVICE, "not enough GPUs for the QR microbenchmark");
    int prev = 0;
    QRT_CUDA(cudaGetDevice(&prev));
    const int n = nl + g;
    const std::uint64_t amps = 1ull << nl;
    std::vector<amp_t*> b0(static_cast<std::size_t>(n_gpus), nullptr), b1(static_cast<std::size_t>(n_gpus), nullptr);
    std::vector<cudaStream_t> str(static_cast<std::size_t>(n_gpus), nullptr);
    std::vector<cudaEvent_t> e0(static_cast<std::size_t>(n_gpus), nullptr), e1(static_cast<std::size_t>(n_gpus), nullptr);
    std::vector<int> sms(static_cast<std::size_t>(n_gpus), 148);
    auto cleanup = [&] {
        for (int d = 0; d < n_gpus; ++d) {
            cudaSetDevice(d);
            cudaDeviceSynchronize();
            if (b0[static_cast<std::size_t>(d)]) cudaFree(b0[static_cast<std::size_t>(d)]);
            if (b1[static_cast<std::size_t>(d)]) cudaFree(b1[static_cast<std::size_t>(d)]);
            if (e0[static_cast<std::size_t>(d)]) cudaEventDestroy(e0[static_cast<std::size_t>(d)]);
            if (e1[static_cast<std::size_t>(d)]) cudaEventDestroy(e1[static_cast<std::size_t>(d)]);
            if (str[static_cast<std::size_t>(d)]) cudaStreamDestroy(str[static_cast<std::size_t>(d)]);
        }
        cudaSetDevice(prev);
    };
    try {
        for (int d = 0; d < n_gpus; ++d) {
            const auto D = static_cast<std::size_t>(d);
            QRT_CUDA(cudaSetDevice(d));
            QRT_CUDA(cudaDeviceGetAttribute(&sms[D], cudaDevAttrMultiProcessorCount, d));
            QRT_CUDA(cudaStreamCreateWithFlags(&str[D], cudaStreamNonBlocking));
            QRT_CUDA(cudaEventCreate(&e0[D]));
            QRT_CUDA(cudaEventCreate(&e1[D]));
            QRT_CUDA(cudaMalloc(&b0[D], amps * sizeof(amp_t)));
            QRT_CUDA(cudaMemset(b0[D], 0, amps * sizeof(amp_t)));
            if (!inplace) QRT_CUDA(cudaMalloc(&b1[D], amps * sizeof(amp_t)));
            for (int o = 0; o < n_gpus; ++o) {
                if (o == d) continue;
                const cudaError_t e = cudaDeviceEnablePeerAccess(o, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else QRT_CUDA(e);
            }
        }
        std::vector<int> dest(static_cast<std::size_t>(n));
        std::iota(dest.begin(), dest.end(), 0);
        for (int i = 0; i < k; ++i) {
            dest[static_cast<std::size_t>(nl - 1 - i)] = nl + i;
            dest[static_cast<std::size_t>(nl + i)] = nl - 1 - i;
        }
        std::vector<QrArgs> pa(static_cast<std::size_t>(n_gpus));
        std::vector<XchgArgs> xa(static_cast<std::size_t>(n_gpus));
        std::uint64_t relocated = 0;
        for (int d = 0; d < n_gpus; ++d) {
            const auto D = static_cast<std::size_t>(d);
            bool identity = false;
            relocated = build_map(n, nl, d, dest.data(), pa[D].m, identity);
            pa[D].src[0] = b0[D];
            for (int pe = 0; pe < n_gpus; ++pe) pa[D].dst[pe] = b1[static_cast<std::size_t>(pe)];
            const InplacePlan P = plan_inplace(n, nl, dest.data());
            XchgArgs& a = xa[D];
            a.pe_begin = d;
            a.k = static_cast<int>(P.cross.size());
            std::vector<char> used(static_cast<std::size_t>(nl), 0);
            for (int i = 0; i < a.k; ++i) {
                a.d_pos[i] = P.cross[static_cast<std::size_t>(i)].first;
                a.pe_bit[i] = P.cross[static_cast<std::size_t>(i)].second;
                used[static_cast<std::size_t>(a.d_pos[i])] = 1;
            }
            a.f = -1;
            for (int x = nl - 1; x >= 0; --x)
                if (!used[static_cast<std::size_t>(x)]) {
                    a.f = x;
                    used[static_cast<std::size_t>(x)] = 1;
                    break;
                }
            std::vector<int> rest;
            for (int x = 0; x < nl; ++x)
                if (!used[static_cast<std::size_t>(x)]) rest.push_back(x);
            make_deposit(rest, a.dep);
            a.nl = nl;
            a.p = n_gpus;
            for (int pe = 0; pe < n_gpus; ++pe) a.pe_ptr[pe] = b0[static_cast<std::size_t>(pe)];
        }
        double total_ms = 0.0;
        for (int it = 0; it <= iters; ++it) {  // iteration 0 warms up
            for (int d = 0; d < n_gpus; ++d) {
                const auto D = static_cast<std::size_t>(d);
                QRT_CUDA(cudaSetDevice(d));
                QRT_CUDA(cudaEventRecord(e0[D], str[D]));
                if (inplace) {
                    const std::uint64_t work = static_cast<std::uint64_t>((1 << xa[D].k) - 1) << xa[D].dep.n_hi;
                    const unsigned gx = static_cast<unsigned>(std::min<std::uint64_t>(work, static_cast<std::uint64_t>(sms[D]) * 8));
                    exchange_kernel<<<dim3(gx, 1), 256, 0, str[D]>>>(xa[D]);
                } else {
                    reorder_kernel<<<dim3(static_cast<unsigned>(1ull << pa[D].m.n_hi), 1), 256, 0, str[D]>>>(pa[D]);
                }
                QRT_CUDA(cudaGetLastError());
                QRT_CUDA(cudaEventRecord(e1[D], str[D]));
            }
            double worst = 0.0;
            for (int d = 0; d < n_gpus; ++d) {
                const auto D = static_cast<std::size_t>(d);
                QRT_CUDA(cudaSetDevice(d));
                QRT_CUDA(cudaEventSynchronize(e1[D]));
                float ms = 0.f;
                QRT_CUDA(cudaEventElapsedTime(&ms, e0[D], e1[D]));
                worst = std::max(worst, static_cast<double>(ms));
            }
            if (it > 0) total_ms += worst;
        }
        const double ms = total_ms / iters;
        const double bytes = 16.0 * static_cast<double>(relocated) / n_gpus;  // sent per GPU = received per GPU
        if (ms_out) *ms_out = ms;
        if (gbs_out) *gbs_out = bytes / (ms * 1e-3) / 1e9;
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
}

// Host-side replay of the kernel's index mapping for one source PE: for every
// source offset, the destination PE and offset the kernel stores it to.
void reorder_plan(int n, int p, const int* dest, int src_pe, std::uint64_t* dst_pe, std::uint64_t* dst_off,
                  std::uint64_t* relocated) {
    if (p < 1 || (p & (p - 1))) fail(QRT_ERR_CONFIG, "p must be a power of two");
    const int nl = n - __builtin_ctz(static_cast<unsigned>(p));
    if (nl < 1 || nl > 30) fail(QRT_ERR_CONFIG, "plan query supports 1 <= n-g <= 30");
    if (src_pe < 0 || src_pe >= p) fail(QRT_ERR_INVALID, "source PE out of range");
    QrMap m{};
    bool identity = false;
    const std::uint64_t rel = build_map(n, nl, 0, dest, m, identity);
    if (relocated) *relocated = rel;
    const std::uint64_t chunks = 1ull << m.n_hi;
    const int E = 1 << m.C, ncls = 1 << m.k;
    for (std::uint64_t chunk = 0; chunk < chunks; ++chunk)
        for (int cls = 0; cls < ncls; ++cls) {
            const Bases b = qr_bases(m, src_pe, chunk, cls);
            for (int e = 0; e < E; ++e) {
                const std::uint64_t so = b.src | qr_src_e(m, e);
                dst_pe[so] = static_cast<std::uint64_t>(b.pe);
                dst_off[so] = b.dst | qr_dst_e(m, e);
            }
        }
}

}  // namespace qrt
