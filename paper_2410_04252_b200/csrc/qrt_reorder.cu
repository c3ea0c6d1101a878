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
        for (int e = threadIdx.x; e < E; e += blockDim.x)
            dst[b.dst | qr_dst_e(a.m, e)] = __ldcs(&src[b.src | qr_src_e(a.m, e)]);
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

}  // namespace

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
        dim3 grid(static_cast<unsigned>(1ull << a.m.n_hi), static_cast<unsigned>(st->pe_count));
        reorder_kernel<<<grid, 256, 0, st->stream>>>(a);
        QRT_CUDA(cudaGetLastError());
        barrier_on_stream(st);
    }
    st->stats[QRT_K_QR].launches++;
    // bytes that cross to another PE (each way), counted for this process's PEs
    st->stats[QRT_K_QR].bytes += 16.0 * static_cast<double>(relocated) * st->pe_count / st->p;
    st->cur = nxt;
}

}  // namespace

std::uint64_t reorder(qrt_state* st, const int* dest) {
    QrMap m{};
    bool identity = false;
    const std::uint64_t relocated = build_map(st->n, st->nl, st->pe_begin, dest, m, identity);
    if (identity) return 0;
    flush_reorder(st);
    // Pulling a tile's sources over NVLink scatters each CTA's reads over the
    // whole peer buffer; past 2^30 amplitudes (16 GiB) per PE the translation
    // misses outweigh the saved exchange (34-qubit HEA on 4 GPUs: 0.31 s
    // slower), so large states keep the push exchange.
    static const int max_log2 = [] {
        const char* e = std::getenv("QRT_FUSED_QR_MAX_LOG2");
        return e ? std::atoi(e) : 30;
    }();
    if (fused_qr_enabled() && st->p > 1 && st->nl <= max_log2) {
        st->qr_pending = true;  // the next gate pass gathers through it
        st->qr_dest.assign(dest, dest + st->n);
        return relocated;
    }
    execute_reorder(st, dest);
    return relocated;
}

void flush_reorder(qrt_state* st) {
    if (!st->qr_pending) return;
    st->qr_pending = false;
    execute_reorder(st, st->qr_dest.data());
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
