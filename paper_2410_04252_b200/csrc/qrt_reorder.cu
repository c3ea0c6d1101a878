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

#include <numeric>

#include "qrt_internal.h"

namespace qrt {

namespace {

struct QrArgs {
    amp_t* dst[kMaxLocalPEs];  // alternate buffer of every PE (p <= 64)
    const amp_t* src[kMaxLocalPEs];
    int pe_begin;
    int C;          // chunk bits (destination-contiguous)
    int k;          // destination PE bits fed by source-local bits
    int n_hi;       // u_lo bits above the chunk
    // contribution tables for the low chunk bits (two 6-bit halves)
    std::uint64_t tab_src[2][64];
    std::uint64_t tab_dst[2][64];
    int hi_src_pos[64];  // for u_lo bits >= C: source / destination positions
    int hi_dst_pos[64];
    int cls_src_pos[8];  // for u_hi bits: source local position, destination PE bit
    int cls_dst_pe_bit[8];
    int g;               // global bits
    int j_dst_pos[8];    // source PE bit b -> destination position (local < nl or nl + pe bit)
    int nl;
};

__global__ void __launch_bounds__(256) reorder_kernel(const QrArgs a) {
    const int lpe = blockIdx.y;
    const int j = a.pe_begin + lpe;
    const std::uint64_t chunk = blockIdx.x;

    // constant parts from the chunk index and the source PE
    std::uint64_t src_base = 0, dst_base = 0;
    int pe_base = 0;
    for (int i = 0; i < a.n_hi; ++i) {
        const std::uint64_t bit = (chunk >> i) & 1ull;
        src_base |= bit << a.hi_src_pos[i];
        dst_base |= bit << a.hi_dst_pos[i];
    }
    for (int b = 0; b < a.g; ++b) {
        const int bit = (j >> b) & 1;
        const int t = a.j_dst_pos[b];
        if (t < a.nl)
            dst_base |= static_cast<std::uint64_t>(bit) << t;
        else
            pe_base |= bit << (t - a.nl);
    }
    const amp_t* __restrict__ src = a.src[lpe];
    const int E = 1 << a.C;
    const int ncls = 1 << a.k;
    for (int cls = 0; cls < ncls; ++cls) {
        std::uint64_t s_cls = src_base;
        int pe = pe_base;
        for (int i = 0; i < a.k; ++i) {
            const int bit = (cls >> i) & 1;
            s_cls |= static_cast<std::uint64_t>(bit) << a.cls_src_pos[i];
            pe |= bit << a.cls_dst_pe_bit[i];
        }
        amp_t* __restrict__ dst = a.dst[pe];
        for (int e = threadIdx.x; e < E; e += blockDim.x) {
            const std::uint64_t so = s_cls | a.tab_src[0][e & 63] | a.tab_src[1][(e >> 6) & 63];
            const std::uint64_t dof = dst_base | a.tab_dst[0][e & 63] | a.tab_dst[1][(e >> 6) & 63];
            dst[dof] = __ldcs(&src[so]);
        }
    }
    __threadfence_system();  // peer stores visible before the stream-ordered barrier
}

int find(std::vector<int>& parent, int x) {
    while (parent[static_cast<std::size_t>(x)] != x) x = parent[static_cast<std::size_t>(x)] = parent[static_cast<std::size_t>(parent[static_cast<std::size_t>(x)])];
    return x;
}

}  // namespace

std::uint64_t reorder(qrt_state* st, const int* dest) {
    const int n = st->n, nl = st->nl, g = n - nl;
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
        int a = find(parent, t), b = find(parent, src_of[static_cast<std::size_t>(t)]);
        if (a != b) parent[static_cast<std::size_t>(a)] = b;
    }
    int comps = 0;
    for (int x = 0; x < n; ++x) comps += find(parent, x) == x ? 1 : 0;
    const std::uint64_t relocated = (n >= 64 ? 0 : (1ull << n)) - (1ull << comps);

    bool identity = true;
    for (int s = 0; s < n; ++s) identity = identity && dest[s] == s;
    if (identity) return 0;

    if (st->p > kMaxLocalPEs) fail(QRT_ERR_CONFIG, "too many PEs for the reorder kernel");
    ensure_alt(st);

    // destination free positions: local F_L (ascending) and global F_G
    std::vector<int> fl, fg;
    for (int t = 0; t < n; ++t) {
        const int s = src_of[static_cast<std::size_t>(t)];
        if (s >= nl) continue;  // fed by a source PE bit
        (t < nl ? fl : fg).push_back(t);
    }
    const int k = static_cast<int>(fg.size());
    if (k > 8) fail(QRT_ERR_CONFIG, "reorder moves more than 8 local bits to global positions");
    QrArgs a{};
    a.pe_begin = st->pe_begin;
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
    const int nxt = st->cur ^ 1;
    for (int pe = 0; pe < st->p; ++pe) a.dst[pe] = st->peer[nxt][static_cast<std::size_t>(pe)];
    for (int i = 0; i < st->pe_count; ++i) a.src[i] = st->live(i);

    {
        ProfileScope prof(st, QRT_K_QR);
        dim3 grid(static_cast<unsigned>(1ull << a.n_hi), static_cast<unsigned>(st->pe_count));
        reorder_kernel<<<grid, 256, 0, st->stream>>>(a);
        QRT_CUDA(cudaGetLastError());
        barrier_on_stream(st);
    }
    st->stats[QRT_K_QR].launches++;
    // bytes that cross to another PE (each way), counted for this process's PEs
    st->stats[QRT_K_QR].bytes += 16.0 * static_cast<double>(relocated) * st->pe_count / st->p;
    st->cur = nxt;
    return relocated;
}

}  // namespace qrt
