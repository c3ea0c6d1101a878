// libqrt — C ABI entry points (include/qrt.h), device state management,
// the one-process-per-GPU communicator (NCCL for barriers / gathers, CUDA IPC
// for direct NVLink peer stores) and measurement plumbing.
//
// Reference mapping: qrt_state_create/set_zero <- init_state
// (dist_sim.cpp:122-131); upload/download <- init_state(ref)/flatten
// (:133-161, position order); qrt_norm <- DistributedState::norm (:115-120).

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include <unistd.h>

#include "qrt_internal.h"

namespace qrt {

namespace {
thread_local std::string g_last_error;

// QRT_TRACE=<path>: every traced ABI call appends "name t_begin_us t_end_us"
// (host wall clock, process-relative) — the host side of the timeline.
struct Tracer {
    std::FILE* f = nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    std::mutex mu;
    Tracer() {
        if (const char* path = std::getenv("QRT_TRACE")) {
            std::string name = std::string(path) + "." + std::to_string(static_cast<long>(getpid()));
            f = std::fopen(name.c_str(), "w");
        }
    }
    ~Tracer() {
        if (f) std::fclose(f);
    }
    double now_us() const {
        return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    }
};
Tracer& tracer() {
    static Tracer t;
    return t;
}
struct TraceScope {
    const char* name;
    double b;
    explicit TraceScope(const char* n) : name(n), b(tracer().f ? tracer().now_us() : 0.0) {}
    ~TraceScope() {
        Tracer& t = tracer();
        if (!t.f) return;
        std::lock_guard<std::mutex> lk(t.mu);
        std::fprintf(t.f, "%s %.1f %.1f\n", name, b, t.now_us());
        std::fflush(t.f);
    }
};

template <class F>
qrt_status guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return QRT_OK;
    } catch (const Failure& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        g_last_error = "host out of memory";
        return QRT_ERR_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return QRT_ERR_INVALID;
    }
}

void require(bool ok, qrt_status s, const std::string& msg) {
    if (!ok) fail(s, msg);
}

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        QRT_CUDA(cudaGetDevice(&prev));
        if (prev != dev) QRT_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

__global__ void zero_state_kernel(amp_t* __restrict__ v, std::uint64_t count, int set_first) {
    std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
    for (; i < count; i += stride) v[i] = make_double2((set_first && i == 0) ? 1.0 : 0.0, 0.0);
}

// Parked states, reused by qrt_state_create with the same (n, p, device,
// comm): a VQE loop creates one state per iteration (evaluate_energy,
// dist_sim.cpp:357-363), and re-allocating tens of GiB plus re-opening IPC
// peer mappings every iteration would dominate small steps.  Every rank
// parks and reuses in the same order, so peer mappings stay valid.
std::mutex g_cache_mu;
std::vector<qrt_state*> g_cache;
// Communicators alive now, by generation id: a parked state is reused only by
// the communicator that created it (a new one allocated at the same address
// has a new id), and a state whose communicator is gone is freed, not parked.
std::uint64_t g_comm_gen = 0;
std::vector<std::pair<const qrt_comm*, std::uint64_t>> g_live_comms;

bool comm_alive(const qrt_comm* c, std::uint64_t gen) {
    if (!c) return true;
    for (auto& [p, g] : g_live_comms)
        if (p == c && g == gen) return true;
    return false;
}

void free_state(qrt_state* st) {
    DeviceGuard g(st->device);
    if (st->stream) cudaStreamSynchronize(st->stream);
    for (void* ptr : st->ipc_opened) cudaIpcCloseMemHandle(ptr);
    for (int b = 0; b < 2; ++b)
        for (auto* ptr : st->bufs[b])
            if (ptr) cudaFree(ptr);
    if (st->d_red) cudaFree(st->d_red);
    if (st->d_ops) cudaFree(st->d_ops);
    if (st->h_pinned) cudaFreeHost(st->h_pinned);
    if (st->d_flag) cudaFree(st->d_flag);
    if (st->ev0) cudaEventDestroy(st->ev0);
    if (st->ev1) cudaEventDestroy(st->ev1);
    if (st->ev2) cudaEventDestroy(st->ev2);
    if (st->ev3) cudaEventDestroy(st->ev3);
    if (st->stream) cudaStreamDestroy(st->stream);
    delete st;
}

qrt_state* take_cached(int n, int p, int device, qrt_comm* comm, int inplace) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (std::size_t i = 0; i < g_cache.size(); ++i) {
        qrt_state* st = g_cache[i];
        if (st->n == n && st->p == p && st->device == device && st->comm == comm &&
            (inplace < 0 || st->inplace == (inplace != 0)) &&
            (!comm || st->comm_gen == comm->gen)) {
            g_cache.erase(g_cache.begin() + static_cast<std::ptrdiff_t>(i));
            return st;
        }
    }
    return nullptr;
}

int grid_for(std::uint64_t items, int threads, int sms) {
    std::uint64_t want = (items + threads - 1) / threads;
    std::uint64_t cap = static_cast<std::uint64_t>(sms) * 8;
    return static_cast<int>(want < cap ? (want == 0 ? 1 : want) : cap);
}

// Single-buffer (in-place QR) policy (QRT_QR_INPLACE: 0 never, 1 always,
// unset = auto).  The second buffer only serves the fused (pull) QR, which is
// used up to 2^30 amplitudes per PE; every executed QR runs in place anyway
// (qrt_reorder.cu execute_qr).  So auto keeps one buffer when the fused QR
// cannot apply, or when this process's sub-vectors twice over would not fit
// in the device memory free now (minus 4 GiB of headroom), e.g. 34 qubits on
// 2 GPUs (2 x 128 GiB per GPU).
int forced_inplace(int p) {  // -1: automatic
    if (p < 2) return 0;
    const char* e = std::getenv("QRT_QR_INPLACE");
    if (e && *e) return std::atoi(e) != 0 ? 1 : 0;
    return -1;
}

bool choose_inplace(int p, int nl, std::uint64_t state_bytes) {
    const int f = forced_inplace(p);
    if (f >= 0) return f != 0;
    if (!fused_qr_enabled() || nl > fused_qr_max_log2()) return true;
    std::size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    const std::uint64_t headroom = 4ull << 30;
    return 2 * state_bytes + headroom > free_b;
}

}  // namespace

void fail(qrt_status s, const std::string& msg) { throw Failure(s, msg); }

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    qrt_status s = (e == cudaErrorMemoryAllocation) ? QRT_ERR_OOM
                   : (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) ? QRT_ERR_NO_DEVICE
                                                                                   : QRT_ERR_CUDA;
    fail(s, std::string(cudaGetErrorString(e)) + " in " + what + " at " + file + ":" + std::to_string(line));
}

void nccl_check(ncclResult_t r, const char* what, const char* file, int line) {
    if (r == ncclSuccess) return;
    fail(QRT_ERR_NCCL, std::string(ncclGetErrorString(r)) + " in " + what + " at " + file + ":" + std::to_string(line));
}

ProfileScope::ProfileScope(qrt_state* s, int f, bool inner_scope) : st(s), fam(f), inner(inner_scope) {
    if (st->profile) QRT_CUDA(cudaEventRecord(inner ? st->ev2 : st->ev0, st->stream));
}
ProfileScope::~ProfileScope() {
    if (!st->profile) return;
    // Destructors must not throw (this one may run during unwinding): a
    // failure here leaves the timing out and is caught by the next checked call.
    float ms = 0.f;
    cudaEvent_t b = inner ? st->ev2 : st->ev0, e = inner ? st->ev3 : st->ev1;
    if (cudaEventRecord(e, st->stream) == cudaSuccess && cudaEventSynchronize(e) == cudaSuccess &&
        cudaEventElapsedTime(&ms, b, e) == cudaSuccess)
        st->stats[fam].ms += ms;
}

void ensure_alt(qrt_state* st) {
    if (!st->bufs[1].empty() && st->bufs[1][0] != nullptr) return;
    st->bufs[1].assign(static_cast<std::size_t>(st->pe_count), nullptr);
    for (int i = 0; i < st->pe_count; ++i) QRT_CUDA(cudaMalloc(&st->bufs[1][static_cast<std::size_t>(i)], st->amps * sizeof(amp_t)));
    // single-process: the peer tables are the local buffers
    for (int b = 0; b < 2; ++b)
        for (int i = 0; i < st->pe_count; ++i)
            st->peer[b][static_cast<std::size_t>(st->pe_begin + i)] = st->bufs[b][static_cast<std::size_t>(i)];
}

void* ensure_ops(qrt_state* st, std::size_t bytes) {
    if (bytes > st->ops_cap) {
        if (st->d_ops) QRT_CUDA(cudaFree(st->d_ops));
        std::size_t cap = bytes < (1u << 20) ? (1u << 20) : bytes + bytes / 2;
        QRT_CUDA(cudaMalloc(&st->d_ops, cap));
        st->ops_cap = cap;
    }
    return st->d_ops;
}

void* ensure_pinned(qrt_state* st, std::size_t bytes) {
    if (bytes > st->pinned_cap) {
        if (st->h_pinned) {
            QRT_CUDA(cudaStreamSynchronize(st->stream));
            QRT_CUDA(cudaFreeHost(st->h_pinned));
        }
        std::size_t cap = bytes < (1u << 20) ? (1u << 20) : bytes + bytes / 2;
        QRT_CUDA(cudaMallocHost(&st->h_pinned, cap));
        st->pinned_cap = cap;
    }
    return st->h_pinned;
}

double* ensure_red(qrt_state* st, std::size_t doubles) {
    if (doubles > st->red_cap) {
        if (st->d_red) QRT_CUDA(cudaFree(st->d_red));
        QRT_CUDA(cudaMalloc(&st->d_red, doubles * sizeof(double)));
        st->red_cap = doubles;
    }
    return st->d_red;
}

void barrier_on_stream(qrt_state* st) {
    if (!st->comm || st->comm->world == 1) return;
    QRT_NCCL(ncclAllReduce(st->d_flag, st->d_flag, 1, ncclInt32, ncclSum, st->comm->nccl, st->stream));
    st->spare_busy = false;  // work enqueued before this point is complete on every rank
}

}  // namespace qrt

using namespace qrt;

// ============================================================================
extern "C" {

const char* qrt_last_error(void) { return g_last_error.c_str(); }
int qrt_abi_version(void) { return QRT_ABI_VERSION; }
int qrt_build_flags(void) { return kBuildFlags; }

qrt_status qrt_device_count(int* out) {
    return guarded([&] {
        require(out != nullptr, QRT_ERR_INVALID, "null out");
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) {
            cudaGetLastError();
            *out = 0;
            return;
        }
        int good = 0;
        for (int d = 0; d < n; ++d) {
            cudaDeviceProp prop{};
            if (cudaGetDeviceProperties(&prop, d) == cudaSuccess && prop.major == 10) ++good;
        }
        *out = good;
    });
}

qrt_status qrt_comm_unique_id(unsigned char id[128]) {
    return guarded([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId uid;
        QRT_NCCL(ncclGetUniqueId(&uid));
        std::memcpy(id, &uid, 128);
    });
}

qrt_status qrt_comm_init(int rank, int world, int device, const unsigned char id[128], qrt_comm** out) {
    return guarded([&] {
        require(out && world >= 1 && rank >= 0 && rank < world, QRT_ERR_INVALID, "bad communicator arguments");
        auto* c = new qrt_comm;
        c->rank = rank;
        c->world = world;
        c->device = device;
        DeviceGuard g(device);
        if (world > 1) {
            ncclUniqueId uid;
            std::memcpy(&uid, id, 128);
            QRT_NCCL(ncclCommInitRank(&c->nccl, world, uid, rank));
            QRT_CUDA(cudaMalloc(&c->d_flag, sizeof(int)));
            QRT_CUDA(cudaMemset(c->d_flag, 0, sizeof(int)));
        }
        {
            std::lock_guard<std::mutex> lk(g_cache_mu);
            c->gen = ++g_comm_gen;
            g_live_comms.emplace_back(c, c->gen);
        }
        *out = c;
    });
}

qrt_status qrt_comm_barrier(qrt_comm* comm) {
    return guarded([&] {
        require(comm != nullptr, QRT_ERR_INVALID, "null comm");
        if (comm->world == 1) return;
        DeviceGuard g(comm->device);
        QRT_NCCL(ncclAllReduce(comm->d_flag, comm->d_flag, 1, ncclInt32, ncclSum, comm->nccl, nullptr));
        QRT_CUDA(cudaStreamSynchronize(nullptr));
    });
}

qrt_status qrt_comm_destroy(qrt_comm* comm) {
    return guarded([&] {
        if (!comm) return;
        // Parked states of this communicator: every rank parks in the same
        // order, so meet once (no peer still reads an IPC-exported buffer),
        // then free them.
        std::vector<qrt_state*> mine;
        {
            std::lock_guard<std::mutex> lk(g_cache_mu);
            for (auto it = g_cache.begin(); it != g_cache.end();) {
                if ((*it)->comm == comm && (*it)->comm_gen == comm->gen) {
                    mine.push_back(*it);
                    it = g_cache.erase(it);
                } else {
                    ++it;
                }
            }
            for (auto it = g_live_comms.begin(); it != g_live_comms.end(); ++it)
                if (it->first == comm && it->second == comm->gen) {
                    g_live_comms.erase(it);
                    break;
                }
        }
        if (!mine.empty() && comm->world > 1) {
            DeviceGuard g(comm->device);
            QRT_NCCL(ncclAllReduce(comm->d_flag, comm->d_flag, 1, ncclInt32, ncclSum, comm->nccl, nullptr));
            QRT_CUDA(cudaStreamSynchronize(nullptr));
        }
        for (qrt_state* st : mine) free_state(st);
        if (comm->d_flag) {
            DeviceGuard g(comm->device);
            cudaFree(comm->d_flag);
        }
        if (comm->nccl) ncclCommDestroy(comm->nccl);
        delete comm;
    });
}

qrt_status qrt_state_create(int n, int p, int device, qrt_comm* comm, qrt_state** out) {
    TraceScope trace_("qrt_state_create");
    return guarded([&] {
        require(out != nullptr, QRT_ERR_INVALID, "null out");
        require(p >= 1 && (p & (p - 1)) == 0, QRT_ERR_CONFIG, "p must be a power of two");
        require(n >= 1 && n <= 62, QRT_ERR_CONFIG, "qubit count out of range");
        int g = __builtin_ctz(static_cast<unsigned>(p));
        require(n - g >= 1, QRT_ERR_TOO_MANY_PES, "p = " + std::to_string(p) + " leaves no local qubit");
        int world = comm ? comm->world : 1;
        int rank = comm ? comm->rank : 0;
        require(p % world == 0, QRT_ERR_CONFIG, "p must be a multiple of the world size");
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            fail(QRT_ERR_NO_DEVICE, "no CUDA device visible");
        }
        require(device >= 0 && device < ndev, QRT_ERR_NO_DEVICE, "device index out of range");
        DeviceGuard dg(device);
        // FusedSource / QrArgs / XchgArgs address every PE of a multi-process
        // state through fixed 64-entry tables.
        require(world == 1 || p <= kMaxLocalPEs, QRT_ERR_CONFIG,
                "p = " + std::to_string(p) + " exceeds the 64-PE limit of a multi-process state");
        const std::uint64_t state_bytes = (1ull << (n - g)) * sizeof(amp_t) * static_cast<std::uint64_t>(p / world);
        // a parked state of the same shape is reused whatever its QR mode
        // (unless QRT_QR_INPLACE forces one): its memory is what the
        // automatic choice would otherwise miss
        if (qrt_state* cached = take_cached(n, p, device, comm, forced_inplace(p))) {
            // buffer parity is kept (peers address the same physical buffers)
            cached->profile = false;
            for (auto& sct : cached->stats) sct = qrt_kernel_stats{};
            for (int i = 0; i < cached->pe_count; ++i)
                zero_state_kernel<<<grid_for(cached->amps, 256, cached->sm_count), 256, 0, cached->stream>>>(
                    cached->live(i), cached->amps, cached->pe_begin + i == 0);
            QRT_CUDA(cudaGetLastError());
            cached->stats[QRT_K_MISC].launches += static_cast<std::uint64_t>(cached->pe_count);
            barrier_on_stream(cached);  // collective, like a fresh create
            QRT_CUDA(cudaStreamSynchronize(cached->stream));
            *out = cached;
            return;
        }

        const bool inplace = choose_inplace(p, n - g, state_bytes);
        auto st = new qrt_state;
        st->n = n;
        st->p = p;
        st->nl = n - g;
        st->device = device;
        st->comm = comm;
        st->comm_gen = comm ? comm->gen : 0;
        st->inplace = inplace;
        QRT_CUDA(cudaDeviceGetAttribute(&st->sm_count, cudaDevAttrMultiProcessorCount, device));
        st->pe_count = p / world;
        require(st->pe_count <= kMaxLocalPEs, QRT_ERR_CONFIG, "too many PEs per process");
        st->pe_begin = rank * st->pe_count;
        st->amps = 1ull << st->nl;
        try {
            QRT_CUDA(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking));
            QRT_CUDA(cudaEventCreate(&st->ev0));
            QRT_CUDA(cudaEventCreate(&st->ev1));
            QRT_CUDA(cudaEventCreate(&st->ev2));
            QRT_CUDA(cudaEventCreate(&st->ev3));
            QRT_CUDA(cudaMalloc(&st->d_flag, sizeof(int)));
            QRT_CUDA(cudaMemsetAsync(st->d_flag, 0, sizeof(int), st->stream));
            if (comm && world > 1) {  // every rank must take the same QR mode
                int v = st->inplace ? 1 : 0;
                QRT_CUDA(cudaMemcpyAsync(st->d_flag, &v, sizeof(int), cudaMemcpyHostToDevice, st->stream));
                QRT_NCCL(ncclAllReduce(st->d_flag, st->d_flag, 1, ncclInt32, ncclMax, comm->nccl, st->stream));
                QRT_CUDA(cudaMemcpyAsync(&v, st->d_flag, sizeof(int), cudaMemcpyDeviceToHost, st->stream));
                QRT_CUDA(cudaStreamSynchronize(st->stream));
                st->inplace = v != 0;
            }
            for (int b = 0; b < 2; ++b) {
                st->bufs[b].assign(static_cast<std::size_t>(st->pe_count), nullptr);
                st->peer[b].assign(static_cast<std::size_t>(p), nullptr);
            }
            const bool multi = comm && world > 1;
            // multi-process: both buffers up front (IPC-exported); in-place
            // QR states never allocate the second one
            const int nb = (multi && !st->inplace) ? 2 : 1;
            for (int b = 0; b < nb; ++b)
                for (int i = 0; i < st->pe_count; ++i)
                    QRT_CUDA(cudaMalloc(&st->bufs[b][static_cast<std::size_t>(i)], st->amps * sizeof(amp_t)));
            for (int b = 0; b < nb; ++b)
                for (int i = 0; i < st->pe_count; ++i)
                    st->peer[b][static_cast<std::size_t>(st->pe_begin + i)] = st->bufs[b][static_cast<std::size_t>(i)];
            if (multi) {
                // Exchange IPC handles of the buffers of every PE (all-gather).
                const std::size_t per = static_cast<std::size_t>(nb * st->pe_count) * sizeof(cudaIpcMemHandle_t);
                std::vector<cudaIpcMemHandle_t> mine(static_cast<std::size_t>(nb * st->pe_count));
                for (int b = 0; b < nb; ++b)
                    for (int i = 0; i < st->pe_count; ++i)
                        QRT_CUDA(cudaIpcGetMemHandle(&mine[static_cast<std::size_t>(b * st->pe_count + i)],
                                                     st->bufs[b][static_cast<std::size_t>(i)]));
                char* d_all = nullptr;
                QRT_CUDA(cudaMalloc(&d_all, per * static_cast<std::size_t>(world)));
                QRT_CUDA(cudaMemcpyAsync(d_all + per * static_cast<std::size_t>(rank), mine.data(), per,
                                         cudaMemcpyHostToDevice, st->stream));
                QRT_NCCL(ncclAllGather(d_all + per * static_cast<std::size_t>(rank), d_all, per, ncclChar,
                                       comm->nccl, st->stream));
                std::vector<cudaIpcMemHandle_t> all(static_cast<std::size_t>(nb * st->pe_count * world));
                QRT_CUDA(cudaMemcpyAsync(all.data(), d_all, per * static_cast<std::size_t>(world), cudaMemcpyDeviceToHost,
                                         st->stream));
                QRT_CUDA(cudaStreamSynchronize(st->stream));
                QRT_CUDA(cudaFree(d_all));
                for (int r = 0; r < world; ++r) {
                    if (r == rank) continue;
                    for (int b = 0; b < nb; ++b)
                        for (int i = 0; i < st->pe_count; ++i) {
                            void* ptr = nullptr;
                            QRT_CUDA(cudaIpcOpenMemHandle(
                                &ptr, all[static_cast<std::size_t>((r * nb + b) * st->pe_count + i)],
                                cudaIpcMemLazyEnablePeerAccess));
                            st->peer[b][static_cast<std::size_t>(r * st->pe_count + i)] = static_cast<amp_t*>(ptr);
                            st->ipc_opened.push_back(ptr);
                        }
                }
            }
            for (int i = 0; i < st->pe_count; ++i)
                zero_state_kernel<<<grid_for(st->amps, 256, st->sm_count), 256, 0, st->stream>>>(
                    st->bufs[0][static_cast<std::size_t>(i)], st->amps, st->pe_begin + i == 0);
            QRT_CUDA(cudaGetLastError());
            st->stats[QRT_K_MISC].launches += static_cast<std::uint64_t>(st->pe_count);
            QRT_CUDA(cudaStreamSynchronize(st->stream));
            if (multi) {
                barrier_on_stream(st);
                QRT_CUDA(cudaStreamSynchronize(st->stream));
            }
        } catch (...) {
            free_state(st);
            throw;
        }
        *out = st;
    });
}

qrt_status qrt_state_destroy(qrt_state* st) {
    TraceScope trace_("qrt_state_destroy");
    return guarded([&] {
        if (!st) return;
        st->qr_pending = false;
        {
            DeviceGuard g(st->device);
            QRT_CUDA(cudaStreamSynchronize(st->stream));
        }
        std::lock_guard<std::mutex> lk(g_cache_mu);
        if (!comm_alive(st->comm, st->comm_gen)) {
            free_state(st);  // its communicator is gone: never reusable
            return;
        }
        g_cache.push_back(st);  // parked; qrt_release_cache / qrt_comm_destroy free
    });
}

qrt_status qrt_release_cache(void) {
    return guarded([&] {
        std::vector<qrt_state*> all;
        {
            std::lock_guard<std::mutex> lk(g_cache_mu);
            all.swap(g_cache);
        }
        // Multi-process states: meet first so no peer still reads a buffer
        // this rank exported (every rank releases the same parked states).
        for (qrt_state* st : all)
            if (st->comm && st->comm->world > 1 && comm_alive(st->comm, st->comm_gen)) {
                DeviceGuard g(st->device);
                barrier_on_stream(st);
                QRT_CUDA(cudaStreamSynchronize(st->stream));
            }
        for (qrt_state* st : all) free_state(st);
    });
}

qrt_status qrt_state_mode(const qrt_state* st, int* inplace_qr, int* sm_count) {
    return guarded([&] {
        require(st != nullptr, QRT_ERR_INVALID, "null state");
        if (inplace_qr) *inplace_qr = st->inplace ? 1 : 0;
        if (sm_count) *sm_count = st->sm_count;
    });
}

qrt_status qrt_state_info(const qrt_state* st, int* n, int* p, int* pe_begin, int* pe_count) {
    return guarded([&] {
        require(st != nullptr, QRT_ERR_INVALID, "null state");
        if (n) *n = st->n;
        if (p) *p = st->p;
        if (pe_begin) *pe_begin = st->pe_begin;
        if (pe_count) *pe_count = st->pe_count;
    });
}

qrt_status qrt_state_set_zero(qrt_state* st) {
    return guarded([&] {
        require(st != nullptr, QRT_ERR_INVALID, "null state");
        DeviceGuard g(st->device);
        st->qr_pending = false;  // |0...0> is the same in every layout
        for (int i = 0; i < st->pe_count; ++i)
            zero_state_kernel<<<grid_for(st->amps, 256, st->sm_count), 256, 0, st->stream>>>(st->live(i), st->amps,
                                                                               st->pe_begin + i == 0);
        QRT_CUDA(cudaGetLastError());
        st->stats[QRT_K_MISC].launches += static_cast<std::uint64_t>(st->pe_count);
        QRT_CUDA(cudaStreamSynchronize(st->stream));
    });
}

qrt_status qrt_state_upload(qrt_state* st, int pe, const double* amps) {
    TraceScope trace_("qrt_state_upload");
    return guarded([&] {
        require(st && amps, QRT_ERR_INVALID, "null argument");
        require(pe >= st->pe_begin && pe < st->pe_begin + st->pe_count, QRT_ERR_INVALID, "PE not owned by this process");
        DeviceGuard g(st->device);
        flush_reorder(st);
        QRT_CUDA(cudaMemcpyAsync(st->live(pe - st->pe_begin), amps, st->amps * sizeof(amp_t), cudaMemcpyHostToDevice,
                                 st->stream));
        QRT_CUDA(cudaStreamSynchronize(st->stream));
    });
}

qrt_status qrt_state_download(const qrt_state* st, int pe, double* amps) {
    TraceScope trace_("qrt_state_download");
    return guarded([&] {
        require(st && amps, QRT_ERR_INVALID, "null argument");
        require(pe >= st->pe_begin && pe < st->pe_begin + st->pe_count, QRT_ERR_INVALID, "PE not owned by this process");
        DeviceGuard g(st->device);
        flush_reorder(const_cast<qrt_state*>(st));
        QRT_CUDA(cudaMemcpyAsync(amps, st->live(pe - st->pe_begin), st->amps * sizeof(amp_t), cudaMemcpyDeviceToHost,
                                 st->stream));
        QRT_CUDA(cudaStreamSynchronize(st->stream));
    });
}

qrt_status qrt_apply_gates(qrt_state* st, int n_gates, const int* arity, const int* pos, const double* mats,
                           const unsigned* flags) {
    TraceScope trace_("qrt_apply_gates");
    return guarded([&] {
        require(st != nullptr, QRT_ERR_INVALID, "null state");
        if (n_gates == 0) return;
        require(arity && pos, QRT_ERR_INVALID, "null gate arrays");
        require(mats != nullptr, QRT_ERR_MISSING_PAYLOAD, "gate payloads missing");
        DeviceGuard g(st->device);
        st->stats[QRT_K_GATES].calls++;
        apply_gates(st, n_gates, arity, pos, mats, flags);
        QRT_CUDA(cudaStreamSynchronize(st->stream));
    });
}

qrt_status qrt_reorder(qrt_state* st, const int* dest, std::uint64_t* relocated) {
    TraceScope trace_("qrt_reorder");
    return guarded([&] {
        require(st && dest, QRT_ERR_INVALID, "null argument");
        DeviceGuard g(st->device);
        st->stats[QRT_K_QR].calls++;
        std::uint64_t moved = reorder(st, dest);
        QRT_CUDA(cudaStreamSynchronize(st->stream));
        if (relocated) *relocated = moved;
    });
}

qrt_status qrt_qr_bench(int n_gpus, int n_local, int k, int inplace, int iters, double* ms_per_qr,
                        double* gbs_per_direction) {
    return guarded([&] { qr_bench(n_gpus, n_local, k, inplace, iters, ms_per_qr, gbs_per_direction); });
}

qrt_status qrt_reorder_inplace_plan(int n, int p, const int* dest, int* local_pairs0, int* n0, int* local_pairs1,
                                    int* n1, int* cross_pairs, int* k) {
    return guarded([&] {
        require(dest && local_pairs0 && n0 && local_pairs1 && n1 && cross_pairs && k, QRT_ERR_INVALID, "null argument");
        require(n >= 1 && n <= 62, QRT_ERR_CONFIG, "qubit count out of range");
        reorder_inplace_plan(n, p, dest, local_pairs0, n0, local_pairs1, n1, cross_pairs, k);
    });
}

qrt_status qrt_reorder_plan(int n, int p, const int* dest, int src_pe, std::uint64_t* dst_pe, std::uint64_t* dst_off,
                            std::uint64_t* relocated) {
    return guarded([&] {
        require(dest && dst_pe && dst_off, QRT_ERR_INVALID, "null argument");
        reorder_plan(n, p, dest, src_pe, dst_pe, dst_off, relocated);
    });
}

qrt_status qrt_pauli_expectation(qrt_state* st, int n_terms, const std::uint64_t* x, const std::uint64_t* y,
                                 const std::uint64_t* z, const std::uint64_t* gz, const double* coeffs,
                                 double* partial) {
    TraceScope trace_("qrt_pauli_expectation");
    return guarded([&] {
        require(st && partial, QRT_ERR_INVALID, "null argument");
        require(n_terms == 0 || (x && y && z && gz && coeffs), QRT_ERR_INVALID, "null term arrays");
        DeviceGuard g(st->device);
        st->stats[QRT_K_PAULI].calls++;
        flush_reorder(st);
        pauli_expectation(st, n_terms, x, y, z, gz, coeffs, partial);
    });
}

qrt_status qrt_pauli_plan_info(int n_local, int n_terms, const std::uint64_t* x, const std::uint64_t* y,
                               const std::uint64_t* z, const std::uint64_t* gz, const double* coeffs, int* passes,
                               int* groups, int* wide_groups, double* seconds) {
    return guarded([&] {
        require(n_local >= 1 && n_local <= 62, QRT_ERR_INVALID, "n_local out of range");
        require(n_terms == 0 || (x && y && z && gz && coeffs), QRT_ERR_INVALID, "null term arrays");
        pauli_plan_info(n_local, n_terms, x, y, z, gz, coeffs, passes, groups, wide_groups, seconds);
    });
}

qrt_status qrt_gate_plan_info(int n_local, int n_gates, const int* arity, const int* pos, const double* mats,
                              const unsigned* flags, int* passes, int* light_passes, int* light_stages, int* fused) {
    return guarded([&] {
        require(n_gates >= 0 && (n_gates == 0 || (arity && pos && mats)), QRT_ERR_INVALID, "null gate arrays");
        gate_plan_info(n_local, n_gates, arity, pos, mats, flags, passes, light_passes, light_stages, fused);
    });
}

qrt_status qrt_norm(qrt_state* st, double* out) {
    TraceScope trace_("qrt_norm");
    return guarded([&] {
        require(st && out, QRT_ERR_INVALID, "null argument");
        DeviceGuard g(st->device);
        flush_reorder(st);
        *out = norm(st);
    });
}

qrt_status qrt_profile_enable(qrt_state* st, int on) {
    return guarded([&] {
        require(st != nullptr, QRT_ERR_INVALID, "null state");
        st->profile = on != 0;
    });
}

qrt_status qrt_stats(const qrt_state* st, qrt_kernel_stats out[QRT_K_COUNT]) {
    return guarded([&] {
        require(st && out, QRT_ERR_INVALID, "null argument");
        for (int i = 0; i < QRT_K_COUNT; ++i) out[i] = st->stats[i];
    });
}

qrt_status qrt_stats_reset(qrt_state* st) {
    return guarded([&] {
        require(st != nullptr, QRT_ERR_INVALID, "null state");
        for (auto& s : st->stats) s = qrt_kernel_stats{};
    });
}

qrt_status qrt_state_stream(const qrt_state* st, void** stream) {
    return guarded([&] {
        require(st && stream, QRT_ERR_INVALID, "null argument");
        *stream = st->stream;
    });
}

qrt_status qrt_synchronize(qrt_state* st) {
    return guarded([&] {
        require(st != nullptr, QRT_ERR_INVALID, "null state");
        DeviceGuard g(st->device);
        QRT_CUDA(cudaStreamSynchronize(st->stream));
    });
}

}  // extern "C"
