// Internal declarations of libqrt (the C ABI in include/qrt.h).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "qrt.h"

namespace qrt {

// Thrown inside the library, converted to a status + qrt_last_error() at the
// ABI boundary.
struct Failure : std::runtime_error {
    qrt_status status;
    Failure(qrt_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] void fail(qrt_status s, const std::string& msg);
void cuda_check(cudaError_t e, const char* what, const char* file, int line);
void nccl_check(ncclResult_t r, const char* what, const char* file, int line);
#define QRT_CUDA(x) ::qrt::cuda_check((x), #x, __FILE__, __LINE__)
#define QRT_NCCL(x) ::qrt::nccl_check((x), #x, __FILE__, __LINE__)

using amp_t = double2;  // (re, im), 16 B, the HBM unit

// Checked build (libqrt_checked.so, -DQRT_CHECKS): device-side bounds and
// invariant checks in the kernels; a failure prints the condition and traps
// (the call then fails with QRT_ERR_CUDA).  compute-sanitizer is closed on
// the GPU pool, so tests run the small parity cases through this build.
#ifdef QRT_CHECKS
#define QRT_DCHECK(cond)                                                                        \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("QRT_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
inline constexpr int kBuildFlags = 1;
#else
#define QRT_DCHECK(cond) ((void)0)
inline constexpr int kBuildFlags = 0;
#endif

inline constexpr int kMaxLocalPEs = 64;  // PEs one process may own
inline constexpr int kTileBits = 12;     // smem tile: 2^12 amplitudes = 64 KiB
inline constexpr int kCoalBits = 4;      // low positions always inside a tile (256 B runs)
inline constexpr int kMaxTileGateK = 7;  // dense gates up to 7 qubits run inside a tile
inline constexpr int kThreads = 256;

}  // namespace qrt

struct qrt_comm {
    int rank = 0;
    int world = 1;
    int device = 0;
    ncclComm_t nccl = nullptr;
    int* d_flag = nullptr;  // barrier word of qrt_comm_barrier (allocated once)
    std::uint64_t gen = 0;  // generation id: keys the parked-state cache
};

struct KernelCounters {
    qrt_kernel_stats s{};
};

struct qrt_state {
    int n = 0;
    int p = 1;
    int nl = 0;  // local positions
    int device = 0;
    qrt_comm* comm = nullptr;
    std::uint64_t comm_gen = 0;
    int pe_begin = 0;
    int pe_count = 0;
    std::uint64_t amps = 0;  // amplitudes per PE

    // Two buffers per owned PE; `cur` selects the live one.  In multi-process
    // mode both are allocated up front and IPC-shared; otherwise the second
    // is allocated on first use (QR / out-of-place gate).
    std::vector<qrt::amp_t*> bufs[2];
    int cur = 0;
    // Base pointer of every PE's buffers (all p PEs; remote ones IPC-mapped).
    std::vector<qrt::amp_t*> peer[2];
    std::vector<void*> ipc_opened;  // pointers to close on destroy

    cudaStream_t stream = nullptr;

    // Scratch: per-CTA reduction slots and small uploads.
    double* d_red = nullptr;
    std::size_t red_cap = 0;
    void* d_ops = nullptr;  // op/pass descriptors + matrices of the current call
    std::size_t ops_cap = 0;
    void* h_pinned = nullptr;  // pinned staging for descriptor uploads
    std::size_t pinned_cap = 0;
    int* d_flag = nullptr;  // barrier word for NCCL

    // A QR recorded but not yet executed: the next gate pass gathers its tile
    // through it (qrt_fused.h); any other access executes it first.
    bool qr_pending = false;
    std::vector<int> qr_dest;
    // In-place QR (one buffer per PE; qrt_reorder.cu execute_inplace): set at
    // create when two sub-vectors per PE do not fit (or QRT_QR_INPLACE=1).
    // Disables the fused (pull) QR, which writes the spare buffer.
    bool inplace = false;
    // A fused pass flipped buffers: peers may still read the new spare (our
    // old live buffer) until the next barrier; writers of the spare wait.
    bool spare_busy = false;
    int sm_count = 148;

    // Measurement.
    bool profile = false;
    qrt_kernel_stats stats[QRT_K_COUNT]{};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // ProfileScope (outer: one ABI call's family)
    cudaEvent_t ev2 = nullptr, ev3 = nullptr;  // ProfileScope(inner): kernels only, e.g. QR without barriers

    qrt::amp_t* live(int local_pe) const { return bufs[cur][static_cast<std::size_t>(local_pe)]; }
};

namespace qrt {

// Scoped profiling region: records events around the launches of one kernel
// family on the state's stream when profiling is on.
struct ProfileScope {
    qrt_state* st;
    int fam;
    bool inner;
    ProfileScope(qrt_state* s, int f, bool inner_scope = false);
    ~ProfileScope();  // never throws: a failed event query is recorded, not raised
};

void ensure_alt(qrt_state* st);
void* ensure_ops(qrt_state* st, std::size_t bytes);
void* ensure_pinned(qrt_state* st, std::size_t bytes);
double* ensure_red(qrt_state* st, std::size_t doubles);
void barrier_on_stream(qrt_state* st);  // NCCL all-reduce of one int (no-op single process)

// Families implemented in the .cu files.
void apply_gates(qrt_state* st, int n_gates, const int* arity, const int* pos, const double* mats,
                 const unsigned* flags);
std::uint64_t reorder(qrt_state* st, const int* dest);
void flush_reorder(qrt_state* st);  // execute a pending QR (no-op if none)
bool fused_qr_enabled();
int fused_qr_max_log2();  // largest log2(amplitudes per PE) the fused (pull) QR is used for
void reorder_plan(int n, int p, const int* dest, int src_pe, std::uint64_t* dst_pe, std::uint64_t* dst_off,
                  std::uint64_t* relocated);
void qr_bench(int n_gpus, int nl, int k, int inplace, int iters, double* ms_out, double* gbs_out);
void reorder_inplace_plan(int n, int p, const int* dest, int* pairs0, int* n0, int* pairs1, int* n1, int* cross,
                          int* k);
void pauli_expectation(qrt_state* st, int n_terms, const std::uint64_t* x, const std::uint64_t* y,
                       const std::uint64_t* z, const std::uint64_t* gz, const double* coeffs, double* partial);
double norm(qrt_state* st);
void gate_plan_info(int nl, int n_gates, const int* arity, const int* pos, const double* mats, const unsigned* flags,
                    int* passes, int* light_passes, int* light_stages, int* fused);
void pauli_plan_info(int nl, int n_terms, const std::uint64_t* x, const std::uint64_t* y, const std::uint64_t* z,
                     const std::uint64_t* gz, const double* coeffs, int* passes, int* groups, int* wide_groups,
                     double* seconds);

// Host helpers shared by planners.
inline std::uint64_t deposit_bits(std::uint64_t value, const int* positions, int count) {
    std::uint64_t out = 0;
    for (int i = 0; i < count; ++i) out |= ((value >> i) & 1ull) << positions[i];
    return out;
}

}  // namespace qrt
