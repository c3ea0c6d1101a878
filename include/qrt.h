/*
 * qrt.h — C ABI of the B200-native QSU / QR / EVC hot path (libqrt.so).
 *
 * The reference (/root/reference/proj) has no FFI layer: its hot path is the
 * C++ function API of include/qrtile/dist_sim.hpp:43-92.  This header is the
 * boundary that API is re-routed through: the host C++
 * layer (paper_2410_04252_b200/host, namespace qrtile) keeps the reference
 * signatures and does all qubit bookkeeping; everything below works purely in
 * *position space* on sm_100a device memory.  No torch types, plain pointers
 * and sizes, caller-owned arrays copied during the call, calls synchronous at
 * return (the reference's barrier semantics).
 *
 * Amplitudes are complex<double>, interleaved (re, im), 16 B each.  A state of
 * n qubits on p = 2^g PEs stores 2^(n-g) amplitudes per PE; positions
 * [0, n-g) are the offset inside a PE, positions [n-g, n) the PE index
 * (dist_sim.hpp:23-27).  One process drives one GPU and owns a contiguous
 * block of PEs; with a communicator (one process per GPU, NCCL + CUDA IPC
 * over NVLink 5) the PEs of all ranks form one distributed state.
 */
#ifndef QRT_H
#define QRT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QRT_ABI_VERSION 2

/* Status codes; the host layer maps each to the reference exception type
 * (types.hpp:35-53). */
typedef enum {
    QRT_OK = 0,
    QRT_ERR_INVALID = 1,            /* bad argument (qrtile::Error)           */
    QRT_ERR_ACCESS_VIOLATION = 2,   /* AccessViolation   dist_sim.cpp:166     */
    QRT_ERR_MISSING_PAYLOAD = 3,    /* MissingPayload    dist_sim.cpp:164-165 */
    QRT_ERR_LAYOUT_MISMATCH = 4,    /* LayoutMismatch    dist_sim.cpp:204     */
    QRT_ERR_NOT_DIAGONALIZABLE = 5, /* NotDiagonalizable dist_sim.cpp:74      */
    QRT_ERR_TOO_MANY_PES = 6,       /* TooManyPEs        layout.cpp:32        */
    QRT_ERR_CONFIG = 7,             /* ConfigError                            */
    QRT_ERR_OOM = 8,                /* device allocation failed               */
    QRT_ERR_CUDA = 9,               /* CUDA runtime / launch failure          */
    QRT_ERR_NCCL = 10,              /* NCCL failure                           */
    QRT_ERR_NO_DEVICE = 11          /* no usable sm_100 device                */
} qrt_status;

typedef struct qrt_comm qrt_comm;   /* one-process-per-GPU communicator      */
typedef struct qrt_state qrt_state; /* distributed state: buffers, streams   */

/* Message of the last failing call on this thread ("" if none). */
const char* qrt_last_error(void);
int qrt_abi_version(void);
/* Build flags: bit 0 = checked build (libqrt_checked.so: device-side bounds
 * and pipeline invariant checks, QRT_CHECKS). */
int qrt_build_flags(void);
/* Number of visible CUDA devices of compute capability 10.x. */
qrt_status qrt_device_count(int* out);

/* ------------------------------------------------------------ communicator
 * Rank 0 creates a unique id; the caller distributes the 128 bytes by any
 * out-of-band means (torch.distributed, MPI, a file) and every rank calls
 * qrt_comm_init.  Collective: all ranks must call it. */
qrt_status qrt_comm_unique_id(unsigned char id[128]);
qrt_status qrt_comm_init(int rank, int world, int device, const unsigned char id[128], qrt_comm** out);
qrt_status qrt_comm_barrier(qrt_comm* comm);
qrt_status qrt_comm_destroy(qrt_comm* comm);

/* ------------------------------------------------------------------- state
 * Collective calls.  With a communicator, qrt_state_create, qrt_reorder and
 * qrt_release_cache are collective.  qrt_reorder may only *record* the QR
 * (fused into the next gate pass); while one is pending, the next
 * qrt_apply_gates, qrt_state_upload, qrt_state_download, qrt_norm and
 * qrt_pauli_expectation execute it first and are then collective as well,
 * and qrt_pauli_expectation / qrt_norm always are (they gather per-PE
 * partials).  Every rank must make the same sequence of these calls. */
/* init_state (dist_sim.cpp:122-131): zero state |0...0> on p PEs.  comm may
 * be NULL (single process, all p PEs on `device`); otherwise p must be a
 * multiple of the world size and rank r owns PEs [r*p/w, (r+1)*p/w).
 * Collective when comm != NULL. */
qrt_status qrt_state_create(int n, int p, int device, qrt_comm* comm, qrt_state** out);
/* Releases the state.  Its device buffers are parked and reused by the next
 * qrt_state_create of the same (n, p, device, comm) (a VQE loop creates one
 * state per iteration); qrt_release_cache frees all parked states
 * (collective when they were created with a communicator). */
qrt_status qrt_state_destroy(qrt_state* st);
qrt_status qrt_release_cache(void);
qrt_status qrt_state_info(const qrt_state* st, int* n, int* p, int* pe_begin, int* pe_count);
qrt_status qrt_state_set_zero(qrt_state* st);
/* Copy one owned PE's 2^(n-g) amplitudes (position order) in / out. */
qrt_status qrt_state_upload(qrt_state* st, int pe, const double* amps);
qrt_status qrt_state_download(const qrt_state* st, int pe, double* amps);

/* apply_gate_narrow (dist_sim.cpp:163-201), batched: a sequence of gates whose
 * targets are all local, applied in order (gates on disjoint targets may be
 * fused into one HBM pass; dependent gates never reorder).
 *   arity[i]   k_i (1 <= k_i <= n-g)
 *   pos        concatenated target positions; pos[j] of gate i <-> matrix bit j
 *   mats       concatenated payloads, interleaved complex: dense gates carry
 *              the row-major 2^k x 2^k matrix, diagonal gates (flags bit 0)
 *              carry only the 2^k diagonal entries
 *   flags      per gate; bit 0 = QRT_GATE_DIAGONAL (may be NULL) */
#define QRT_GATE_DIAGONAL 1u
qrt_status qrt_apply_gates(qrt_state* st, int n_gates, const int* arity, const int* pos,
                           const double* mats, const unsigned* flags);

/* perform_qr (dist_sim.cpp:203-240): permute index bits, dest[p] = new
 * position of the bit at position p (a permutation of [0, n)).  Amplitudes
 * change PE over NVLink; collective when comm != NULL.  *relocated receives
 * the number of amplitudes (all PEs) whose owning PE changed. */
qrt_status qrt_reorder(qrt_state* st, const int* dest, uint64_t* relocated);

/* QR mode of a state: *inplace_qr = 1 when qrt_reorder runs in place (one
 * buffer per PE: local bit-transposition passes + a pairwise NVLink swap of
 * slot classes), 0 for the two-buffer push / fused pull
 * exchange.  Chosen at qrt_state_create: QRT_QR_INPLACE=1/0 forces it, unset
 * picks in-place when two sub-vectors per PE do not fit in free device
 * memory (e.g. 34 qubits on 2 GPUs); all ranks agree (collective).
 * *sm_count = multiprocessors of the state's device (grid sizing). */
qrt_status qrt_state_mode(const qrt_state* st, int* inplace_qr, int* sm_count);

/* NVLink microbenchmark of the QR exchange (diagnostics, single process):
 * n_gpus GPUs (2/4/8) with one PE of 2^n_local amplitudes each swap their k
 * highest local positions with k PE bits through CUDA peer access, using the
 * push kernel (inplace = 0, two buffers) or the in-place exchange
 * (inplace = 1).  Returns the mean over `iters` of the slowest GPU's kernel
 * time and the per-direction NVLink rate (bytes each GPU sends / that time).
 * Meant to run under ncu (one process) for the NVLink counters. */
qrt_status qrt_qr_bench(int n_gpus, int n_local, int k, int inplace, int iters, double* ms_per_qr,
                        double* gbs_per_direction);

/* Host-only: the in-place decomposition of a reorder map (no device).
 * local_pairs0 / local_pairs1 receive n0 / n1 disjoint local position
 * transpositions (a, c) applied in that order, cross_pairs k (local slot,
 * PE-index bit) transpositions exchanged between PEs.  Arrays of 2*64 ints.
 * Fails with QRT_ERR_CONFIG when a global position would move to another
 * global position. */
qrt_status qrt_reorder_inplace_plan(int n, int p, const int* dest, int* local_pairs0, int* n0, int* local_pairs1,
                                    int* n1, int* cross_pairs, int* k);

/* Host-only replay of qrt_reorder's index mapping (no device needed): for
 * each of the 2^(n-g) amplitudes of source PE `src_pe`, the destination PE
 * and offset the kernel stores it to.  Used to emulate and check the
 * multi-process exchange on CPU. */
qrt_status qrt_reorder_plan(int n, int p, const int* dest, int src_pe, uint64_t* dst_pe, uint64_t* dst_off,
                            uint64_t* relocated);

/* The per-PE accumulation of expectation() for one plan tile
 * (dist_sim.cpp:84-97, 289-295):
 *   partial[pe] = sum_t coeff_t * (-1)^{popc(pe & gz_t)} * i^{popc(y_t)}
 *                 * sum_i (-1)^{popc(i & (z_t|y_t))} conj(v[i ^ (x_t|y_t)]) v[i]
 * masks are over local positions (gz over PE-index bits); coeffs interleaved
 * complex.  partial receives 2*p doubles for ALL p PEs (gathered over ranks). */
qrt_status qrt_pauli_expectation(qrt_state* st, int n_terms, const uint64_t* x, const uint64_t* y,
                                 const uint64_t* z, const uint64_t* gz, const double* coeffs,
                                 double* partial);

/* Host-only: the EVC pass plan qrt_pauli_expectation would build for these
 * masks on a PE of n_local positions (passes, flip-mask groups, full-vector
 * groups, planning seconds).  No device needed. */
qrt_status qrt_pauli_plan_info(int n_local, int n_terms, const uint64_t* x, const uint64_t* y, const uint64_t* z,
                               const uint64_t* gz, const double* coeffs, int* passes, int* groups, int* wide_groups,
                               double* seconds);

/* Host-only: the pass plan qrt_apply_gates would build for these gates on a
 * PE of n_local positions: HBM passes, light (register-resident) passes and
 * their register stages, and 1-qubit gates fused into a neighbour on the
 * host.  No device needed. */
qrt_status qrt_gate_plan_info(int n_local, int n_gates, const int* arity, const int* pos, const double* mats,
                              const unsigned* flags, int* passes, int* light_passes, int* light_stages, int* fused);

/* sqrt(sum |amp|^2) over all PEs (DistributedState::norm, dist_sim.cpp:115). */
qrt_status qrt_norm(qrt_state* st, double* out);

/* ------------------------------------------------------------ measurement
 * Per kernel family: launches and device time measured with CUDA events on
 * the stream the kernels run on (enabled by qrt_profile_enable), plus
 * algorithmic byte / flop counters (always on). */
typedef struct {
    uint64_t launches;      /* kernels launched                                 */
    double ms;              /* summed event time (profiling enabled only)      */
    double bytes;           /* algorithmic HBM bytes (gates/EVC) or NVLink bytes (QR) */
    double flops;           /* algorithmic fp64 flops                          */
    uint64_t calls;         /* ABI calls                                       */
} qrt_kernel_stats;

/* QRT_K_QR times a whole QR (barriers included); QRT_K_QR_XFER only its
 * exchange kernels (the NVLink transfer), so the barrier cost is their
 * difference. */
enum { QRT_K_GATES = 0, QRT_K_QR = 1, QRT_K_PAULI = 2, QRT_K_MISC = 3, QRT_K_QR_XFER = 4, QRT_K_COUNT = 5 };

qrt_status qrt_profile_enable(qrt_state* st, int on);
qrt_status qrt_stats(const qrt_state* st, qrt_kernel_stats out[QRT_K_COUNT]);
qrt_status qrt_stats_reset(qrt_state* st);
/* The cudaStream_t all work of `st` is issued on (as void*). */
qrt_status qrt_state_stream(const qrt_state* st, void** stream);
qrt_status qrt_synchronize(qrt_state* st);

#ifdef __cplusplus
}
#endif
#endif /* QRT_H */
