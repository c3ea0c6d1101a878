#pragma once
// B200 qrtile drop-in — the distributed state vector, now resident in B200
// HBM and driven through the C ABI in include/qrt.h.
// Reference interface: /root/reference/proj/include/qrtile/dist_sim.hpp
// (ReferenceState :16-22, DistributedState :28-41, init_state :43-44,
//  flatten :48, apply_gate_narrow :53, perform_qr :57, run_qsu :61,
//  diag_expectation_term :65, expectation :69, dense oracle :75-78,
//  evaluate_energy :84, state dump :90-91).
//
// Differences a caller can observe, all deliberate:
//  * `sub` lives on the GPU.  Read it with `sub_vectors()` / `sub_of(pe)`
//    (download, reference position order) and write it with `set_sub`.
//  * The state is move-only (device memory); use `clone()` for a copy.
//  * `workers` is accepted and ignored: parallelism is the GPU.
//  * The dense oracle (dense_oracle_apply / dense_oracle_expectation) is test
//    infrastructure and lives in oracle/, not in the product.

#include <iosfwd>
#include <memory>

#include "qrtile/evc_scheduler.hpp"
#include "qrtile/schedule.hpp"

struct qrt_state;
struct qrt_comm;

namespace qrtile {

// Dense canonical-order state (bit q of the index = qubit q).
struct ReferenceState {
    int n = 0;
    std::vector<Amp> amps;

    static ReferenceState zero(int n);
    double norm() const;
};

// ---- device context --------------------------------------------------------
// One process drives one GPU.  With world > 1 the PEs of a state are split
// evenly over the ranks (rank r owns PEs [r*p/w, (r+1)*p/w)) and QRs move
// amplitudes over NVLink.  The default context is rank 0 of 1 on device 0.
struct DeviceContext {
    int rank = 0;
    int world = 1;
    int device = 0;
    qrt_comm* comm = nullptr;
};
// Collective over all ranks when world > 1.  `unique_id` comes from
// device_unique_id() on rank 0, distributed by the caller.
void init_device(int rank, int world, int device, const std::string& unique_id = {});
std::string device_unique_id();
const DeviceContext& device_context();
void shutdown_device();

// Owner of the device buffers plus the *physical* layout: global positions
// always equal the logical ones, local positions are permuted freely so QRs
// move contiguous blocks.
struct DeviceState {
    qrt_state* handle = nullptr;
    std::vector<int> phys_pos_of;    // qubit -> physical position
    std::vector<int> phys_qubit_at;  // physical position -> qubit
    int pe_begin = 0;
    int pe_count = 0;

    DeviceState() = default;
    DeviceState(const DeviceState&) = delete;
    DeviceState& operator=(const DeviceState&) = delete;
    ~DeviceState();
};

struct DistributedState {
    int n = 0;
    ClusterShape shape;
    QubitLayout layout;  // logical layout, identical to the reference's

    std::uint64_t last_relocated = 0;
    std::uint64_t total_relocated = 0;
    std::vector<std::pair<int, std::uint64_t>> qr_log;  // (swap pairs, relocated)

    std::unique_ptr<DeviceState> device;

    int n_local() const { return layout.n_local; }
    double norm() const;

    int pe_begin() const { return device ? device->pe_begin : 0; }
    int pe_count() const { return device ? device->pe_count : 0; }
    bool owns(int pe) const { return pe >= pe_begin() && pe < pe_begin() + pe_count(); }

    // Reference-order (logical positions) copy of one owned PE / all PEs.
    std::vector<Amp> sub_of(int pe) const;
    std::vector<std::vector<Amp>> sub_vectors() const;  // single-process only
    void set_sub(int pe, const std::vector<Amp>& amps);

    DistributedState clone() const;
};

DistributedState init_state(int n, const ClusterShape& shape);
DistributedState init_state(const ReferenceState& ref, const ClusterShape& shape);

ReferenceState flatten(const DistributedState& state);

void apply_gate_narrow(DistributedState& state, const Operator& gate, int workers = 1);
// Batched form used by run_qsu: the listed gates in order, fused on device.
void apply_gates_narrow(DistributedState& state, const Circuit& circuit, const std::vector<int>& ids);

std::uint64_t perform_qr(DistributedState& state, const QrEvent& event);

// The device-side position permutation perform_qr issues for `event` given the
// current physical layout (qubit -> physical position): returns dest[p] for
// qrt_reorder and the new physical layout.  Exposed for tests / ABI callers.
std::vector<int> physical_reorder_plan(const QrEvent& event, const std::vector<int>& phys_pos_of,
                                       std::vector<int>& new_phys_pos_of);

void run_qsu(DistributedState& state, const Circuit& circuit, const Schedule& schedule, int workers = 1);

double diag_expectation_term(const DistributedState& state, const PauliTerm& term);

Amp expectation(DistributedState& state, const PauliTilePlan& plan, const std::vector<PauliTerm>& terms,
                int workers = 1);

inline constexpr int kOracleMaxQubits = 14;

double evaluate_energy(const Circuit& circuit, const Schedule& schedule, const std::vector<PauliTerm>& terms,
                       const PauliTilePlan& plan, int workers = 1);

void write_state_dump(std::ostream& out, const ReferenceState& ref, int p);
ReferenceState read_state_dump(std::istream& in, int* p_out = nullptr);

}  // namespace qrtile
