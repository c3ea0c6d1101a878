// B200 qrtile drop-in — DistributedState on B200 HBM.
//
// The reference dist-sim (/root/reference/proj/src/dist_sim.cpp) keeps p
// host vectors and loops over them on CPU threads.  This file keeps the
// reference's control flow and error behaviour (the checks of :164-168,
// :204-206, :268-288) but routes every numeric loop through the C ABI of
// include/qrt.h:
//   apply_gate_narrow / run_qsu   -> qrt_apply_gates   (fused gate passes)
//   perform_qr                    -> qrt_reorder       (NVLink push exchange)
//   expectation / diag_expectation_term -> qrt_pauli_expectation
// It also owns the *physical* layout: global positions are the logical
// ones, local positions are chosen so a QR moves contiguous runs (see
// physical_plan below and DESIGN.md).

#include <algorithm>
#include <cstring>
#include <istream>
#include <numeric>
#include <ostream>

#include "qrt.h"
#include "qrtile/dist_sim.hpp"

namespace qrtile {

namespace {

DeviceContext g_ctx;

[[noreturn]] void raise(qrt_status s, const std::string& where) {
    const std::string msg = where + ": " + qrt_last_error();
    switch (s) {
        case QRT_ERR_ACCESS_VIOLATION: throw AccessViolation(msg);
        case QRT_ERR_MISSING_PAYLOAD: throw MissingPayload(msg);
        case QRT_ERR_LAYOUT_MISMATCH: throw LayoutMismatch(msg);
        case QRT_ERR_NOT_DIAGONALIZABLE: throw NotDiagonalizable(msg);
        case QRT_ERR_TOO_MANY_PES: throw TooManyPEs(msg);
        case QRT_ERR_CONFIG: throw ConfigError(msg);
        case QRT_ERR_INVALID: throw Error(msg);
        default: throw DeviceError(msg);
    }
}

void ok(qrt_status s, const char* where) {
    if (s != QRT_OK) raise(s, where);
}

// Masked Pauli word in physical position space (reference MaskedTerm, :54-58).
struct Masked {
    std::uint64_t x = 0, y = 0, z = 0, gz = 0;
};

// mask_term (:60-81): the *logical* layout decides local vs global (and the
// NotDiagonalizable error); the bit positions come from the physical layout.
Masked mask_term(const PauliTerm& term, const DistributedState& st) {
    Masked m;
    const QubitLayout& l = st.layout;
    for (int q = 0; q < term.n(); ++q) {
        const char c = term.letters[static_cast<std::size_t>(q)];
        if (c == 'I') continue;
        const int pos = l.pos_of[static_cast<std::size_t>(q)];
        if (pos < l.n_local) {
            const std::uint64_t bit = std::uint64_t{1} << st.device->phys_pos_of[static_cast<std::size_t>(q)];
            if (c == 'X') m.x |= bit;
            if (c == 'Y') m.y |= bit;
            if (c == 'Z') m.z |= bit;
        } else {
            if (c != 'Z')
                throw NotDiagonalizable(std::string("letter ") + c + " on global qubit " + std::to_string(q));
            m.gz |= std::uint64_t{1} << (pos - l.n_local);
        }
    }
    return m;
}

// Physical permutation for a logical QR event.  Global positions follow the
// logical layout exactly.  A qubit that stays local keeps its physical
// position.  An arriving qubit takes the physical slot of a departing one,
// except that departing slots below 2^4 are refilled by the highest staying
// qubit (which moves down) and the arriving qubit goes to that high slot, so
// both sides of the exchange move runs of >= 16 contiguous amplitudes.
std::vector<int> physical_plan_impl(const QrEvent& ev, const std::vector<int>& phys, std::vector<int>& new_phys) {
    const int n = ev.before.n, nl = ev.before.n_local;
    std::vector<int> phys_qubit_at(static_cast<std::size_t>(n));
    for (int q = 0; q < n; ++q) phys_qubit_at[static_cast<std::size_t>(phys[static_cast<std::size_t>(q)])] = q;
    constexpr int kLowRun = 4;
    new_phys.assign(static_cast<std::size_t>(n), -1);
    std::vector<int> arriving, freed;
    std::vector<char> taken(static_cast<std::size_t>(nl), 0);
    for (int q = 0; q < n; ++q) {
        const int before = ev.before.pos_of[static_cast<std::size_t>(q)];
        const int after = ev.after.pos_of[static_cast<std::size_t>(q)];
        if (after >= nl) {
            new_phys[static_cast<std::size_t>(q)] = after;
            if (before < nl) freed.push_back(phys[static_cast<std::size_t>(q)]);
        } else if (before < nl) {
            new_phys[static_cast<std::size_t>(q)] = phys[static_cast<std::size_t>(q)];
            taken[static_cast<std::size_t>(phys[static_cast<std::size_t>(q)])] = 1;
        } else {
            arriving.push_back(q);
        }
    }
    std::sort(freed.begin(), freed.end());
    std::sort(arriving.begin(), arriving.end(), [&](int a, int b) {
        return ev.before.pos_of[static_cast<std::size_t>(a)] < ev.before.pos_of[static_cast<std::size_t>(b)];
    });
    if (freed.size() != arriving.size()) throw Error("unbalanced local exchange in QR event");
    // refill low freed slots from the top staying qubits
    std::vector<int> slots;  // where arriving qubits go
    int hi = nl - 1;
    for (int f : freed) {
        if (f >= kLowRun) {
            slots.push_back(f);
            continue;
        }
        while (hi >= kLowRun && !taken[static_cast<std::size_t>(hi)]) --hi;
        if (hi < kLowRun) {
            slots.push_back(f);
            continue;
        }
        const int mover = phys_qubit_at[static_cast<std::size_t>(hi)];
        new_phys[static_cast<std::size_t>(mover)] = f;
        taken[static_cast<std::size_t>(hi)] = 0;
        taken[static_cast<std::size_t>(f)] = 1;
        slots.push_back(hi);
        --hi;
    }
    std::sort(slots.begin(), slots.end());
    for (std::size_t i = 0; i < arriving.size(); ++i) new_phys[static_cast<std::size_t>(arriving[i])] = slots[i];
    std::vector<int> dest(static_cast<std::size_t>(n));
    for (int q = 0; q < n; ++q)
        dest[static_cast<std::size_t>(phys[static_cast<std::size_t>(q)])] = new_phys[static_cast<std::size_t>(q)];
    return dest;
}

std::vector<int> physical_plan(const DistributedState& st, const QrEvent& ev, std::vector<int>& new_phys) {
    return physical_plan_impl(ev, st.device->phys_pos_of, new_phys);
}

// Logical offset (reference position order) <-> physical offset inside a PE.
std::vector<std::uint64_t> logical_to_physical_map(const DistributedState& st) {
    const int nl = st.layout.n_local;
    std::vector<int> lp(static_cast<std::size_t>(nl));  // logical position -> physical position
    bool same = true;
    for (int p = 0; p < nl; ++p) {
        const int q = st.layout.qubit_at[static_cast<std::size_t>(p)];
        lp[static_cast<std::size_t>(p)] = st.device->phys_pos_of[static_cast<std::size_t>(q)];
        same = same && lp[static_cast<std::size_t>(p)] == p;
    }
    if (same) return {};
    std::vector<std::uint64_t> map(std::size_t{1} << nl);
    for (std::uint64_t o = 0; o < map.size(); ++o) {
        std::uint64_t r = 0;
        for (int p = 0; p < nl; ++p) r |= ((o >> p) & 1u) << lp[static_cast<std::size_t>(p)];
        map[o] = r;
    }
    return map;
}

void check_gate(const Operator& gate, const QubitLayout& layout) {
    if (gate.kind != OpKind::Gate) throw MissingPayload("operator is not a gate");
    if (!gate.payload) throw MissingPayload("gate " + std::to_string(gate.id) + " has no payload");
    if (classify_access(gate, layout) == Access::Wide)
        throw AccessViolation("gate " + std::to_string(gate.id) + " targets a global qubit; reorder first");
}

void submit_gates(DistributedState& st, const std::vector<const Operator*>& gates) {
    std::vector<int> arity, pos;
    std::vector<unsigned> flags;
    std::vector<double> mats;
    arity.reserve(gates.size());
    flags.reserve(gates.size());
    for (const Operator* g : gates) {
        check_gate(*g, st.layout);
        const GateMatrix& u = *g->payload;
        if (u.dim != (1 << g->arity())) throw Error("payload dimension mismatch in gate " + std::to_string(g->id));
        arity.push_back(g->arity());
        for (int t : g->targets) pos.push_back(st.device->phys_pos_of[static_cast<std::size_t>(t)]);
        const bool diag = u.is_diagonal();
        flags.push_back(diag ? QRT_GATE_DIAGONAL : 0u);
        if (diag) {
            for (int r = 0; r < u.dim; ++r) {
                mats.push_back(u.at(r, r).real());
                mats.push_back(u.at(r, r).imag());
            }
        } else {
            for (const Amp& a : u.a) {
                mats.push_back(a.real());
                mats.push_back(a.imag());
            }
        }
    }
    if (gates.empty()) return;
    ok(qrt_apply_gates(st.device->handle, static_cast<int>(gates.size()), arity.data(), pos.data(), mats.data(),
                       flags.data()),
       "qrt_apply_gates");
}

}  // namespace

std::vector<int> physical_reorder_plan(const QrEvent& event, const std::vector<int>& phys_pos_of,
                                       std::vector<int>& new_phys_pos_of) {
    return physical_plan_impl(event, phys_pos_of, new_phys_pos_of);
}

// ---------------------------------------------------------------- context

void init_device(int rank, int world, int device, const std::string& unique_id) {
    shutdown_device();
    g_ctx.rank = rank;
    g_ctx.world = world;
    g_ctx.device = device;
    if (world > 1) {
        if (unique_id.size() != 128) throw ConfigError("device unique id must be 128 bytes");
        qrt_comm* c = nullptr;
        ok(qrt_comm_init(rank, world, device, reinterpret_cast<const unsigned char*>(unique_id.data()), &c),
           "qrt_comm_init");
        g_ctx.comm = c;
    }
}

std::string device_unique_id() {
    std::string id(128, '\0');
    ok(qrt_comm_unique_id(reinterpret_cast<unsigned char*>(id.data())), "qrt_comm_unique_id");
    return id;
}

const DeviceContext& device_context() { return g_ctx; }

void shutdown_device() {
    qrt_release_cache();
    if (g_ctx.comm) qrt_comm_destroy(g_ctx.comm);
    g_ctx = DeviceContext{};
}

DeviceState::~DeviceState() {
    if (handle) qrt_state_destroy(handle);
}

// ------------------------------------------------------------------ states

ReferenceState ReferenceState::zero(int n) {
    ReferenceState r;
    r.n = n;
    r.amps.assign(std::size_t{1} << n, Amp{0.0, 0.0});
    r.amps[0] = 1.0;
    return r;
}

double ReferenceState::norm() const {
    double s = 0.0;
    for (const Amp& a : amps) s += std::norm(a);
    return std::sqrt(s);
}

double DistributedState::norm() const {
    double out = 0.0;
    ok(qrt_norm(device->handle, &out), "qrt_norm");
    return out;
}

DistributedState init_state(int n, const ClusterShape& shape) {
    DistributedState st;
    st.n = n;
    st.shape = shape;
    st.layout = QubitLayout::identity(n, shape);  // validates; TooManyPEs
    st.device = std::make_unique<DeviceState>();
    qrt_state* h = nullptr;
    ok(qrt_state_create(n, shape.p, g_ctx.device, g_ctx.comm, &h), "qrt_state_create");
    st.device->handle = h;
    ok(qrt_state_info(h, nullptr, nullptr, &st.device->pe_begin, &st.device->pe_count), "qrt_state_info");
    st.device->phys_pos_of.resize(static_cast<std::size_t>(n));
    std::iota(st.device->phys_pos_of.begin(), st.device->phys_pos_of.end(), 0);
    st.device->phys_qubit_at = st.device->phys_pos_of;
    return st;
}

DistributedState init_state(const ReferenceState& ref, const ClusterShape& shape) {
    DistributedState st = init_state(ref.n, shape);
    const std::size_t per = std::size_t{1} << st.layout.n_local;
    for (int i = 0; i < st.pe_count(); ++i) {
        const int pe = st.pe_begin() + i;
        ok(qrt_state_upload(st.device->handle, pe, reinterpret_cast<const double*>(ref.amps.data() + per * static_cast<std::size_t>(pe))),
           "qrt_state_upload");
    }
    return st;
}

std::vector<Amp> DistributedState::sub_of(int pe) const {
    if (!owns(pe)) throw Error("PE " + std::to_string(pe) + " is not owned by this process");
    const std::size_t per = std::size_t{1} << layout.n_local;
    std::vector<Amp> phys(per);
    ok(qrt_state_download(device->handle, pe, reinterpret_cast<double*>(phys.data())), "qrt_state_download");
    const auto map = logical_to_physical_map(*this);
    if (map.empty()) return phys;
    std::vector<Amp> out(per);
    for (std::size_t o = 0; o < per; ++o) out[o] = phys[map[o]];
    return out;
}

std::vector<std::vector<Amp>> DistributedState::sub_vectors() const {
    std::vector<std::vector<Amp>> all;
    for (int pe = 0; pe < shape.p; ++pe) all.push_back(sub_of(pe));
    return all;
}

void DistributedState::set_sub(int pe, const std::vector<Amp>& amps) {
    if (!owns(pe)) throw Error("PE " + std::to_string(pe) + " is not owned by this process");
    const std::size_t per = std::size_t{1} << layout.n_local;
    if (amps.size() != per) throw Error("sub-vector size mismatch");
    const auto map = logical_to_physical_map(*this);
    if (map.empty()) {
        ok(qrt_state_upload(device->handle, pe, reinterpret_cast<const double*>(amps.data())), "qrt_state_upload");
        return;
    }
    std::vector<Amp> phys(per);
    for (std::size_t o = 0; o < per; ++o) phys[map[o]] = amps[o];
    ok(qrt_state_upload(device->handle, pe, reinterpret_cast<const double*>(phys.data())), "qrt_state_upload");
}

DistributedState DistributedState::clone() const {
    DistributedState c = init_state(n, shape);
    c.layout = layout;
    c.last_relocated = last_relocated;
    c.total_relocated = total_relocated;
    c.qr_log = qr_log;
    c.device->phys_pos_of = device->phys_pos_of;
    c.device->phys_qubit_at = device->phys_qubit_at;
    const std::size_t per = std::size_t{1} << layout.n_local;
    std::vector<double> buf(2 * per);
    for (int i = 0; i < pe_count(); ++i) {
        const int pe = pe_begin() + i;
        ok(qrt_state_download(device->handle, pe, buf.data()), "qrt_state_download");
        ok(qrt_state_upload(c.device->handle, pe, buf.data()), "qrt_state_upload");
    }
    return c;
}

ReferenceState flatten(const DistributedState& state) {
    if (state.pe_count() != state.shape.p) throw Error("flatten needs every PE in this process");
    ReferenceState ref;
    ref.n = state.n;
    ref.amps.assign(std::size_t{1} << state.n, Amp{0.0, 0.0});
    const int nl = state.layout.n_local;
    const std::size_t per = std::size_t{1} << nl;
    const std::vector<int>& qat = state.device->phys_qubit_at;
    std::vector<Amp> phys(per);
    for (int pe = 0; pe < state.shape.p; ++pe) {
        ok(qrt_state_download(state.device->handle, pe, reinterpret_cast<double*>(phys.data())), "qrt_state_download");
        std::uint64_t pe_bits = 0;
        for (int b = 0; b < state.n - nl; ++b)
            if ((pe >> b) & 1) pe_bits |= qbit(qat[static_cast<std::size_t>(nl + b)]);
        for (std::uint64_t off = 0; off < per; ++off) {
            std::uint64_t canon = pe_bits;
            for (std::uint64_t rest = off; rest; rest &= rest - 1)
                canon |= qbit(qat[static_cast<std::size_t>(std::countr_zero(rest))]);
            ref.amps[canon] = phys[off];
        }
    }
    return ref;
}

void apply_gate_narrow(DistributedState& state, const Operator& gate, int /*workers*/) {
    check_gate(gate, state.layout);
    submit_gates(state, {&gate});
}

void apply_gates_narrow(DistributedState& state, const Circuit& circuit, const std::vector<int>& ids) {
    std::vector<const Operator*> gates;
    gates.reserve(ids.size());
    for (int id : ids) gates.push_back(&circuit.op(id));
    submit_gates(state, gates);
}

std::uint64_t perform_qr(DistributedState& state, const QrEvent& event) {
    if (!(event.before == state.layout)) throw LayoutMismatch("event does not start from the current layout");
    event.after.check();
    std::vector<int> new_phys;
    std::vector<int> dest = physical_plan(state, event, new_phys);
    std::uint64_t relocated = 0;
    ok(qrt_reorder(state.device->handle, dest.data(), &relocated), "qrt_reorder");
    state.device->phys_pos_of = new_phys;
    for (int q = 0; q < state.n; ++q)
        state.device->phys_qubit_at[static_cast<std::size_t>(new_phys[static_cast<std::size_t>(q)])] = q;
    state.layout = event.after;
    state.last_relocated = relocated;
    state.total_relocated += relocated;
    state.qr_log.emplace_back(static_cast<int>(event.swaps.size()), relocated);
    return relocated;
}

void run_qsu(DistributedState& state, const Circuit& circuit, const Schedule& schedule, int /*workers*/) {
    std::size_t next = 0;
    for (int t = 0; t < static_cast<int>(schedule.tiles.size()); ++t) {
        while (next < schedule.qr_events.size() && schedule.qr_events[next].before_tile == t)
            perform_qr(state, schedule.qr_events[next++]);
        apply_gates_narrow(state, circuit, schedule.tiles[static_cast<std::size_t>(t)].gates);
    }
}

namespace {
// Per-PE partials of one tile's terms, all PEs (gathered across ranks).
std::vector<Amp> tile_partials(DistributedState& st, const std::vector<Masked>& masked, const std::vector<Amp>& coeffs) {
    const std::size_t nt = masked.size();
    std::vector<std::uint64_t> x(nt), y(nt), z(nt), gz(nt);
    std::vector<double> c(2 * nt);
    for (std::size_t i = 0; i < nt; ++i) {
        x[i] = masked[i].x;
        y[i] = masked[i].y;
        z[i] = masked[i].z;
        gz[i] = masked[i].gz;
        c[2 * i] = coeffs[i].real();
        c[2 * i + 1] = coeffs[i].imag();
    }
    std::vector<Amp> partial(static_cast<std::size_t>(st.shape.p));
    ok(qrt_pauli_expectation(st.device->handle, static_cast<int>(nt), x.data(), y.data(), z.data(), gz.data(),
                             c.data(), reinterpret_cast<double*>(partial.data())),
       "qrt_pauli_expectation");
    return partial;
}
}  // namespace

double diag_expectation_term(const DistributedState& state, const PauliTerm& term) {
    auto& st = const_cast<DistributedState&>(state);
    Masked m = mask_term(term, st);  // NotDiagonalizable on a global X/Y
    std::vector<Amp> partial = tile_partials(st, {m}, {Amp{1.0, 0.0}});
    Amp acc = 0.0;
    for (const Amp& a : partial) acc += a;
    return acc.real();
}

Amp expectation(DistributedState& state, const PauliTilePlan& plan, const std::vector<PauliTerm>& terms,
                int /*workers*/) {
    std::vector<Amp> partial(static_cast<std::size_t>(state.shape.p), Amp{0.0, 0.0});
    for (const PauliTile& tile : plan.tiles) {
        if (state.layout.local_set() != tile.local_qubits)
            if (auto ev = make_qr_event(state.layout, tile.local_qubits)) perform_qr(state, *ev);
        std::vector<Masked> masked;
        std::vector<Amp> coeffs;
        masked.reserve(tile.terms.size());
        coeffs.reserve(tile.terms.size());
        for (int id : tile.terms) {
            const PauliTerm& term = terms[static_cast<std::size_t>(id)];
            Masked m;
            try {
                m = mask_term(term, state);
            } catch (const NotDiagonalizable& e) {
                throw AccessViolation(std::string("term not narrow in its tile: ") + e.what());
            }
            if (!plan.diagonalized && m.gz != 0)
                throw AccessViolation("term has a global Z but the plan is not diagonalized");
            masked.push_back(m);
            coeffs.push_back(term.coeff);
        }
        const std::vector<Amp> part = tile_partials(state, masked, coeffs);
        for (std::size_t pe = 0; pe < partial.size(); ++pe) partial[pe] += part[pe];
    }
    Amp total = 0.0;
    for (const Amp& a : partial) total += a;  // ascending PE order (:297-298)
    return total;
}

double evaluate_energy(const Circuit& circuit, const Schedule& schedule, const std::vector<PauliTerm>& terms,
                       const PauliTilePlan& plan, int workers) {
    DistributedState st = init_state(circuit.n, schedule.shape);
    run_qsu(st, circuit, schedule, workers);
    return expectation(st, plan, terms, workers).real();
}

// --------------------------------------------------------------- state dump
// Two little-endian u64 (n, p), then canonical (re, im) doubles
// (reference :365-403).

void write_state_dump(std::ostream& out, const ReferenceState& ref, int p) {
    auto put = [&](std::uint64_t v) {
        unsigned char b[8];
        for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
        out.write(reinterpret_cast<const char*>(b), 8);
    };
    put(static_cast<std::uint64_t>(ref.n));
    put(static_cast<std::uint64_t>(p));
    out.write(reinterpret_cast<const char*>(ref.amps.data()), static_cast<std::streamsize>(ref.amps.size() * sizeof(Amp)));
}

ReferenceState read_state_dump(std::istream& in, int* p_out) {
    auto get = [&]() {
        unsigned char b[8] = {};
        in.read(reinterpret_cast<char*>(b), 8);
        std::uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= static_cast<std::uint64_t>(b[i]) << (8 * i);
        return v;
    };
    ReferenceState ref;
    ref.n = static_cast<int>(get());
    const std::uint64_t p = get();
    if (p_out) *p_out = static_cast<int>(p);
    if (ref.n < 0 || ref.n > kMaxQubits) throw ParseError("corrupt state dump header");
    ref.amps.resize(std::size_t{1} << ref.n);
    in.read(reinterpret_cast<char*>(ref.amps.data()), static_cast<std::streamsize>(ref.amps.size() * sizeof(Amp)));
    if (!in) throw ParseError("truncated state dump");
    return ref;
}

}  // namespace qrtile
