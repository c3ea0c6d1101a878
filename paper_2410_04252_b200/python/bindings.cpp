// Python bindings of the B200 qrtile drop-in (module paper_2410_04252_b200._qrtile).
// Names, argument meaning and error types mirror the reference C++ API so the
// parity tests read like the reference's own tests (proj/tests/*.cpp).

#include <pybind11/complex.h>
#include <pybind11/functional.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <sstream>

#include "qrt.h"
#include "qrtile/dist_sim.hpp"
#include "qrtile/evc_scheduler.hpp"
#include "qrtile/models.hpp"
#include "qrtile/qsu_scheduler.hpp"

namespace py = pybind11;
using namespace qrtile;

namespace {

using CArray = py::array_t<std::complex<double>, py::array::c_style | py::array::forcecast>;

CArray to_numpy(const std::vector<Amp>& v) {
    CArray out(static_cast<py::ssize_t>(v.size()));
    std::memcpy(out.mutable_data(), v.data(), v.size() * sizeof(Amp));
    return out;
}

std::vector<Amp> from_numpy(const CArray& a) {
    std::vector<Amp> v(static_cast<std::size_t>(a.size()));
    std::memcpy(v.data(), a.data(), v.size() * sizeof(Amp));
    return v;
}

GatePayload payload_from(const py::object& m) {
    if (m.is_none()) return nullptr;
    CArray a = m.cast<CArray>();
    if (a.ndim() != 2 || a.shape(0) != a.shape(1)) throw ConfigError("payload must be a square matrix");
    auto g = std::make_shared<GateMatrix>(static_cast<int>(a.shape(0)));
    std::memcpy(g->a.data(), a.data(), g->a.size() * sizeof(Amp));
    return g;
}

py::object payload_to(const GatePayload& p) {
    if (!p) return py::none();
    CArray a({p->dim, p->dim});
    std::memcpy(a.mutable_data(), p->a.data(), p->a.size() * sizeof(Amp));
    return a;
}

}  // namespace

PYBIND11_MODULE(_qrtile, m) {
    m.doc() = "B200-native qrtile drop-in: schedulers (host) + QSU/QR/EVC on sm_100a via libqrt";

    // ---- exceptions (reference types.hpp:35-53) -------------------------------
    static py::exception<Error> exc_base(m, "Error", PyExc_RuntimeError);
#define QRT_EXC(Name) static py::exception<Name> exc_##Name(m, #Name, exc_base.ptr())
    QRT_EXC(InvalidSchedule);
    QRT_EXC(GateTooWide);
    QRT_EXC(SchedulerStuck);
    QRT_EXC(DegenerateQr);
    QRT_EXC(TooManyPEs);
    QRT_EXC(AccessViolation);
    QRT_EXC(LayoutMismatch);
    QRT_EXC(NotDiagonalizable);
    QRT_EXC(OracleTooLarge);
    QRT_EXC(MissingPayload);
    QRT_EXC(ParseError);
    QRT_EXC(IndexError);
    QRT_EXC(TermTooWide);
    QRT_EXC(CircuitTooSmall);
    QRT_EXC(ConfigError);
    QRT_EXC(DeviceError);
#undef QRT_EXC
    py::register_exception_translator([](std::exception_ptr p) {
        // most-derived first; DeviceError and friends all derive from Error
        try {
            if (p) std::rethrow_exception(p);
        } catch (const InvalidSchedule& e) { py::set_error(exc_InvalidSchedule, e.what());
        } catch (const GateTooWide& e) { py::set_error(exc_GateTooWide, e.what());
        } catch (const SchedulerStuck& e) { py::set_error(exc_SchedulerStuck, e.what());
        } catch (const DegenerateQr& e) { py::set_error(exc_DegenerateQr, e.what());
        } catch (const TooManyPEs& e) { py::set_error(exc_TooManyPEs, e.what());
        } catch (const AccessViolation& e) { py::set_error(exc_AccessViolation, e.what());
        } catch (const LayoutMismatch& e) { py::set_error(exc_LayoutMismatch, e.what());
        } catch (const NotDiagonalizable& e) { py::set_error(exc_NotDiagonalizable, e.what());
        } catch (const OracleTooLarge& e) { py::set_error(exc_OracleTooLarge, e.what());
        } catch (const MissingPayload& e) { py::set_error(exc_MissingPayload, e.what());
        } catch (const ParseError& e) { py::set_error(exc_ParseError, e.what());
        } catch (const IndexError& e) { py::set_error(exc_IndexError, e.what());
        } catch (const TermTooWide& e) { py::set_error(exc_TermTooWide, e.what());
        } catch (const CircuitTooSmall& e) { py::set_error(exc_CircuitTooSmall, e.what());
        } catch (const ConfigError& e) { py::set_error(exc_ConfigError, e.what());
        } catch (const DeviceError& e) { py::set_error(exc_DeviceError, e.what());
        } catch (const Error& e) { py::set_error(exc_base, e.what());
        }
    });

    // ---- types ---------------------------------------------------------------
    py::class_<ClusterShape>(m, "ClusterShape")
        .def(py::init<>())
        .def_static("flat", &ClusterShape::flat)
        .def_static("two_level", &ClusterShape::two_level)
        .def_readwrite("p", &ClusterShape::p)
        .def_readwrite("n_node", &ClusterShape::n_node)
        .def_readwrite("n_gpn", &ClusterShape::n_gpn)
        .def("global_bits", &ClusterShape::global_bits)
        .def("validate", &ClusterShape::validate)
        .def("__eq__", [](const ClusterShape& a, const ClusterShape& b) { return a == b; });

    py::class_<QubitLayout>(m, "QubitLayout")
        .def_static("identity", &QubitLayout::identity)
        .def_readonly("n", &QubitLayout::n)
        .def_readonly("n_local", &QubitLayout::n_local)
        .def_readonly("intra_bits", &QubitLayout::intra_bits)
        .def_readonly("pos_of", &QubitLayout::pos_of)
        .def_readonly("qubit_at", &QubitLayout::qubit_at)
        .def("local_set", &QubitLayout::local_set)
        .def("intra_set", &QubitLayout::intra_set)
        .def("inter_set", &QubitLayout::inter_set)
        .def("check", &QubitLayout::check)
        .def("__eq__", [](const QubitLayout& a, const QubitLayout& b) { return a == b; });

    py::enum_<QrClass>(m, "QrClass").value("Intra", QrClass::Intra).value("Inter", QrClass::Inter);

    py::class_<QrEvent>(m, "QrEvent")
        .def_readonly("swaps", &QrEvent::swaps)
        .def_readonly("before", &QrEvent::before)
        .def_readonly("after", &QrEvent::after)
        .def_readonly("cls", &QrEvent::cls)
        .def_readonly("before_tile", &QrEvent::before_tile);

    py::class_<Operator>(m, "Operator")
        .def_readonly("id", &Operator::id)
        .def_readonly("targets", &Operator::targets)
        .def_readonly("letters", &Operator::letters)
        .def_property_readonly("is_gate", [](const Operator& o) { return o.kind == OpKind::Gate; })
        .def_property_readonly("payload", [](const Operator& o) { return payload_to(o.payload); })
        .def("arity", &Operator::arity)
        .def("target_mask", &Operator::target_mask);

    m.def("make_gate", [](int id, std::vector<int> targets, py::object mat) {
        return make_gate(id, std::move(targets), payload_from(mat));
    }, py::arg("id"), py::arg("targets"), py::arg("matrix") = py::none());
    m.def("make_pauli_op", &make_pauli_op);

    py::class_<Circuit>(m, "Circuit")
        .def(py::init([](int n, std::vector<Operator> ops) {
                 Circuit c;
                 c.n = n;
                 c.operators = std::move(ops);
                 return c;
             }),
             py::arg("n"), py::arg("operators") = std::vector<Operator>{})
        .def_readonly("n", &Circuit::n)
        .def_readonly("operators", &Circuit::operators)
        .def("size", &Circuit::size)
        .def("validate", &Circuit::validate)
        .def("__len__", &Circuit::size);

    py::class_<DependencyGraph>(m, "DependencyGraph")
        .def_readonly("edges", &DependencyGraph::edges)
        .def_readonly("depth", &DependencyGraph::depth)
        .def("reaches", &DependencyGraph::reaches);
    m.def("build_dependency_graph", &build_dependency_graph);
    m.def("depth_sort", &depth_sort);

    py::class_<PauliTerm>(m, "PauliTerm")
        .def(py::init([](Amp c, std::string letters) { return PauliTerm{c, std::move(letters)}; }))
        .def_readwrite("coeff", &PauliTerm::coeff)
        .def_readwrite("letters", &PauliTerm::letters)
        .def("plain_targets", &PauliTerm::plain_targets)
        .def("xy_targets", &PauliTerm::xy_targets)
        .def("z_targets", &PauliTerm::z_targets);

    py::class_<Tile>(m, "Tile").def_readonly("gates", &Tile::gates).def_readonly("local_qubits", &Tile::local_qubits);
    py::class_<Schedule>(m, "Schedule")
        .def_readonly("n", &Schedule::n)
        .def_readonly("n_local", &Schedule::n_local)
        .def_readonly("shape", &Schedule::shape)
        .def_readonly("order", &Schedule::order)
        .def_readonly("tiles", &Schedule::tiles)
        .def_readonly("qr_events", &Schedule::qr_events);
    py::class_<QrCounts>(m, "QrCounts")
        .def_readonly("total", &QrCounts::total)
        .def_readonly("intra", &QrCounts::intra)
        .def_readonly("inter", &QrCounts::inter);
    py::class_<CostWeights>(m, "CostWeights")
        .def(py::init([](double a, double b) { return CostWeights{a, b}; }), py::arg("w_intra") = 1.0,
             py::arg("w_inter") = 24.0)
        .def_readwrite("w_intra", &CostWeights::w_intra)
        .def_readwrite("w_inter", &CostWeights::w_inter)
        .def("validate", &CostWeights::validate);

    m.def("flat_tiling", &flat_tiling);
    m.def("hierarchical_tiling", &hierarchical_tiling);
    m.def("adhoc_schedule", &adhoc_schedule);
    m.def("tile_construction", &tile_construction);
    m.def("qubit_mapping", &qubit_mapping);
    m.def("hierarchical_qubit_mapping", &hierarchical_qubit_mapping);
    m.def("validate_schedule", [](const Circuit& c, const DependencyGraph& d, const Schedule& s) -> py::object {
        auto v = validate_schedule(c, d, s);
        if (!v) return py::none();
        return py::make_tuple(v->before, v->after);
    });
    m.def("schedule_is_narrow", &schedule_is_narrow);
    m.def("count_qrs", &count_qrs);
    m.def("qr_cost", &qr_cost);
    m.def("schedule_to_json", [](const Schedule& s) { return schedule_to_json(s).dump(); });
    m.def("qr_data_volume", &qr_data_volume);
    m.def("make_qr_event", [](const QubitLayout& l, QubitSet locals, std::optional<QubitSet> wanted) {
        return make_qr_event(l, locals, wanted);
    }, py::arg("before"), py::arg("new_locals"), py::arg("wanted_intra") = std::nullopt);
    m.def("make_qr_event_from_pairs", &make_qr_event_from_pairs);

    py::class_<PauliTermGroup>(m, "PauliTermGroup")
        .def_readonly("representative", &PauliTermGroup::representative)
        .def_readonly("members", &PauliTermGroup::members);
    py::class_<PauliTile>(m, "PauliTile")
        .def_readonly("local_qubits", &PauliTile::local_qubits)
        .def_readonly("groups", &PauliTile::groups)
        .def_readonly("terms", &PauliTile::terms);
    py::class_<PauliTilePlan>(m, "PauliTilePlan")
        .def_readonly("tiles", &PauliTilePlan::tiles)
        .def_readonly("qr_events", &PauliTilePlan::qr_events)
        .def_readonly("diagonalized", &PauliTilePlan::diagonalized)
        .def("qr_count", &PauliTilePlan::qr_count);
    py::class_<BaselineResult>(m, "BaselineResult").def_readonly("n_qr", &BaselineResult::n_qr);
    m.def("effective_targets", &effective_targets);
    m.def("merge_terms", &merge_terms);
    m.def("tiling_pauli_strings", &tiling_pauli_strings, py::arg("groups"), py::arg("n"), py::arg("shape"),
          py::arg("diagonalized"), py::arg("workers") = 1, py::arg("restrict_candidates") = false);
    m.def("plan_evc", &plan_evc, py::arg("terms"), py::arg("n"), py::arg("shape"), py::arg("diagonalize"),
          py::arg("workers") = 1, py::arg("restrict_candidates") = false);
    m.def("index_order_baseline", &index_order_baseline);
    m.def("plan_to_json", [](const PauliTilePlan& p) { return plan_to_json(p).dump(); });

    // ---- generators ------------------------------------------------------------
    m.def("random_unitary", [](int k, std::uint64_t seed) { return payload_to(std::make_shared<GateMatrix>(random_unitary(k, seed))); });
    m.def("gen_gatefabric", [](int n, int layers, std::uint64_t seed, bool payloads) {
        return gen_gatefabric(GateFabricSpec{n, layers, seed, payloads});
    }, py::arg("n"), py::arg("layers"), py::arg("seed") = 1, py::arg("payloads") = true);
    m.def("gatefabric_block_count", &gatefabric_block_count);
    m.def("gen_hea", [](int n, int depth, std::uint64_t seed, bool payloads) {
        return gen_hea(HeaSpec{n, depth, seed, payloads});
    }, py::arg("n"), py::arg("depth"), py::arg("seed") = 1, py::arg("payloads") = true);
    m.def("gen_synthetic_jw", &gen_synthetic_jw, py::arg("n"), py::arg("seed"), py::arg("max_span") = 0);
    m.def("synthetic_jw_term_count", &synthetic_jw_term_count, py::arg("n"), py::arg("max_span") = 0);
    m.def("gen_uniform_words", &gen_uniform_words, py::arg("n"), py::arg("count"), py::arg("seed") = 2024);
    m.def("gen_random_circuit", &gen_random_circuit, py::arg("n"), py::arg("m"), py::arg("seed"),
          py::arg("max_arity") = 2, py::arg("payloads") = true);
    m.def("random_state", [](int n, std::uint64_t seed) { return to_numpy(random_state(n, seed).amps); });
    m.def("seed_payloads", [](Circuit c, std::uint64_t seed) {
        seed_payloads(c, seed);
        return c;
    });
    m.def("fixture_circuit", &fixture_circuit, py::arg("name"), py::arg("seed") = 1);
    m.def("fixture_shape", &fixture_shape);
    m.def("fixture_hamiltonian", [](const std::string& name) {
        int n = 0;
        auto t = fixture_hamiltonian(name, &n);
        return py::make_tuple(t, n);
    });
    m.def("rng_stream", [](std::uint64_t seed, int count) {
        Rng r(seed);
        std::vector<std::uint64_t> out;
        for (int i = 0; i < count; ++i) out.push_back(r.next());
        return out;
    });

    // ---- device state (dist_sim) -------------------------------------------------
    m.def("init_device", &init_device, py::arg("rank") = 0, py::arg("world") = 1, py::arg("device") = 0,
          py::arg("unique_id") = py::bytes());
    m.def("device_unique_id", []() { return py::bytes(device_unique_id()); });
    m.def("device_context", []() {
        const auto& c = device_context();
        return py::make_tuple(c.rank, c.world, c.device);
    });
    m.def("shutdown_device", &shutdown_device);
    m.def("device_count", []() {
        int n = 0;
        qrt_device_count(&n);
        return n;
    });

    py::class_<DistributedState>(m, "DistributedState")
        .def_readonly("n", &DistributedState::n)
        .def_readonly("shape", &DistributedState::shape)
        .def_readonly("layout", &DistributedState::layout)
        .def_readonly("last_relocated", &DistributedState::last_relocated)
        .def_readonly("total_relocated", &DistributedState::total_relocated)
        .def_readonly("qr_log", &DistributedState::qr_log)
        .def("n_local", &DistributedState::n_local)
        .def("norm", &DistributedState::norm)
        .def("pe_begin", &DistributedState::pe_begin)
        .def("pe_count", &DistributedState::pe_count)
        .def("sub_of", [](const DistributedState& s, int pe) { return to_numpy(s.sub_of(pe)); })
        .def_property_readonly("sub", [](const DistributedState& s) {
            py::list out;
            for (auto& v : s.sub_vectors()) out.append(to_numpy(v));
            return out;
        })
        .def("set_sub", [](DistributedState& s, int pe, const CArray& a) { s.set_sub(pe, from_numpy(a)); })
        .def("clone", &DistributedState::clone)
        .def_property_readonly("phys_pos_of", [](const DistributedState& s) { return s.device->phys_pos_of; })
        .def("stats", [](const DistributedState& s) {
            qrt_kernel_stats st[QRT_K_COUNT];
            qrt_stats(s.device->handle, st);
            py::dict d;
            const char* names[QRT_K_COUNT] = {"gates", "qr", "pauli", "misc", "qr_xfer"};
            for (int i = 0; i < QRT_K_COUNT; ++i) {
                py::dict e;
                e["launches"] = st[i].launches;
                e["ms"] = st[i].ms;
                e["bytes"] = st[i].bytes;
                e["flops"] = st[i].flops;
                e["calls"] = st[i].calls;
                d[names[i]] = e;
            }
            return d;
        })
        .def("reset_stats", [](DistributedState& s) { qrt_stats_reset(s.device->handle); })
        .def("profile", [](DistributedState& s, bool on) { qrt_profile_enable(s.device->handle, on ? 1 : 0); })
        .def("stream", [](const DistributedState& s) {
            void* p = nullptr;
            qrt_state_stream(s.device->handle, &p);
            return reinterpret_cast<std::uintptr_t>(p);
        })
        .def("synchronize", [](DistributedState& s) { qrt_synchronize(s.device->handle); })
        .def("handle", [](const DistributedState& s) { return reinterpret_cast<std::uintptr_t>(s.device->handle); });

    m.def("init_state", [](int n, const ClusterShape& shape) { return init_state(n, shape); });
    m.def("init_state_from", [](const CArray& amps, const ClusterShape& shape) {
        ReferenceState r;
        r.amps = from_numpy(amps);
        int n = 0;
        while ((std::size_t{1} << n) < r.amps.size()) ++n;
        if ((std::size_t{1} << n) != r.amps.size()) throw ConfigError("amplitude count must be a power of two");
        r.n = n;
        return init_state(r, shape);
    });
    m.def("flatten", [](const DistributedState& s) { return to_numpy(flatten(s).amps); });
    m.def("apply_gate_narrow", &apply_gate_narrow, py::arg("state"), py::arg("gate"), py::arg("workers") = 1);
    m.def("apply_gates_narrow", &apply_gates_narrow);
    m.def("perform_qr", &perform_qr);
    m.def("physical_reorder_plan", [](const QrEvent& ev, const std::vector<int>& phys) {
        std::vector<int> np;
        std::vector<int> dest = physical_reorder_plan(ev, phys, np);
        return py::make_tuple(dest, np);
    });
    m.def("run_qsu", &run_qsu, py::arg("state"), py::arg("circuit"), py::arg("schedule"), py::arg("workers") = 1);
    m.def("diag_expectation_term", &diag_expectation_term);
    m.def("expectation", &expectation, py::arg("state"), py::arg("plan"), py::arg("terms"), py::arg("workers") = 1);
    m.def("evaluate_energy", &evaluate_energy, py::arg("circuit"), py::arg("schedule"), py::arg("terms"),
          py::arg("plan"), py::arg("workers") = 1);
    m.def("write_state_dump", [](const CArray& amps, int p) {
        ReferenceState r;
        r.amps = from_numpy(amps);
        while ((std::size_t{1} << r.n) < r.amps.size()) ++r.n;
        std::ostringstream out;
        write_state_dump(out, r, p);
        return py::bytes(out.str());
    });
    m.def("read_state_dump", [](const py::bytes& b) {
        std::istringstream in{std::string(b)};
        int p = 0;
        ReferenceState r = read_state_dump(in, &p);
        return py::make_tuple(to_numpy(r.amps), r.n, p);
    });
    m.attr("kOracleMaxQubits") = kOracleMaxQubits;
    m.attr("QRT_ABI_VERSION") = QRT_ABI_VERSION;
    m.def("build_flags", []() { return qrt_build_flags(); });
}
