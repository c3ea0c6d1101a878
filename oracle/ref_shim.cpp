// TEST INFRASTRUCTURE ONLY — not part of the product.
//
// A C-ABI shim over the *unmodified* reference library (qrtile, compiled
// straight from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libqrtile_ref.so).  It lets the Python test-suite and the
// bench's CPU-baseline leg drive the reference's own code path:
//   schedulers  qsu_scheduler.cpp:186-249, evc_scheduler.cpp:238-280
//   dist-sim    dist_sim.cpp:122-363 (init_state, run_qsu, expectation,
//               evaluate_energy, dense oracle)
//   generators  models.cpp:37-206
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it.  Every entry point catches C++
// exceptions and reports them through ref_last_error().

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "qrtile/dist_sim.hpp"
#include "qrtile/evc_scheduler.hpp"
#include "qrtile/models.hpp"
#include "qrtile/qsu_scheduler.hpp"
#include "qrtile/schedule.hpp"

using namespace qrtile;

namespace {

thread_local std::string g_err;

struct Terms {
    int n = 0;
    std::vector<PauliTerm> terms;
};

ClusterShape shape_of(int p, int n_node, int n_gpn) {
    if (n_node > 0 && n_gpn > 0) return ClusterShape::two_level(n_node, n_gpn);
    return ClusterShape::flat(p);
}

Schedule pick(const char* name, const Circuit& c, const DependencyGraph& d, const ClusterShape& s) {
    std::string k(name);
    if (k == "flat") return flat_tiling(c, d, s);
    if (k == "hierarchical") return hierarchical_tiling(c, d, s);
    if (k == "adhoc") return adhoc_schedule(c, d, s);
    throw ConfigError("unknown scheduler " + k);
}

char* dup(const std::string& s) {
    char* out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(out, s.data(), s.size() + 1);
    return out;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

double secs() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// ---------------------------------------------------------------- circuits
void* ref_circuit_gatefabric(int n, int layers, uint64_t seed, int payloads) {
    Circuit* c = nullptr;
    guarded([&] { c = new Circuit(gen_gatefabric(GateFabricSpec{n, layers, seed, payloads != 0})); });
    return c;
}

// The HEA of SURVEY.md §8d C4 (absent from the reference): per layer RY(theta)
// on every qubit, RZ(theta) on every qubit, CZ(q, q+1) for even q then odd q,
// theta ~ uniform(0, 2 pi) from the reference's Rng(seed) in gate order —
// built from reference types so the reference arm never loads the product.
void* ref_circuit_hea(int n, int depth, uint64_t seed) {
    Circuit* c = nullptr;
    guarded([&] {
        auto out = std::make_unique<Circuit>();
        out->n = n;
        Rng rng(seed);
        auto angle = [&] { return rng.uniform(0.0, 2.0 * 3.14159265358979323846); };
        auto push = [&](std::vector<int> t, GatePayload pl) {
            out->operators.push_back(make_gate(static_cast<int>(out->operators.size()), std::move(t), std::move(pl)));
        };
        auto cz = std::make_shared<GateMatrix>(4);
        cz->at(0, 0) = 1.0;
        cz->at(1, 1) = 1.0;
        cz->at(2, 2) = 1.0;
        cz->at(3, 3) = -1.0;
        for (int layer = 0; layer < depth; ++layer) {
            for (int q = 0; q < n; ++q) {
                const double th = angle();
                auto m = std::make_shared<GateMatrix>(2);
                m->at(0, 0) = std::cos(th / 2);
                m->at(0, 1) = -std::sin(th / 2);
                m->at(1, 0) = std::sin(th / 2);
                m->at(1, 1) = std::cos(th / 2);
                push({q}, m);
            }
            for (int q = 0; q < n; ++q) {
                const double th = angle();
                auto m = std::make_shared<GateMatrix>(2);
                m->at(0, 0) = std::polar(1.0, -th / 2);
                m->at(1, 1) = std::polar(1.0, th / 2);
                push({q}, m);
            }
            for (int parity = 0; parity < 2; ++parity)
                for (int q = parity; q + 1 < n; q += 2) push({q, q + 1}, cz);
        }
        c = out.release();
    });
    return c;
}

void* ref_circuit_random(int n, int m, uint64_t seed, int max_arity, int payloads) {
    Circuit* c = nullptr;
    guarded([&] { c = new Circuit(gen_random_circuit(n, m, seed, max_arity, payloads != 0)); });
    return c;
}

void* ref_circuit_fixture(const char* name, uint64_t seed) {
    Circuit* c = nullptr;
    guarded([&] { c = new Circuit(fixture_circuit(name, seed)); });
    return c;
}

// Builds a circuit from flat arrays; mats may be NULL (payload-free).
void* ref_circuit_from_arrays(int n, int m, const int* arity, const int* targets, const double* mats) {
    Circuit* c = nullptr;
    guarded([&] {
        auto out = std::make_unique<Circuit>();
        out->n = n;
        std::size_t t = 0, off = 0;
        for (int i = 0; i < m; ++i) {
            std::vector<int> tg(targets + t, targets + t + arity[i]);
            t += static_cast<std::size_t>(arity[i]);
            GatePayload pl;
            if (mats) {
                int dim = 1 << arity[i];
                auto g = std::make_shared<GateMatrix>(dim);
                for (int e = 0; e < dim * dim; ++e) g->a[static_cast<std::size_t>(e)] = Amp{mats[off + 2 * e], mats[off + 2 * e + 1]};
                off += static_cast<std::size_t>(2 * dim * dim);
                pl = g;
            }
            out->operators.push_back(make_gate(i, tg, pl));
        }
        c = out.release();
    });
    return c;
}

void ref_circuit_free(void* h) { delete static_cast<Circuit*>(h); }
int ref_circuit_n(void* h) { return static_cast<Circuit*>(h)->n; }
int ref_circuit_m(void* h) { return static_cast<Circuit*>(h)->size(); }
int ref_circuit_total_targets(void* h) {
    int s = 0;
    for (auto& o : static_cast<Circuit*>(h)->operators) s += o.arity();
    return s;
}
int64_t ref_circuit_total_mat_doubles(void* h) {
    int64_t s = 0;
    for (auto& o : static_cast<Circuit*>(h)->operators)
        if (o.payload) s += 2LL * o.payload->dim * o.payload->dim;
    return s;
}
// Exports targets (and payloads when mats != NULL and present).
int ref_circuit_export(void* h, int* arity, int* targets, double* mats) {
    auto* c = static_cast<Circuit*>(h);
    std::size_t t = 0, off = 0;
    for (auto& o : c->operators) {
        arity[o.id] = o.arity();
        for (int q : o.targets) targets[t++] = q;
        if (mats && o.payload)
            for (const Amp& a : o.payload->a) {
                mats[off++] = a.real();
                mats[off++] = a.imag();
            }
    }
    return 0;
}

// ------------------------------------------------------------------ terms
void* ref_terms_jw(int n, uint64_t seed, int max_span) {
    Terms* t = nullptr;
    guarded([&] {
        t = new Terms{n, gen_synthetic_jw(n, seed, max_span)};
    });
    return t;
}
// C5 stress words drawn with the reference's own Rng
// (models.hpp:15-31, models.cpp:26-35): letters "IXYZ"[below(4)] per qubit,
// then the coefficient uniform(-1, 1).
void* ref_terms_uniform(int n, int count, uint64_t seed) {
    Terms* t = nullptr;
    guarded([&] {
        Rng rng(seed);
        std::vector<PauliTerm> ts;
        for (int i = 0; i < count; ++i) {
            std::string letters(static_cast<std::size_t>(n), 'I');
            for (int q = 0; q < n; ++q) letters[static_cast<std::size_t>(q)] = "IXYZ"[rng.below(4)];
            ts.push_back(PauliTerm{Amp{rng.uniform(-1.0, 1.0), 0.0}, letters});
        }
        t = new Terms{n, std::move(ts)};
    });
    return t;
}
void* ref_terms_fixture(const char* name) {
    Terms* t = nullptr;
    guarded([&] {
        int n = 0;
        auto ts = fixture_hamiltonian(name, &n);
        t = new Terms{n, ts};
    });
    return t;
}
void* ref_terms_from_arrays(int n, int count, const char* letters, const double* coeffs) {
    Terms* t = nullptr;
    guarded([&] {
        auto out = std::make_unique<Terms>();
        out->n = n;
        for (int i = 0; i < count; ++i)
            out->terms.push_back(PauliTerm{Amp{coeffs[2 * i], coeffs[2 * i + 1]},
                                           std::string(letters + static_cast<std::size_t>(i) * n, static_cast<std::size_t>(n))});
        t = out.release();
    });
    return t;
}
void ref_terms_free(void* h) { delete static_cast<Terms*>(h); }
int ref_terms_count(void* h) { return static_cast<int>(static_cast<Terms*>(h)->terms.size()); }
int ref_terms_n(void* h) { return static_cast<Terms*>(h)->n; }
void ref_terms_export(void* h, char* letters, double* coeffs) {
    auto* t = static_cast<Terms*>(h);
    for (std::size_t i = 0; i < t->terms.size(); ++i) {
        std::memcpy(letters + i * static_cast<std::size_t>(t->n), t->terms[i].letters.data(), static_cast<std::size_t>(t->n));
        coeffs[2 * i] = t->terms[i].coeff.real();
        coeffs[2 * i + 1] = t->terms[i].coeff.imag();
    }
}

// -------------------------------------------------------------- schedules
// Returns malloc'd JSON: {"schedule": schedule_to_json, "counts": {...},
// "layouts": [after.pos_of per event], "tile_sizes": [...]}
char* ref_schedule_json(void* circ, const char* name, int p, int n_node, int n_gpn) {
    char* out = nullptr;
    guarded([&] {
        auto* c = static_cast<Circuit*>(circ);
        DependencyGraph d = build_dependency_graph(*c);
        ClusterShape s = shape_of(p, n_node, n_gpn);
        Schedule sch = pick(name, *c, d, s);
        QrCounts q = count_qrs(sch);
        nlohmann::json j;
        j["schedule"] = schedule_to_json(sch);
        j["counts"] = {{"total", q.total}, {"intra", q.intra}, {"inter", q.inter}};
        nlohmann::json lay = nlohmann::json::array();
        for (auto& ev : sch.qr_events) lay.push_back({{"before_tile", ev.before_tile}, {"after_pos_of", ev.after.pos_of}});
        j["events"] = lay;
        j["valid"] = !validate_schedule(*c, d, sch).has_value();
        j["narrow"] = schedule_is_narrow(*c, sch);
        out = dup(j.dump());
    });
    return out;
}

char* ref_depth_sort_json(void* circ) {
    char* out = nullptr;
    guarded([&] {
        auto* c = static_cast<Circuit*>(circ);
        DependencyGraph d = build_dependency_graph(*c);
        nlohmann::json j;
        j["order"] = depth_sort(*c, d);
        j["depth"] = d.depth;
        j["edges"] = d.edges;
        out = dup(j.dump());
    });
    return out;
}

char* ref_plan_json(void* terms, int n, int p, int n_node, int n_gpn, int diagonalize, int workers) {
    char* out = nullptr;
    guarded([&] {
        auto* t = static_cast<Terms*>(terms);
        ClusterShape s = shape_of(p, n_node, n_gpn);
        auto groups = merge_terms(t->terms, diagonalize != 0);
        PauliTilePlan plan = tiling_pauli_strings(groups, n, s, diagonalize != 0, workers);
        BaselineResult base = index_order_baseline(t->terms, n, s);
        nlohmann::json j;
        j["plan"] = plan_to_json(plan);
        j["qr_count"] = plan.qr_count();
        j["baseline_qr"] = base.n_qr;
        j["n_groups"] = static_cast<int>(groups.size());
        nlohmann::json g = nlohmann::json::array();
        for (auto& gr : groups) g.push_back({{"rep", gr.representative}, {"members", gr.members}});
        j["groups"] = g;
        out = dup(j.dump());
    });
    return out;
}

// ------------------------------------------------------------- simulation
int ref_random_state(int n, uint64_t seed, double* out) {
    return guarded([&] {
        ReferenceState r = random_state(n, seed);
        std::memcpy(out, r.amps.data(), r.amps.size() * sizeof(Amp));
    });
}

// Runs the reference QSU from the zero state; writes flatten() into out
// (2^n complex) and the qr_log relocation counts into qr_moved (may be NULL).
int ref_run_qsu(void* circ, const char* sched, int p, int n_node, int n_gpn, int workers,
                double* out, uint64_t* qr_moved, int* qr_k, int* n_qr) {
    return guarded([&] {
        auto* c = static_cast<Circuit*>(circ);
        DependencyGraph d = build_dependency_graph(*c);
        ClusterShape s = shape_of(p, n_node, n_gpn);
        Schedule sch = pick(sched, *c, d, s);
        DistributedState st = init_state(c->n, s);
        run_qsu(st, *c, sch, workers);
        ReferenceState r = flatten(st);
        std::memcpy(out, r.amps.data(), r.amps.size() * sizeof(Amp));
        if (n_qr) *n_qr = static_cast<int>(st.qr_log.size());
        for (std::size_t i = 0; i < st.qr_log.size(); ++i) {
            if (qr_k) qr_k[i] = st.qr_log[i].first;
            if (qr_moved) qr_moved[i] = st.qr_log[i].second;
        }
    });
}

int ref_dense_qsu(void* circ, double* out) {
    return guarded([&] {
        auto* c = static_cast<Circuit*>(circ);
        ReferenceState r = ReferenceState::zero(c->n);
        for (auto& op : c->operators) dense_oracle_apply(r, op);
        std::memcpy(out, r.amps.data(), r.amps.size() * sizeof(Amp));
    });
}

int ref_dense_expectation(const double* canon, int n, void* terms, double* out2) {
    return guarded([&] {
        ReferenceState r;
        r.n = n;
        r.amps.assign(reinterpret_cast<const Amp*>(canon), reinterpret_cast<const Amp*>(canon) + (std::size_t{1} << n));
        Amp e = dense_oracle_expectation(r, static_cast<Terms*>(terms)->terms);
        out2[0] = e.real();
        out2[1] = e.imag();
    });
}

// Expectation of `terms` on a canonical state distributed with
// init_state(ref, shape); also reports the executed QR count and the
// post-EVC flatten (out_after may be NULL).
int ref_expectation(const double* canon, int n, void* terms, int p, int n_node, int n_gpn,
                    int diagonalize, int workers, double* out2, int* n_qr, double* out_after) {
    return guarded([&] {
        ReferenceState r;
        r.n = n;
        r.amps.assign(reinterpret_cast<const Amp*>(canon), reinterpret_cast<const Amp*>(canon) + (std::size_t{1} << n));
        ClusterShape s = shape_of(p, n_node, n_gpn);
        DistributedState st = init_state(r, s);
        auto& ts = static_cast<Terms*>(terms)->terms;
        PauliTilePlan plan = plan_evc(ts, n, s, diagonalize != 0, workers);
        Amp e = expectation(st, plan, ts, workers);
        out2[0] = e.real();
        out2[1] = e.imag();
        if (n_qr) *n_qr = static_cast<int>(st.qr_log.size());
        if (out_after) {
            ReferenceState f = flatten(st);
            std::memcpy(out_after, f.amps.data(), f.amps.size() * sizeof(Amp));
        }
    });
}

// One VQE iteration (evaluate_energy, dist_sim.cpp:357) plus the executed
// QR totals of QSU and EVC.
int ref_evaluate_energy(void* circ, void* terms, const char* sched, int p, int n_node, int n_gpn,
                        int diagonalize, int workers, double* energy, int* qsu_qr, int* evc_qr) {
    return guarded([&] {
        auto* c = static_cast<Circuit*>(circ);
        auto& ts = static_cast<Terms*>(terms)->terms;
        DependencyGraph d = build_dependency_graph(*c);
        ClusterShape s = shape_of(p, n_node, n_gpn);
        Schedule sch = pick(sched, *c, d, s);
        PauliTilePlan plan = plan_evc(ts, c->n, s, diagonalize != 0, workers);
        *energy = evaluate_energy(*c, sch, ts, plan, workers);
        DistributedState st = init_state(c->n, s);
        run_qsu(st, *c, sch, workers);
        if (qsu_qr) *qsu_qr = static_cast<int>(st.qr_log.size());
        std::size_t before = st.qr_log.size();
        (void)expectation(st, plan, ts, workers);
        if (evc_qr) *evc_qr = static_cast<int>(st.qr_log.size() - before);
    });
}

// ------------------------------------------------------- CPU-baseline timing
// Times the reference's hot loops on a bounded sample: apply_gate_narrow on
// the first `n_gates` gates of `circ` that are narrow under the identity
// layout, then `n_terms` expectation terms (diagonalized plan restricted to
// the first tile's terms).  Returns seconds per gate and per term.
int ref_time_sample(void* circ, void* terms, int p, int workers, int n_gates, int n_terms,
                    double* sec_per_gate, double* sec_per_term) {
    return guarded([&] {
        auto* c = static_cast<Circuit*>(circ);
        ClusterShape s = ClusterShape::flat(p);
        DistributedState st = init_state(c->n, s);
        int done = 0;
        double t0 = secs();
        for (auto& op : c->operators) {
            if (done >= n_gates) break;
            if (classify_access(op, st.layout) != Access::Narrow) continue;
            apply_gate_narrow(st, op, workers);
            ++done;
        }
        double t1 = secs();
        *sec_per_gate = done ? (t1 - t0) / done : 0.0;
        *sec_per_term = 0.0;
        if (terms && n_terms > 0) {
            auto& all = static_cast<Terms*>(terms)->terms;
            std::vector<PauliTerm> pick_terms;
            for (auto& t : all) {
                bool ok = true;
                for (int q = 0; q < t.n(); ++q) {
                    char ch = t.letters[static_cast<std::size_t>(q)];
                    if (ch != 'I' && ch != 'Z' && st.layout.pos_of[static_cast<std::size_t>(q)] >= st.layout.n_local) ok = false;
                }
                if (ok) pick_terms.push_back(t);
                if (static_cast<int>(pick_terms.size()) >= n_terms) break;
            }
            PauliTilePlan plan;
            plan.n = c->n;
            plan.n_local = st.layout.n_local;
            plan.shape = s;
            plan.diagonalized = true;
            PauliTile tile;
            tile.local_qubits = st.layout.local_set();
            for (int i = 0; i < static_cast<int>(pick_terms.size()); ++i) tile.terms.push_back(i);
            plan.tiles.push_back(tile);
            double t2 = secs();
            (void)expectation(st, plan, pick_terms, workers);
            double t3 = secs();
            *sec_per_term = pick_terms.empty() ? 0.0 : (t3 - t2) / static_cast<double>(pick_terms.size());
        }
    });
}

// The reference arm's bounded sample (SURVEY.md §8d "CPU timing beside it"):
// on an identity-layout state of circ->n qubits and flat(p), time
//   * apply_gate_narrow (dist_sim.cpp:163-201) on the first `per_arity`
//     narrow gates of each arity 1..4 -> sec_per_gate[arity-1] (0 if none),
//   * expectation (dist_sim.cpp:263-300) on the first `n_terms` terms that
//     need no QR under the identity layout -> *sec_per_term,
//   * perform_qr (dist_sim.cpp:203-240; single-threaded) once for each k in
//     1..log2 p, swapping the k highest local qubits with the k globals ->
//     sec_per_qr[k-1].
int ref_time_prefix(void* circ, void* terms, int p, int workers, int per_arity, int n_terms,
                    double* sec_per_gate, double* sec_per_term, double* sec_per_qr) {
    return guarded([&] {
        auto* c = static_cast<Circuit*>(circ);
        ClusterShape s = ClusterShape::flat(p);
        DistributedState st = init_state(c->n, s);
        for (int a = 1; a <= 4; ++a) {
            int done = 0;
            double t0 = secs();
            for (auto& op : c->operators) {
                if (done >= per_arity) break;
                if (op.arity() != a || classify_access(op, st.layout) != Access::Narrow) continue;
                apply_gate_narrow(st, op, workers);
                ++done;
            }
            sec_per_gate[a - 1] = done ? (secs() - t0) / done : 0.0;
        }
        *sec_per_term = 0.0;
        if (terms && n_terms > 0) {
            auto& all = static_cast<Terms*>(terms)->terms;
            std::vector<PauliTerm> pick_terms;
            for (auto& t : all) {
                bool ok = true;
                for (int q = 0; q < t.n(); ++q) {
                    char ch = t.letters[static_cast<std::size_t>(q)];
                    if (ch != 'I' && ch != 'Z' && st.layout.pos_of[static_cast<std::size_t>(q)] >= st.layout.n_local) ok = false;
                }
                if (ok) pick_terms.push_back(t);
                if (static_cast<int>(pick_terms.size()) >= n_terms) break;
            }
            PauliTilePlan plan;
            plan.n = c->n;
            plan.n_local = st.layout.n_local;
            plan.shape = s;
            plan.diagonalized = true;
            PauliTile tile;
            tile.local_qubits = st.layout.local_set();
            for (int i = 0; i < static_cast<int>(pick_terms.size()); ++i) tile.terms.push_back(i);
            plan.tiles.push_back(tile);
            double t2 = secs();
            (void)expectation(st, plan, pick_terms, workers);
            double t3 = secs();
            *sec_per_term = pick_terms.empty() ? 0.0 : (t3 - t2) / static_cast<double>(pick_terms.size());
        }
        const int g = s.global_bits();
        for (int k = 1; k <= g; ++k) {
            QubitSet locals = st.layout.local_set();
            const int nl = st.layout.n_local;
            for (int j = 0; j < k; ++j) {
                locals &= ~(QubitSet{1} << st.layout.qubit_at[static_cast<std::size_t>(nl - 1 - j)]);
                locals |= QubitSet{1} << st.layout.qubit_at[static_cast<std::size_t>(nl + j)];
            }
            auto ev = make_qr_event(st.layout, locals);
            double t0 = secs();
            if (ev) perform_qr(st, *ev);
            sec_per_qr[k - 1] = secs() - t0;
        }
    });
}

}  // extern "C"
