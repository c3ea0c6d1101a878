// B200 qrtile drop-in — deterministic synthetic inputs.  Bit-identical to the
// reference generators for equal seeds (/root/reference/proj/src/models.cpp:
// Rng :12-35, random_unitary :37-59, GateFabric :61-89, JW :91-162,
// random circuits/states :164-197, seed_payloads :199-206, fixtures
// :208-276), plus the hardware-efficient ansatz the reference lacks
// (SURVEY.md §8d, config C4).

#include <algorithm>
#include <numbers>

#include "qrtile/models.hpp"

namespace qrtile {

double Rng::normal() {
    if (have_spare_) {
        have_spare_ = false;
        return spare_;
    }
    const double u = 1.0 - uniform();  // (0, 1]
    const double v = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u));
    const double angle = 2.0 * std::numbers::pi * v;
    spare_ = radius * std::sin(angle);
    have_spare_ = true;
    return radius * std::cos(angle);
}

int Rng::below(int bound) {
    if (bound <= 0) throw ConfigError("rng bound must be positive");
    const std::uint64_t b = static_cast<std::uint64_t>(bound);
    const std::uint64_t top = ~std::uint64_t{0};
    const std::uint64_t reject = (top % b + 1) % b;  // size of the biased tail
    for (;;) {
        const std::uint64_t x = next();
        if (reject == 0 || x <= top - reject) return static_cast<int>(x % b);
    }
}

GateMatrix random_unitary(int k_qubits, std::uint64_t seed) {
    const int dim = 1 << k_qubits;
    Rng rng(seed);
    GateMatrix u(dim);
    for (int r = 0; r < dim; ++r)
        for (int c = 0; c < dim; ++c) {
            const double re = rng.normal();
            const double im = rng.normal();
            u.at(r, c) = Amp{re, im};
        }
    // Modified Gram-Schmidt over the columns, two passes.
    for (int pass = 0; pass < 2; ++pass)
        for (int c = 0; c < dim; ++c) {
            for (int j = 0; j < c; ++j) {
                Amp proj = 0.0;
                for (int r = 0; r < dim; ++r) proj += std::conj(u.at(r, j)) * u.at(r, c);
                for (int r = 0; r < dim; ++r) u.at(r, c) -= proj * u.at(r, j);
            }
            double norm2 = 0.0;
            for (int r = 0; r < dim; ++r) norm2 += std::norm(u.at(r, c));
            const double len = std::sqrt(norm2);
            for (int r = 0; r < dim; ++r) u.at(r, c) /= len;
        }
    return u;
}

int gatefabric_block_count(int n, int layers) { return layers * (n / 4 + (n - 2) / 4); }

Circuit gen_gatefabric(const GateFabricSpec& spec) {
    if (spec.n < 4) throw CircuitTooSmall("GateFabric needs at least 4 qubits");
    if (spec.n % 2 != 0) throw ConfigError("GateFabric needs an even qubit count");
    if (spec.layers < 1) throw ConfigError("GateFabric needs at least one layer");
    Circuit c;
    c.n = spec.n;
    Rng master(spec.seed);
    auto block = [&](int first) {
        GatePayload pl;
        if (spec.payloads) pl = std::make_shared<GateMatrix>(random_unitary(4, master.next()));
        c.operators.push_back(make_gate(c.size(), {first, first + 1, first + 2, first + 3}, std::move(pl)));
    };
    for (int layer = 0; layer < spec.layers; ++layer) {
        for (int first = 0; first + 3 < spec.n; first += 4) block(first);  // even bricks
        for (int first = 2; first + 3 < spec.n; first += 4) block(first);  // offset bricks
    }
    return c;
}

namespace {
// n letters 'I', Z on the open interval of every chain, then explicit letters.
std::string word(int n, std::initializer_list<std::pair<int, char>> put,
                 std::initializer_list<std::pair<int, int>> chains = {}) {
    std::string s(static_cast<std::size_t>(n), 'I');
    for (const auto& [lo, hi] : chains)
        for (int q = lo + 1; q < hi; ++q) s[static_cast<std::size_t>(q)] = 'Z';
    for (const auto& [q, ch] : put) s[static_cast<std::size_t>(q)] = ch;
    return s;
}
}  // namespace

std::vector<PauliTerm> gen_synthetic_jw(int n, std::uint64_t seed, int max_span) {
    if (n < 2) throw ConfigError("Hamiltonian generator needs at least 2 qubits");
    const int span = max_span > 0 ? max_span : n;
    Rng rng(seed);
    std::vector<PauliTerm> out;
    auto add = [&](std::string letters) { out.push_back(PauliTerm{Amp{rng.uniform(-1.0, 1.0), 0.0}, std::move(letters)}); };

    add(std::string(static_cast<std::size_t>(n), 'I'));
    for (int i = 0; i < n; ++i) add(word(n, {{i, 'Z'}}));
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n && j - i + 1 <= span; ++j) add(word(n, {{i, 'Z'}, {j, 'Z'}}));
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n && j - i + 1 <= span; ++j) {
            add(word(n, {{i, 'X'}, {j, 'X'}}, {{i, j}}));
            add(word(n, {{i, 'Y'}, {j, 'Y'}}, {{i, j}}));
        }
    static constexpr char kPatterns[4][4] = {{'X', 'X', 'X', 'X'}, {'X', 'X', 'Y', 'Y'},
                                             {'Y', 'Y', 'X', 'X'}, {'Y', 'Y', 'Y', 'Y'}};
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j)
            for (int k = j + 1; k < n; ++k)
                for (int l = k + 1; l < n && l - i + 1 <= span; ++l)
                    for (const auto& pat : kPatterns)
                        add(word(n, {{i, pat[0]}, {j, pat[1]}, {k, pat[2]}, {l, pat[3]}}, {{i, j}, {k, l}}));
    return out;
}

std::uint64_t synthetic_jw_term_count(int n, int max_span) {
    const int span = max_span > 0 ? max_span : n;
    std::uint64_t count = 1 + static_cast<std::uint64_t>(n);
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n && j - i + 1 <= span; ++j) count += 3;
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j)
            for (int k = j + 1; k < n; ++k)
                for (int l = k + 1; l < n && l - i + 1 <= span; ++l) count += 4;
    return count;
}

Circuit gen_random_circuit(int n, int m, std::uint64_t seed, int max_arity, bool payloads) {
    if (max_arity < 1 || max_arity > n) throw ConfigError("bad gate arity bound");
    Rng rng(seed);
    Circuit c;
    c.n = n;
    for (int id = 0; id < m; ++id) {
        const int arity = 1 + rng.below(max_arity);
        std::vector<int> targets;
        while (static_cast<int>(targets.size()) < arity) {
            const int q = rng.below(n);
            if (std::find(targets.begin(), targets.end(), q) == targets.end()) targets.push_back(q);
        }
        GatePayload pl;
        if (payloads) pl = std::make_shared<GateMatrix>(random_unitary(arity, rng.next()));
        c.operators.push_back(make_gate(id, std::move(targets), std::move(pl)));
    }
    return c;
}

ReferenceState random_state(int n, std::uint64_t seed) {
    Rng rng(seed);
    ReferenceState ref;
    ref.n = n;
    ref.amps.resize(std::size_t{1} << n);
    double norm2 = 0.0;
    for (Amp& a : ref.amps) {
        const double re = rng.normal();
        const double im = rng.normal();
        a = Amp{re, im};
        norm2 += std::norm(a);
    }
    const double len = std::sqrt(norm2);
    for (Amp& a : ref.amps) a /= len;
    return ref;
}

void seed_payloads(Circuit& circuit, std::uint64_t seed) {
    Rng master(seed);
    for (Operator& op : circuit.operators) {
        const std::uint64_t s = master.next();  // drawn for every operator
        if (op.kind == OpKind::Gate && !op.payload)
            op.payload = std::make_shared<GateMatrix>(random_unitary(op.arity(), s));
    }
}

Circuit gen_hea(const HeaSpec& spec) {
    if (spec.n < 2) throw CircuitTooSmall("HEA needs at least 2 qubits");
    if (spec.depth < 1) throw ConfigError("HEA needs at least one layer");
    Circuit c;
    c.n = spec.n;
    Rng rng(spec.seed);
    auto angle = [&] { return rng.uniform(0.0, 2.0 * std::numbers::pi); };
    auto push = [&](std::vector<int> t, GatePayload pl) {
        c.operators.push_back(make_gate(c.size(), std::move(t), spec.payloads ? std::move(pl) : nullptr));
    };
    static const GatePayload cz = [] {
        auto m = std::make_shared<GateMatrix>(4);
        m->at(0, 0) = 1.0;
        m->at(1, 1) = 1.0;
        m->at(2, 2) = 1.0;
        m->at(3, 3) = -1.0;
        return m;
    }();
    for (int layer = 0; layer < spec.depth; ++layer) {
        for (int q = 0; q < spec.n; ++q) {  // RY(theta) = exp(-i theta Y / 2)
            const double th = angle();
            auto m = std::make_shared<GateMatrix>(2);
            m->at(0, 0) = std::cos(th / 2);
            m->at(0, 1) = -std::sin(th / 2);
            m->at(1, 0) = std::sin(th / 2);
            m->at(1, 1) = std::cos(th / 2);
            push({q}, m);
        }
        for (int q = 0; q < spec.n; ++q) {  // RZ(theta) = diag(e^{-i theta/2}, e^{i theta/2})
            const double th = angle();
            auto m = std::make_shared<GateMatrix>(2);
            m->at(0, 0) = std::polar(1.0, -th / 2);
            m->at(1, 1) = std::polar(1.0, th / 2);
            push({q}, m);
        }
        for (int parity = 0; parity < 2; ++parity)
            for (int q = parity; q + 1 < spec.n; q += 2) push({q, q + 1}, cz);
    }
    return c;
}

std::vector<PauliTerm> gen_uniform_words(int n, int count, std::uint64_t seed) {
    if (n < 1) throw ConfigError("uniform words need at least 1 qubit");
    if (count < 0) throw ConfigError("uniform word count must be non-negative");
    Rng rng(seed);
    std::vector<PauliTerm> terms;
    terms.reserve(static_cast<std::size_t>(count));
    for (int t = 0; t < count; ++t) {
        std::string letters(static_cast<std::size_t>(n), 'I');
        for (int q = 0; q < n; ++q) letters[static_cast<std::size_t>(q)] = "IXYZ"[rng.below(4)];
        terms.push_back(PauliTerm{Amp{rng.uniform(-1.0, 1.0), 0.0}, std::move(letters)});
    }
    return terms;
}

// ---------------------------------------------------------------- fixtures

std::vector<std::string> fixture_circuit_names() { return {"fig2", "fig3", "fig7", "gatefabric-fig6"}; }

Circuit fixture_circuit(const std::string& name, std::uint64_t seed) {
    auto from_targets = [](int n, std::vector<std::vector<int>> targets) {
        Circuit c;
        c.n = n;
        for (auto& t : targets) c.operators.push_back(make_gate(c.size(), std::move(t)));
        return c;
    };
    Circuit c;
    if (name == "fig2")
        c = from_targets(4, {{0, 1}, {2, 3}, {1, 2}, {1}, {2}});
    else if (name == "fig3")
        c = from_targets(4, {{0, 1}, {2, 3}, {1, 2}, {0, 1}, {0, 3}});
    else if (name == "fig7")
        c = from_targets(6, {{0, 1}, {2, 3}, {4, 5}, {0, 1}, {3, 4}, {0, 2}, {2, 3}, {4, 5}});
    else if (name == "gatefabric-fig6")
        return gen_gatefabric(GateFabricSpec{16, 6, seed, true});
    else
        throw ConfigError("unknown circuit fixture: " + name);
    seed_payloads(c, seed);
    return c;
}

ClusterShape fixture_shape(const std::string& name) {
    if (name == "fig2" || name == "fig3" || name == "fig7") return ClusterShape::flat(4);
    if (name == "gatefabric-fig6") return ClusterShape::two_level(4, 4);
    throw ConfigError("unknown circuit fixture: " + name);
}

std::vector<std::string> fixture_hamiltonian_names() { return {"evc-diagram", "three-term", "jw8", "jw10", "jw12"}; }

std::vector<PauliTerm> fixture_hamiltonian(const std::string& name, int* n_out) {
    std::vector<PauliTerm> terms;
    int n = 0;
    if (name == "evc-diagram") {
        n = 8;
        terms = {{1.0, word(n, {{0, 'Z'}, {1, 'Y'}, {3, 'X'}, {4, 'Y'}, {7, 'Z'}})},
                 {1.0, word(n, {{2, 'X'}, {6, 'Z'}, {7, 'X'}})},
                 {1.0, word(n, {{0, 'X'}, {3, 'Y'}, {4, 'Z'}, {6, 'X'}})}};
    } else if (name == "three-term") {
        n = 4;
        terms = {{1.0, word(n, {{0, 'Z'}, {1, 'Z'}})}, {1.0, word(n, {{0, 'X'}, {1, 'X'}})},
                 {1.0, word(n, {{2, 'X'}, {3, 'X'}})}};
    } else if (name == "jw8" || name == "jw10" || name == "jw12") {
        n = std::stoi(name.substr(2));
        terms = gen_synthetic_jw(n, 1);
    } else {
        throw ConfigError("unknown Hamiltonian fixture: " + name);
    }
    if (n_out) *n_out = n;
    return terms;
}

}  // namespace qrtile
