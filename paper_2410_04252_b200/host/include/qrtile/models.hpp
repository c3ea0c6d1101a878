#pragma once
// B200 qrtile drop-in — deterministic synthetic inputs.
// Reference interface: /root/reference/proj/include/qrtile/models.hpp
// (Rng :15-31, random_unitary :35, GateFabricSpec/gen_gatefabric :42-52,
//  gen_synthetic_jw :60, gen_random_circuit :63, random_state :65,
//  fixtures :71-78, seed_payloads :90).  Payload bits are identical to the
//  reference for the same seeds (mt19937_64 + hand-rolled Box-Muller).
//
// Added (absent from the reference): gen_hea, a
// hardware-efficient ansatz of RY / RZ / CZ layers.

#include <cmath>
#include <random>

#include "qrtile/circuit.hpp"
#include "qrtile/dist_sim.hpp"

namespace qrtile {

struct Rng {
    std::mt19937_64 engine;

    explicit Rng(std::uint64_t seed) : engine(seed) {}

    std::uint64_t next() { return engine(); }
    double uniform() { return std::ldexp(static_cast<double>(engine() >> 11), -53); }  // [0,1)
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double normal();          // Box-Muller, caches the second variate
    int below(int bound);     // unbiased integer in [0, bound)

  private:
    bool have_spare_ = false;
    double spare_ = 0.0;
};

GateMatrix random_unitary(int k_qubits, std::uint64_t seed);

struct GateFabricSpec {
    int n = 4;
    int layers = 1;
    std::uint64_t seed = 1;
    bool payloads = true;
};
Circuit gen_gatefabric(const GateFabricSpec& spec);
int gatefabric_block_count(int n, int layers);

std::vector<PauliTerm> gen_synthetic_jw(int n, std::uint64_t seed, int max_span = 0);
std::uint64_t synthetic_jw_term_count(int n, int max_span = 0);

// C5 stress Hamiltonian: per word, letters "IXYZ"[rng.below(4)]
// for q = 0..n-1 (the letter draw of acceptance.cpp:251 / test_evc_scheduler.cpp:133
// over the whole word), then coefficient rng.uniform(-1, 1); one Rng(seed) stream.
std::vector<PauliTerm> gen_uniform_words(int n, int count, std::uint64_t seed);

Circuit gen_random_circuit(int n, int m, std::uint64_t seed, int max_arity = 2, bool payloads = true);
ReferenceState random_state(int n, std::uint64_t seed);

// Hardware-efficient ansatz: per layer RY(theta) on every
// qubit, RZ(theta) on every qubit, CZ(q,q+1) for even q, then odd q.
// theta ~ U[0, 2pi) drawn from Rng(seed) in gate order.
struct HeaSpec {
    int n = 4;
    int depth = 1;
    std::uint64_t seed = 1;
    bool payloads = true;
};
Circuit gen_hea(const HeaSpec& spec);

std::vector<std::string> fixture_circuit_names();
Circuit fixture_circuit(const std::string& name, std::uint64_t seed = 1);
ClusterShape fixture_shape(const std::string& name);
std::vector<std::string> fixture_hamiltonian_names();
std::vector<PauliTerm> fixture_hamiltonian(const std::string& name, int* n_out);

void seed_payloads(Circuit& circuit, std::uint64_t seed);

}  // namespace qrtile
