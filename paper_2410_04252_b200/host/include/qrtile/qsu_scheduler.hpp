#pragma once
// B200 qrtile drop-in — QSU schedulers (host planning; bit-exact with the
// reference).  Reference interface: /root/reference/proj/include/qrtile/qsu_scheduler.hpp
// (flat_tiling :17, hierarchical_tiling :22, adhoc_schedule :27, building
//  blocks :36-56).  Algorithms: PAPER.md Alg. 1-5, reference
//  qsu_scheduler.cpp:14-249.

#include "qrtile/schedule.hpp"

namespace qrtile {

// Lazy QR by time-space tiling: maximal tile (P1), then greedy remap (P2).
Schedule flat_tiling(const Circuit& circuit, const DependencyGraph& deps, const ClusterShape& shape);

// Flat tiling with a two-phase remap that prefers intra-node exchanges.
Schedule hierarchical_tiling(const Circuit& circuit, const DependencyGraph& deps,
                             const ClusterShape& shape);

// Eager baseline: depth order, remap on demand before each wide gate.
Schedule adhoc_schedule(const Circuit& circuit, const DependencyGraph& deps, const ClusterShape& shape);

// Building blocks over a depth-ordered id list.
std::vector<int> tile_construction(QubitSet q_local, const Circuit& circuit,
                                   const std::vector<int>& remaining);
QubitSet qubit_mapping(QubitSet universe, const Circuit& circuit, const std::vector<int>& remaining,
                       int n_local);
std::pair<QubitSet, QubitSet> hierarchical_qubit_mapping(QubitSet universe, const Circuit& circuit,
                                                         const std::vector<int>& remaining,
                                                         QubitSet q_local, QubitSet q_intra);

}  // namespace qrtile
