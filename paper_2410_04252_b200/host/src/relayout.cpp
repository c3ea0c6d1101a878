// B200 qrtile drop-in — cluster shapes, qubit layouts, QR events, schedule
// bookkeeping and JSON.  The QR event construction fixes the qubit
// permutation sequence and must agree bit-exactly with
// /root/reference/proj/src/layout.cpp:96-161; counting and JSON follow
// /root/reference/proj/src/schedule.cpp:8-94.

#include <algorithm>

#include "qrtile/schedule.hpp"

namespace qrtile {

namespace {
bool pow2(int v) { return v >= 1 && (v & (v - 1)) == 0; }

QubitSet positions_to_qubits(const QubitLayout& l, int lo, int hi) {
    QubitSet s = 0;
    for (int p = lo; p < hi; ++p) s |= qbit(l.qubit_at[static_cast<std::size_t>(p)]);
    return s;
}
}  // namespace

void ClusterShape::validate() const {
    if (!pow2(p) || !pow2(n_node) || !pow2(n_gpn)) throw ConfigError("cluster shape entries must be powers of two");
    if (p != n_node * n_gpn) throw ConfigError("cluster shape requires p = n_node * n_gpn");
}

void CostWeights::validate() const {
    if (w_intra < 0.0 || w_inter < 0.0) throw ConfigError("cost weights must be non-negative");
    if (w_inter < w_intra) throw ConfigError("inter weight must be at least the intra weight");
}

QubitLayout QubitLayout::identity(int n, const ClusterShape& shape) {
    shape.validate();
    if (n < 1 || n > kMaxQubits) throw ConfigError("qubit count out of range");
    QubitLayout l;
    l.n = n;
    l.n_local = n - shape.global_bits();
    l.intra_bits = shape.intra_bits();
    if (l.n_local < 1) throw TooManyPEs("p = " + std::to_string(shape.p) + " leaves no local qubit");
    l.pos_of.resize(static_cast<std::size_t>(n));
    for (int q = 0; q < n; ++q) l.pos_of[static_cast<std::size_t>(q)] = q;
    l.qubit_at = l.pos_of;
    return l;
}

QubitSet QubitLayout::local_set() const { return positions_to_qubits(*this, 0, n_local); }
QubitSet QubitLayout::intra_set() const { return positions_to_qubits(*this, n_local, inter_start()); }
QubitSet QubitLayout::inter_set() const { return positions_to_qubits(*this, inter_start(), n); }

void QubitLayout::check() const {
    std::vector<char> used(static_cast<std::size_t>(n), 0);
    for (int q = 0; q < n; ++q) {
        const int p = pos_of[static_cast<std::size_t>(q)];
        if (p < 0 || p >= n || qubit_at[static_cast<std::size_t>(p)] != q) throw Error("layout is not a bijection");
        if (used[static_cast<std::size_t>(p)]++) throw Error("layout position used twice");
    }
}

Access classify_access(const Operator& op, const QubitLayout& layout) {
    const bool wide = std::any_of(op.targets.begin(), op.targets.end(), [&](int t) {
        return layout.pos_of[static_cast<std::size_t>(t)] >= layout.n_local;
    });
    return wide ? Access::Wide : Access::Narrow;
}

QrClass classify_qr(const QrEvent& event) {
    if (event.swaps.empty()) throw DegenerateQr("empty swap set");
    bool global = false, inter = false;
    for (const auto& pr : event.swaps)
        for (int q : {pr.first, pr.second}) {
            const Region r = event.before.region_of(event.before.pos_of[static_cast<std::size_t>(q)]);
            global = global || r != Region::Local;
            inter = inter || r == Region::Inter;
        }
    if (!global) throw DegenerateQr("swaps confined to local positions");
    return inter ? QrClass::Inter : QrClass::Intra;
}

std::uint64_t qr_data_volume(int k, int n) {
    return k <= 0 ? 0 : (std::uint64_t{1} << n) - (std::uint64_t{1} << (n - k));
}

QrEvent make_qr_event_from_pairs(const QubitLayout& before, const std::vector<std::pair<int, int>>& pairs) {
    QrEvent ev;
    ev.swaps = pairs;
    ev.before = before;
    ev.after = before;
    QubitLayout& a = ev.after;
    for (const auto& [dep, arr] : pairs) {
        const int pd = a.pos_of[static_cast<std::size_t>(dep)];
        const int pa = a.pos_of[static_cast<std::size_t>(arr)];
        a.pos_of[static_cast<std::size_t>(dep)] = pa;
        a.pos_of[static_cast<std::size_t>(arr)] = pd;
        a.qubit_at[static_cast<std::size_t>(pd)] = arr;
        a.qubit_at[static_cast<std::size_t>(pa)] = dep;
    }
    ev.cls = classify_qr(ev);
    return ev;
}

std::optional<QrEvent> make_qr_event(const QubitLayout& before, QubitSet new_locals,
                                     std::optional<QubitSet> wanted_intra) {
    const QubitSet old_locals = before.local_set();
    if (new_locals == old_locals) return std::nullopt;
    if (set_size(new_locals) != before.n_local) throw Error("new local set has wrong size");
    const std::vector<int> leaving = set_to_vector(old_locals & ~new_locals);
    const std::vector<int> entering = set_to_vector(new_locals & ~old_locals);
    if (leaving.size() != entering.size()) throw Error("unbalanced local exchange");

    std::vector<std::pair<int, int>> pairs;
    const bool routed = wanted_intra.has_value() && before.intra_bits > 0 && before.inter_start() < before.n;
    if (!routed) {
        // Flat pairing: both lists ascending, matched index by index.
        for (std::size_t i = 0; i < leaving.size(); ++i) pairs.emplace_back(leaving[i], entering[i]);
        return make_qr_event_from_pairs(before, pairs);
    }

    // Hierarchical routing: a leaving qubit the caller wants in the intra
    // region takes the position of an entering qubit that currently sits in
    // the intra region, and likewise for inter; leftovers pair up in
    // ascending order.  Globals that stay global never move.
    std::vector<int> enter_intra, enter_inter, leave_intra, leave_inter;
    for (int q : entering)
        (before.region_of(before.pos_of[static_cast<std::size_t>(q)]) == Region::Intra ? enter_intra : enter_inter)
            .push_back(q);
    for (int q : leaving) (contains(*wanted_intra, q) ? leave_intra : leave_inter).push_back(q);

    auto match = [&pairs](const std::vector<int>& l, const std::vector<int>& e, std::vector<int>& l_rest,
                          std::vector<int>& e_rest) {
        const std::size_t k = std::min(l.size(), e.size());
        for (std::size_t i = 0; i < k; ++i) pairs.emplace_back(l[i], e[i]);
        l_rest.insert(l_rest.end(), l.begin() + static_cast<std::ptrdiff_t>(k), l.end());
        e_rest.insert(e_rest.end(), e.begin() + static_cast<std::ptrdiff_t>(k), e.end());
    };
    std::vector<int> leave_rest, enter_rest;
    match(leave_intra, enter_intra, leave_rest, enter_rest);
    match(leave_inter, enter_inter, leave_rest, enter_rest);
    std::sort(leave_rest.begin(), leave_rest.end());
    std::sort(enter_rest.begin(), enter_rest.end());
    for (std::size_t i = 0; i < leave_rest.size(); ++i) pairs.emplace_back(leave_rest[i], enter_rest[i]);
    std::sort(pairs.begin(), pairs.end());
    return make_qr_event_from_pairs(before, pairs);
}

// ---------------------------------------------------------------- schedule

void Schedule::index_tiles() {
    tile_of.assign(order.size(), -1);
    for (std::size_t t = 0; t < tiles.size(); ++t)
        for (int id : tiles[t].gates) tile_of[static_cast<std::size_t>(id)] = static_cast<int>(t);
}

std::optional<ScheduleViolation> validate_schedule(const Circuit& circuit, const DependencyGraph& deps,
                                                   const Schedule& schedule) {
    const int m = circuit.size();
    if (static_cast<int>(schedule.order.size()) != m)
        throw InvalidSchedule("order covers " + std::to_string(schedule.order.size()) + " of " + std::to_string(m) +
                              " operators");
    std::vector<int> slot(static_cast<std::size_t>(m), -1);
    for (int x = 0; x < m; ++x) {
        const int id = schedule.order[static_cast<std::size_t>(x)];
        if (id < 0 || id >= m || slot[static_cast<std::size_t>(id)] != -1)
            throw InvalidSchedule("order is not a permutation of operator ids");
        slot[static_cast<std::size_t>(id)] = x;
    }
    std::vector<std::pair<int, int>> edges = deps.edges;
    std::sort(edges.begin(), edges.end());
    for (const auto& [i, j] : edges)
        if (slot[static_cast<std::size_t>(i)] > slot[static_cast<std::size_t>(j)]) return ScheduleViolation{i, j};
    return std::nullopt;
}

bool schedule_is_narrow(const Circuit& circuit, const Schedule& schedule) {
    return std::all_of(schedule.order.begin(), schedule.order.end(), [&](int id) {
        return is_subset(circuit.op(id).target_mask(), schedule.mapping_of(id));
    });
}

QrCounts count_qrs(const Schedule& schedule) {
    QrCounts c;
    QubitSet prev = schedule.initial_mapping();
    for (int id : schedule.order) {
        const QubitSet cur = schedule.mapping_of(id);
        c.total += cur != prev ? 1 : 0;
        prev = cur;
    }
    if (c.total != static_cast<int>(schedule.qr_events.size()))
        throw InvalidSchedule("event list disagrees with mapping sequence: " +
                              std::to_string(schedule.qr_events.size()) + " events, " + std::to_string(c.total) +
                              " mapping changes");
    for (const QrEvent& ev : schedule.qr_events) ++(ev.cls == QrClass::Intra ? c.intra : c.inter);
    return c;
}

double qr_cost(const QrCounts& counts, const CostWeights& weights) {
    weights.validate();
    return weights.w_intra * counts.intra + weights.w_inter * counts.inter;
}

nlohmann::json qr_event_to_json(const QrEvent& event, const Schedule& schedule) {
    nlohmann::json swaps = nlohmann::json::array();
    for (const auto& [a, b] : event.swaps) swaps.push_back({a, b});
    int before_gate = 0;
    if (event.before_tile < static_cast<int>(schedule.tiles.size())) {
        const Tile& t = schedule.tiles[static_cast<std::size_t>(event.before_tile)];
        if (!t.gates.empty()) {
            auto it = std::find(schedule.order.begin(), schedule.order.end(), t.gates.front());
            if (it != schedule.order.end()) before_gate = static_cast<int>(it - schedule.order.begin());
        }
    }
    return nlohmann::json{{"swaps", swaps},
                          {"class", event.cls == QrClass::Intra ? "intra" : "inter"},
                          {"before_gate", before_gate}};
}

nlohmann::json schedule_to_json(const Schedule& schedule) {
    nlohmann::json tiles = nlohmann::json::array();
    for (const Tile& t : schedule.tiles)
        tiles.push_back({{"gates", t.gates}, {"local_qubits", set_to_vector(t.local_qubits)}});
    nlohmann::json events = nlohmann::json::array();
    for (const QrEvent& ev : schedule.qr_events) events.push_back(qr_event_to_json(ev, schedule));
    return nlohmann::json{{"order", schedule.order}, {"tiles", tiles}, {"qr_events", events}};
}

}  // namespace qrtile
