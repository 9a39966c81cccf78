#include "host_model.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <set>
#include <utility>

namespace isingb200 {

namespace {

uint32_t bits_of(float v) {
    uint32_t b;
    std::memcpy(&b, &v, sizeof b);
    return b;
}

std::string at_spin(uint32_t i) { return "spin " + std::to_string(i); }

// Is half-edge slot k of spin i one of its trailing tau slots?
bool slot_is_tau(const HostModel& m, uint32_t i, uint32_t e) {
    return e >= m.offsets[i + 1] - m.tau_counts[i];
}

void check_symmetry(const HostModel& m) {
    for (uint32_t i = 0; i < m.n_spins; ++i) {
        if (m.tau_counts[i] > m.degree(i)) {
            throw Error("validate_model: " + at_spin(i) + " tau_count exceeds degree");
        }
        for (uint32_t e = m.offsets[i]; e < m.offsets[i + 1]; ++e) {
            const uint32_t t = m.targets[e];
            if (t >= m.n_spins) throw Error("validate_model: " + at_spin(i) + " edge target out of range");
            if (t == i) throw Error("validate_model: self edge at " + at_spin(i));
            const bool tau = slot_is_tau(m, i, e);
            bool matched = false;
            for (uint32_t r = m.offsets[t]; r < m.offsets[t + 1] && !matched; ++r) {
                matched = m.targets[r] == i && slot_is_tau(m, t, r) == tau &&
                          bits_of(m.couplings[r]) == bits_of(m.couplings[e]);
            }
            if (!matched) {
                throw Error("validate_model: edge " + std::to_string(i) + "-" + std::to_string(t) +
                            " has no matching reverse record");
            }
        }
    }
}

void check_layered(const HostModel& m) {
    const uint32_t L = m.layers, P = m.per_layer;
    if (uint64_t(L) * P != m.n_spins) throw Error("validate_model: layers * per_layer != n_spins");
    for (uint32_t i = 0; i < m.n_spins; ++i) {
        if (m.tau_counts[i] != 2) {
            throw Error("validate_model: layered " + at_spin(i) + " has tau_count " +
                        std::to_string(m.tau_counts[i]));
        }
        const uint32_t l = i / P, pos = i % P;
        const uint32_t up = ((l + 1) % L) * P + pos, down = ((l + L - 1) % L) * P + pos;
        const uint32_t end = m.offsets[i + 1];
        const uint32_t t0 = m.targets[end - 2], t1 = m.targets[end - 1];
        if (!((t0 == up && t1 == down) || (t0 == down && t1 == up))) {
            throw Error("validate_model: " + at_spin(i) + " tau edges do not link adjacent layers");
        }
        for (uint32_t e = m.offsets[i]; e + 2 < end; ++e) {
            if (m.targets[e] / P != l) throw Error("validate_model: space edge leaves layer at " + at_spin(i));
        }
        if (l == 0) continue;
        // every layer repeats layer 0's space edges
        if (m.degree(i) != m.degree(pos)) {
            throw Error("validate_model: layers differ in degree at position " + std::to_string(pos));
        }
        for (uint32_t k = 0; k + 2 < m.degree(i); ++k) {
            const uint32_t ea = m.offsets[i] + k, eb = m.offsets[pos] + k;
            if (m.targets[ea] % P != m.targets[eb] % P ||
                bits_of(m.couplings[ea]) != bits_of(m.couplings[eb])) {
                throw Error("validate_model: layers are not identical at position " + std::to_string(pos));
            }
        }
    }
}

// Decide whether the tau field can be rebuilt from spin bits (see HostModel::layered_uniform)
// and extract the single-layer graph the layered kernel keeps on chip.
void analyse_layers(HostModel& m) {
    m.layered_uniform = false;
    if (m.layers == 0) return;
    const uint32_t L = m.layers, P = m.per_layer;
    std::vector<float> jt(P);
    for (uint32_t i = 0; i < m.n_spins; ++i) {
        const uint32_t l = i / P, pos = i % P, end = m.offsets[i + 1];
        const uint32_t up = ((l + 1) % L) * P + pos, down = ((l + L - 1) % L) * P + pos;
        if (m.targets[end - 2] != up || m.targets[end - 1] != down) return;  // slot order
        if (bits_of(m.couplings[end - 2]) != bits_of(m.couplings[end - 1])) return;
        if (l == 0) jt[pos] = m.couplings[end - 1];
        else if (bits_of(jt[pos]) != bits_of(m.couplings[end - 1])) return;
        if (!std::isfinite(2.0f * m.couplings[end - 1])) return;
    }
    m.layer_offsets.assign(P + 1, 0);
    m.layer_targets.clear();
    m.layer_couplings.clear();
    for (uint32_t pos = 0; pos < P; ++pos) {
        m.layer_offsets[pos] = uint32_t(m.layer_targets.size());
        for (uint32_t e = m.offsets[pos]; e + 2 < m.offsets[pos + 1]; ++e) {
            const uint32_t t = m.targets[e] % P;
            // the kernel batches a flip's neighbour updates, so a repeated target must not occur
            for (uint32_t k = m.layer_offsets[pos]; k < m.layer_targets.size(); ++k) {
                if (m.layer_targets[k] == t) return;
            }
            if (!std::isfinite(2.0f * m.couplings[e])) return;
            m.layer_targets.push_back(t);
            m.layer_couplings.push_back(m.couplings[e]);
        }
    }
    m.layer_offsets[P] = uint32_t(m.layer_targets.size());
    m.layer_tau = std::move(jt);
    m.layered_uniform = true;
}

}  // namespace

void finalize_model(HostModel& m) {
    if (m.h.size() != m.n_spins || m.offsets.size() != size_t(m.n_spins) + 1 ||
        m.tau_counts.size() != m.n_spins) {
        throw Error("validate_model: field/adjacency size mismatch");
    }
    if (m.offsets[0] != 0) throw Error("validate_model: offsets must start at 0");
    for (uint32_t i = 0; i < m.n_spins; ++i) {
        if (m.offsets[i + 1] < m.offsets[i]) throw Error("validate_model: offsets must not decrease");
    }
    if (m.offsets[m.n_spins] != m.targets.size() || m.targets.size() != m.couplings.size()) {
        throw Error("validate_model: field/adjacency size mismatch");
    }
    check_symmetry(m);
    if (m.layers != 0) check_layered(m);
    m.has_tau = false;
    m.max_degree = 0;
    for (uint32_t i = 0; i < m.n_spins; ++i) {
        m.has_tau = m.has_tau || m.tau_counts[i] != 0;
        m.max_degree = std::max(m.max_degree, m.degree(i));
    }
    analyse_layers(m);
}

HostModel model_from_csr(uint32_t n, const float* h, const uint32_t* offsets,
                         const uint32_t* targets, const float* couplings,
                         const uint8_t* tau_counts, uint32_t layers, uint32_t per_layer) {
    if (n != 0 && (h == nullptr || offsets == nullptr)) throw Error("null argument");
    HostModel m;
    m.n_spins = n;
    m.h.assign(h, h + n);
    if (offsets != nullptr) m.offsets.assign(offsets, offsets + n + 1);
    else m.offsets.assign(1, 0);
    const uint32_t edges = m.offsets[n];
    if (edges != 0 && (targets == nullptr || couplings == nullptr)) throw Error("null argument");
    m.targets.assign(targets, targets + edges);
    m.couplings.assign(couplings, couplings + edges);
    if (tau_counts != nullptr) m.tau_counts.assign(tau_counts, tau_counts + n);
    else m.tau_counts.assign(n, 0);
    m.layers = layers;
    m.per_layer = layers ? per_layer : 0;
    finalize_model(m);
    return m;
}

HostModel build_layered_model(uint32_t positions, const float* h, uint32_t n_edges,
                              const uint32_t* p, const uint32_t* q, const float* j,
                              uint32_t n_layers, float j_tau) {
    if (n_layers < 4) throw Error("build_layered_model: need at least 4 layers");
    if (positions == 0) throw Error("build_layered_model: empty layer");
    if (h == nullptr || (n_edges != 0 && (p == nullptr || q == nullptr || j == nullptr))) {
        throw Error("null argument");
    }
    // one layer's adjacency, each list ascending by target
    std::vector<std::vector<std::pair<uint32_t, float>>> nbr(positions);
    std::set<std::pair<uint32_t, uint32_t>> seen;
    for (uint32_t e = 0; e < n_edges; ++e) {
        if (p[e] >= positions || q[e] >= positions) throw Error("build_layered_model: edge endpoint out of range");
        if (p[e] == q[e]) throw Error("build_layered_model: self edge at position " + std::to_string(p[e]));
        if (!seen.insert(std::minmax(p[e], q[e])).second) {
            throw Error("build_layered_model: duplicate or asymmetric edge " + std::to_string(p[e]) +
                        "-" + std::to_string(q[e]));
        }
        nbr[p[e]].emplace_back(q[e], j[e]);
        nbr[q[e]].emplace_back(p[e], j[e]);
    }
    for (auto& list : nbr) {
        std::stable_sort(list.begin(), list.end(),
                         [](const auto& a, const auto& b) { return a.first < b.first; });
    }
    HostModel m;
    m.n_spins = n_layers * positions;
    m.layers = n_layers;
    m.per_layer = positions;
    m.h.resize(m.n_spins);
    m.offsets.reserve(size_t(m.n_spins) + 1);
    m.tau_counts.assign(m.n_spins, 2);
    for (uint32_t l = 0; l < n_layers; ++l) {
        const uint32_t base = l * positions;
        const uint32_t up = ((l + 1) % n_layers) * positions;
        const uint32_t down = ((l + n_layers - 1) % n_layers) * positions;
        for (uint32_t pos = 0; pos < positions; ++pos) {
            m.h[base + pos] = h[pos];
            m.offsets.push_back(uint32_t(m.targets.size()));
            for (const auto& [t, c] : nbr[pos]) {
                m.targets.push_back(base + t);
                m.couplings.push_back(c);
            }
            m.targets.push_back(up + pos);
            m.couplings.push_back(j_tau);
            m.targets.push_back(down + pos);
            m.couplings.push_back(j_tau);
        }
    }
    m.offsets.push_back(uint32_t(m.targets.size()));
    finalize_model(m);
    return m;
}

double total_cost(const HostModel& m, const int8_t* spins, uint32_t count) {
    if (count != m.n_spins) throw Error("total_cost: spin count mismatch");
    for (uint32_t i = 0; i < count; ++i) {
        if (spins[i] != 1 && spins[i] != -1) throw Error("total_cost: spin " + std::to_string(i) + " not +/-1");
    }
    double cost = 0.0;
    for (uint32_t i = 0; i < m.n_spins; ++i) {
        cost -= double(m.h[i]) * double(spins[i]);
        for (uint32_t e = m.offsets[i]; e < m.offsets[i + 1]; ++e) {
            const uint32_t t = m.targets[e];
            if (t > i) cost -= double(m.couplings[e]) * double(spins[i]) * double(spins[t]);
        }
    }
    return cost;
}

}  // namespace isingb200
