// Host-side model for the B200 batch engine: graph + fields in the flattened form the device
// consumes.  Mirrors the *meaning* of the reference's SpinModel / LayerSpec /
// build_layered_model / total_cost / validate_model (ref: proj/include/isingmc/model.hpp:18-130,
// proj/src/model.cpp:52-126,246-349) but is CSR-first: the per-spin edge lists the reference
// keeps as vectors of records live here as one offsets/targets/couplings triple, which is what
// gets uploaded verbatim.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace isingb200 {

struct Error : std::runtime_error {  // maps to ISING_ERR_ARGUMENT at the C boundary
    using std::runtime_error::runtime_error;
};

struct LayerEdge {  // ref: model.hpp:62-68
    uint32_t p, q;
    float coupling;
};

struct HostModel {
    uint32_t n_spins = 0;
    std::vector<float> h;             // n_spins
    std::vector<uint32_t> offsets;    // n_spins + 1
    std::vector<uint32_t> targets;    // half-edges
    std::vector<float> couplings;     // half-edges
    std::vector<uint8_t> tau_counts;  // trailing tau edges per spin
    uint32_t layers = 0;              // 0: generic model
    uint32_t per_layer = 0;

    // derived by finalize()
    bool has_tau = false;
    uint32_t max_degree = 0;
    // True when the on-chip layered kernel applies: layered, every layer's space edges are the
    // same (validate_model guarantees it), tau slots are (next layer, previous layer), and for
    // every position the two tau couplings are one value shared by all layers.  Then the tau
    // field J*(s_up + s_dn) takes only the values {2J, +0, -2J}, every incremental update of it
    // is exact, and it can be rebuilt from two spin bits instead of being stored.
    bool layered_uniform = false;
    std::vector<uint32_t> layer_offsets;  // per_layer + 1 : space edges of one layer (CSR)
    std::vector<uint32_t> layer_targets;  // target position inside the layer
    std::vector<float> layer_couplings;
    std::vector<float> layer_tau;         // per position tau coupling J

    uint32_t degree(uint32_t i) const { return offsets[i + 1] - offsets[i]; }
    uint64_t half_edges() const { return targets.size(); }
};

// Structural checks equal to the reference's validate_model; throws Error naming the first
// violation.  Then fills the derived members.
void finalize_model(HostModel& m);

HostModel model_from_csr(uint32_t n, const float* h, const uint32_t* offsets,
                         const uint32_t* targets, const float* couplings,
                         const uint8_t* tau_counts, uint32_t layers, uint32_t per_layer);

HostModel build_layered_model(uint32_t positions, const float* h, uint32_t n_edges,
                              const uint32_t* p, const uint32_t* q, const float* j,
                              uint32_t n_layers, float j_tau);

// -sum h_i s_i - sum_{t>i} J s_i s_t in f64, index order (ref: model.cpp:108-126).
double total_cost(const HostModel& m, const int8_t* spins, uint32_t count);

}  // namespace isingb200
