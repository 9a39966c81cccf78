// TEST INFRASTRUCTURE ONLY.  A thin extern "C" window onto the UNMODIFIED reference
// sources (compiled where they lie under /root/reference/proj by oracle/build_ref.sh into
// oracle/_ref/libisingref.so).  Nothing here restates an algorithm: every call forwards to
// the reference's own C++ API (include/isingmc/{rng,fastexp,model,sweep}.hpp).  Used to pin
// oracle/ising_oracle.c, to generate tests/golden/, and as the "reference" CPU baseline.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "isingmc/fastexp.hpp"
#include "isingmc/model.hpp"
#include "isingmc/model_io.hpp"
#include "isingmc/rng.hpp"
#include "isingmc/oracle.hpp"
#include "isingmc/sweep.hpp"

using namespace isingmc;

namespace {
thread_local std::string g_err;

ExpKind exp_of(int k) {
    return k == 1 ? ExpKind::exact : (k == 2 ? ExpKind::fast : ExpKind::accurate);
}
EngineKind engine_of(int e) {
    switch (e) {
        case 0: return EngineKind::reference;
        case 1: return EngineKind::basic;
        case 2: return EngineKind::vector4;
        default: return EngineKind::coalesced;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- numeric primitives
void ref_mt_fill(uint32_t seed, uint32_t* out, size_t count) {
    Mt19937 g(seed);  // blockwise twist + bulk tempering
    g.fill(std::span<uint32_t>(out, count));
}
void ref_mt_next_stream(uint32_t seed, uint32_t* out, size_t count) {
    Mt19937 g(seed, TwistImpl::plain);
    for (size_t i = 0; i < count; ++i) out[i] = g.next_u32();
}
float ref_u32_to_unit(uint32_t x) { return u32_to_unit(x); }
float ref_exp_fast(float x) { return exp_fast(x); }
float ref_exp_accurate(float x) { return exp_accurate(x); }
float ref_exp_exact(float x) { return static_cast<float>(std::exp(double(x))); }
void ref_initial_spins(uint32_t n, uint32_t seed, int8_t* out) {
    const auto v = initial_spins(n, seed);
    std::memcpy(out, v.data(), n);
}

// ---- models
void* ref_model_from_csr(uint32_t n, const float* h, const uint32_t* offsets,
                         const uint32_t* targets, const float* couplings,
                         const uint8_t* tau_counts, uint32_t layers, uint32_t per_layer) {
    auto* m = new SpinModel;
    m->n_spins = n;
    m->h.assign(h, h + n);
    m->adjacency.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
        for (uint32_t e = offsets[i]; e < offsets[i + 1]; ++e) {
            m->adjacency[i].edges.push_back({targets[e], couplings[e]});
        }
        m->adjacency[i].tau_count = tau_counts ? tau_counts[i] : 0;
    }
    if (layers) m->layered = LayeredMeta{layers, per_layer, Ordering::identity, 0};
    return m;
}

void* ref_build_layered(uint32_t positions, const float* h, uint32_t n_edges, const uint32_t* p,
                        const uint32_t* q, const float* j, uint32_t layers, float j_tau) {
    try {
        LayerSpec spec;
        spec.positions = positions;
        spec.h.assign(h, h + positions);
        for (uint32_t e = 0; e < n_edges; ++e) spec.edges.push_back({p[e], q[e], j[e]});
        return new SpinModel(build_layered_model(spec, layers, j_tau));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_model_free(void* m) { delete static_cast<SpinModel*>(m); }

// prepare_model_for_engine (sweep_state.cpp:292-323): the permuted copy an engine needs, and the
// permutation (forward[old] = new) it was built with.
void* ref_prepare_model(const void* m, int engine, uint32_t* forward) {
    try {
        auto prepared = prepare_model_for_engine(*static_cast<const SpinModel*>(m), engine_of(engine));
        if (forward != nullptr) std::copy(prepared.second.forward.begin(), prepared.second.forward.end(), forward);
        return new SpinModel(std::move(prepared.first));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// `ising-model v1` documents through the reference's own reader and writer (model_io.cpp).
// to_string: returns the length, copies at most `capacity` bytes; -1 on error.
long ref_model_to_string(const void* m, char* out, size_t capacity) {
    try {
        const std::string text = model_to_string(*static_cast<const SpinModel*>(m));
        if (out != nullptr && capacity != 0) std::memcpy(out, text.data(), std::min(capacity, text.size()));
        return long(text.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}
void* ref_model_from_string(const char* text) {
    try {
        return new SpinModel(model_from_string(text));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

int ref_model_validate(const void* m) {
    try {
        validate_model(*static_cast<const SpinModel*>(m));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

uint32_t ref_model_spins(const void* m) { return static_cast<const SpinModel*>(m)->n_spins; }
uint64_t ref_model_half_edges(const void* m) {
    return 2 * static_cast<const SpinModel*>(m)->edge_count();
}
// Writes the CSR view (same order as the engines' flatten()).
void ref_model_export(const void* mp, float* h, uint32_t* offsets, uint32_t* targets,
                      float* couplings, uint8_t* tau_counts) {
    const auto& m = *static_cast<const SpinModel*>(mp);
    uint32_t k = 0;
    for (uint32_t i = 0; i < m.n_spins; ++i) {
        h[i] = m.h[i];
        offsets[i] = k;
        tau_counts[i] = uint8_t(m.adjacency[i].tau_count);
        for (const EdgeRecord& e : m.adjacency[i].edges) {
            targets[k] = e.target_spin;
            couplings[k] = e.coupling;
            ++k;
        }
    }
    offsets[m.n_spins] = k;
}

double ref_total_cost(const void* m, const float* spins) {
    const auto& model = *static_cast<const SpinModel*>(m);
    return total_cost(model, std::span<const float>(spins, model.n_spins));
}
uint64_t ref_checksum(const float* spins, uint32_t n) {
    return state_checksum(std::span<const float>(spins, n));
}

// ---- chains
void* ref_chain_create(const void* m, int engine, uint32_t seed, float beta, float tau_scale,
                       int exp_kind, const int8_t* initial) {
    try {
        const auto& model = *static_cast<const SpinModel*>(m);
        EngineConfig cfg;
        cfg.engine = engine_of(engine);
        cfg.params.beta = beta;
        cfg.params.tau_scale = tau_scale;
        cfg.params.exp_kind = exp_of(exp_kind);
        cfg.seed = seed;
        if (initial) {
            return new SweepState(
                init_state(model, cfg, std::span<const int8_t>(initial, model.n_spins)));
        }
        return new SweepState(init_state(model, cfg));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_chain_free(void* s) { delete static_cast<SweepState*>(s); }
void ref_chain_sweep(void* s, const void* m, uint64_t sweeps) {
    run_sweeps(*static_cast<SweepState*>(s), *static_cast<const SpinModel*>(m), sweeps);
}
void ref_chain_set_beta(void* s, float beta) { static_cast<SweepState*>(s)->params.beta = beta; }
void ref_chain_read(const void* sp, float* spins, float* hs, float* ht, uint64_t* flips,
                    uint64_t* attempts) {
    const auto& s = *static_cast<const SweepState*>(sp);
    if (spins) std::memcpy(spins, s.spins.data(), s.n_spins * sizeof(float));
    if (hs) std::memcpy(hs, s.h_eff_space.data(), s.n_spins * sizeof(float));
    if (ht) std::memcpy(ht, s.h_eff_tau.data(), s.n_spins * sizeof(float));
    if (flips) *flips = s.stats.flips;
    if (attempts) *attempts = s.stats.attempts;
}
uint64_t ref_chain_coherence(const void* s, const void* m) {
    return field_coherence_ulp(*static_cast<const SweepState*>(s),
                               *static_cast<const SpinModel*>(m));
}
float ref_flip_probability(const void* s, uint32_t spin) {
    return flip_probability(*static_cast<const SweepState*>(s), spin);
}

// ---- CPU baseline: ladders of chains on a thread pool with an atomic work counter (the
// scheme of src/bench.cpp:72-84), every sweep done by the reference's run_sweeps.  The
// reference has no tempering and exposes no per-flip hook, so the swap step here uses
// total_cost() energies at the swap point (same pair schedule and draw as the oracle's
// definition); it is <2% of the CPU time and is timing scaffolding, not a parity path.
struct RefLadders {
    struct Ladder {
        const SpinModel* model;
        std::vector<SweepState> chains;
        std::vector<uint32_t> at_slot;
        Mt19937 swap_rng{0};
        uint64_t round = 0;
    };
    std::vector<Ladder> ladders;
    std::vector<float> betas;
    int exp_kind = 2;
    uint64_t sweeps_done = 0;
};

void* ref_ladders_create(const void* const* models, uint32_t n_ladders, uint32_t n_betas,
                         const float* betas, const uint32_t* seeds, const uint32_t* swap_seeds,
                         float tau_scale, int exp_kind, int engine) {
    try {
        auto* set = new RefLadders;
        set->betas.assign(betas, betas + n_betas);
        set->exp_kind = exp_kind;
        set->ladders.resize(n_ladders);
        for (uint32_t l = 0; l < n_ladders; ++l) {
            auto& lad = set->ladders[l];
            lad.model = static_cast<const SpinModel*>(models[l]);
            lad.swap_rng.reseed((swap_seeds ? swap_seeds[l] : 0u) ^ 0x85EBCA6Bu);
            for (uint32_t k = 0; k < n_betas; ++k) {
                EngineConfig cfg;
                cfg.engine = engine_of(engine);
                cfg.params = {betas[k], tau_scale, exp_of(exp_kind)};
                cfg.seed = seeds[size_t(l) * n_betas + k];
                lad.chains.push_back(init_state(*lad.model, cfg));
                lad.at_slot.push_back(k);
            }
        }
        return set;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_ladders_free(void* p) { delete static_cast<RefLadders*>(p); }

// Runs `sweeps` more sweeps of every chain (swap round after every swap_interval-th sweep,
// counted since creation) on `threads` workers; returns the seconds spent.
double ref_ladders_run(void* p, uint64_t sweeps, uint32_t swap_interval, uint32_t threads) {
    auto& set = *static_cast<RefLadders*>(p);
    const uint32_t nb = uint32_t(set.betas.size());
    const uint64_t base = set.sweeps_done;
    std::atomic<uint32_t> next{0};
    const auto work = [&]() {
        for (;;) {
            const uint32_t l = next.fetch_add(1);
            if (l >= set.ladders.size()) return;
            auto& lad = set.ladders[l];
            const SpinModel& model = *lad.model;
            if (swap_interval == 0 || nb < 2) {
                for (auto& c : lad.chains) run_sweeps(c, model, sweeps);
                continue;
            }
            uint64_t left = sweeps, done = base;
            while (left > 0) {
                const uint64_t step = std::min<uint64_t>(left, swap_interval - done % swap_interval);
                for (auto& c : lad.chains) run_sweeps(c, model, step);
                left -= step;
                done += step;
                if (done % swap_interval != 0) continue;
                for (uint32_t k = uint32_t(lad.round & 1u); k + 1 < nb; k += 2) {
                    const uint32_t a = lad.at_slot[k], b = lad.at_slot[k + 1];
                    const float u = u32_to_unit(lad.swap_rng.next_u32());
                    const double ea = total_cost(model, std::span<const float>(lad.chains[a].spins));
                    const double eb = total_cost(model, std::span<const float>(lad.chains[b].spins));
                    const float x = float((double(set.betas[k]) - double(set.betas[k + 1])) * (ea - eb));
                    const float pr = set.exp_kind == 2   ? exp_fast(x)
                                     : set.exp_kind == 3 ? exp_accurate(x)
                                                         : float(std::exp(double(x)));
                    if (u < pr) {
                        std::swap(lad.at_slot[k], lad.at_slot[k + 1]);
                        lad.chains[a].params.beta = set.betas[k + 1];
                        lad.chains[b].params.beta = set.betas[k];
                    }
                }
                ++lad.round;
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (uint32_t t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    set.sweeps_done += sweeps;
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void ref_ladders_read(const void* p, uint64_t* flips_out, double* energy_out) {
    const auto& set = *static_cast<const RefLadders*>(p);
    size_t c = 0;
    for (const auto& lad : set.ladders) {
        for (const SweepState& s : lad.chains) {
            if (flips_out) flips_out[c] = s.stats.flips;
            if (energy_out) energy_out[c] = total_cost(*lad.model, std::span<const float>(s.spins));
            ++c;
        }
    }
}

// ---- the reference's own validators (src/oracle.cpp:64-174): exact enumeration and the
// replicate-means z-test, for pinning what can be pinned of the tempering sampler.
// probabilities: 2^n entries, state index bit i set <=> s_i = +1 (oracle.hpp:13); moments[3] =
// {mean_cost, mean_magnetization, log_partition}.  Returns 0, or -1 with ref_last_error().
int ref_enumerate_boltzmann(const void* m, double beta, double* probabilities, double* moments) {
    try {
        const ExactDistribution d = enumerate_boltzmann(*static_cast<const SpinModel*>(m), beta);
        if (probabilities) std::copy(d.probabilities.begin(), d.probabilities.end(), probabilities);
        if (moments) {
            moments[0] = d.mean_cost;
            moments[1] = d.mean_magnetization;
            moments[2] = d.log_partition;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// out[9] = {exact_cost, exact_magnetization, est_cost, est_magnetization, se_cost, se_magnetization,
// z_cost, z_magnetization, pass}
int ref_chain_statistics(const void* m, int engine, float beta, float tau_scale, int exp_kind, uint64_t sweeps,
                         uint64_t burn_in, uint32_t replicates, uint32_t base_seed, double z_threshold, double* out) {
    try {
        ChainStatsConfig cfg;
        cfg.engine = engine_of(engine);
        cfg.params = {beta, tau_scale, exp_of(exp_kind)};
        cfg.sweeps = sweeps;
        cfg.burn_in = burn_in;
        cfg.replicates = replicates;
        cfg.base_seed = base_seed;
        cfg.z_threshold = z_threshold;
        const ChainStatsReport r = chain_statistics_test(*static_cast<const SpinModel*>(m), cfg);
        const double v[9] = {r.exact_cost, r.exact_magnetization, r.est_cost, r.est_magnetization, r.se_cost,
                             r.se_magnetization, r.z_cost, r.z_magnetization, r.pass ? 1.0 : 0.0};
        std::copy(v, v + 9, out);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
