// extern "C" boundary of libisingb200.so (declared in include/isingmc_b200.h).  Follows the
// reference's conventions (ref: proj/src/capi.cpp:21-65): opaque heap handles, a thread-local
// last-error string, and an exception firewall that maps argument errors to
// ISING_ERR_ARGUMENT and everything else (CUDA failures included) to ISING_ERR_INTERNAL.
#include "isingmc_b200.h"

#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <sys/utsname.h>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "batch.hpp"
#include "coalesced.hpp"
#include "host_model.hpp"
#include "model_text.hpp"

using namespace isingb200;

extern "C" {
struct ising_b200_model {
    HostModel model;
};
struct ising_batch {
    Batch* impl;
};
struct ising_coalesced {
    CoalescedBatch* impl;
};
}

namespace {

thread_local std::string g_last_error;

template <typename F>
ising_status guarded(F&& body) {
    try {
        return body();
    } catch (const ParseError& e) {
        g_last_error = e.what();
        return ISING_ERR_PARSE;
    } catch (const IoError& e) {
        g_last_error = e.what();
        return ISING_ERR_IO;
    } catch (const Error& e) {
        g_last_error = e.what();
        return ISING_ERR_ARGUMENT;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return ISING_ERR_ARGUMENT;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return ISING_ERR_INTERNAL;
    }
}

void require(const void* p) {
    if (p == nullptr) throw Error("null argument");
}

Batch& impl_of(ising_batch* b) {
    require(b);
    return *b->impl;
}

char* dup_string(const std::string& text) {
    char* out = new (std::nothrow) char[text.size() + 1];
    if (out != nullptr) std::memcpy(out, text.c_str(), text.size() + 1);
    return out;
}

// One chain on the device: what ising_b200_run and ising_b200_run_json share.
struct SingleRun {
    ising_b200_run_report report;
    int exp_kind;
    int family;
};

int resolve_exp_kind(int kind);

SingleRun run_single(const ising_b200_model* model, const ising_b200_run_params* params) {
    require(model);
    require(params);
    BatchConfig cfg;
    cfg.n_ladders = 1;
    cfg.n_betas = 1;
    cfg.betas = {params->beta};
    cfg.seeds = {params->seed};
    cfg.swap_seeds = {0u};
    cfg.tau_scale = params->tau_scale;
    cfg.exp_kind = resolve_exp_kind(params->exp_kind);
    cfg.device = params->device;
    Batch batch({&model->model}, {0u}, cfg, nullptr);
    batch.run(params->sweeps, 0);
    uint64_t flips = 0, attempts = 0, checksum = 0;
    double cost = 0.0;
    batch.read_stats(&flips, &attempts);
    batch.read_energies(&cost);
    batch.read_checksums(&checksum);
    SingleRun out{};
    out.report.final_cost = cost;
    out.report.flips = flips;
    out.report.attempts = attempts;
    out.report.flip_rate = attempts ? double(flips) / double(attempts) : 0.0;
    out.report.checksum = checksum;
    out.exp_kind = cfg.exp_kind;
    out.family = int(batch.family());
    return out;
}

// Shortest decimal text that reads back as the same double (JSON number).
std::string json_number(double v) {
    char buf[40];
    for (int digits = 1; digits <= 17; ++digits) {
        std::snprintf(buf, sizeof buf, "%.*g", digits, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string text = buf;
    if (text.find_first_of(".eEn") == std::string::npos) text += ".0";
    return text;
}

int resolve_exp_kind(int kind) {
    if (kind == ISING_EXP_ENGINE_DEFAULT) return ISING_EXP_FAST;  // ref: default_exp_kind, sweep_state.cpp:29-31
    if (kind < ISING_EXP_EXACT || kind > ISING_EXP_ACCURATE) {
        throw Error("invalid exp_kind value " + std::to_string(kind));
    }
    return kind;
}

}  // namespace

extern "C" {

const char* ising_b200_last_error(void) { return g_last_error.c_str(); }

int ising_b200_device_count(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return count;
}

// ---------------------------------------------------------------- models

ising_status ising_b200_model_from_csr(uint32_t n_spins, const float* h, const uint32_t* offsets,
                                       const uint32_t* targets, const float* couplings,
                                       const uint8_t* tau_counts, uint32_t layers,
                                       uint32_t per_layer, ising_b200_model** out) {
    return guarded([&]() {
        require(out);
        *out = new ising_b200_model{
            model_from_csr(n_spins, h, offsets, targets, couplings, tau_counts, layers, per_layer)};
        return ISING_OK;
    });
}

ising_status ising_b200_model_build_layered(uint32_t positions, const float* h, uint32_t n_edges,
                                            const uint32_t* p, const uint32_t* q, const float* j,
                                            uint32_t n_layers, float j_tau,
                                            ising_b200_model** out) {
    return guarded([&]() {
        require(out);
        *out = new ising_b200_model{build_layered_model(positions, h, n_edges, p, q, j, n_layers, j_tau)};
        return ISING_OK;
    });
}

void ising_b200_model_free(ising_b200_model* model) { delete model; }

uint32_t ising_b200_model_spins(const ising_b200_model* model) {
    return model ? model->model.n_spins : 0;
}

uint64_t ising_b200_model_half_edges(const ising_b200_model* model) {
    return model ? model->model.half_edges() : 0;
}

int ising_b200_model_layers(const ising_b200_model* model, uint32_t* layers, uint32_t* per_layer) {
    if (model == nullptr || model->model.layers == 0) return 0;
    if (layers != nullptr) *layers = model->model.layers;
    if (per_layer != nullptr) *per_layer = model->model.per_layer;
    return 1;
}

ising_status ising_b200_model_export_csr(const ising_b200_model* model, float* h, uint32_t* offsets,
                                         uint32_t* targets, float* couplings, uint8_t* tau_counts) {
    return guarded([&]() {
        require(model);
        const HostModel& m = model->model;
        if (h) std::memcpy(h, m.h.data(), m.h.size() * sizeof(float));
        if (offsets) std::memcpy(offsets, m.offsets.data(), m.offsets.size() * sizeof(uint32_t));
        if (targets) std::memcpy(targets, m.targets.data(), m.targets.size() * sizeof(uint32_t));
        if (couplings) std::memcpy(couplings, m.couplings.data(), m.couplings.size() * sizeof(float));
        if (tau_counts) std::memcpy(tau_counts, m.tau_counts.data(), m.tau_counts.size());
        return ISING_OK;
    });
}

ising_status ising_b200_model_cost(const ising_b200_model* model, const int8_t* spins, uint32_t n,
                                   double* cost) {
    return guarded([&]() {
        require(model);
        require(cost);
        if (n != 0) require(spins);
        *cost = total_cost(model->model, spins, n);
        return ISING_OK;
    });
}

// ---------------------------------------------------------------- batches

ising_status ising_batch_create(const ising_b200_model* const* models, uint32_t n_models,
                                const uint32_t* model_of_ladder, const ising_batch_params* params,
                                ising_batch** out) {
    return guarded([&]() {
        require(models);
        require(params);
        require(out);
        if (n_models == 0) throw Error("init_state: no model given");
        std::vector<const HostModel*> host_models;
        for (uint32_t k = 0; k < n_models; ++k) {
            require(models[k]);
            host_models.push_back(&models[k]->model);
        }
        BatchConfig cfg;
        cfg.n_ladders = params->n_ladders;
        cfg.n_betas = params->n_betas;
        if (cfg.n_ladders == 0 || cfg.n_betas == 0) throw Error("init_state: batch needs at least one chain");
        require(params->betas);
        cfg.betas.assign(params->betas, params->betas + params->n_betas);
        const uint64_t chains = uint64_t(cfg.n_ladders) * cfg.n_betas;
        if (chains > 0x7fffffffull) throw Error("init_state: too many chains for one batch");
        cfg.seeds.resize(chains);
        for (uint64_t c = 0; c < chains; ++c) {
            cfg.seeds[c] = params->seeds ? params->seeds[c]
                                         : uint32_t(params->base_seed + params->first_ladder * cfg.n_betas + c);
        }
        cfg.swap_seeds.resize(cfg.n_ladders);
        for (uint32_t l = 0; l < cfg.n_ladders; ++l) {
            cfg.swap_seeds[l] = params->swap_seeds ? params->swap_seeds[l]
                                                   : uint32_t(params->swap_base_seed + params->first_ladder + l);
        }
        cfg.tau_scale = params->tau_scale;
        cfg.exp_kind = resolve_exp_kind(params->exp_kind);
        cfg.device = params->device;
        cfg.kernel = params->kernel;
        std::vector<uint32_t> of_ladder(cfg.n_ladders, 0);
        if (model_of_ladder != nullptr) {
            of_ladder.assign(model_of_ladder, model_of_ladder + cfg.n_ladders);
        } else if (n_models == cfg.n_ladders && n_models > 1) {
            for (uint32_t l = 0; l < cfg.n_ladders; ++l) of_ladder[l] = l;
        } else if (n_models != 1) {
            throw Error("init_state: model_of_ladder is required when n_models is neither 1 nor n_ladders");
        }
        auto* handle = new ising_batch{nullptr};
        try {
            handle->impl = new Batch(host_models, of_ladder, cfg, params->initial_spins);
        } catch (...) {
            delete handle;
            throw;
        }
        *out = handle;
        return ISING_OK;
    });
}

void ising_batch_free(ising_batch* batch) {
    if (batch == nullptr) return;
    delete batch->impl;
    delete batch;
}

ising_status ising_batch_run(ising_batch* batch, uint64_t sweeps, uint32_t swap_interval) {
    return guarded([&]() {
        impl_of(batch).run(sweeps, swap_interval);
        return ISING_OK;
    });
}

ising_status ising_batch_swap(ising_batch* batch) {
    return guarded([&]() {
        impl_of(batch).swap_round();
        return ISING_OK;
    });
}

ising_status ising_batch_sync(ising_batch* batch) {
    return guarded([&]() {
        impl_of(batch).sync();
        return ISING_OK;
    });
}

ising_status ising_batch_read_spins(ising_batch* batch, uint64_t first_chain, uint64_t n_chains,
                                    int8_t* out) {
    return guarded([&]() {
        impl_of(batch).read_spins(first_chain, n_chains, out);
        return ISING_OK;
    });
}

ising_status ising_batch_read_fields(ising_batch* batch, uint64_t chain, float* h_space, float* h_tau) {
    return guarded([&]() {
        impl_of(batch).read_fields(chain, h_space, h_tau);
        return ISING_OK;
    });
}

ising_status ising_batch_read_energies(ising_batch* batch, double* out) {
    return guarded([&]() {
        impl_of(batch).read_energies(out);
        return ISING_OK;
    });
}

ising_status ising_batch_read_running_energies(ising_batch* batch, double* out) {
    return guarded([&]() {
        impl_of(batch).read_running_energies(out);
        return ISING_OK;
    });
}

ising_status ising_batch_resync_energies(ising_batch* batch) {
    return guarded([&]() {
        impl_of(batch).resync_energies();
        return ISING_OK;
    });
}

ising_status ising_batch_read_stats(ising_batch* batch, uint64_t* flips, uint64_t* attempts) {
    return guarded([&]() {
        impl_of(batch).read_stats(flips, attempts);
        return ISING_OK;
    });
}

ising_status ising_batch_checksums(ising_batch* batch, uint64_t* out) {
    return guarded([&]() {
        impl_of(batch).read_checksums(out);
        return ISING_OK;
    });
}

ising_status ising_batch_field_coherence(ising_batch* batch, uint64_t* out) {
    return guarded([&]() {
        impl_of(batch).read_coherence(out);
        return ISING_OK;
    });
}

ising_status ising_batch_read_slots(ising_batch* batch, uint32_t* slot_of_chain) {
    return guarded([&]() {
        impl_of(batch).read_slots(slot_of_chain);
        return ISING_OK;
    });
}

ising_status ising_batch_read_swap_stats(ising_batch* batch, uint64_t* accepts, uint64_t* attempts) {
    return guarded([&]() {
        impl_of(batch).read_swap_stats(accepts, attempts);
        return ISING_OK;
    });
}

ising_status ising_batch_pack_results(ising_batch* batch, void* device_out) {
    return guarded([&]() {
        impl_of(batch).pack_results(device_out);
        return ISING_OK;
    });
}

ising_status ising_batch_all_gather_results(ising_batch* batch, void* nccl_comm, void* device_out_all) {
    return guarded([&]() {
        impl_of(batch).all_gather_results(nccl_comm, device_out_all);
        return ISING_OK;
    });
}

ising_status ising_batch_set_timing(ising_batch* batch, int timing) {
    return guarded([&]() {
        impl_of(batch).set_timing(timing != 0);
        return ISING_OK;
    });
}

ising_status ising_batch_record_wait(ising_batch* batch, int on) {
    return guarded([&]() {
        impl_of(batch).record_wait(on != 0);
        return ISING_OK;
    });
}

ising_status ising_batch_read_wait_stats(ising_batch* batch, uint32_t n_widths, const uint32_t* widths,
                                         double* probability, uint64_t* groups, uint64_t* with_flip) {
    return guarded([&]() {
        std::vector<uint64_t> g(n_widths), f(n_widths);
        impl_of(batch).read_wait(n_widths, widths, g.data(), f.data());
        for (uint32_t i = 0; i < n_widths; ++i) {
            if (probability != nullptr) probability[i] = g[i] ? double(f[i]) / double(g[i]) : 0.0;
            if (groups != nullptr) groups[i] = g[i];
            if (with_flip != nullptr) with_flip[i] = f[i];
        }
        return ISING_OK;
    });
}

ising_status ising_batch_get_info(ising_batch* batch, ising_batch_info* out) {
    return guarded([&]() {
        Batch& b = impl_of(batch);
        require(out);
        out->n_chains = b.n_chains();
        out->n_spins = b.n_spins();
        out->n_tiles = b.n_tiles();
        out->kernel = int(b.family());
        out->sweeps_done = b.sweeps_done();
        out->device_bytes = b.device_bytes();
        out->sweep_launches = b.sweep_launches;
        out->swap_launches = b.swap_launches;
        out->other_launches = b.other_launches;
        out->sweep_ms = b.sweep_ms();
        out->swap_ms = b.swap_ms();
        out->last_run_ms = b.last_run_ms();
        out->generic_variant = b.generic_variant();
        out->strands = b.strands();
        return ISING_OK;
    });
}

void* ising_batch_stream(ising_batch* batch) {
    return batch ? static_cast<void*>(batch->impl->stream()) : nullptr;
}

// ---------------------------------------------------------------- one-shot

ising_status ising_b200_run(const ising_b200_model* model, const ising_b200_run_params* params,
                            ising_b200_run_report* out) {
    return guarded([&]() {
        require(out);
        *out = run_single(model, params).report;
        return ISING_OK;
    });
}

ising_status ising_b200_run_json(const ising_b200_model* model, const ising_b200_run_params* params,
                                 ising_b200_run_report* out_report, char** out_json) {
    return guarded([&]() {
        require(out_json);
        const SingleRun run = run_single(model, params);
        if (out_report != nullptr) *out_report = run.report;
        static const char* const exp_names[] = {"?", "exact", "fast", "accurate"};
        utsname u{};
        std::string env = "unknown";
        if (uname(&u) == 0) env = std::string(u.nodename) + " " + u.sysname + " " + u.release + " " + u.machine;
        cudaDeviceProp prop{};
        if (cudaGetDeviceProperties(&prop, params->device) == cudaSuccess) env += std::string("; device=") + prop.name;
        env += "; build=optimized; compiler=nvcc " + std::to_string(__CUDACC_VER_MAJOR__) + "." +
               std::to_string(__CUDACC_VER_MINOR__);
        char checksum[24];
        std::snprintf(checksum, sizeof checksum, "%016" PRIx64, run.report.checksum);
        // the keys of the reference's report (ref: capi.cpp:237-258), in its (alphabetical) dump order
        std::string j = "{\n";
        j += "  \"attempts\": " + std::to_string(run.report.attempts) + ",\n";
        j += "  \"beta\": " + json_number(double(params->beta)) + ",\n";
        j += std::string("  \"checksum\": \"") + checksum + "\",\n";
        j += std::string("  \"engine\": \"") + (run.family == 3 ? "b200-strand" : run.family == 2 ? "b200-layered" : "b200-generic") + "\",\n";
        j += "  \"environment\": \"" + env + "\",\n";
        j += std::string("  \"exp\": \"") + exp_names[run.exp_kind] + "\",\n";
        j += "  \"final_cost\": " + json_number(run.report.final_cost) + ",\n";
        j += "  \"flip_rate\": " + json_number(run.report.flip_rate) + ",\n";
        j += "  \"flips\": " + std::to_string(run.report.flips) + ",\n";
        j += "  \"seed\": " + std::to_string(params->seed) + ",\n";
        j += "  \"spins\": " + std::to_string(model->model.n_spins) + ",\n";
        j += "  \"sweeps\": " + std::to_string(params->sweeps) + ",\n";
        j += "  \"tau_scale\": " + json_number(double(params->tau_scale)) + ",\n";
        j += "  \"wait\": {},\n";  // one chain fills one lane: no lockstep groups to wait in
        j += "  \"workers\": 1\n}";
        *out_json = dup_string(j);
        return *out_json != nullptr ? ISING_OK : ISING_ERR_INTERNAL;
    });
}

// ---------------------------------------------------------------- coalesced (intra-system) batches

ising_status ising_coalesced_create(const ising_b200_model* model, const ising_coalesced_params* params,
                                    ising_coalesced** out) {
    return guarded([&]() {
        require(model);
        require(params);
        require(out);
        if (params->n_chains == 0 || params->betas == nullptr) throw Error("null argument");
        CoalescedConfig cfg;
        cfg.betas.assign(params->betas, params->betas + params->n_chains);
        cfg.seeds.resize(params->n_chains);
        for (uint32_t c = 0; c < params->n_chains; ++c) {
            cfg.seeds[c] = params->seeds != nullptr ? params->seeds[c] : params->base_seed + c * (model->model.layers / 2);
        }
        cfg.tau_scale = params->tau_scale;
        cfg.exp_kind = resolve_exp_kind(params->exp_kind);
        cfg.device = params->device;
        auto impl = std::make_unique<CoalescedBatch>(model->model, cfg, params->initial_spins);
        *out = new ising_coalesced{impl.release()};
        return ISING_OK;
    });
}

void ising_coalesced_free(ising_coalesced* batch) {
    if (batch != nullptr) {
        delete batch->impl;
        delete batch;
    }
}

namespace {
CoalescedBatch& coalesced_of(ising_coalesced* b) {
    require(b);
    return *b->impl;
}
}  // namespace

ising_status ising_coalesced_run(ising_coalesced* batch, uint64_t sweeps) {
    return guarded([&]() {
        coalesced_of(batch).run(sweeps);
        return ISING_OK;
    });
}

ising_status ising_coalesced_read_spins(ising_coalesced* batch, uint64_t chain, int8_t* out) {
    return guarded([&]() {
        coalesced_of(batch).read_spins(chain, out);
        return ISING_OK;
    });
}

ising_status ising_coalesced_read_fields(ising_coalesced* batch, uint64_t chain, float* hs, float* ht) {
    return guarded([&]() {
        coalesced_of(batch).read_fields(chain, hs, ht);
        return ISING_OK;
    });
}

ising_status ising_coalesced_read_stats(ising_coalesced* batch, uint64_t* flips, uint64_t* attempts) {
    return guarded([&]() {
        coalesced_of(batch).read_stats(flips, attempts);
        return ISING_OK;
    });
}

ising_status ising_coalesced_read_energies(ising_coalesced* batch, double* out) {
    return guarded([&]() {
        coalesced_of(batch).read_energies(out);
        return ISING_OK;
    });
}

ising_status ising_coalesced_checksums(ising_coalesced* batch, uint64_t* out) {
    return guarded([&]() {
        coalesced_of(batch).read_checksums(out);
        return ISING_OK;
    });
}

ising_status ising_coalesced_get_info(ising_coalesced* batch, ising_coalesced_info* out) {
    return guarded([&]() {
        CoalescedBatch& b = coalesced_of(batch);
        require(out);
        out->n_chains = b.n_chains();
        out->n_spins = b.n_spins();
        out->lanes = b.lanes();
        out->sweeps_done = b.sweeps_done();
        out->launches = b.launches;
        out->last_run_ms = b.last_run_ms();
        return ISING_OK;
    });
}

// ---------------------------------------------------------------- model text I/O

void ising_b200_string_free(char* text) { delete[] text; }

ising_status ising_b200_model_from_string(const char* text, ising_b200_model** out) {
    return guarded([&]() {
        require(text);
        require(out);
        *out = new ising_b200_model{model_from_text(text)};
        return ISING_OK;
    });
}

ising_status ising_b200_model_to_string(const ising_b200_model* model, char** out) {
    return guarded([&]() {
        require(model);
        require(out);
        *out = dup_string(model_to_text(model->model));
        return *out != nullptr ? ISING_OK : ISING_ERR_INTERNAL;
    });
}

ising_status ising_b200_model_load(const char* path, ising_b200_model** out) {
    return guarded([&]() {
        require(path);
        require(out);
        *out = new ising_b200_model{load_model_text(path)};
        return ISING_OK;
    });
}

ising_status ising_b200_model_save(const ising_b200_model* model, const char* path) {
    return guarded([&]() {
        require(model);
        require(path);
        save_model_text(model->model, path);
        return ISING_OK;
    });
}

}  // extern "C"
