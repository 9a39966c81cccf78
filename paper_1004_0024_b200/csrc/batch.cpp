#include "batch.hpp"

#include <algorithm>
#include <cmath>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <dlfcn.h>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>

namespace isingb200 {

void cuda_check(cudaError_t status, const char* what) {
    if (status != cudaSuccess) {
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(status));
    }
}

DeviceBuffer::~DeviceBuffer() {
    if (ptr_ != nullptr) cudaFree(ptr_);
}

void DeviceBuffer::allocate(size_t bytes, size_t& tally) {
    if (ptr_ != nullptr) {
        cudaFree(ptr_);
        ptr_ = nullptr;
    }
    bytes_ = 0;
    if (bytes == 0) return;
    cuda_check(cudaMalloc(&ptr_, bytes), "cudaMalloc");
    bytes_ = bytes;  // (only once the memory exists: a failed allocation leaves an empty buffer)
    tally += bytes;
}

namespace {

template <typename T>
void upload(DeviceBuffer& buf, const std::vector<T>& host, size_t& tally, cudaStream_t stream) {
    buf.allocate(host.size() * sizeof(T), tally);
    if (!host.empty()) {
        cuda_check(cudaMemcpyAsync(buf.as<void>(), host.data(), host.size() * sizeof(T),
                                   cudaMemcpyHostToDevice, stream),
                   "upload");
    }
}

// Host-side image of DevLayerGraph (see device_batch.hpp for the meaning of every array).
struct HostLayerGraph {
    std::vector<uint4> pos, band_pm, chunks;
    std::vector<uint4> far;        // {target position, 7 - attempt index in its chunk, bits of 2J, 0}
    std::vector<uint32_t> groups;  // edge begin | edge count << 16
};

bool is_band(uint32_t p, uint32_t t) { return (t > p ? t - p : p - t) <= 2; }

uint32_t bits(float v) {
    uint32_t b;
    std::memcpy(&b, &v, sizeof b);
    return b;
}

HostLayerGraph build_layer_graph(const HostModel& m, float tau_scale) {
    const uint32_t P = m.per_layer;
    HostLayerGraph out;
    out.pos.resize(P);
    out.band_pm.resize(2 * size_t(P));
    out.chunks.resize(P / 8);
    std::vector<uint4>&pos = out.pos, &band_pm = out.band_pm, &chunks = out.chunks;
    std::vector<uint4>& far = out.far;
    std::vector<uint32_t>& groups = out.groups;
        // Far (non-band) edges are split by who applies them.  The FAR warp, which trails the sweep
    // warp by whole 8-attempt chunks, takes every target the sweep warp is not going to read
    // soon: backward targets (already out of its register window) and forward targets that
    // enter the window at least two chunks after the flipping attempt's chunk.  The sweep warp
    // keeps the NEAR forward targets.  A near target inside the columns the chunk has already
    // loaded (<= 8c+10) makes the chunk CAREFUL: it runs the per-attempt loop, with per-position
    // near lists.  Otherwise the chunk is LEAN and applies its near edges, like the far warp,
    // in groups after its last attempt.
    const auto delegated = [](uint32_t p, uint32_t t) { return t < p || (t - 3) / 8 >= p / 8 + 2; };
    struct Edge { uint32_t k, t, j2; };
    // a group is up to 8 edges with distinct targets, applied with their loads batched
    // A group is padded to 8 edges when the layer has columns to spare for it: a padding edge
    // is tied to attempt 8 (no such attempt: nobody accepts it, it adds -0.0) and targets a
    // column that no real edge of the group uses and that the sweep warp does not write while
    // the group can be applied (it retires columns up to 8c+13 meanwhile): one at least a chunk
    // behind chunk c, else one at least three chunks ahead.
    const auto emit_groups = [&](const std::vector<Edge>& edges, uint32_t chunk, bool pad) {
        const uint32_t first_group = uint32_t(groups.size());
        std::vector<Edge> cur;
        const auto close = [&]() {
            if (cur.empty()) return;
            const uint32_t begin = uint32_t(far.size());
            std::vector<uint32_t> used;
            for (const Edge& e : cur) used.push_back(e.t);
            for (uint32_t col = 0; pad && col < P && cur.size() < 8; ++col) {
                const bool safe = col + 9 <= 8 * chunk || col >= 8 * chunk + 24;
                if (!safe || std::find(used.begin(), used.end(), col) != used.end()) continue;
                cur.push_back({8, col, 0x80000000u});
                used.push_back(col);
            }
            for (const Edge& e : cur) far.push_back(make_uint4(e.t, e.k < 8 ? 7u - e.k : 15u, e.j2, 0u));  // shift 15: a bit nobody sets
            groups.push_back(begin | uint32_t(cur.size()) << 16);
            cur.clear();
        };
        for (const Edge& e : edges) {
            const bool clash = std::any_of(cur.begin(), cur.end(), [&](const Edge& o) { return o.t == e.t; });
            if (cur.size() == 8 || clash) close();
            cur.push_back(e);
        }
        close();
        return first_group | (uint32_t(groups.size()) - first_group) << 16;
    };
    for (uint32_t p0 = 0; p0 < P; p0 += 8) {
        std::vector<Edge> for_far_warp, near_all;
        std::vector<std::vector<Edge>> near_of(8);
        bool careful = false;
        for (uint32_t k = 0; k < 8; ++k) {
            const uint32_t p = p0 + k;
            uint32_t j2[4] = {0, 0, 0, 0}, mask[4] = {0x80000000u, 0x80000000u, 0x80000000u, 0x80000000u};
            for (uint32_t e = m.layer_offsets[p]; e < m.layer_offsets[p + 1]; ++e) {
                const uint32_t t = m.layer_targets[e];
                const uint32_t doubled = bits(2.0f * m.layer_couplings[e]);  // exact
                if (is_band(p, t)) {
                    const int off = int(t) - int(p);             // -2, -1, +1, +2
                    const int slot = off < 0 ? off + 2 : off + 1;  //  0,  1,  2,  3
                    j2[slot] = doubled;
                    mask[slot] = 0;
                } else if (delegated(p, t)) {
                    for_far_warp.push_back({k, t, doubled});
                } else {
                    near_of[k].push_back({k, t, doubled});
                    near_all.push_back({k, t, doubled});
                    careful = careful || t <= p0 + 10;
                }
            }
            const float tau2 = 2.0f * m.layer_tau[p];
            const float tau2g = tau_scale * tau2;  // f32 product, as gamma * h_tau in the reference
            pos[p] = make_uint4(bits(tau2g), bits(tau2), 0, 0);
            // what a flip of s adds to the four band neighbours: -(2s)*J, i.e. 2J with the sign
            // of -s; an empty slot adds -0.0.  Entry 2p is for s = -1 (sign bit of -2*beta*s
            // clear), entry 2p+1 for s = +1.
            for (uint32_t neg = 0; neg < 2; ++neg) {
                const uint32_t flip = neg ? 0x80000000u : 0u;
                band_pm[2 * size_t(p) + neg] = make_uint4((j2[0] ^ flip) | mask[0], (j2[1] ^ flip) | mask[1],
                                                         (j2[2] ^ flip) | mask[2], (j2[3] ^ flip) | mask[3]);
            }
        }
        uint32_t near_groups = 0;
        if (careful) {
            for (uint32_t k = 0; k < 8; ++k) {
                pos[p0 + k].z = uint32_t(far.size()) | uint32_t(near_of[k].size()) << 16;
                for (const Edge& e : near_of[k]) far.push_back(make_uint4(e.t, e.k < 8 ? 7u - e.k : 15u, e.j2, 0u));  // shift 15: a bit nobody sets
            }
        } else {
            near_groups = emit_groups(near_all, p0 / 8, false);  // rare and short: not worth padding
        }
        // flags: bit 0 careful; bit 1 lean but first or last chunk of the layer
        const bool odd = !careful && (p0 == 0 || p0 + 8 >= P);
        chunks[p0 / 8] = make_uint4(emit_groups(for_far_warp, p0 / 8, true), near_groups,
                                    (careful ? 1u : 0u) | (odd ? 2u : 0u), 0u);
    }
    if (far.size() > 0xffffu || groups.size() > 0xffffu) throw Error("init_state: layer graph too large for the layered kernel");
    return out;
}


// Host-side image of DevStrandGraph (see device_batch.hpp and kernels_strand.cu).
struct HostStrandGraph {
    std::vector<uint4> pos, band_pm, chunks, edges, inslots;
    std::vector<uint32_t> tau;
};

HostStrandGraph build_strand_graph(const HostModel& m, float tau_scale) {
    const uint32_t P = m.per_layer;
    HostStrandGraph out;
    out.pos.resize(P);
    out.band_pm.resize(2 * size_t(P));
    out.chunks.resize(P / 8);
    struct NearEdge { uint32_t k, t, j2; };
    // A far edge q -> t is PULLED by its target: {q, index in q's list, 2J} per target, in the order the
    // reference applies them to h[t] between two attempts of t — sources after t (the sweep before),
    // then sources before t (this sweep), each group in attempt order.
    struct InEdge { uint32_t q, e, j2; };
    std::vector<std::vector<InEdge>> incoming(P);
    std::vector<std::vector<NearEdge>> near_of(P);
    for (uint32_t p = 0; p < P; ++p) {
        const uint32_t p0 = p / 8 * 8;
        uint32_t j2[4] = {0, 0, 0, 0}, mask[4] = {0x80000000u, 0x80000000u, 0x80000000u, 0x80000000u};
        for (uint32_t e = m.layer_offsets[p]; e < m.layer_offsets[p + 1]; ++e) {
            const uint32_t t = m.layer_targets[e];
            const uint32_t doubled = bits(2.0f * m.layer_couplings[e]);  // exact
            if (is_band(p, t)) {
                const int off = int(t) - int(p);               // -2, -1, +1, +2
                const int slot = off < 0 ? off + 2 : off + 1;  //  0,  1,  2,  3
                j2[slot] = doubled;
                mask[slot] = 0;
            } else if (t > p && t <= p0 + 10) {
                // the target column is on its way into the register window already (the chunk loads
                // p0+3 .. p0+10 at its start and pulls their far updates then): pushed, through the scratch
                near_of[p].push_back({p - p0, t, doubled});
            } else {
                incoming[t].push_back({p, e, doubled});
            }
        }
        const float tau2g = tau_scale * (2.0f * m.layer_tau[p]);  // f32 product, as gamma * h_tau in the reference
        out.pos[p] = make_uint4(bits(tau2g), 0, 0, 0);
        out.tau.push_back(bits(tau2g));
        // what a flip of s adds to the four band neighbours: -(2s)*J, i.e. 2J with the sign of -s; an
        // empty slot adds -0.0.  Entry 2p is for s = -1, entry 2p+1 for s = +1.
        for (uint32_t neg = 0; neg < 2; ++neg) {
            const uint32_t flip = neg ? 0x80000000u : 0u;
            out.band_pm[2 * size_t(p) + neg] = make_uint4((j2[0] ^ flip) | mask[0], (j2[1] ^ flip) | mask[1],
                                                         (j2[2] ^ flip) | mask[2], (j2[3] ^ flip) | mask[3]);
        }
    }
    // slot: {bits of 2J, meta}; meta = shift | byte offset of the source chunk's cell row << 8, the shift
    // (23 - bit) moving the source's spin bit (8 + bit of its cell) to bit 31 and its flip bit to bit 23.
    // The null slot shifts by 31 (bit 23 ends up clear: never flipped) and adds -0.0.
    const uint32_t null_j2 = 0x80000000u, null_meta = 31u;
    const auto slot_of = [](const InEdge& in) { return (23u - (in.q & 7u)) | ((in.q / 8u) * 64u) << 8; };
    std::vector<bool> extra_in(P, false);
    out.inslots.assign(size_t(P) + 8, make_uint4(null_j2, null_meta, null_j2, null_meta));
    for (uint32_t t = 0; t < P; ++t) {
        std::vector<InEdge>& in = incoming[t];
        std::stable_sort(in.begin(), in.end(), [t](const InEdge& a, const InEdge& b) {
            const bool a_after = a.q > t, b_after = b.q > t;  // sources after t come first (older sweep)
            if (a_after != b_after) return a_after;
            return a.q != b.q ? a.q < b.q : a.e < b.e;
        });
        uint4 s = make_uint4(null_j2, null_meta, null_j2, null_meta);
        if (in.size() > 0) { s.x = in[0].j2; s.y = slot_of(in[0]); }
        if (in.size() > 1) { s.z = in[1].j2; s.w = slot_of(in[1]); }
        out.inslots[t] = s;
        // further far edges into t: a list in `edges`, applied by the careful path
        const uint32_t more = in.size() > 2 ? uint32_t(in.size() - 2) : 0u;
        out.pos[t].z = uint32_t(out.edges.size()) | more << 16;
        for (size_t i = 2; i < in.size(); ++i) out.edges.push_back(make_uint4(in[i].j2, slot_of(in[i]), 0u, 0u));
        extra_in[t] = more != 0;
    }
    for (uint32_t p0 = 0; p0 < P; p0 += 8) {
        bool careful = false;
        for (uint32_t k = 0; k < 8; ++k) {
            const std::vector<NearEdge>& near = near_of[p0 + k];
            out.pos[p0 + k].y = uint32_t(out.edges.size()) | uint32_t(near.size()) << 16;
            for (const NearEdge& e : near) out.edges.push_back(make_uint4(e.t, e.k, e.j2, 0u));
            careful = careful || !near.empty();
            // the columns entering the window during this chunk
            const uint32_t entering = p0 + 3 + k;
            careful = careful || (entering < P && extra_in[entering]);
        }
        out.chunks[p0 / 8] = make_uint4(0u, 0u, careful ? 1u : 0u, 0u);
    }
    return out;
}

// An unsigned value from the environment (tuning knobs of the strand family), 0 when unset or malformed.
uint32_t env_u32(const char* name) {
    const char* text = std::getenv(name);
    if (text == nullptr || *text == 0) return 0;
    char* end = nullptr;
    const unsigned long v = std::strtoul(text, &end, 10);
    return (end != nullptr && *end == 0 && v <= 0xfffffffful) ? uint32_t(v) : 0u;
}
}  // namespace

// Runs fn(0) .. fn(count - 1) on up to 16 host threads (the per-model graph analysis of a batch with
// many distinct instances); the first exception is rethrown on the calling thread.
template <typename Fn>
static void parallel_for(size_t count, Fn&& fn) {
    const size_t workers = std::min<size_t>({count, size_t(std::max(1u, std::thread::hardware_concurrency())), size_t(16)});
    if (workers <= 1) {
        for (size_t k = 0; k < count; ++k) fn(k);
        return;
    }
    std::atomic<size_t> next{0};
    std::exception_ptr failure;
    std::mutex failure_lock;
    std::vector<std::thread> pool;
    for (size_t w = 0; w < workers; ++w) {
        pool.emplace_back([&]() {
            for (size_t k = next.fetch_add(1); k < count; k = next.fetch_add(1)) {
                try {
                    fn(k);
                } catch (...) {
                    std::lock_guard<std::mutex> hold(failure_lock);
                    if (!failure) failure = std::current_exception();
                }
            }
        });
    }
    for (std::thread& t : pool) t.join();
    if (failure) std::rethrow_exception(failure);
}

void Batch::bind_device() const { cuda_check(cudaSetDevice(device_), "cudaSetDevice"); }

// total_cost (ref: model.cpp:108-126) as the flat sequence of terms its two loops visit: for every
// spin the field term, then its edges towards higher indices in adjacency order.  Terms with a zero
// field are left out (cost - (+-0) == cost for every cost the sum can hold), the tail is padded
// with zero coefficients to a multiple of 32 so that a warp can always take 32 terms at a time.
static std::vector<uint4> build_cost_terms(const HostModel& m, float tau_scale = 1.0f) {
    std::vector<uint4> terms;
    terms.reserve(size_t(m.n_spins) + m.targets.size() / 2 + 32);
    const auto bits = [](float v) {
        uint32_t pattern;
        std::memcpy(&pattern, &v, sizeof pattern);
        return pattern;
    };
    for (uint32_t i = 0; i < m.n_spins; ++i) {
        if (m.h[i] != 0.0f) terms.push_back(make_uint4(i, kFieldTerm, bits(m.h[i]), 0));
        const uint32_t first_tau = m.offsets[i + 1] - m.tau_counts[i];
        for (uint32_t e = m.offsets[i]; e < m.offsets[i + 1]; ++e) {
            // tempering energy: the tau coupling as the sweep sees it, gamma * J in f32
            const float j = e >= first_tau ? tau_scale * m.couplings[e] : m.couplings[e];
            if (m.targets[e] > i) terms.push_back(make_uint4(i, m.targets[e], bits(j), 0));
        }
    }
    do {
        terms.push_back(make_uint4(0, kFieldTerm, 0, 0));
    } while (terms.size() % 32 != 0);
    return terms;
}

Batch::Batch(const std::vector<const HostModel*>& models,
             const std::vector<uint32_t>& model_of_ladder, const BatchConfig& cfg,
             const int8_t* initial_spins) {
    // The destructor does not run for an object whose constructor throws: release what the body had
    // created by then (stream, events; the DeviceBuffer members clean up after themselves).
    try {
        construct(models, model_of_ladder, cfg, initial_spins);
    } catch (...) {
        release_cuda_objects();
        throw;
    }
}

void Batch::release_cuda_objects() {
    for (TimedLaunch& t : pending_) {
        cudaEventDestroy(t.start);
        cudaEventDestroy(t.stop);
    }
    pending_.clear();
    if (run_start_ != nullptr) cudaEventDestroy(run_start_);
    if (run_stop_ != nullptr) cudaEventDestroy(run_stop_);
    if (stream_ != nullptr) cudaStreamDestroy(stream_);
    run_start_ = run_stop_ = nullptr;
    stream_ = nullptr;
}

void Batch::construct(const std::vector<const HostModel*>& models,
                      const std::vector<uint32_t>& model_of_ladder, const BatchConfig& cfg,
                      const int8_t* initial_spins) {
    const auto t_begin = std::chrono::steady_clock::now();
    // ---- argument checks (ref: check_engine_model, sweep_state.cpp:108-158)
    if (models.empty()) throw Error("init_state: no model given");
    if (cfg.n_ladders == 0 || cfg.n_betas == 0) throw Error("init_state: batch needs at least one chain");
    if (cfg.betas.size() != cfg.n_betas) throw Error("init_state: betas count mismatch");
    for (float beta : cfg.betas) {
        if (!(beta >= 0.0f) || !std::isfinite(beta)) throw Error("init_state: beta must be finite and >= 0");
    }
    if (!std::isfinite(cfg.tau_scale)) throw Error("init_state: tau_scale must be finite");
    if (cfg.exp_kind < 1 || cfg.exp_kind > 3) throw Error("invalid exp_kind value " + std::to_string(cfg.exp_kind));
    const uint64_t chains64 = uint64_t(cfg.n_ladders) * cfg.n_betas;
    if (chains64 > 0x7fffffffull) throw Error("init_state: too many chains for one batch");
    if (cfg.seeds.size() != chains64 || cfg.swap_seeds.size() != cfg.n_ladders) {
        throw Error("init_state: seed count mismatch");
    }
    if (model_of_ladder.size() != cfg.n_ladders) throw Error("init_state: model_of_ladder count mismatch");
    const uint32_t n = models[0]->n_spins;
    bool any_tau = false;
    for (const HostModel* m : models) {
        if (m == nullptr) throw Error("null argument");
        if (m->n_spins != n) throw Error("init_state: all models of a batch must have the same spin count");
        any_tau = any_tau || m->has_tau;
    }
    for (uint32_t idx : model_of_ladder) {
        if (idx >= models.size()) throw Error("init_state: model_of_ladder entry out of range");
    }
    if (cfg.kernel < 0 || cfg.kernel > 3) throw Error("invalid kernel value " + std::to_string(cfg.kernel));
    // The layered family needs every model to qualify (HostModel::layered_uniform) and one layer
    // to fit the on-chip window: <= 512 positions (TMEM columns) and the graph within shared memory.
    uint32_t max_per_layer = 0, max_far_edges = 0, max_groups = 0;
    bool layered_ok = true;
    for (const HostModel* m : models) {
        layered_ok = layered_ok && m->layered_uniform && m->per_layer % 8 == 0;
        max_per_layer = std::max(max_per_layer, m->per_layer);
        if (!m->layered_uniform) continue;
        for (uint32_t p = 0; p < m->per_layer; ++p) {
            uint32_t far_here = 0;
            for (uint32_t e = m->layer_offsets[p]; e < m->layer_offsets[p + 1]; ++e) {
                far_here += is_band(p, m->layer_targets[e]) ? 0u : 1u;
            }
            layered_ok = layered_ok && far_here < 16;  // 4-bit edge counts in DevLayerGraph::pos
        }
    }
    // The strand family needs identical-layer models with one tau coupling per position as well, but
    // nothing on chip: any per_layer that is a multiple of 8 (two chunks at least).
    bool strand_ok = true;
    uint32_t common_layers = 0;  // gcd of the models' layer counts: the strand count must divide it
    uint32_t min_chunks = 0xffffffffu;
    for (const HostModel* m : models) {
        strand_ok = strand_ok && m->layered_uniform && m->per_layer % 8 == 0 && m->per_layer >= 16;
        if (!strand_ok) break;
        uint32_t a = common_layers, c = m->layers;
        while (c != 0) { const uint32_t r = a % c; a = c; c = r; }
        common_layers = a;
        min_chunks = std::min(min_chunks, m->per_layer / 8);
    }
    if (cfg.kernel == int(KernelFamily::strand) && !strand_ok) {
        throw Error("init_state: the strand kernel needs identical-layer models with equal tau couplings "
                    "and a multiple of 8, at least 16, positions per layer");
    }
    // AUTO: the strand family whenever the batch qualifies (the fastest on every layered workload
    // measured); the Tensor Memory family only on request.
    const bool use_strand = cfg.kernel == int(KernelFamily::strand) || (cfg.kernel == 0 && strand_ok);
    std::vector<HostLayerGraph> host_graphs;
    if (layered_ok && !use_strand && cfg.kernel != int(KernelFamily::generic)) {
        host_graphs.resize(models.size());
        parallel_for(models.size(), [&](size_t k) { host_graphs[k] = build_layer_graph(*models[k], cfg.tau_scale); });
        for (const HostLayerGraph& hg : host_graphs) {
            layered_ok = layered_ok && hg.far.size() <= 0xffffu && hg.groups.size() <= 0xffffu;
            max_far_edges = std::max(max_far_edges, uint32_t(hg.far.size()));
            max_groups = std::max(max_groups, uint32_t(hg.groups.size()));
        }
    }
    const bool graph_shared = models.size() == 1;
    const size_t layered_smem = layered_ok ? layered_smem_bytes(max_per_layer, max_far_edges, max_groups, graph_shared) : 0;
    layered_ok = layered_ok && layered_smem != 0;
    if (cfg.kernel == int(KernelFamily::layered) && !layered_ok) {
        throw Error("init_state: the layered kernel needs identical-layer models with equal tau couplings "
                    "and a multiple of 8, at most 512, positions per layer");
    }
    family_ = use_strand ? KernelFamily::strand
              : (cfg.kernel != int(KernelFamily::generic) && layered_ok) ? KernelFamily::layered
                                                                         : KernelFamily::generic;
    if (family_ != KernelFamily::generic) any_tau = false;  // the tau field is rebuilt, never stored

    if (initial_spins != nullptr) {  // (host-side validation first: nothing to release on failure)
        const size_t total = size_t(chains64) * n;
        for (size_t k = 0; k < total; ++k) {
            if (initial_spins[k] != 1 && initial_spins[k] != -1) throw Error("init_state: spins must be +/-1");
        }
    }

    const auto t_checked = std::chrono::steady_clock::now();
    // ---- device
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        throw CudaError("no CUDA device available (this engine has no CPU fallback)");
    }
    if (cfg.device < 0 || cfg.device >= count) throw Error("invalid device ordinal " + std::to_string(cfg.device));
    device_ = cfg.device;
    bind_device();
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreate(&run_start_), "cudaEventCreate");
    cuda_check(cudaEventCreate(&run_stop_), "cudaEventCreate");

    // ---- tiles: runs of consecutive ladders sharing a model, cut every 32 chains
    std::vector<uint32_t> tile_first, tile_count, tile_model, chain_loc(chains64);
    {
        uint32_t l = 0;
        while (l < cfg.n_ladders) {
            uint32_t r = l;
            while (r < cfg.n_ladders && model_of_ladder[r] == model_of_ladder[l]) ++r;
            const uint32_t first = l * cfg.n_betas, last = r * cfg.n_betas;
            for (uint32_t c = first; c < last; c += 32) {
                const uint32_t cnt = std::min<uint32_t>(32, last - c);
                for (uint32_t k = 0; k < cnt; ++k) chain_loc[c + k] = uint32_t(tile_first.size()) * 32 + k;
                tile_first.push_back(c);
                tile_count.push_back(cnt);
                tile_model.push_back(model_of_ladder[l]);
            }
            l = r;
        }
    }

    // ---- models
    std::vector<DevModel> dev_models;
    const auto keep = [&](auto const& host_vec) {
        model_storage_.push_back(std::make_unique<DeviceBuffer>());
        upload(*model_storage_.back(), host_vec, device_bytes_, stream_);
        return model_storage_.back().get();
    };
    struct Prepared {  // what the kernels want to know about a model, worked out on the host
        uint32_t distinct_targets = 1u, reduction_safe = 1u;
        std::vector<float> window;  // empty: unusable
        std::vector<uint4> terms, tempering_terms;  // the second stays empty when tau_scale is 1
    };
    std::vector<Prepared> prepared(models.size());
    const bool generic_family = family_ == KernelFamily::generic;
    parallel_for(models.size(), [&](size_t k) {
        const HostModel* m = models[k];
        Prepared& out = prepared[k];
        for (uint32_t i = 0; i < m->n_spins && out.distinct_targets; ++i) {
            for (uint32_t a = m->offsets[i]; a < m->offsets[i + 1] && out.distinct_targets; ++a) {
                for (uint32_t b = a + 1; b < m->offsets[i + 1]; ++b) {
                    if (m->targets[a] == m->targets[b]) out.distinct_targets = 0u;
                }
            }
        }
        const auto tiny = [](float v) { return v != 0.0f && std::fabs(v) < 0x1p-100f; };
        for (float v : m->h) out.reduction_safe &= tiny(v) ? 0u : 1u;
        for (float v : m->couplings) out.reduction_safe &= tiny(v) ? 0u : 1u;
        if (generic_family && out.reduction_safe) {
            out.window.assign(size_t(m->n_spins) * 8, 0.0f);
            bool usable = true;
            for (uint32_t i = 0; i < m->n_spins && usable; ++i) {
                const uint32_t end = m->offsets[i + 1], first_tau = end - m->tau_counts[i];
                for (uint32_t e = m->offsets[i]; e < end; ++e) {
                    const uint32_t t = m->targets[e];
                    if (t <= i || t / 8 != i / 8) continue;
                    float& slot = out.window[size_t(i) * 8 + (t - i)];
                    if (e >= first_tau || slot != 0.0f) usable = false;
                    slot = m->couplings[e];
                }
            }
            if (!usable) out.window.clear();
        }
        out.terms = build_cost_terms(*m);
        if (cfg.tau_scale != 1.0f && m->has_tau) out.tempering_terms = build_cost_terms(*m, cfg.tau_scale);
    });
    for (size_t k = 0; k < models.size(); ++k) {
        const HostModel* m = models[k];
        const Prepared& ready = prepared[k];
        DevModel d{};
        d.n_spins = m->n_spins;
        d.has_tau = m->has_tau ? 1u : 0u;
        d.distinct_targets = ready.distinct_targets;
        d.reduction_safe = ready.reduction_safe;
        d.window = ready.window.empty() ? nullptr : keep(ready.window)->as<float>();
        d.h = keep(m->h)->as<float>();
        d.offsets = keep(m->offsets)->as<uint32_t>();
        d.targets = keep(m->targets)->as<uint32_t>();
        d.couplings = keep(m->couplings)->as<float>();
        d.tau_counts = keep(m->tau_counts)->as<uint8_t>();
        d.cost_terms = keep(ready.terms)->as<uint4>();
        d.n_cost_terms = uint32_t(ready.terms.size());
        // (scaling a coupling never changes which terms exist: the two lists have one length)
        d.tempering_terms = ready.tempering_terms.empty() ? d.cost_terms : keep(ready.tempering_terms)->as<uint4>();
        d.energy_block = (m->layers != 0 && m->per_layer != 0) ? m->per_layer : m->n_spins;
        dev_models.push_back(d);
    }
    upload(models_, dev_models, device_bytes_, stream_);
    dev_.generic_reduce = 1u;
    bool all_windows = true;
    for (const DevModel& d : dev_models) {
        dev_.generic_reduce &= d.reduction_safe;
        all_windows = all_windows && d.window != nullptr;
    }
    dev_.generic_windows = dev_.generic_reduce && all_windows ? 1u : 0u;
    generic_variant_ = family_ != KernelFamily::generic ? 0u : !dev_.generic_reduce ? 0u : all_windows ? 2u : 1u;

    if (family_ == KernelFamily::layered) {
        cudaDeviceProp prop{};
        cuda_check(cudaGetDeviceProperties(&prop, device_), "cudaGetDeviceProperties");
        if (prop.major != 10) throw CudaError("the layered kernel needs an sm_100 device (tcgen05 tensor memory)");
        sm_count_ = prop.multiProcessorCount;
        std::vector<DevLayerGraph> graphs;
        for (size_t k = 0; k < models.size(); ++k) {
            HostLayerGraph& hg = host_graphs[k];
            DevLayerGraph g{};
            g.per_layer = models[k]->per_layer;
            g.layers = models[k]->layers;
            g.n_far = uint32_t(hg.far.size());
            g.n_groups = uint32_t(hg.groups.size());
            if (hg.far.empty()) hg.far.push_back(make_uint4(0, 0, 0, 0));
            if (hg.groups.empty()) hg.groups.push_back(0);
            g.pos = keep(hg.pos)->as<uint4>();
            g.band_pm = keep(hg.band_pm)->as<uint4>();
            g.chunks = keep(hg.chunks)->as<uint4>();
            g.groups = keep(hg.groups)->as<uint32_t>();
            g.far = keep(hg.far)->as<uint4>();
            graphs.push_back(g);
        }
        cuda_check(cudaStreamSynchronize(stream_), "upload layer graphs");  // host_graphs die with the constructor
        upload(layer_graphs_, graphs, device_bytes_, stream_);
        cuda_check(cudaStreamSynchronize(stream_), "upload layer graphs");
        dev_.layer_graphs = layer_graphs_.as<DevLayerGraph>();
        dev_.max_far_edges = max_far_edges;
        dev_.max_groups = max_groups;
        dev_.max_per_layer = max_per_layer;
        dev_.graph_shared = graph_shared ? 1u : 0u;
        dev_.layered_stages = layered_stage_count(max_per_layer, max_far_edges, max_groups, graph_shared);
        dev_.layered_smem = uint32_t(layered_smem);
        cuda_check(prepare_layered_kernels(layered_smem), "cudaFuncSetAttribute");
    }

    if (family_ == KernelFamily::strand) {
        cudaDeviceProp prop{};
        cuda_check(cudaGetDeviceProperties(&prop, device_), "cudaGetDeviceProperties");
        sm_count_ = prop.multiProcessorCount;
        std::vector<HostStrandGraph> strand_host(models.size());
        parallel_for(models.size(), [&](size_t k) { strand_host[k] = build_strand_graph(*models[k], cfg.tau_scale); });
        std::vector<DevStrandGraph> graphs;
        for (size_t k = 0; k < models.size(); ++k) {
            HostStrandGraph& hg = strand_host[k];
            if (hg.edges.size() > 0xffffu) throw Error("init_state: layer graph too large for the strand kernel");
            DevStrandGraph g{};
            g.per_layer = models[k]->per_layer;
            g.layers = models[k]->layers;
            g.n_edges = uint32_t(hg.edges.size());
            if (hg.edges.empty()) hg.edges.push_back(make_uint4(0, 0, 0, 0));
            g.pos = keep(hg.pos)->as<uint4>();
            g.band_pm = keep(hg.band_pm)->as<uint4>();
            g.tau = keep(hg.tau)->as<uint4>();
            g.chunks = keep(hg.chunks)->as<uint4>();
            g.inslots = keep(hg.inslots)->as<uint4>();
            g.edges = keep(hg.edges)->as<uint4>();
            graphs.push_back(g);
        }
        cuda_check(cudaStreamSynchronize(stream_), "upload strand graphs");  // strand_host dies with this block
        upload(strand_graphs_, graphs, device_bytes_, stream_);
        cuda_check(cudaStreamSynchronize(stream_), "upload strand graphs");
        dev_.strand_graphs = strand_graphs_.as<DevStrandGraph>();
        // one model: its graph is staged in every CTA's shared memory, next to the strands' landing stages
        // and cell rows, when the launcher finds room (launch_sweep_strand)
        // (several models: only when every CTA hosts warps of one tile — small batches, see launch_sweep_strand)
        dev_.strand_graph_smem = 0;
        for (const DevStrandGraph& g : graphs) {
            dev_.strand_graph_smem = std::max(dev_.strand_graph_smem, uint32_t(strand_graph_bytes(g.per_layer, g.n_edges)));
        }
        dev_.strand_single_model = graphs.size() == 1 ? 1u : 0u;
        // How many layers of a tile are swept at once.  Every strand and producer of a round must be
        // resident, sm_count * warps of them; more strands hide more latency, fewer keep the tape ring
        // (S * per_layer rows per tile) small.  ISING_B200_STRANDS / ISING_B200_STRAND_WARPS override.
        const uint32_t tiles = uint32_t(tile_first.size());
        strand_warps_ = env_u32("ISING_B200_STRAND_WARPS");
        if (strand_warps_ == 0 || strand_warps_ > strand_max_warps()) strand_warps_ = strand_max_warps();
        const uint32_t capacity = uint32_t(sm_count_) * strand_warps_;
        const uint32_t limit = std::min<uint32_t>({common_layers, 32u, std::max(1u, min_chunks / 2)});
        uint32_t strands = env_u32("ISING_B200_STRANDS");
        if (strands == 0) {
            strands = 1;
            for (uint32_t s = 2; s <= limit; ++s) {
                // (measured on c4, 32 tiles of 512 x 64: 8 strands 2.8e10, 16 strands 4.1e10, 32 strands 4.0e10)
                if (common_layers % s == 0 && uint64_t(tiles) * (s + 1) <= capacity && s <= 16) strands = s;
            }
        }
        if (strands > limit || common_layers % strands != 0 || strands + 1 > capacity) {
            throw Error("init_state: invalid strand count " + std::to_string(strands));
        }
        dev_.strands = strands;
        // a publication costs a device-scope fence (~4000 cycles): as rarely as the wavefront allows — the
        // strands of a tile may trail each other by min_chunks / strands chunks
        dev_.strand_pub = std::max(1u, std::min(16u, min_chunks / (2 * strands)));
        if (env_u32("ISING_B200_STRAND_PUB") != 0) dev_.strand_pub = env_u32("ISING_B200_STRAND_PUB");
        dev_.max_per_layer = max_per_layer;
        dev_.max_layers = 0;
        for (const HostModel* m : models) dev_.max_layers = std::max(dev_.max_layers, m->layers);
        dev_.tape_rows = (strands * max_per_layer + 1024 + 31) / 32 * 32;
        tape_.allocate(size_t(tiles) * dev_.tape_rows * 32 * sizeof(uint32_t), device_bytes_);
        spin_cells_.allocate(std::max<size_t>(1, size_t(tiles) * (n / 8) * 32 * sizeof(uint16_t)), device_bytes_);
        strand_flags_.allocate(size_t(strand_flag_words(tiles, strands)) * sizeof(uint32_t), device_bytes_);
        dev_.tape = tape_.as<uint32_t>();
        spin_nbr_.allocate(std::max<size_t>(1, size_t(tiles) * (n / 8) * 32 * sizeof(uint16_t)), device_bytes_);
        dev_.spin_cells = spin_cells_.as<uint16_t>();
        dev_.spin_nbr = spin_nbr_.as<uint16_t>();
        dev_.strand_flags = strand_flags_.as<uint32_t>();
    }

    const auto t_graphs = std::chrono::steady_clock::now();
    // ---- batch description
    dev_.n_spins = n;
    dev_.n_tiles = uint32_t(tile_first.size());
    dev_.n_chains = uint32_t(chains64);
    dev_.n_ladders = cfg.n_ladders;
    dev_.n_betas = cfg.n_betas;
    dev_.tau_scale = cfg.tau_scale;
    dev_.exp_kind = cfg.exp_kind;
    upload(tile_first_, tile_first, device_bytes_, stream_);
    upload(tile_count_, tile_count, device_bytes_, stream_);
    upload(tile_model_, tile_model, device_bytes_, stream_);
    upload(chain_loc_, chain_loc, device_bytes_, stream_);
    upload(seeds_, cfg.seeds, device_bytes_, stream_);
    upload(betas_, cfg.betas, device_bytes_, stream_);
    upload(swap_seeds_, cfg.swap_seeds, device_bytes_, stream_);
    dev_.models = models_.as<DevModel>();
    dev_.tile_first = tile_first_.as<uint32_t>();
    dev_.tile_count = tile_count_.as<uint32_t>();
    dev_.tile_model = tile_model_.as<uint32_t>();
    dev_.chain_loc = chain_loc_.as<uint32_t>();
    dev_.seeds = seeds_.as<uint32_t>();
    dev_.betas = betas_.as<float>();
    dev_.swap_seeds = swap_seeds_.as<uint32_t>();

    const size_t tiles = dev_.n_tiles, chains = dev_.n_chains, ladders = dev_.n_ladders;
    const size_t field_elems = std::max<size_t>(1, tiles * n * 32);
    slot_of_chain_.allocate(chains * sizeof(uint32_t), device_bytes_);
    chain_at_slot_.allocate(chains * sizeof(uint32_t), device_bytes_);
    hs_.allocate(field_elems * sizeof(float), device_bytes_);
    if (any_tau) ht_.allocate(field_elems * sizeof(float), device_bytes_);
    spin_bits_.allocate(std::max<size_t>(1, tiles * n) * sizeof(uint32_t), device_bytes_);
    mt_.allocate(tiles * kMtWords * 32 * sizeof(uint32_t), device_bytes_);
    mt_pos_.allocate(tiles * sizeof(uint32_t), device_bytes_);
    e_run_.allocate(chains * sizeof(double), device_bytes_);
    flips_.allocate(chains * sizeof(unsigned long long), device_bytes_);
    swap_mt_.allocate(ladders * kMtWords * sizeof(uint32_t), device_bytes_);
    swap_pos_.allocate(ladders * sizeof(uint32_t), device_bytes_);
    swap_acc_.allocate(chains * sizeof(unsigned long long), device_bytes_);
    swap_att_.allocate(chains * sizeof(unsigned long long), device_bytes_);
    dev_.slot_of_chain = slot_of_chain_.as<uint32_t>();
    dev_.chain_at_slot = chain_at_slot_.as<uint32_t>();
    dev_.hs = hs_.as<float>();
    dev_.ht = any_tau ? ht_.as<float>() : nullptr;
    dev_.spin_bits = spin_bits_.as<uint32_t>();
    dev_.mt = mt_.as<uint32_t>();
    dev_.mt_pos = mt_pos_.as<uint32_t>();
    dev_.e_run = e_run_.as<double>();
    dev_.flips = flips_.as<unsigned long long>();
    dev_.swap_mt = swap_mt_.as<uint32_t>();
    dev_.swap_pos = swap_pos_.as<uint32_t>();
    dev_.swap_acc = swap_acc_.as<unsigned long long>();
    dev_.swap_att = swap_att_.as<unsigned long long>();

    // ---- initial state, on the device
    DeviceBuffer initial_dev;
    size_t ignored = 0;
    if (initial_spins != nullptr) {
        const size_t total = chains * n;
        initial_dev.allocate(std::max<size_t>(1, total), ignored);
        cuda_check(cudaMemcpyAsync(initial_dev.as<void>(), initial_spins, total, cudaMemcpyHostToDevice,
                                   stream_),
                   "upload initial spins");
    }
    const auto t_host = std::chrono::steady_clock::now();
    cuda_check(launch_init(dev_, initial_spins ? initial_dev.as<int8_t>() : nullptr, stream_), "init kernel");
    other_launches += 2;
    cuda_check(cudaStreamSynchronize(stream_), "init");
    if (std::getenv("ISING_B200_TRACE") != nullptr) {  // where batch creation spends its time (profiles/init_time.py)
        const auto t_done = std::chrono::steady_clock::now();
        const auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "ising_batch_create: checks and tiling %.2f ms, model and graph uploads (+ family buffers) %.2f ms, "
                             "state allocation and uploads %.2f ms, init kernels %.2f ms\n",
                     ms(t_begin, t_checked), ms(t_checked, t_graphs), ms(t_graphs, t_host), ms(t_host, t_done));
    }

    // The MT19937 states (2,496 B per chain) are re-read and re-written every 624 attempts while
    // 8 B per attempt of field data stream past them.  Ask for them to persist in L2 so they stop
    // costing HBM traffic; this is a hint, so failure (older driver, MIG, ...) is not an error.
    // The set-aside is a device-wide limit: it is only ever raised here (a smaller batch must not shrink
    // it under a live larger one), and the stream's window goes away with the batch (see ~Batch).  The
    // strand family reads the states once per launch and needs no window.
    if (family_ != KernelFamily::strand) {
        cudaDeviceProp prop{};
        if (cudaGetDeviceProperties(&prop, device_) == cudaSuccess && prop.persistingL2CacheMaxSize > 0 &&
            prop.accessPolicyMaxWindowSize > 0) {
            const size_t want = std::min<size_t>(mt_.bytes(), size_t(prop.persistingL2CacheMaxSize));
            const size_t window = std::min<size_t>(mt_.bytes(), size_t(prop.accessPolicyMaxWindowSize));
            size_t have = 0;
            if (cudaDeviceGetLimit(&have, cudaLimitPersistingL2CacheSize) != cudaSuccess) have = 0;
            const bool limit_ok = have >= want || cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess;
            if (limit_ok && window > 0) {
                l2_window_set_ = true;
                cudaStreamAttrValue attr{};
                attr.accessPolicyWindow.base_ptr = mt_.as<void>();
                attr.accessPolicyWindow.num_bytes = window;
                attr.accessPolicyWindow.hitRatio = float(std::min(1.0, double(want) / double(window)));
                attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                cudaStreamSetAttribute(stream_, cudaStreamAttributeAccessPolicyWindow, &attr);
            }
        }
        cudaGetLastError();  // a refused hint must not poison later error checks
    }
}

Batch::~Batch() {
    cudaSetDevice(device_);
    if (stream_ != nullptr) cudaStreamSynchronize(stream_);
    if (l2_window_set_ && stream_ != nullptr) {
        // drop the access-policy window and let the lines it pinned go back to normal use
        cudaStreamAttrValue attr{};
        attr.accessPolicyWindow.num_bytes = 0;
        cudaStreamSetAttribute(stream_, cudaStreamAttributeAccessPolicyWindow, &attr);
        cudaCtxResetPersistingL2Cache();
        cudaGetLastError();
    }
    release_cuda_objects();
}

void Batch::begin_timed(bool is_swap) {
    if (!timing_) return;
    TimedLaunch t{};
    t.is_swap = is_swap;
    cuda_check(cudaEventCreate(&t.start), "cudaEventCreate");
    cuda_check(cudaEventCreate(&t.stop), "cudaEventCreate");
    cuda_check(cudaEventRecord(t.start, stream_), "cudaEventRecord");
    pending_.push_back(t);
}

void Batch::end_timed() {
    if (!timing_) return;
    cuda_check(cudaEventRecord(pending_.back().stop, stream_), "cudaEventRecord");
}

void Batch::drain_timings() {
    for (TimedLaunch& t : pending_) {
        float ms = 0.0f;
        cuda_check(cudaEventSynchronize(t.stop), "cudaEventSynchronize");
        cuda_check(cudaEventElapsedTime(&ms, t.start, t.stop), "cudaEventElapsedTime");
        (t.is_swap ? swap_ms_ : sweep_ms_) += double(ms);
        cudaEventDestroy(t.start);
        cudaEventDestroy(t.stop);
    }
    pending_.clear();
}

void Batch::launch_sweeps(uint32_t sweeps) {
    if (sweeps == 0) return;
    begin_timed(false);
    if (family_ == KernelFamily::strand) {
        // the cells stay authoritative between strand launches (settle() restores the canonical state)
        dev_.strand_epoch = uint32_t(sweeps_done_ & 0xffu);
        cuda_check(launch_sweep_strand(dev_, sweeps, sm_count_, strand_warps_, !strand_live_, stream_),
                   "strand sweep kernel");
        if (!strand_live_) ++other_launches;  // spin words -> cells
        strand_live_ = true;
    } else if (family_ == KernelFamily::layered) {
        cuda_check(launch_sweep_layered(dev_, sweeps, sm_count_, stream_), "layered sweep kernel");
    } else {
        cuda_check(launch_sweep_generic(dev_, sweeps, stream_), "sweep kernel");
    }
    end_timed();
    ++sweep_launches;
    sweeps_done_ += sweeps;
}

void Batch::settle() {
    if (!strand_live_) return;
    cuda_check(launch_strand_settle(dev_, stream_), "strand settle kernels");
    other_launches += 2;  // pending far updates into the fields, cells -> spin words
    strand_live_ = false;
}

void Batch::launch_swap_round() {
    begin_timed(true);
    cuda_check(launch_swap(dev_, swap_rounds_, stream_), "swap kernel");
    end_timed();
    ++swap_launches;
    ++swap_rounds_;
}

void Batch::run(uint64_t sweeps, uint32_t swap_interval) {
    bind_device();
    cuda_check(cudaEventRecord(run_start_, stream_), "cudaEventRecord");
    const bool swapping = swap_interval != 0 && dev_.n_betas > 1;
    uint64_t left = sweeps;
    while (left > 0) {
        uint64_t step = left;
        if (swapping) step = std::min<uint64_t>(left, swap_interval - sweeps_done_ % swap_interval);
        // the kernels count a launch's flips in 32 bits: keep sweeps * n_spins below 2^32
        step = std::min<uint64_t>(step, std::max<uint64_t>(1, 0xFFFFFFFFull / std::max<uint32_t>(1, dev_.n_spins)));
        step = std::min<uint64_t>(step, 1u << 20);
        // the strand family indexes a launch's draws (sweeps * n_spins + 624 tape rows) in 32 bits
        if (family_ == KernelFamily::strand) {
            step = std::min<uint64_t>(step, std::max<uint64_t>(1, 0x7FFFFFFFull / std::max<uint32_t>(1, dev_.n_spins)));
        }
        launch_sweeps(uint32_t(step));
        left -= step;
        if (swapping && sweeps_done_ % swap_interval == 0) launch_swap_round();
    }
    cuda_check(cudaEventRecord(run_stop_, stream_), "cudaEventRecord");
    run_timed_ = true;
}

void Batch::swap_round() {
    bind_device();
    if (dev_.n_betas > 1) launch_swap_round();
}

void Batch::sync() {
    bind_device();
    cuda_check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
    drain_timings();
}

double Batch::sweep_ms() {
    sync();
    return sweep_ms_;
}
double Batch::swap_ms() {
    sync();
    return swap_ms_;
}
double Batch::last_run_ms() {
    sync();
    if (!run_timed_) return 0.0;
    float ms = 0.0f;
    cuda_check(cudaEventElapsedTime(&ms, run_start_, run_stop_), "cudaEventElapsedTime");
    return double(ms);
}

// ---- readout -------------------------------------------------------------------------

namespace {
template <typename T>
void download(T* host, const void* dev, size_t count, cudaStream_t stream) {
    if (count == 0) return;
    cuda_check(cudaMemcpyAsync(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost, stream), "download");
    cuda_check(cudaStreamSynchronize(stream), "download");
}
}  // namespace

void Batch::read_spins(uint64_t first_chain, uint64_t n_chains, int8_t* out) {
    bind_device();
    settle();
    if (first_chain > dev_.n_chains || n_chains > dev_.n_chains - first_chain) {
        throw Error("read_spins: chain range out of bounds");
    }
    if (n_chains != 0 && out == nullptr) throw Error("null argument");
    // stage through a bounded scratch buffer so that huge batches do not double their footprint
    const size_t n = dev_.n_spins;
    const uint64_t per_pass = std::max<uint64_t>(1, (256ull << 20) / std::max<size_t>(1, n));
    size_t ignored = 0;
    for (uint64_t done = 0; done < n_chains; done += per_pass) {
        const uint64_t cnt = std::min<uint64_t>(per_pass, n_chains - done);
        if (scratch_.bytes() < cnt * n) scratch_.allocate(cnt * n, ignored);
        cuda_check(launch_unpack_spins(dev_, uint32_t(first_chain + done), uint32_t(cnt),
                                       scratch_.as<int8_t>(), stream_),
                   "unpack kernel");
        ++other_launches;
        download(out + done * n, scratch_.as<void>(), cnt * n, stream_);
    }
}

void Batch::read_fields(uint64_t chain, float* hs, float* ht) {
    bind_device();
    settle();
    if (chain >= dev_.n_chains) throw Error("read_fields: chain out of range");
    if (hs == nullptr || ht == nullptr) throw Error("null argument");
    const size_t n = dev_.n_spins;
    size_t ignored = 0;
    if (scratch_.bytes() < 2 * n * sizeof(float)) scratch_.allocate(2 * n * sizeof(float), ignored);
    float* d = scratch_.as<float>();
    cuda_check(launch_gather_fields(dev_, uint32_t(chain), d, d + n, stream_), "gather kernel");
    ++other_launches;
    download(hs, d, n, stream_);
    download(ht, d + n, n, stream_);
}

void Batch::read_energies(double* out) {
    bind_device();
    settle();
    if (out == nullptr) throw Error("null argument");
    size_t ignored = 0;
    if (scratch_.bytes() < dev_.n_chains * sizeof(double)) scratch_.allocate(dev_.n_chains * sizeof(double), ignored);
    cuda_check(launch_energies(dev_, scratch_.as<double>(), stream_), "energy kernel");
    ++other_launches;
    download(out, scratch_.as<void>(), dev_.n_chains, stream_);
}

void Batch::resync_energies() {
    bind_device();
    settle();
    cuda_check(launch_resync_energies(dev_, stream_), "energy resync kernel");
    ++other_launches;
}

void Batch::read_running_energies(double* out) {
    bind_device();
    if (out == nullptr) throw Error("null argument");
    download(out, dev_.e_run, dev_.n_chains, stream_);
}

void Batch::read_stats(uint64_t* flips, uint64_t* attempts) {
    bind_device();
    if (flips != nullptr) download(flips, dev_.flips, dev_.n_chains, stream_);
    else sync();
    if (attempts != nullptr) {
        for (uint32_t c = 0; c < dev_.n_chains; ++c) attempts[c] = sweeps_done_ * dev_.n_spins;
    }
}

void Batch::record_wait(bool on) {
    bind_device();
    sync();
    if (!on) {
        dev_.wait_counts = nullptr;  // counters stay readable until recording is switched on again
        return;
    }
    const size_t bytes = size_t(dev_.n_tiles) * kWaitSlots * sizeof(unsigned long long);
    if (wait_counts_.bytes() < bytes) wait_counts_.allocate(bytes, device_bytes_);
    cuda_check(cudaMemsetAsync(wait_counts_.as<void>(), 0, bytes, stream_), "cudaMemsetAsync");
    dev_.wait_counts = wait_counts_.as<unsigned long long>();
}

void Batch::read_wait(uint32_t n_widths, const uint32_t* widths, uint64_t* groups, uint64_t* with_flip) {
    bind_device();
    if (n_widths != 0 && (widths == nullptr || groups == nullptr || with_flip == nullptr)) throw Error("null argument");
    if (wait_counts_.bytes() == 0) throw Error("collect_wait_stats: wait statistics were not recorded");
    std::vector<unsigned long long> host(size_t(dev_.n_tiles) * kWaitSlots);
    download(host.data(), wait_counts_.as<void>(), host.size(), stream_);
    unsigned long long total[kWaitSlots] = {};
    for (uint32_t t = 0; t < dev_.n_tiles; ++t) {
        for (uint32_t k = 0; k < kWaitSlots; ++k) total[k] += host[size_t(t) * kWaitSlots + k];
    }
    for (uint32_t i = 0; i < n_widths; ++i) {
        uint32_t slot = 0;
        while (slot < 6 && (1u << slot) != widths[i]) ++slot;
        if (slot == 6) {  // ref: collect_wait_stats throws for widths that were not recorded
            throw Error("collect_wait_stats: width " + std::to_string(widths[i]) + " was not recorded");
        }
        groups[i] = total[6] * (32u >> slot);  // attempts per lane x groups of that width in a tile
        with_flip[i] = total[slot];
    }
}

void Batch::read_checksums(uint64_t* out) {
    bind_device();
    settle();
    if (out == nullptr) throw Error("null argument");
    size_t ignored = 0;
    if (scratch_.bytes() < dev_.n_chains * sizeof(uint64_t)) scratch_.allocate(dev_.n_chains * sizeof(uint64_t), ignored);
    cuda_check(launch_checksums(dev_, scratch_.as<unsigned long long>(), stream_), "checksum kernel");
    ++other_launches;
    download(out, scratch_.as<void>(), dev_.n_chains, stream_);
}

void Batch::read_coherence(uint64_t* out) {
    bind_device();
    settle();
    if (out == nullptr) throw Error("null argument");
    size_t ignored = 0;
    if (scratch_.bytes() < dev_.n_chains * sizeof(uint64_t)) scratch_.allocate(dev_.n_chains * sizeof(uint64_t), ignored);
    cuda_check(launch_coherence(dev_, scratch_.as<unsigned long long>(), stream_), "coherence kernel");
    ++other_launches;
    download(out, scratch_.as<void>(), dev_.n_chains, stream_);
}

void Batch::read_slots(uint32_t* out) {
    bind_device();
    if (out == nullptr) throw Error("null argument");
    download(out, dev_.slot_of_chain, dev_.n_chains, stream_);
}

void Batch::read_swap_stats(uint64_t* acc, uint64_t* att) {
    bind_device();
    if (acc != nullptr) download(acc, dev_.swap_acc, dev_.n_chains, stream_);
    if (att != nullptr) download(att, dev_.swap_att, dev_.n_chains, stream_);
}

void Batch::pack_results(void* device_out) {
    bind_device();
    settle();
    if (device_out == nullptr) throw Error("null argument");
    cuda_check(launch_pack_results(dev_, device_out, stream_), "pack kernel");
    ++other_launches;
    cuda_check(cudaStreamSynchronize(stream_), "pack");
}

}  // namespace isingb200

namespace isingb200 {

// NCCL, found at run time: the copy the process has loaded already (the caller's communicator belongs
// to it), else the system's.  ncclAllGather(send, recv, count, datatype, comm, stream); ncclInt64 == 4.
void Batch::all_gather_results(void* nccl_comm, void* device_out_all) {
    bind_device();
    if (nccl_comm == nullptr || device_out_all == nullptr) throw Error("null argument");
    using AllGather = int (*)(const void*, void*, size_t, int, void*, cudaStream_t);
    using ErrorString = const char* (*)(int);
    static void* handle = nullptr;
    static AllGather all_gather = nullptr;
    static ErrorString error_string = nullptr;
    if (all_gather == nullptr) {
        handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (handle == nullptr) handle = dlopen("libnccl.so.2", RTLD_NOW);
        if (handle == nullptr) handle = dlopen("libnccl.so", RTLD_NOW);
        if (handle == nullptr) throw CudaError("NCCL not found (libnccl.so.2): " + std::string(dlerror() ? dlerror() : ""));
        all_gather = reinterpret_cast<AllGather>(dlsym(handle, "ncclAllGather"));
        error_string = reinterpret_cast<ErrorString>(dlsym(handle, "ncclGetErrorString"));
        if (all_gather == nullptr) throw CudaError("NCCL has no ncclAllGather");
    }
    const size_t bytes = size_t(dev_.n_chains) * 32;
    size_t ignored = 0;
    if (gather_send_.bytes() < bytes) gather_send_.allocate(std::max<size_t>(bytes, 32), ignored);
    settle();
    cuda_check(launch_pack_results(dev_, gather_send_.as<void>(), stream_), "pack kernel");
    ++other_launches;
    const int rc = all_gather(gather_send_.as<void>(), device_out_all, size_t(dev_.n_chains) * 4, /*ncclInt64*/ 4, nccl_comm,
                              stream_);
    if (rc != 0) throw CudaError(std::string("ncclAllGather: ") + (error_string ? error_string(rc) : "error"));
    cuda_check(cudaStreamSynchronize(stream_), "all-gather");
}

}  // namespace isingb200
