#include "coalesced.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>

namespace isingb200 {

namespace {

template <typename T>
void upload_vec(DeviceBuffer& buf, const std::vector<T>& host, size_t& tally, cudaStream_t stream) {
    buf.allocate(std::max<size_t>(1, host.size()) * sizeof(T), tally);
    if (!host.empty()) {
        cuda_check(cudaMemcpyAsync(buf.as<void>(), host.data(), host.size() * sizeof(T), cudaMemcpyHostToDevice,
                                   stream),
                   "upload");
    }
}

template <typename T>
std::vector<T> download_vec(const T* device, size_t count, cudaStream_t stream) {
    std::vector<T> host(count);
    if (count != 0) {
        cuda_check(cudaMemcpyAsync(host.data(), device, count * sizeof(T), cudaMemcpyDeviceToHost, stream), "download");
    }
    cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    return host;
}

}  // namespace

void CoalescedBatch::bind_device() const { cuda_check(cudaSetDevice(device_), "cudaSetDevice"); }

CoalescedBatch::CoalescedBatch(const HostModel& m, const CoalescedConfig& cfg, const int8_t* initial)
    : model_(m) {
    // ---- what the reference checks (prepare_model_for_engine, sweep_state.cpp:292-323;
    // check_engine_model, :120-146)
    if (m.layers == 0) throw Error("prepare_model_for_engine: coalesced needs a layered model");
    if (m.layers % 2 != 0) throw Error("prepare_model_for_engine: coalesced needs an even layer count");
    const uint32_t n = m.n_spins, W = m.layers / 2, P = m.per_layer, L = m.layers;
    if (cfg.betas.empty() || cfg.betas.size() != cfg.seeds.size()) {
        throw Error("init_state: coalesced batch needs one beta and one seed per chain");
    }
    for (float beta : cfg.betas) {
        if (!(beta >= 0.0f) || !std::isfinite(beta)) throw Error("init_state: beta must be finite and >= 0");
    }
    if (!std::isfinite(cfg.tau_scale)) throw Error("init_state: tau_scale must be finite");
    // the kernel applies tau updates as global f32 reductions, which flush subnormals: with every
    // non-zero value at least 2^-100 no field (a sum of multiples of 2^-123) can be subnormal
    const auto tiny = [](float v) { return v != 0.0f && std::fabs(v) < 0x1p-100f; };
    if (std::any_of(m.h.begin(), m.h.end(), tiny) || std::any_of(m.couplings.begin(), m.couplings.end(), tiny)) {
        throw Error("init_state: the coalesced kernel needs non-zero fields and couplings of magnitude >= 2^-100");
    }
    if (cfg.exp_kind < 1 || cfg.exp_kind > 3) throw Error("invalid exp_kind value " + std::to_string(cfg.exp_kind));
    for (uint32_t i = 0; i < n; ++i) {
        const uint32_t l = i / P, pos = i % P, end = m.offsets[i + 1];
        if (m.tau_counts[i] != 2) throw Error("init_state: coalesced model needs 2 tau edges per spin");
        if (m.targets[end - 2] != ((l + 1) % L) * P + pos || m.targets[end - 1] != ((l + L - 1) % L) * P + pos) {
            throw Error("init_state: coalesced tau slots out of order at spin " + std::to_string(i));
        }
        for (uint32_t e = m.offsets[i]; e + 2 < end; ++e) {
            if (m.targets[e] / P != l) throw Error("init_state: coalesced model has a space edge leaving its layer");
        }
    }
    // one layer's space graph, if every layer carries the same one (targets and coupling bits)
    std::vector<uint32_t> layer_offsets(size_t(P) + 1, 0);
    std::vector<uint2> layer_edges;
    bool same_layers = true;
    for (uint32_t pos = 0; pos < P; ++pos) {
        layer_offsets[pos] = uint32_t(layer_edges.size());
        for (uint32_t e = m.offsets[pos]; e + 2 < m.offsets[pos + 1]; ++e) {
            uint32_t bits;
            std::memcpy(&bits, &m.couplings[e], sizeof bits);
            layer_edges.push_back(make_uint2(m.targets[e] % P, bits));
        }
    }
    layer_offsets[P] = uint32_t(layer_edges.size());
    for (uint32_t i = P; i < n && same_layers; ++i) {
        const uint32_t pos = i % P, first = layer_offsets[pos], count = layer_offsets[pos + 1] - first;
        same_layers = m.offsets[i + 1] - m.offsets[i] == count + 2;
        for (uint32_t k = 0; k < count && same_layers; ++k) {
            uint32_t bits;
            std::memcpy(&bits, &m.couplings[m.offsets[i] + k], sizeof bits);
            same_layers = m.targets[m.offsets[i] + k] % P == layer_edges[first + k].x && bits == layer_edges[first + k].y;
        }
    }
    if (!same_layers) layer_edges.clear();
    // band / far split of the layer for the register-window variant
    std::vector<uint4> band_pm;
    std::vector<uint32_t> far_offsets;
    std::vector<uint2> far_edges;
    bool windowed = same_layers && P % 8 == 0;
    if (windowed) {
        band_pm.resize(2 * size_t(P));
        far_offsets.assign(size_t(P) + 1, 0);
        for (uint32_t pos = 0; pos < P; ++pos) {
            uint32_t twice[4] = {0, 0, 0, 0}, empty[4] = {0x80000000u, 0x80000000u, 0x80000000u, 0x80000000u};
            far_offsets[pos] = uint32_t(far_edges.size());
            for (uint32_t e = layer_offsets[pos]; e < layer_offsets[pos + 1]; ++e) {
                const uint32_t t = layer_edges[e].x;
                const uint32_t distance = t > pos ? t - pos : pos - t;
                if (distance <= 2) {
                    float j;
                    std::memcpy(&j, &layer_edges[e].y, sizeof j);
                    const float doubled = 2.0f * j;  // exact
                    const int slot = t < pos ? int(t + 2 - pos) : int(t - pos + 1);  // -2,-1,+1,+2 -> 0..3
                    if (empty[slot] == 0) windowed = false;  // a neighbour listed twice: the table holds one
                    std::memcpy(&twice[slot], &doubled, sizeof doubled);
                    empty[slot] = 0;
                    windowed = windowed && std::isfinite(doubled);
                } else {
                    far_edges.push_back(layer_edges[e]);
                }
            }
            for (uint32_t positive = 0; positive < 2; ++positive) {  // a flip of s adds -(2s)*J
                const uint32_t flip = positive ? 0x80000000u : 0u;
                band_pm[2 * size_t(pos) + positive] =
                    make_uint4((twice[0] ^ flip) | empty[0], (twice[1] ^ flip) | empty[1],
                               (twice[2] ^ flip) | empty[2], (twice[3] ^ flip) | empty[3]);
            }
        }
        far_offsets[P] = uint32_t(far_edges.size());
        if (windowed && coalesced_window_smem_bytes(W, P, uint32_t(far_edges.size())) == 0) windowed = false;
    }
    smem_bytes_ = windowed ? coalesced_window_smem_bytes(W, P, uint32_t(far_edges.size()))
                           : coalesced_smem_bytes(W, P, uint32_t(layer_edges.size()));
    if (smem_bytes_ == 0 && same_layers) {  // the graph copy does not fit next to the region: walk the CSR
        same_layers = false;
        layer_edges.clear();
        smem_bytes_ = coalesced_smem_bytes(W, P, 0);
    }
    if (smem_bytes_ == 0) {
        throw Error("init_state: the coalesced kernel needs at most 64 layers and one region (half the spins) "
                    "within 227 KB of shared memory at 5 bytes per spin");
    }

    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        throw CudaError("no CUDA device available (this engine has no CPU fallback)");
    }
    if (cfg.device < 0 || cfg.device >= count) throw Error("invalid device ordinal " + std::to_string(cfg.device));
    device_ = cfg.device;
    bind_device();
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreate(&start_), "cudaEventCreate");
    cuda_check(cudaEventCreate(&stop_), "cudaEventCreate");

    // ---- coalesce_permutation + apply_permutation (model.cpp:190-245)
    forward_.resize(n);
    std::vector<uint32_t> inverse(n);
    for (uint32_t l = 0; l < L; ++l) {
        for (uint32_t p = 0; p < P; ++p) {
            const uint32_t fresh = W * ((l % 2) * P + p) + l / 2;
            forward_[l * P + p] = fresh;
            inverse[fresh] = l * P + p;
        }
    }
    std::vector<uint32_t> offsets(size_t(n) + 1), targets(m.targets.size());
    std::vector<float> couplings(m.couplings.size()), h(n);
    uint32_t at = 0;
    for (uint32_t fresh = 0; fresh < n; ++fresh) {
        const uint32_t old = inverse[fresh];
        h[fresh] = m.h[old];
        offsets[fresh] = at;
        for (uint32_t e = m.offsets[old]; e < m.offsets[old + 1]; ++e, ++at) {
            targets[at] = forward_[m.targets[e]];
            couplings[at] = m.couplings[e];
        }
    }
    offsets[n] = at;
    std::vector<float> tau_up(n), tau_down(n);
    for (uint32_t i = 0; i < n; ++i) {
        tau_up[i] = couplings[offsets[i + 1] - 2];
        tau_down[i] = couplings[offsets[i + 1] - 1];
    }

    // ---- init_state on the permuted model, per chain (sweep_state.cpp:160-234)
    const size_t chains = cfg.betas.size();
    std::vector<int8_t> spins(chains * n);
    std::vector<float> hs(chains * n), ht(chains * n);
    std::vector<uint32_t> mt(chains * size_t(kMtWords) * W), mt_pos(chains, 0);
    for (size_t c = 0; c < chains; ++c) {
        int8_t* sp = spins.data() + c * n;
        if (initial != nullptr) {
            for (uint32_t old = 0; old < n; ++old) {
                const int8_t v = initial[c * n + old];
                if (v != 1 && v != -1) throw Error("init_state: spins must be +/-1");
                sp[forward_[old]] = v;
            }
        } else {  // initial_spins(n, seed): bit 31 of each draw of Mt19937(seed ^ 0x9E3779B9), new index order
            std::mt19937 init_rng(cfg.seeds[c] ^ 0x9E3779B9u);
            for (uint32_t i = 0; i < n; ++i) sp[i] = (init_rng() >> 31) ? -1 : 1;
        }
        // recompute_fields (sweep_state.cpp:236-255): f32, adjacency order, h_i first
        float* fs = hs.data() + c * n;
        float* ft = ht.data() + c * n;
        for (uint32_t i = 0; i < n; ++i) {
            float acc_s = h[i], acc_t = 0.0f;
            const uint32_t end = offsets[i + 1];
            for (uint32_t e = offsets[i]; e + 2 < end; ++e) acc_s += couplings[e] * float(sp[targets[e]]);
            for (uint32_t e = end - 2; e < end; ++e) acc_t += couplings[e] * float(sp[targets[e]]);
            fs[i] = acc_s;
            ft[i] = acc_t;
        }
        // InterlacedMt::with_base_seed(seed, W): word w of lane k at [w*W + k] (rng.cpp:128-148)
        uint32_t* state = mt.data() + c * size_t(kMtWords) * W;
        for (uint32_t k = 0; k < W; ++k) {
            uint32_t prev = cfg.seeds[c] + k;
            state[k] = prev;
            for (uint32_t w = 1; w < kMtWords; ++w) {
                prev = 1812433253u * (prev ^ (prev >> 30)) + w;
                state[size_t(w) * W + k] = prev;
            }
        }
    }

    upload_vec(offsets_, offsets, device_bytes_, stream_);
    upload_vec(targets_, targets, device_bytes_, stream_);
    upload_vec(couplings_, couplings, device_bytes_, stream_);
    upload_vec(tau_up_, tau_up, device_bytes_, stream_);
    upload_vec(tau_down_, tau_down, device_bytes_, stream_);
    upload_vec(layer_offsets_, layer_offsets, device_bytes_, stream_);
    upload_vec(layer_edges_, layer_edges, device_bytes_, stream_);
    upload_vec(band_pm_, band_pm, device_bytes_, stream_);
    upload_vec(far_offsets_, far_offsets, device_bytes_, stream_);
    upload_vec(far_edges_, far_edges, device_bytes_, stream_);
    upload_vec(hs_, hs, device_bytes_, stream_);
    upload_vec(ht_, ht, device_bytes_, stream_);
    upload_vec(spins_, spins, device_bytes_, stream_);
    upload_vec(mt_, mt, device_bytes_, stream_);
    upload_vec(mt_pos_, mt_pos, device_bytes_, stream_);
    upload_vec(betas_, cfg.betas, device_bytes_, stream_);
    upload_vec(flips_, std::vector<unsigned long long>(chains, 0ull), device_bytes_, stream_);
    cuda_check(cudaStreamSynchronize(stream_), "upload");  // the host vectors die here

    dev_.n_spins = n;
    dev_.lanes = W;
    dev_.per_layer = P;
    dev_.n_chains = uint32_t(chains);
    dev_.tau_scale = cfg.tau_scale;
    dev_.exp_kind = cfg.exp_kind;
    dev_.offsets = offsets_.as<uint32_t>();
    dev_.targets = targets_.as<uint32_t>();
    dev_.couplings = couplings_.as<float>();
    dev_.tau_up = tau_up_.as<float>();
    dev_.tau_down = tau_down_.as<float>();
    dev_.layer_offsets = same_layers ? layer_offsets_.as<uint32_t>() : nullptr;
    dev_.layer_edges = same_layers ? layer_edges_.as<uint2>() : nullptr;
    dev_.n_layer_edges = uint32_t(layer_edges.size());
    dev_.band_pm = windowed ? band_pm_.as<uint4>() : nullptr;
    dev_.far_offsets = far_offsets_.as<uint32_t>();
    dev_.far_edges = far_edges_.as<uint2>();
    dev_.n_far_edges = uint32_t(far_edges.size());
    dev_.hs = hs_.as<float>();
    dev_.ht = ht_.as<float>();
    dev_.spins = spins_.as<int8_t>();
    dev_.mt = mt_.as<uint32_t>();
    dev_.mt_pos = mt_pos_.as<uint32_t>();
    dev_.betas = betas_.as<float>();
    dev_.flips = flips_.as<unsigned long long>();
    cuda_check(prepare_coalesced_kernels(smem_bytes_), "cudaFuncSetAttribute");
}

CoalescedBatch::~CoalescedBatch() {
    if (stream_ != nullptr) {
        cudaSetDevice(device_);
        cudaStreamSynchronize(stream_);
        cudaEventDestroy(start_);
        cudaEventDestroy(stop_);
        cudaStreamDestroy(stream_);
    }
}

void CoalescedBatch::run(uint64_t sweeps) {
    bind_device();
    cuda_check(cudaEventRecord(start_, stream_), "cudaEventRecord");
    uint64_t left = sweeps;
    while (left != 0) {  // a launch's per-chain flip counter is 64-bit; bound the launch length anyway
        const uint32_t part = uint32_t(std::min<uint64_t>(left, 1u << 20));
        cuda_check(launch_sweep_coalesced(dev_, part, smem_bytes_, stream_), "coalesced sweep kernel");
        ++launches;
        left -= part;
    }
    cuda_check(cudaEventRecord(stop_, stream_), "cudaEventRecord");
    timed_ = true;
    sweeps_done_ += sweeps;
}

void CoalescedBatch::sync() {
    bind_device();
    cuda_check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
}

double CoalescedBatch::last_run_ms() {
    if (!timed_) return 0.0;
    sync();
    float ms = 0.0f;
    cuda_check(cudaEventElapsedTime(&ms, start_, stop_), "cudaEventElapsedTime");
    return double(ms);
}

void CoalescedBatch::read_spins(uint64_t chain, int8_t* out) {
    bind_device();
    if (out == nullptr) throw Error("null argument");
    if (chain >= dev_.n_chains) throw Error("chain index out of range");
    const std::vector<int8_t> fresh = download_vec(dev_.spins + chain * dev_.n_spins, dev_.n_spins, stream_);
    for (uint32_t old = 0; old < dev_.n_spins; ++old) out[old] = fresh[forward_[old]];
}

void CoalescedBatch::read_fields(uint64_t chain, float* hs, float* ht) {
    bind_device();
    if (hs == nullptr || ht == nullptr) throw Error("null argument");
    if (chain >= dev_.n_chains) throw Error("chain index out of range");
    const std::vector<float> fs = download_vec(dev_.hs + chain * dev_.n_spins, dev_.n_spins, stream_);
    const std::vector<float> ft = download_vec(dev_.ht + chain * dev_.n_spins, dev_.n_spins, stream_);
    for (uint32_t old = 0; old < dev_.n_spins; ++old) {
        hs[old] = fs[forward_[old]];
        ht[old] = ft[forward_[old]];
    }
}

void CoalescedBatch::read_stats(uint64_t* flips, uint64_t* attempts) {
    bind_device();
    if (flips != nullptr) {
        const auto host = download_vec(dev_.flips, dev_.n_chains, stream_);
        for (uint32_t c = 0; c < dev_.n_chains; ++c) flips[c] = host[c];
    } else {
        sync();
    }
    if (attempts != nullptr) {
        for (uint32_t c = 0; c < dev_.n_chains; ++c) attempts[c] = sweeps_done_ * dev_.n_spins;
    }
}

void CoalescedBatch::read_energies(double* out) {
    if (out == nullptr) throw Error("null argument");
    std::vector<int8_t> spins(dev_.n_spins);
    for (uint32_t c = 0; c < dev_.n_chains; ++c) {
        read_spins(c, spins.data());
        out[c] = total_cost(model_, spins.data(), dev_.n_spins);
    }
}

void CoalescedBatch::read_checksums(uint64_t* out) {
    if (out == nullptr) throw Error("null argument");
    std::vector<int8_t> spins(dev_.n_spins);
    for (uint32_t c = 0; c < dev_.n_chains; ++c) {
        read_spins(c, spins.data());
        uint64_t hash = 1469598103934665603ull;  // FNV-1a over the sign bits, original order
        for (uint32_t i = 0; i < dev_.n_spins; ++i) {
            hash ^= uint64_t(spins[i] > 0 ? 1 : 0);
            hash *= 1099511628211ull;
        }
        out[c] = hash;
    }
}

}  // namespace isingb200
