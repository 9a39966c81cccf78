// The INTRA-SYSTEM ("coalesced") schedule on the device: one warp per chain,
// lane t owns layers 2t and 2t+1 of a layered model with L = 2W <= 64 layers, and the W lanes
// attempt W spins of ONE chain in lockstep.  It is the regime of few chains and large systems,
// where the replica-parallel families (lane = chain) cannot fill the machine.  Semantics are the
// reference's `coalesced` engine bit for bit (ref: proj/src/sweep_coalesced.cpp:10-124): spin
// (l, p) lives at new index W*((l%2)*P + p) + l/2 (ref: coalesce_permutation, model.cpp:190-215),
// a sweep is even flips (space edges + tau edge to the previous layer), deferred tau edges to the
// next layer, odd flips, deferred; lane t draws from Mt19937(seed + t) (ref: sweep_state.cpp:193-199).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include <cuda_runtime.h>

#include "batch.hpp"
#include "host_model.hpp"

namespace isingb200 {

struct CoalescedDev {
    uint32_t n_spins, lanes, per_layer, n_chains;
    float tau_scale;
    int exp_kind;
    // permuted model (shared by all chains): CSR in the new index order
    const uint32_t* offsets;
    const uint32_t* targets;
    const float* couplings;
    // the two tau couplings of every spin (new index order): next layer, previous layer
    const float* tau_up;
    const float* tau_down;
    // one layer's space graph when all layers carry the same one (else nullptr: the kernel walks the CSR):
    // edges of position p are layer_edges[layer_offsets[p] .. layer_offsets[p+1]) = {position, bits of J}
    const uint32_t* layer_offsets;  // per_layer + 1
    const uint2* layer_edges;
    uint32_t n_layer_edges;
    // the same layer split for the REGISTER WINDOW variant (per_layer % 8 == 0): what a flip adds to the
    // fields at p-2, p-1, p+1, p+2 (two entries per position, by the sign of the flipped spin: 2p for
    // s = -1, 2p+1 for s = +1; an empty slot holds -0.0), and the remaining ("far") edges as a CSR list
    const uint4* band_pm;           // 2 * per_layer, or nullptr
    const uint32_t* far_offsets;    // per_layer + 1
    const uint2* far_edges;
    uint32_t n_far_edges;
    // per chain, new index order
    float* hs;        // [chain][n]
    float* ht;        // [chain][n]
    int8_t* spins;    // [chain][n]
    uint32_t* mt;     // [chain][624][lanes]  (the reference's InterlacedMt layout, rng.hpp:51-53)
    uint32_t* mt_pos; // [chain]
    const float* betas;             // [chain]
    unsigned long long* flips;      // [chain]
};

size_t coalesced_smem_bytes(uint32_t lanes, uint32_t per_layer, uint32_t n_layer_edges);
// the register-window variant: band table + far list next to the region
size_t coalesced_window_smem_bytes(uint32_t lanes, uint32_t per_layer, uint32_t n_far_edges);
cudaError_t prepare_coalesced_kernels(size_t smem_bytes);
cudaError_t launch_sweep_coalesced(const CoalescedDev& d, uint32_t sweeps, size_t smem_bytes, cudaStream_t stream);

struct CoalescedConfig {
    std::vector<float> betas;     // one per chain
    std::vector<uint32_t> seeds;  // one per chain: lane t of chain c draws from Mt19937(seeds[c] + t)
    float tau_scale = 1.0f;
    int exp_kind = 2;
    int device = 0;
};

class CoalescedBatch {
  public:
    // initial_spins: nullptr (initial_spins(n, seed) in the NEW index order, as the reference's
    // init_state on the permuted model does) or [chains][n] of +/-1 in the ORIGINAL spin order
    CoalescedBatch(const HostModel& model, const CoalescedConfig& cfg, const int8_t* initial_spins);
    ~CoalescedBatch();
    CoalescedBatch(const CoalescedBatch&) = delete;
    CoalescedBatch& operator=(const CoalescedBatch&) = delete;

    void run(uint64_t sweeps);
    void sync();
    // readouts, all in the ORIGINAL spin order
    void read_spins(uint64_t chain, int8_t* out);
    void read_fields(uint64_t chain, float* hs, float* ht);
    void read_stats(uint64_t* flips, uint64_t* attempts);
    void read_energies(double* out);     // total_cost of the current spins (host, f64)
    void read_checksums(uint64_t* out);  // ref: state_checksum with the permutation, sweep_state.cpp:325-336

    uint64_t n_chains() const { return dev_.n_chains; }
    uint32_t n_spins() const { return dev_.n_spins; }
    uint32_t lanes() const { return dev_.lanes; }
    uint64_t sweeps_done() const { return sweeps_done_; }
    uint64_t launches = 0;
    double last_run_ms();

  private:
    void bind_device() const;
    const HostModel& model_;
    int device_ = 0;
    cudaStream_t stream_ = nullptr;
    cudaEvent_t start_ = nullptr, stop_ = nullptr;
    bool timed_ = false;
    CoalescedDev dev_{};
    size_t smem_bytes_ = 0, device_bytes_ = 0;
    uint64_t sweeps_done_ = 0;
    std::vector<uint32_t> forward_;  // old index -> new index
    DeviceBuffer offsets_, targets_, couplings_, tau_up_, tau_down_, layer_offsets_, layer_edges_;
    DeviceBuffer band_pm_, far_offsets_, far_edges_;
    DeviceBuffer hs_, ht_, spins_, mt_, mt_pos_, betas_, flips_;
};

}  // namespace isingb200
