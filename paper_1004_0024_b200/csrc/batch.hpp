// Host-side batch object: owns the device state of many chains and drives the kernels.
// This is the device-backed counterpart of the reference's SweepState + run_sweeps loop
// (ref: proj/include/isingmc/sweep.hpp:85-157, proj/src/sweep_state.cpp:160-291), one object
// for ALL chains instead of one SweepState per chain.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "device_batch.hpp"
#include "host_model.hpp"

namespace isingb200 {

struct CudaError : std::runtime_error {  // maps to ISING_ERR_INTERNAL at the C boundary
    using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t status, const char* what);

// Plain device allocation with RAII; tracks bytes for the batch's footprint report.
class DeviceBuffer {
  public:
    DeviceBuffer() = default;
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    ~DeviceBuffer();
    void allocate(size_t bytes, size_t& tally);
    template <typename T>
    T* as() const { return static_cast<T*>(ptr_); }
    size_t bytes() const { return bytes_; }

  private:
    void* ptr_ = nullptr;
    size_t bytes_ = 0;
};

enum class KernelFamily : int { generic = 1, layered = 2, strand = 3 };

struct BatchConfig {
    uint32_t n_ladders = 0;
    uint32_t n_betas = 1;
    std::vector<float> betas;
    std::vector<uint32_t> seeds;       // n_chains
    std::vector<uint32_t> swap_seeds;  // n_ladders
    float tau_scale = 1.0f;
    int exp_kind = 2;  // ising_exp_kind: fast
    int device = 0;
    int kernel = 0;  // 0 auto, 1 generic, 2 layered, 3 strand
};

class Batch {
  public:
    Batch(const std::vector<const HostModel*>& models, const std::vector<uint32_t>& model_of_ladder,
          const BatchConfig& cfg, const int8_t* initial_spins);
    ~Batch();
    Batch(const Batch&) = delete;
    Batch& operator=(const Batch&) = delete;

    void run(uint64_t sweeps, uint32_t swap_interval);
    void swap_round();
    void sync();

    void read_spins(uint64_t first_chain, uint64_t n_chains, int8_t* out);
    void read_fields(uint64_t chain, float* hs, float* ht);
    void read_energies(double* out);
    void read_running_energies(double* out);
    void resync_energies();
    void read_stats(uint64_t* flips, uint64_t* attempts);
    void read_checksums(uint64_t* out);
    void read_coherence(uint64_t* out);
    void read_slots(uint32_t* out);
    void read_swap_stats(uint64_t* acc, uint64_t* att);
    void pack_results(void* device_out);
    void all_gather_results(void* nccl_comm, void* device_out_all);

    void set_timing(bool on) { timing_ = on; }
    // wait statistics (ref: FlipStats::group_wait): recording starts (counters zeroed) or stops
    void record_wait(bool on);
    // per requested width (1, 2, 4, 8, 16 or 32): groups seen, groups with at least one flip
    void read_wait(uint32_t n_widths, const uint32_t* widths, uint64_t* groups, uint64_t* with_flip);
    cudaStream_t stream() const { return stream_; }

    // introspection
    uint64_t n_chains() const { return dev_.n_chains; }
    uint32_t n_spins() const { return dev_.n_spins; }
    uint32_t n_tiles() const { return dev_.n_tiles; }
    KernelFamily family() const { return family_; }
    // generic family: 0 read-modify-write, 1 reductions, 2 reductions + own-field window in every model
    uint32_t generic_variant() const { return generic_variant_; }
    // strand family: concurrent layers per tile and warps per persistent CTA (0 for the other families)
    uint32_t strands() const { return dev_.strands; }
    uint32_t strand_warps() const { return strand_warps_; }
    uint64_t sweeps_done() const { return sweeps_done_; }
    uint64_t device_bytes() const { return device_bytes_; }
    uint64_t sweep_launches = 0, swap_launches = 0, other_launches = 0;
    double sweep_ms();
    double swap_ms();
    double last_run_ms();

  private:
    struct TimedLaunch {
        cudaEvent_t start, stop;
        bool is_swap;
    };
    void construct(const std::vector<const HostModel*>& models, const std::vector<uint32_t>& model_of_ladder,
                   const BatchConfig& cfg, const int8_t* initial_spins);
    void release_cuda_objects();
    void bind_device() const;
    void launch_sweeps(uint32_t sweeps);
    void launch_swap_round();
    void begin_timed(bool is_swap);
    void end_timed();
    void drain_timings();

    int device_ = 0;
    cudaStream_t stream_ = nullptr;
    KernelFamily family_ = KernelFamily::generic;
    uint32_t generic_variant_ = 0;
    DevBatch dev_{};
    size_t device_bytes_ = 0;
    uint64_t sweeps_done_ = 0;
    uint64_t swap_rounds_ = 0;

    // device storage
    std::vector<std::unique_ptr<DeviceBuffer>> model_storage_;
    DeviceBuffer models_, tile_first_, tile_count_, tile_model_, chain_loc_, seeds_, betas_;
    DeviceBuffer slot_of_chain_, chain_at_slot_, hs_, ht_, spin_bits_, mt_, mt_pos_, e_run_, flips_;
    DeviceBuffer swap_seeds_, swap_mt_, swap_pos_, swap_acc_, swap_att_;
    DeviceBuffer layer_graphs_, wait_counts_;
    DeviceBuffer strand_graphs_, tape_, spin_cells_, spin_nbr_, strand_flags_;
    bool strand_live_ = false;  // the strand family has run since the last settle(): cells hold the spins, far updates pending
    void settle();              // back to the canonical state (fields complete, spin_bits current); no-op otherwise
    uint32_t strand_warps_ = 0;
    bool l2_window_set_ = false;
    DeviceBuffer scratch_;  // readout staging
    DeviceBuffer gather_send_;  // this rank's packed records on their way into the all-gather
    int sm_count_ = 0;

    // timing
    bool timing_ = false;
    std::vector<TimedLaunch> pending_;
    double sweep_ms_ = 0.0, swap_ms_ = 0.0;
    cudaEvent_t run_start_ = nullptr, run_stop_ = nullptr;
    bool run_timed_ = false;
};

}  // namespace isingb200
