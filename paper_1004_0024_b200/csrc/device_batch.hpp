// Device-side description of a batch and the kernel launchers.  Layout (HBM):
//
//   chains are packed in TILES of 32 — one tile per warp, lane = chain ("replica").  A tile
//   never mixes models, so every graph access of a warp is warp-uniform.
//     hs, ht      f32 [tile][spin][32]     replica-interleaved effective fields
//     spin_bits   u32 [tile][spin]         bit `lane` set <=> that chain's spin is -1
//     mt          u32 [tile][624][32]      replica-interleaved MT19937 state (the reference's
//                                          InterlacedMt layout words[w*K+k], rng.hpp:51-53, K=32)
//     mt_pos      u32 [tile]               next state word to regenerate (all lanes in lockstep)
//   per chain:  slot (beta index), running energy f64, flips u64
//   per ladder: chain_at_slot[n_betas], swap MT state [624][n_ladders], accept/attempt counts
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace isingb200 {

constexpr uint32_t kWaitSlots = 7;  // widths 1, 2, 4, 8, 16, 32, then the attempts (per lane) recorded
constexpr uint32_t kMtWords = 624;  // MT19937 state words per chain (ref: rng.hpp:11)

struct DevModel {
    uint32_t n_spins;
    uint32_t has_tau;
    uint32_t distinct_targets;  // 1: no spin lists a neighbour twice, so a flip's updates may be batched
    // 1: every non-zero field and coupling is at least 2^-100 in magnitude, so no effective field can
    // ever be subnormal (they are sums of multiples of 2^-123) and h[t] -= d may be issued as a global
    // f32 reduction, which rounds like the subtraction but flushes subnormals
    uint32_t reduction_safe;
    // Generic family, own-field window: window[i*8 + q] is the space coupling from spin i to spin i+q
    // when both lie in the same chunk of eight attempts (else 0).  nullptr when the window cannot be
    // used (not reduction_safe, a repeated in-chunk neighbour, an in-chunk tau edge).
    const float* window;
    const float* h;
    const uint32_t* offsets;
    const uint32_t* targets;
    const float* couplings;
    const uint8_t* tau_counts;
    // total_cost as a flat list in the reference's summation order (batch.cpp: build_cost_terms):
    // {spin, partner or kFieldTerm, bits of the coefficient, 0}, padded to a multiple of 32 with
    // zero coefficients.
    const uint4* cost_terms;
    uint32_t n_cost_terms;
    // The same list with every tau coupling replaced by fl32(tau_scale * J): the energy the sweeps
    // sample, which the tempering swap compares (== cost_terms when tau_scale is 1).
    const uint4* tempering_terms;
    // Attempts per partial sum of the running energy: per_layer for layered models, n_spins otherwise
    // (tempering definition, oracle/ising_oracle.h).
    uint32_t energy_block;
};
constexpr uint32_t kFieldTerm = 0xffffffffu;

// One layer of an identical-layer model, as the layered kernel keeps it in shared memory.
// Edge e of position p (layer_offsets[p] <= e < layer_offsets[p+1]) goes to position
// targets[e] of the same layer with doubled coupling j2[e] = 2*J (exact); tau2[p] = 2*J_tau(p)
// and tau2g[p] = fl(tau_scale * tau2[p]) are the two non-zero magnitudes of the tau field.
//
// The in-layer edges of position p are split by distance: the BAND slots are the (up to four)
// neighbours at p-2, p-1, p+1, p+2, which the kernel keeps in a register window; everything else
// is a FAR edge, updated in Tensor Memory.
struct DevLayerGraph {
    uint32_t per_layer;
    uint32_t layers;
    uint32_t n_far;
    // per position: {bits of tau2g, bits of tau2,
    //                near forward edges of a CAREFUL chunk: begin | count << 16 (indices into `far`), 0}
    const uint4* pos;
    // per chunk of 8 positions: {far-warp groups: begin | count << 16 (indices into `groups`),
    //                            near groups of a LEAN chunk: begin | count << 16,
    //                            flags (1 careful, 2 lean but first/last of the layer), 0}
    const uint4* chunks;
    // a group is up to 8 edges with distinct targets: edge begin | edge count << 16
    const uint32_t* groups;
    uint32_t n_groups;
    // per position two entries (2p: flipped spin was -1, 2p+1: it was +1): what the flip adds to the
    // fields at p-2, p-1, p+1, p+2, i.e. -(2s)*J as bits; an empty slot holds -0.0, the additive
    // identity for every float bit pattern, so it costs no predicate.
    const uint4* band_pm;
    const uint4* far;  // {target position, 7 - attempt index in its chunk, bits of 2J, 0}
};

// One layer of an identical-layer model as the strand (layer-wavefront) kernel reads it.  Band slots
// as in DevLayerGraph.  Every other in-layer edge q -> t is either NEAR — t lies among the columns
// q's chunk has already requested, q+3 .. 8*(q/8)+10, pushed through a scratch, which makes the chunk
// CAREFUL — or FAR: the target PULLS it when column t enters the register window, from the source
// chunk's CELL (u16 per chain and chunk of 8 spins: bit k = spin k flipped in the chunk's latest
// sweep, bit 8+k = spin k is -1).  Two far edges per column are fixed slots of the lean path; a column
// with more makes the chunk it enters in careful.
struct DevStrandGraph {
    uint32_t per_layer;
    uint32_t layers;
    const uint4* pos;      // per position: {bits of gamma*2J_tau, near edges begin | count << 16,
                           //                far in-edges beyond the two slots begin | count << 16, 0} (into `edges`)
    const uint4* band_pm;  // as DevLayerGraph::band_pm
    const uint4* tau;      // per position the bits of gamma*2J_tau (u32 [per_layer], read 8 at a time)
    const uint4* chunks;   // per chunk: {0, 0, flags (1 careful), 0}
    // per position, per_layer + 8 entries (the last 8 null): the first two far in-edges in application
    // order (sources after the column — flips of the sweep before — then sources before it), each
    // {bits of 2J, (23 - source bit) | byte offset of the source chunk's cell row << 8}; a null slot is
    // {-0.0, 31}
    const uint4* inslots;
    const uint4* edges;    // near: {target position, attempt index k in its chunk, bits of 2J, 0}; far: {bits of 2J, meta, 0, 0}
    uint32_t n_edges;
};

struct DevBatch {
    const DevLayerGraph* layer_graphs;  // per model; nullptr unless the layered family is used
    uint32_t max_far_edges;             // largest n_far over the batch's models
    uint32_t max_groups;                // largest n_groups over the batch's models
    uint32_t layered_smem;              // dynamic shared memory of one layered-kernel CTA
    uint32_t max_per_layer;             // largest per_layer over the batch's models
    uint32_t graph_shared;              // 1: all tiles use model 0, one shared-memory copy per CTA
    uint32_t layered_stages;            // depth of the producer/sweep stage ring (2, 4 or 8)
    uint32_t n_spins;
    uint32_t n_tiles;
    uint32_t n_chains;
    uint32_t n_ladders;
    uint32_t n_betas;
    float tau_scale;
    int exp_kind;
    const DevModel* models;
    const uint32_t* tile_first;  // first chain of the tile
    const uint32_t* tile_count;  // active lanes
    const uint32_t* tile_model;
    const uint32_t* chain_loc;   // chain -> tile*32 + lane
    const uint32_t* seeds;       // per chain
    const float* betas;          // n_betas
    uint32_t* slot_of_chain;
    uint32_t* chain_at_slot;     // [ladder][n_betas] -> global chain id
    float* hs;
    float* ht;                   // nullptr when no model has tau edges
    uint32_t* spin_bits;
    uint32_t* mt;
    uint32_t* mt_pos;
    double* e_run;
    unsigned long long* flips;
    // wait statistics (ref: FlipStats::group_wait, sweep.hpp:31-44), per tile: groups of w = 1, 2, 4, 8,
    // 16, 32 neighbouring lanes (chains attempting the same spin in lockstep) that held at least one
    // flip, and the attempts recorded; nullptr unless recording was requested
    unsigned long long* wait_counts;  // [tile][kWaitSlots]
    uint32_t generic_reduce;          // every model is reduction_safe: the generic family uses sweep_split_kernel
    uint32_t generic_windows;         // ... and every model has an own-field window: sweep_trio_kernel
    // strand (layer-wavefront) family: kernels_strand.cu
    const DevStrandGraph* strand_graphs;  // per model
    uint32_t strands;       // S: concurrent layers per tile (divides every model's layer count)
    uint32_t max_layers;    // largest layer count over the batch's models
    uint32_t strand_pub;    // a strand publishes its progress every strand_pub chunks
    uint32_t tape_rows;     // R: rows of a tile's MT19937 tape ring (a multiple of 32)
    uint32_t* tape;         // u32 [tile][R][32]: raw MT19937 words in draw order
    uint16_t* spin_cells;   // u16 [tile][spin / 8][32]: bit 8+k of a lane's cell <=> its spin 8c+k is -1, bit k <=> it
                            // flipped in the chunk's latest sweep (DevStrandGraph)
    // u16 [tile][spin / 8][32], what the strands of the neighbouring layers read: bit k <=> spin 8c+k is
    // -1, high byte = low byte of the number of sweeps the chunk has seen (batch lifetime) — spins and
    // their version in one word, so a reader needs no fence between a progress counter and the data
    uint16_t* spin_nbr;
    uint32_t strand_epoch;  // sweeps done before this launch: the version every chunk carries at its start
    uint32_t* strand_flags; // per tile S + 1 progress counters (strand chunks done, tape head), one line each
    uint32_t strand_graph_smem;  // bytes of the largest layer graph as staged in shared memory
    uint32_t strand_single_model;  // 1: every tile uses model 0
    // tempering
    const uint32_t* swap_seeds;  // per ladder
    uint32_t* swap_mt;           // [624][n_ladders]
    uint32_t* swap_pos;          // per ladder
    unsigned long long* swap_acc;  // [ladder][n_betas]
    unsigned long long* swap_att;
};

// All launchers enqueue on `stream` and return the launch error (cudaGetLastError).
cudaError_t launch_init(const DevBatch& b, const int8_t* initial_spins_dev, cudaStream_t stream);
cudaError_t launch_sweep_generic(const DevBatch& b, uint32_t sweeps, cudaStream_t stream);
// Layered family: needs b.layer_graphs; `sm_count` persistent CTAs of 4 sweep warps.
cudaError_t launch_sweep_layered(const DevBatch& b, uint32_t sweeps, int sm_count, cudaStream_t stream);
// Bytes of dynamic shared memory one CTA of the layered kernel needs (0: does not fit).
size_t layered_smem_bytes(uint32_t per_layer, uint32_t max_far_edges, uint32_t max_groups, bool graph_shared);
uint32_t layered_stage_count(uint32_t per_layer, uint32_t max_far_edges, uint32_t max_groups, bool graph_shared);
cudaError_t prepare_layered_kernels(size_t smem_bytes);
// Strand family: needs b.strand_graphs, tape, spin_cells, strand_flags; `warps_per_cta` <= strand_max_warps().
// While the family runs, the cells hold the spins and the fields lack the far updates of each layer's
// latest sweep (they are pulled during the next one): `from_words` builds the cells from spin_bits
// first; launch_strand_settle applies what is pending and writes spin_bits back.
cudaError_t launch_sweep_strand(const DevBatch& b, uint32_t sweeps, int sm_count, uint32_t warps_per_cta,
                                bool from_words, cudaStream_t stream);
cudaError_t launch_strand_settle(const DevBatch& b, cudaStream_t stream);
uint32_t strand_max_warps();
uint32_t strand_warp_smem();  // shared-memory bytes per warp (landing stages, scratch)
uint32_t strand_flag_words(uint32_t n_tiles, uint32_t strands);
size_t strand_graph_bytes(uint32_t per_layer, uint32_t n_edges);
cudaError_t launch_swap(const DevBatch& b, uint64_t round, cudaStream_t stream);
cudaError_t launch_energies(const DevBatch& b, double* out_dev, cudaStream_t stream);
cudaError_t launch_resync_energies(const DevBatch& b, cudaStream_t stream);  // e_run := tempering cost of the spins
cudaError_t launch_checksums(const DevBatch& b, unsigned long long* out_dev, cudaStream_t stream);
cudaError_t launch_coherence(const DevBatch& b, unsigned long long* out_dev, cudaStream_t stream);
cudaError_t launch_unpack_spins(const DevBatch& b, uint32_t first_chain, uint32_t n_chains,
                                int8_t* out_dev, cudaStream_t stream);
cudaError_t launch_gather_fields(const DevBatch& b, uint32_t chain, float* hs_dev, float* ht_dev,
                                 cudaStream_t stream);
cudaError_t launch_pack_results(const DevBatch& b, void* out_dev, cudaStream_t stream);

}  // namespace isingb200
