/* C ABI of the B200 batched sweep engine: the drop-in boundary for the hot path of
 * isingmc (arXiv 1004.0024) — batched Metropolis sweeps over many independent sparse Ising
 * chains under parallel tempering, executed by hand-written sm_100a CUDA kernels.
 *
 * Conventions are those of the reference's C interface (reference:
 * proj/include/isingmc.h:1-38, proj/src/capi.cpp:21-65): every entry point returns an
 * ising_status; on failure ising_b200_last_error() describes the problem for the calling
 * thread (thread-local); handles are opaque and freed by their matching _free; input
 * arrays are borrowed for the duration of the call; output arrays are caller-owned HOST
 * memory; C++ exceptions never cross the boundary.  There is NO CPU fallback: without a
 * usable CUDA device every batch entry point fails with ISING_ERR_INTERNAL.
 *
 * Each declaration cites the reference interface it replaces or extends.  "ref:" paths are
 * relative to /root/reference/proj.
 */
#ifndef ISINGMC_B200_H
#define ISINGMC_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ISING_B200_API __attribute__((visibility("default")))
#else
#define ISING_B200_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#ifndef ISINGMC_H /* same values as ref: include/isingmc.h:15-35 when both headers are used */
typedef enum ising_status {
    ISING_OK = 0,
    ISING_ERR_ARGUMENT = 1,
    ISING_ERR_PARSE = 2,
    ISING_ERR_IO = 3,
    ISING_ERR_INTERNAL = 4
} ising_status;

typedef enum ising_exp_kind {
    ISING_EXP_ENGINE_DEFAULT = 0, /* fast (the default of every non-`reference` engine) */
    ISING_EXP_EXACT = 1,
    ISING_EXP_FAST = 2,
    ISING_EXP_ACCURATE = 3
} ising_exp_kind;
#endif

/* ref: ising_last_error, include/isingmc.h:38 / src/capi.cpp:33,145 */
ISING_B200_API const char* ising_b200_last_error(void);

/* Number of visible CUDA devices (0 if none / driver missing). Never fails. */
ISING_B200_API int ising_b200_device_count(void);

/* ---------------------------------------------------------------- models ---- */

/* Immutable, shareable graph + fields (ref: SpinModel, include/isingmc/model.hpp:52-60). */
typedef struct ising_b200_model ising_b200_model;

/* From the flattened adjacency the reference engines use (ref: FlatEdges,
 * include/isingmc/sweep.hpp:67-72; flatten(), src/sweep_state.cpp:84-106): spin i owns
 * half-edges offsets[i]..offsets[i+1], the last tau_counts[i] of them tau edges.
 * tau_counts may be NULL (all zero).  layers = 0 for a generic model, otherwise the model
 * is declared layered (layers * per_layer == n_spins, ref: LayeredMeta model.hpp:44-50).
 * Runs the structural checks of validate_model (ref: src/model.cpp:246-330). */
ISING_B200_API ising_status ising_b200_model_from_csr(uint32_t n_spins, const float* h, const uint32_t* offsets,
                                       const uint32_t* targets, const float* couplings,
                                       const uint8_t* tau_counts, uint32_t layers,
                                       uint32_t per_layer, ising_b200_model** out);

/* ref: build_layered_model(LayerSpec, n_layers, j_tau), src/model.cpp:52-104: n_layers
 * copies of a `positions`-site layer (undirected space edges p[e]-q[e] with coupling j[e]),
 * spin (l,pos) -> l*positions+pos, tau edges of coupling j_tau to the next then the previous
 * layer in the last two slots.  Same rejections (n_layers < 4, bad/duplicate/self edges). */
ISING_B200_API ising_status ising_b200_model_build_layered(uint32_t positions, const float* h, uint32_t n_edges,
                                            const uint32_t* p, const uint32_t* q, const float* j,
                                            uint32_t n_layers, float j_tau,
                                            ising_b200_model** out);

ISING_B200_API void ising_b200_model_free(ising_b200_model* model); /* ref: ising_model_free */
ISING_B200_API uint32_t ising_b200_model_spins(const ising_b200_model* model); /* ref: ising_model_spins */
ISING_B200_API uint64_t ising_b200_model_half_edges(const ising_b200_model* model);
/* ref: ising_model_layers, include/isingmc.h:53 — returns 1 and fills for layered models. */
ISING_B200_API int ising_b200_model_layers(const ising_b200_model* model, uint32_t* layers, uint32_t* per_layer);
/* Copies the CSR view out (arrays sized by _spins / _half_edges). */
ISING_B200_API ising_status ising_b200_model_export_csr(const ising_b200_model* model, float* h, uint32_t* offsets,
                                         uint32_t* targets, float* couplings, uint8_t* tau_counts);
/* ref: ising_model_cost, include/isingmc.h:55 -> total_cost, src/model.cpp:108-126 (host, f64). */
ISING_B200_API ising_status ising_b200_model_cost(const ising_b200_model* model, const int8_t* spins, uint32_t n,
                                   double* cost);

/* ---------------------------------------------------------------- batches ---- */

/* Which sweep kernel family a batch uses.  All families follow the same trajectories bit for bit. */
typedef enum ising_b200_kernel {
    ISING_KERNEL_AUTO = 0,    /* STRAND when every model qualifies, else GENERIC */
    ISING_KERNEL_GENERIC = 1, /* any graph: state in HBM, replica-interleaved [spin][32 chains] */
    ISING_KERNEL_LAYERED = 2, /* identical-layer models, at most 512 positions per layer: one layer of
                                 fields in Tensor Memory per 32 chains, one sweep warp per tile */
    ISING_KERNEL_STRAND = 3   /* identical-layer models: the layers of a tile swept by several warps in
                                 a wavefront (same order of decisions per chain), state in HBM/L2 */
} ising_b200_kernel;

/* The batch counterpart of EngineConfig + the per-chain SweepParams
 * (ref: include/isingmc/sweep.hpp:25-29,55-63).  Chains are grouped in ladders of n_betas;
 * chain c = ladder * n_betas + k starts in beta slot k (beta = betas[k]).  n_betas = 1 gives
 * plain independent replicas. */
typedef struct ising_batch_params {
    uint32_t n_ladders;
    uint32_t n_betas;
    const float* betas;         /* n_betas, each finite and >= 0 (ref: sweep_state.cpp:148-150) */
    const uint32_t* seeds;      /* n_ladders*n_betas sweep-stream seeds, or NULL: base_seed +
                                   (first_ladder*n_betas + c), the reference's lane-seed rule
                                   (ref: sweep.hpp:59, rng.cpp:144-148) */
    const uint32_t* swap_seeds; /* n_ladders, or NULL: swap_base_seed + first_ladder + l */
    uint32_t base_seed;
    uint32_t swap_base_seed;
    uint64_t first_ladder;      /* global index of this shard's ladder 0 (multi-GPU sharding) */
    float tau_scale;            /* ref: SweepParams::tau_scale, must be finite */
    int exp_kind;               /* ising_exp_kind */
    int device;                 /* CUDA device ordinal */
    int kernel;                 /* ising_b200_kernel */
    const int8_t* initial_spins; /* NULL: initial_spins(n, seed) per chain (ref:
                                    sweep_state.cpp:211-223); else [chains][n_spins] of +/-1
                                    (ref: init_state(model,cfg,initial), sweep_state.cpp:225-234) */
} ising_batch_params;

typedef struct ising_batch ising_batch;

/* ref: init_state(model, cfg) for every chain (src/sweep_state.cpp:160-234): uploads the
 * models, then ON THE DEVICE seeds each chain's MT19937, draws its initial spins, sums the
 * effective fields in the reference's order and the initial energy.  models[model_of_ladder[l]]
 * is ladder l's graph; model_of_ladder may be NULL when n_models == 1 (shared graph) or
 * n_models == n_ladders (ladder l uses models[l]).  All models must have equal n_spins. */
ISING_B200_API ising_status ising_batch_create(const ising_b200_model* const* models, uint32_t n_models,
                                const uint32_t* model_of_ladder, const ising_batch_params* params,
                                ising_batch** out);
ISING_B200_API void ising_batch_free(ising_batch* batch);

/* ref: run_sweeps(state, model, n), src/sweep_state.cpp:272-291, for every chain; after each
 * swap_interval-th sweep (counted since creation) one tempering swap round runs.
 * swap_interval = 0: never swap.  Asynchronous on the batch's stream; reads synchronise. */
ISING_B200_API ising_status ising_batch_run(ising_batch* batch, uint64_t sweeps, uint32_t swap_interval);
/* One swap round now (new: the reference has no tempering). */
ISING_B200_API ising_status ising_batch_swap(ising_batch* batch);
ISING_B200_API ising_status ising_batch_sync(ising_batch* batch);

/* --- readout: all outputs are host buffers, chains in global order --- */
/* ref: SweepState::spins (sweep.hpp:92) as +/-1 int8, [n_chains][n_spins], original order. */
ISING_B200_API ising_status ising_batch_read_spins(ising_batch* batch, uint64_t first_chain, uint64_t n_chains,
                                    int8_t* out);
/* ref: SweepState::h_eff_space / h_eff_tau (sweep.hpp:93-94) of one chain. */
ISING_B200_API ising_status ising_batch_read_fields(ising_batch* batch, uint64_t chain, float* h_space,
                                     float* h_tau);
/* ref: total_cost(model, state.spins) per chain (capi.cpp:119), f64, reference summation order. */
ISING_B200_API ising_status ising_batch_read_energies(ising_batch* batch, double* out);
/* Running energy used by the swap rule (initial cost + sum of flip energies). */
ISING_B200_API ising_status ising_batch_read_running_energies(ising_batch* batch, double* out);
/* Recomputes every chain's running energy from its spins (the tempering cost: total_cost with the
 * tau couplings scaled by tau_scale, oracle: orc_tempering_cost), discarding the rounding the flip
 * energies have accumulated.  New: the reference has no running energy.  Optional — a long
 * tempering run may call it every few thousand sweeps; a parity run sets the oracle chain's e_run to
 * orc_tempering_cost at the same sweep counts. */
ISING_B200_API ising_status ising_batch_resync_energies(ising_batch* batch);
/* ref: FlipStats::flips / attempts (sweep.hpp:38-44). Either pointer may be NULL. */
ISING_B200_API ising_status ising_batch_read_stats(ising_batch* batch, uint64_t* flips, uint64_t* attempts);
/* ref: state_checksum (sweep_state.cpp:325-336): FNV-1a over the sign sequence. */
ISING_B200_API ising_status ising_batch_checksums(ising_batch* batch, uint64_t* out);
/* ref: field_coherence_ulp (sweep_state.cpp:346-354) per chain. */
ISING_B200_API ising_status ising_batch_field_coherence(ising_batch* batch, uint64_t* out);
/* Current beta slot of each chain; per ladder and slot pair k,(k+1) the accept / attempt
 * counts ([n_ladders][n_betas], last column unused). Either swap pointer may be NULL. */
ISING_B200_API ising_status ising_batch_read_slots(ising_batch* batch, uint32_t* slot_of_chain);
ISING_B200_API ising_status ising_batch_read_swap_stats(ising_batch* batch, uint64_t* accepts, uint64_t* attempts);

/* Packs per-chain {energy f64, running energy f64, flips u64, checksum u64} (32 B per chain)
 * into a DEVICE buffer (e.g. a torch CUDA tensor) so a multi-GPU caller can gather results
 * with one NCCL all-gather and no host round trip.  device_out: n_chains * 32 bytes. */
ISING_B200_API ising_status ising_batch_pack_results(ising_batch* batch, void* device_out);
/* The same records of EVERY rank's shard, gathered over NCCL (NVLink / NVSwitch) on the batch's own
 * stream: packs this rank's records and calls ncclAllGather on `nccl_comm` (an ncclComm_t of the
 * caller, every rank holding the same number of chains — the weak-scaling layout of the bench).
 * device_out_all: n_ranks * n_chains * 32 bytes of DEVICE memory, rank-major.  This is the data
 * path's only collective; it replaces the shared-memory result vectors of the reference's chain
 * pool (ref: src/bench.cpp:51-84: one RepetitionResult per chain, filled by the workers).  NCCL is
 * looked up at run time (the libnccl.so.2 the process has loaded, else the system's): the library
 * has no link-time dependency on it.  ISING_ERR_INTERNAL when NCCL is missing or reports an error. */
ISING_B200_API ising_status ising_batch_all_gather_results(ising_batch* batch, void* nccl_comm, void* device_out_all);

/* --- introspection / measurement --- */
typedef struct ising_batch_info {
    uint64_t n_chains;
    uint32_t n_spins;
    uint32_t n_tiles;        /* warps' worth of chains (32 per tile) */
    int kernel;              /* ising_b200_kernel actually used */
    uint64_t sweeps_done;
    uint64_t device_bytes;   /* HBM held by this batch */
    uint64_t sweep_launches; /* sweep kernel launches so far */
    uint64_t swap_launches;
    uint64_t other_launches; /* init / readout kernels */
    double sweep_ms;         /* CUDA-event time summed over sweep launches (needs timing on) */
    double swap_ms;
    double last_run_ms;      /* CUDA-event time of the last ising_batch_run call, whole call */
    /* generic family only: 0 read-modify-write updates (some coupling or field is below 2^-100 in
     * magnitude), 1 updates as f32 reductions, 2 reductions + own-field window for every model */
    uint32_t generic_variant;
    uint32_t strands;        /* strand family: layers of a tile swept concurrently (0 otherwise) */
} ising_batch_info;
/* timing = 1 brackets every sweep/swap launch with CUDA events on the batch's stream. */
ISING_B200_API ising_status ising_batch_set_timing(ising_batch* batch, int timing);
ISING_B200_API ising_status ising_batch_get_info(ising_batch* batch, ising_batch_info* out); /* synchronises */

/* Wait statistics (ref: FlipStats::group_wait / collect_wait_stats, include/isingmc/sweep.hpp:31-53,
 * src/sweep_state.cpp:33-44; ising_run_report.wait_*, include/isingmc.h:94-96).  The reference
 * groups w consecutively processed spins of ONE chain (its SIMD lanes); here the lanes of a warp are
 * w NEIGHBOURING CHAINS attempting the same spin in lockstep, so the probability that a w-wide group
 * holds at least one flip is measured on the real ballots.  Widths 1, 2, 4, 8, 16, 32 (1 = the
 * flip rate); tiles with fewer than 32 chains are not recorded.  record_wait(1) zeroes the counters
 * and starts recording for the following ising_batch_run calls; record_wait(0) stops it.
 * probability/groups/with_flip: n_widths entries each, any may be NULL. */
ISING_B200_API ising_status ising_batch_record_wait(ising_batch* batch, int on);
ISING_B200_API ising_status ising_batch_read_wait_stats(ising_batch* batch, uint32_t n_widths,
                                                         const uint32_t* widths, double* probability,
                                                         uint64_t* groups, uint64_t* with_flip);
/* The batch's cudaStream_t, for callers that want to record their own events on it. */
ISING_B200_API void* ising_batch_stream(ising_batch* batch);

/* ---------------------------------------------------------------- one-shot ---- */
/* Single-chain counterpart of ising_run (ref: include/isingmc.h:74-106, capi.cpp:96-139,
 * 221-228) with the basic engine's semantics: same fields as ising_run_params /
 * ising_run_report minus the CPU-tier knobs (engine, workers, wait statistics). */
typedef struct ising_b200_run_params {
    uint64_t sweeps;
    float beta;
    float tau_scale;
    int exp_kind;
    uint32_t seed;
    int device;
} ising_b200_run_params;

typedef struct ising_b200_run_report {
    double final_cost;
    double flip_rate;
    uint64_t flips;
    uint64_t attempts;
    uint64_t checksum;
} ising_b200_run_report;

ISING_B200_API ising_status ising_b200_run(const ising_b200_model* model, const ising_b200_run_params* params,
                            ising_b200_run_report* out);
/* ref: ising_run_json, include/isingmc.h:108-112, src/capi.cpp:230-262: the same run, plus a JSON
 * document with the reference's keys (engine, exp, spins, sweeps, beta, tau_scale, seed, workers,
 * final_cost, flip_rate, flips, attempts, wait, checksum as 16 hex digits, environment).  `engine`
 * names the kernel family used ("b200-generic" / "b200-layered" / "b200-strand"); `wait` is empty for a single
 * chain (see ising_batch_read_wait_stats).  *out_json is freed with ising_b200_string_free;
 * out_report may be NULL. */
ISING_B200_API ising_status ising_b200_run_json(const ising_b200_model* model, const ising_b200_run_params* params,
                                                 ising_b200_run_report* out_report, char** out_json);

/* ------------------------------------------- coalesced (intra-system) batches ---- */
/* The reference's `coalesced` engine on the device (ref: EngineKind::coalesced, include/isingmc/
 * sweep.hpp:16; src/sweep_coalesced.cpp:10-124; prepare_model_for_engine + coalesce_permutation,
 * src/sweep_state.cpp:292-323, src/model.cpp:190-215): one warp per chain, W = layers/2 lanes, lane t
 * owns layers 2t and 2t+1 and draws from Mt19937(seed + t); four phases per sweep.  For few chains
 * of a large layered system, where one chain per lane cannot fill the GPU.  The model is the
 * ORIGINAL identity-ordered layered model (the permutation is applied internally, every readout is
 * in the original spin order) and must stay alive as long as the batch.  Needs an even layer count
 * <= 64 and half the spins within 227 KB of shared memory at 5 bytes per spin.  Chains are
 * independent (this engine has no tempering in the reference either). */
typedef struct ising_coalesced_params {
    uint32_t n_chains;
    const float* betas;          /* n_chains */
    const uint32_t* seeds;       /* n_chains, or NULL: base_seed + c * (layers/2) (disjoint lane seeds) */
    uint32_t base_seed;
    float tau_scale;
    int exp_kind;                /* ising_exp_kind */
    int device;
    const int8_t* initial_spins; /* NULL: initial_spins(n, seed) in the permuted order, exactly what the
                                    reference's init_state(permuted model, cfg) draws; else
                                    [n_chains][n_spins] of +/-1 in the ORIGINAL order */
} ising_coalesced_params;

typedef struct ising_coalesced_info {
    uint64_t n_chains;
    uint32_t n_spins;
    uint32_t lanes;
    uint64_t sweeps_done;
    uint64_t launches;
    double last_run_ms; /* CUDA-event time of the last ising_coalesced_run call */
} ising_coalesced_info;

typedef struct ising_coalesced ising_coalesced;

ISING_B200_API ising_status ising_coalesced_create(const ising_b200_model* model,
                                                    const ising_coalesced_params* params, ising_coalesced** out);
ISING_B200_API void ising_coalesced_free(ising_coalesced* batch);
/* ref: run_sweeps_coalesced, src/sweep_coalesced.cpp:139-178 (asynchronous; readouts synchronise) */
ISING_B200_API ising_status ising_coalesced_run(ising_coalesced* batch, uint64_t sweeps);
ISING_B200_API ising_status ising_coalesced_read_spins(ising_coalesced* batch, uint64_t chain, int8_t* out);
ISING_B200_API ising_status ising_coalesced_read_fields(ising_coalesced* batch, uint64_t chain, float* hs, float* ht);
ISING_B200_API ising_status ising_coalesced_read_stats(ising_coalesced* batch, uint64_t* flips, uint64_t* attempts);
ISING_B200_API ising_status ising_coalesced_read_energies(ising_coalesced* batch, double* out);
ISING_B200_API ising_status ising_coalesced_checksums(ising_coalesced* batch, uint64_t* out);
ISING_B200_API ising_status ising_coalesced_get_info(ising_coalesced* batch, ising_coalesced_info* out);

/* ------------------------------------------------------- model text documents ---- */
/* `ising-model v1` documents (ref: include/isingmc/model_io.hpp:10-28, src/model_io.cpp:45-226;
 * C entry points ising_model_load / _from_string / _to_string / ising_string_free, include/isingmc.h:
 * 40-53).  Hex-float literals: save -> load is bit-exact; the loader canonicalises the adjacency
 * order and validates.  Malformed documents -> ISING_ERR_PARSE with "line N: ..." (N 1-based),
 * unreadable / unwritable files -> ISING_ERR_IO, structurally invalid models -> ISING_ERR_ARGUMENT. */
ISING_B200_API ising_status ising_b200_model_from_string(const char* text, ising_b200_model** out);
ISING_B200_API ising_status ising_b200_model_to_string(const ising_b200_model* model, char** out);
ISING_B200_API ising_status ising_b200_model_load(const char* path, ising_b200_model** out);
ISING_B200_API ising_status ising_b200_model_save(const ising_b200_model* model, const char* path);
ISING_B200_API void ising_b200_string_free(char* text);

#ifdef __cplusplus
}
#endif
#endif /* ISINGMC_B200_H */
