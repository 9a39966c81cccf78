/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
 *
 * This header and ising_oracle.c restate, in plain C, the algorithm of the
 * reference's scalar sweep tier (`sweep_basic`, bit-identical to
 * `sweep_reference`) and everything it calls, so that the CUDA path can be
 * checked bit-for-bit on a box where /root/reference does not exist.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product library never links it.
 *
 * Pinning: tests/test_oracle_vs_reference.py compares every function here
 * against the reference's own code compiled unmodified into
 * oracle/_ref/libisingref.so (recipe: oracle/build_ref.sh), and
 * tests/golden/ holds vectors generated from that library.  The tempering
 * swap has no counterpart in the reference: for that one
 * function parity is UNPINNED and this file is its definition.
 *
 * Reference citations are relative to /root/reference/proj.
 */
#ifndef ISING_ORACLE_H
#define ISING_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_EXP_EXACT = 1, ORC_EXP_FAST = 2, ORC_EXP_ACCURATE = 3 }; /* isingmc.h:30-35 */

/* ---- MT19937 (src/rng.cpp:22-44, 75-128) ---- */
typedef struct orc_mt {
    uint32_t w[624];
    uint32_t cursor;
} orc_mt;

void orc_mt_seed(orc_mt* g, uint32_t seed);
uint32_t orc_mt_next(orc_mt* g);
void orc_mt_fill(uint32_t seed, uint32_t* out, size_t count);

/* include/isingmc/rng.hpp:87-92 */
float orc_u32_to_unit(uint32_t x);

/* include/isingmc/fastexp.hpp:27-51, src/sweep_kernels.hpp:19-37 */
float orc_exp_fast(float x);
float orc_exp_accurate(float x);
float orc_exp_exact(float x);
float orc_exp_kind(int kind, float x);

/* ---- model view: the flattened CSR of src/sweep_state.cpp:84-106 ---- */
typedef struct orc_model {
    uint32_t n_spins;
    const float* h;             /* n_spins */
    const uint32_t* offsets;    /* n_spins + 1 */
    const uint32_t* targets;    /* offsets[n] half-edges */
    const float* couplings;     /* offsets[n] */
    const uint8_t* tau_counts;  /* n_spins: trailing tau edges per spin */
    uint32_t layers, per_layer; /* LayeredMeta (model.hpp:44-50); 0, 0 for generic models */
} orc_model;

/* src/sweep_state.cpp:211-216 */
void orc_initial_spins(uint32_t n, uint32_t seed, int8_t* out);
/* src/sweep_state.cpp:236-255 */
void orc_recompute_fields(const orc_model* m, const float* spins, float* hs, float* ht);
/* src/model.cpp:108-126 */
double orc_total_cost(const orc_model* m, const float* spins);
/* new (tempering): total_cost with the tau couplings scaled by gamma in f32 (see orc_pt_run) */
double orc_tempering_cost(const orc_model* m, const float* spins, float tau_scale);
/* src/sweep_state.cpp:325-336 (identity permutation) */
uint64_t orc_checksum(const float* spins, uint32_t n);
/* src/sweep_state.cpp:338-354 */
uint64_t orc_field_coherence_ulp(const orc_model* m, const float* spins, const float* hs,
                                 const float* ht);

/* ---- one chain: SweepState for the basic engine (include/isingmc/sweep.hpp:85-121) ---- */
typedef struct orc_chain {
    uint32_t n;
    float beta, tau_scale;
    int exp_kind;
    float* spins; /* +/-1.0f */
    float* hs;
    float* ht;
    orc_mt rng;
    uint64_t flips, attempts;
    double e_run; /* running energy used by the tempering swap (see orc_pt_run) */
    uint32_t energy_block; /* spins per partial sum of the running energy (see orc_pt_run) */
} orc_chain;

/* init_state(model, cfg[, initial]) — src/sweep_state.cpp:218-234.  initial may be NULL. */
orc_chain* orc_chain_create(const orc_model* m, uint32_t seed, float beta, float tau_scale,
                            int exp_kind, const int8_t* initial);
void orc_chain_free(orc_chain* c);
/* run_sweeps on the basic engine — src/sweep_basic.cpp:12-56, src/sweep_state.cpp:272-291 */
void orc_chain_sweep(orc_chain* c, const orc_model* m, uint64_t sweeps);

/* ---- batched run with parallel tempering ----
 * Chains are grouped in ladders of n_betas; chain c = ladder * n_betas + k0 starts in
 * beta slot k0.  NEW SEMANTICS (no reference counterpart):
 *   - after every `swap_interval`-th sweep (counted over the whole run) one swap round r
 *     (r = 0,1,2,...) visits slot pairs (k,k+1), k = r&1, r&1+2, ... in increasing k;
 *   - for the chains a,b holding slots k,k+1: one draw u = u32_to_unit(next) from the
 *     ladder's own Mt19937(swap_seed ^ 0x85EBCA6B), x = (float)((double(beta_k) -
 *     double(beta_k1)) * (E_a - E_b)), accept iff u < exp_kind(x); on accept the two
 *     chains exchange beta slots (spin arrays and sweep RNG streams stay put);
 *   - E is the running value of the energy the sweeps sample, E_space + gamma * E_tau: it starts as
 *     orc_tempering_cost of the initial spins (total_cost with the tau couplings scaled by gamma;
 *     total_cost itself when gamma == 1) and receives, after every ENERGY BLOCK of attempts, the
 *     block's partial sum: starting from 0.0, (double)((2.0f*s)*(hs + gamma*ht)) — the inner factor
 *     of the flip exponent, an f32 — added at each accepted flip in flip order.  A block is one
 *     layer (per_layer spins) of a layered model, the whole sweep otherwise.  Summing per block is
 *     what lets the layers of one chain be swept by different warps (a block's partial sum needs
 *     nothing from the blocks before it); the blocks are added in index order.
 */
/* ---- the intra-system "coalesced" schedule (ref: proj/src/sweep_coalesced.cpp:10-124; model
 * permutation proj/src/model.cpp:190-215; init proj/src/sweep_state.cpp:120-146,193-199).
 * W = layers/2 lanes; lane t owns layers 2t (even region) and 2t+1 (odd region); spin (l,p) lives
 * at new index W*((l%2)*P + p) + l/2.  One sweep = even flips (space edges + tau edge down),
 * deferred tau edges up, odd flips, deferred tau edges up; lane t draws from Mt19937(seed + t).
 * The model given here is the ORIGINAL (identity-ordered) layered model; all arrays of the
 * state are in the new index order, `forward[old] = new`. */
typedef struct orc_coalesced {
    uint32_t n, lanes, per_layer;
    float beta, tau_scale;
    int exp_kind;
    orc_model permuted;   /* owned: CSR of the permuted model (edge order of the original lists) */
    uint32_t* forward;    /* old index -> new index */
    float *spins, *hs, *ht;
    uint8_t* flags;
    orc_mt* lane_rng;     /* lanes generators */
    uint64_t flips, attempts;
} orc_coalesced;

orc_coalesced* orc_coalesced_create(const orc_model* m, uint32_t seed, float beta, float tau_scale,
                                    int exp_kind, const int8_t* initial_new_order);
void orc_coalesced_free(orc_coalesced* c);
void orc_coalesced_sweep(orc_coalesced* c, uint64_t sweeps);
/* spins in the ORIGINAL spin order (+1/-1) */
void orc_coalesced_read_spins(const orc_coalesced* c, int8_t* out);

typedef struct orc_pt_result {
    int8_t* spins;        /* n_chains * n : +/-1 */
    uint64_t* flips;      /* n_chains */
    double* e_run;        /* n_chains */
    double* energy;       /* n_chains : total_cost of final spins */
    uint32_t* slot;       /* n_chains : final beta slot of each chain */
    uint64_t* swap_acc;   /* n_ladders * n_betas (entry k: pair k,k+1; last unused) */
    uint64_t* swap_att;   /* n_ladders * n_betas */
} orc_pt_result;

/* models[l] is the model of ladder l.  seeds: n_chains; swap_seeds: n_ladders.  Any result
 * pointer may be NULL.  threads >= 1 splits ladders over pthreads (results are identical for
 * any thread count).  Returns 0, or -1 on allocation failure / bad arguments. */
int orc_pt_run(const orc_model* const* models, uint32_t n_ladders, uint32_t n_betas,
               const float* betas, const uint32_t* seeds, const uint32_t* swap_seeds,
               float tau_scale, int exp_kind, uint64_t sweeps, uint32_t swap_interval,
               uint32_t threads, const int8_t* initial /* may be NULL */, orc_pt_result* out);

#define ORC_INIT_SPIN_SEED_MIX 0x9E3779B9u /* src/sweep_state.cpp:48 */
#define ORC_SWAP_SEED_MIX 0x85EBCA6Bu      /* new: keeps swap draws off every sweep stream */

#ifdef __cplusplus
}
#endif
#endif
