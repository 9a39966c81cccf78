/* TEST INFRASTRUCTURE ONLY — see ising_oracle.h.  Plain C restatement of the reference's
 * scalar Metropolis sweep and its helpers; compile with
 *   gcc -O2 -ffp-contract=off -fno-math-errno -fPIC -shared -pthread
 * (contraction must stay off: the reference forbids FMA, src/CMakeLists.txt:23-29).
 */
#include "ising_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ MT19937 */

void orc_mt_seed(orc_mt* g, uint32_t seed) { /* rng.cpp:37-44 */
    g->w[0] = seed;
    for (uint32_t i = 1; i < 624; ++i) {
        uint32_t p = g->w[i - 1];
        g->w[i] = 1812433253u * (p ^ (p >> 30)) + i;
    }
    g->cursor = 624;
}

static void mt_regenerate(orc_mt* g) { /* rng.cpp:22-25, 89-96 (plain loop) */
    uint32_t* w = g->w;
    for (uint32_t i = 0; i < 624; ++i) {
        uint32_t y = (w[i] & 0x80000000u) | (w[(i + 1) % 624] & 0x7fffffffu);
        uint32_t v = w[(i + 397) % 624] ^ (y >> 1);
        if (y & 1u) v ^= 0x9908b0dfu;
        w[i] = v;
    }
    g->cursor = 0;
}

uint32_t orc_mt_next(orc_mt* g) { /* rng.cpp:27-33, 99-102 */
    if (g->cursor == 624) mt_regenerate(g);
    uint32_t y = g->w[g->cursor++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

void orc_mt_fill(uint32_t seed, uint32_t* out, size_t count) {
    orc_mt g;
    orc_mt_seed(&g, seed);
    for (size_t i = 0; i < count; ++i) out[i] = orc_mt_next(&g);
}

/* x / 2^32 truncated toward zero: keep the top 24 significant bits (rng.hpp:87-92). */
float orc_u32_to_unit(uint32_t x) {
    if (x == 0) return 0.0f;
    int width = 32 - __builtin_clz(x);
    if (width > 24) x &= ~((1u << (width - 24)) - 1u);
    return (float)x * 0x1p-32f;
}

/* ------------------------------------------------------------------ exponentials */

static const float kTwoLnSq2 = 0.9609060278364028f;   /* fastexp.hpp:15 */
static const float kLog2eP23 = 12102203.161561485f;   /* fastexp.hpp:16 */
static const float kLog2eP25 = 48408812.64624594f;    /* fastexp.hpp:17 */
static const float kAccCutoff = -21.834136187592387f; /* fastexp.hpp:18 */
static const float kImageLo = -1056964608.0f;         /* fastexp.hpp:22 */
static const float kImageHi = 1073741760.0f;          /* fastexp.hpp:23 */

static float image_to_float(float t) { /* fastexp.hpp:29-31 */
    if (t < kImageLo) t = kImageLo; /* std::max(t, lo): x is never NaN on this path */
    if (t > kImageHi) t = kImageHi;
    int32_t i = (int32_t)lrintf(t) + 0x3F800000;
    float f;
    memcpy(&f, &i, sizeof f);
    return f * kTwoLnSq2;
}

float orc_exp_fast(float x) { return image_to_float(x * kLog2eP23); }

float orc_exp_accurate(float x) { /* fastexp.hpp:37-51 */
    if (x >= 0.0f) return 1.0f;
    if (x < kAccCutoff) return 0.0f;
    return sqrtf(sqrtf(image_to_float(x * kLog2eP25)));
}

float orc_exp_exact(float x) { return (float)exp((double)x); } /* sweep_kernels.hpp:22 */

float orc_exp_kind(int kind, float x) {
    switch (kind) {
        case ORC_EXP_EXACT: return orc_exp_exact(x);
        case ORC_EXP_FAST: return orc_exp_fast(x);
        default: return orc_exp_accurate(x);
    }
}

/* ------------------------------------------------------------------ state helpers */

void orc_initial_spins(uint32_t n, uint32_t seed, int8_t* out) {
    orc_mt g;
    orc_mt_seed(&g, seed ^ ORC_INIT_SPIN_SEED_MIX);
    for (uint32_t i = 0; i < n; ++i) out[i] = (orc_mt_next(&g) >> 31) ? -1 : 1;
}

void orc_recompute_fields(const orc_model* m, const float* spins, float* hs, float* ht) {
    for (uint32_t i = 0; i < m->n_spins; ++i) {
        uint32_t end = m->offsets[i + 1], mid = end - m->tau_counts[i];
        float a = m->h[i];
        for (uint32_t e = m->offsets[i]; e < mid; ++e) a += m->couplings[e] * spins[m->targets[e]];
        float b = 0.0f;
        for (uint32_t e = mid; e < end; ++e) b += m->couplings[e] * spins[m->targets[e]];
        hs[i] = a;
        ht[i] = b;
    }
}

double orc_total_cost(const orc_model* m, const float* spins) {
    double cost = 0.0;
    for (uint32_t i = 0; i < m->n_spins; ++i) {
        cost -= (double)m->h[i] * (double)spins[i];
        for (uint32_t e = m->offsets[i]; e < m->offsets[i + 1]; ++e) {
            uint32_t t = m->targets[e];
            if (t > i) cost -= (double)m->couplings[e] * (double)spins[i] * (double)spins[t];
        }
    }
    return cost;
}

/* The energy whose Boltzmann weight the sweeps sample, exp(-beta * (E_space + gamma * E_tau)):
 * total_cost with every tau coupling replaced by the f32 product gamma * J (new: see orc_pt_run;
 * equal to orc_total_cost bit for bit when gamma == 1). */
double orc_tempering_cost(const orc_model* m, const float* spins, float tau_scale) {
    double cost = 0.0;
    for (uint32_t i = 0; i < m->n_spins; ++i) {
        cost -= (double)m->h[i] * (double)spins[i];
        const uint32_t end = m->offsets[i + 1], mid = end - m->tau_counts[i];
        for (uint32_t e = m->offsets[i]; e < end; ++e) {
            uint32_t t = m->targets[e];
            const float j = e >= mid ? tau_scale * m->couplings[e] : m->couplings[e];
            if (t > i) cost -= (double)j * (double)spins[i] * (double)spins[t];
        }
    }
    return cost;
}

uint64_t orc_checksum(const float* spins, uint32_t n) {
    uint64_t h = 1469598103934665603ull;
    for (uint32_t i = 0; i < n; ++i) {
        h ^= (uint64_t)(spins[i] > 0.0f ? 1 : 0);
        h *= 1099511628211ull;
    }
    return h;
}

static int64_t ulp_key(float v) {
    int32_t b;
    memcpy(&b, &v, sizeof b);
    return b < 0 ? (int64_t)0x80000000ll - b : (int64_t)b;
}

uint64_t orc_field_coherence_ulp(const orc_model* m, const float* spins, const float* hs,
                                 const float* ht) {
    float* a = (float*)malloc(sizeof(float) * m->n_spins * 2);
    float* b = a + m->n_spins;
    orc_recompute_fields(m, spins, a, b);
    uint64_t worst = 0;
    for (uint32_t i = 0; i < m->n_spins; ++i) {
        int64_t d1 = ulp_key(hs[i]) - ulp_key(a[i]);
        int64_t d2 = ulp_key(ht[i]) - ulp_key(b[i]);
        if (d1 < 0) d1 = -d1;
        if (d2 < 0) d2 = -d2;
        if ((uint64_t)d1 > worst) worst = (uint64_t)d1;
        if ((uint64_t)d2 > worst) worst = (uint64_t)d2;
    }
    free(a);
    return worst;
}

/* ------------------------------------------------------------------ chains */

orc_chain* orc_chain_create(const orc_model* m, uint32_t seed, float beta, float tau_scale,
                            int exp_kind, const int8_t* initial) {
    orc_chain* c = (orc_chain*)calloc(1, sizeof *c);
    if (!c) return NULL;
    c->n = m->n_spins;
    c->beta = beta;
    c->tau_scale = tau_scale;
    c->exp_kind = exp_kind;
    c->spins = (float*)malloc(sizeof(float) * 3 * (size_t)(c->n ? c->n : 1));
    if (!c->spins) {
        free(c);
        return NULL;
    }
    c->hs = c->spins + c->n;
    c->ht = c->hs + c->n;
    if (initial) {
        for (uint32_t i = 0; i < c->n; ++i) c->spins[i] = (float)initial[i];
    } else {
        int8_t* tmp = (int8_t*)malloc(c->n ? c->n : 1);
        orc_initial_spins(c->n, seed, tmp);
        for (uint32_t i = 0; i < c->n; ++i) c->spins[i] = (float)tmp[i];
        free(tmp);
    }
    orc_recompute_fields(m, c->spins, c->hs, c->ht);
    orc_mt_seed(&c->rng, seed);
    c->e_run = orc_tempering_cost(m, c->spins, tau_scale);
    c->energy_block = (m->layers != 0 && m->per_layer != 0) ? m->per_layer : m->n_spins;
    return c;
}

void orc_chain_free(orc_chain* c) {
    if (!c) return;
    free(c->spins);
    free(c);
}

/* One uniform per spin in index order, accept iff u < p with NO min(1, .) clamp
 * (sweep_basic.cpp:27-50).  The reference pulls uniforms from 624-wide batches; the
 * stream is the same as one next_u32 per attempt. */
void orc_chain_sweep(orc_chain* c, const orc_model* m, uint64_t sweeps) {
    const float beta = c->beta, gamma = c->tau_scale;
    const uint32_t block = c->energy_block ? c->energy_block : c->n;
    for (uint64_t sw = 0; sw < sweeps; ++sw) {
        double e_block = 0.0; /* new: see orc_pt_run */
        for (uint32_t i = 0; i < c->n; ++i) {
            const float u = orc_u32_to_unit(orc_mt_next(&c->rng));
            const float s = c->spins[i];
            const float hs = c->hs[i], ht = c->ht[i];
            const float x = -beta * (2.0f * s * (hs + gamma * ht)); /* sweep_kernels.hpp:14-16 */
            const float p = orc_exp_kind(c->exp_kind, x);
            if (u < p) {
                const float two_s = 2.0f * s;
                const uint32_t end = m->offsets[i + 1], mid = end - m->tau_counts[i];
                for (uint32_t e = m->offsets[i]; e < mid; ++e)
                    c->hs[m->targets[e]] -= two_s * m->couplings[e];
                for (uint32_t e = mid; e < end; ++e)
                    c->ht[m->targets[e]] -= two_s * m->couplings[e];
                c->spins[i] = -s;
                ++c->flips;
                e_block += (double)(two_s * (hs + gamma * ht)); /* the inner factor of x above */
            }
            if ((i + 1) % block == 0 || i + 1 == c->n) {
                c->e_run += e_block;
                e_block = 0.0;
            }
        }
        c->attempts += c->n;
    }
}

/* ------------------------------------------------------------------ tempering driver */

typedef struct pt_job {
    const orc_model* const* models;
    uint32_t n_ladders, n_betas;
    const float* betas;
    const uint32_t* seeds;
    const uint32_t* swap_seeds;
    float tau_scale;
    int exp_kind;
    uint64_t sweeps;
    uint32_t swap_interval;
    const int8_t* initial;
    orc_pt_result* out;
    uint32_t next_ladder; /* shared work counter */
    pthread_mutex_t lock;
    int failed;
} pt_job;

static int run_ladder(pt_job* job, uint32_t l) {
    const uint32_t nb = job->n_betas;
    const orc_model* m = job->models[l];
    const uint32_t n = m->n_spins;
    orc_chain** ch = (orc_chain**)calloc(nb, sizeof *ch);
    uint32_t* at_slot = (uint32_t*)malloc(sizeof(uint32_t) * nb); /* chain holding slot k */
    uint32_t* slot_of = (uint32_t*)malloc(sizeof(uint32_t) * nb); /* slot of chain j */
    if (!ch || !at_slot || !slot_of) return -1;
    for (uint32_t k = 0; k < nb; ++k) {
        size_t c = (size_t)l * nb + k;
        ch[k] = orc_chain_create(m, job->seeds[c], job->betas[k], job->tau_scale, job->exp_kind,
                                 job->initial ? job->initial + c * n : NULL);
        if (!ch[k]) return -1;
        at_slot[k] = slot_of[k] = k;
    }
    orc_mt swap_rng;
    orc_mt_seed(&swap_rng, job->swap_seeds[l] ^ ORC_SWAP_SEED_MIX);
    orc_pt_result* out = job->out;
    uint64_t round = 0;
    for (uint64_t sw = 1; sw <= job->sweeps; ++sw) {
        for (uint32_t j = 0; j < nb; ++j) orc_chain_sweep(ch[j], m, 1);
        if (job->swap_interval == 0 || nb < 2 || sw % job->swap_interval != 0) continue;
        for (uint32_t k = (uint32_t)(round & 1u); k + 1 < nb; k += 2) {
            const uint32_t a = at_slot[k], b = at_slot[k + 1];
            const float u = orc_u32_to_unit(orc_mt_next(&swap_rng));
            const double arg =
                ((double)job->betas[k] - (double)job->betas[k + 1]) * (ch[a]->e_run - ch[b]->e_run);
            const float p = orc_exp_kind(job->exp_kind, (float)arg);
            if (out && out->swap_att) ++out->swap_att[(size_t)l * nb + k];
            if (u < p) {
                at_slot[k] = b;
                at_slot[k + 1] = a;
                slot_of[a] = k + 1;
                slot_of[b] = k;
                ch[a]->beta = job->betas[k + 1];
                ch[b]->beta = job->betas[k];
                if (out && out->swap_acc) ++out->swap_acc[(size_t)l * nb + k];
            }
        }
        ++round;
    }
    for (uint32_t j = 0; j < nb; ++j) {
        size_t c = (size_t)l * nb + j;
        if (out) {
            if (out->spins)
                for (uint32_t i = 0; i < n; ++i) out->spins[c * n + i] = ch[j]->spins[i] > 0 ? 1 : -1;
            if (out->flips) out->flips[c] = ch[j]->flips;
            if (out->e_run) out->e_run[c] = ch[j]->e_run;
            if (out->energy) out->energy[c] = orc_total_cost(m, ch[j]->spins);
            if (out->slot) out->slot[c] = slot_of[j];
        }
        orc_chain_free(ch[j]);
    }
    free(ch);
    free(at_slot);
    free(slot_of);
    return 0;
}

static void* pt_worker(void* arg) {
    pt_job* job = (pt_job*)arg;
    for (;;) {
        pthread_mutex_lock(&job->lock);
        uint32_t l = job->next_ladder++;
        pthread_mutex_unlock(&job->lock);
        if (l >= job->n_ladders) break;
        if (run_ladder(job, l) != 0) job->failed = 1;
    }
    return NULL;
}

int orc_pt_run(const orc_model* const* models, uint32_t n_ladders, uint32_t n_betas,
               const float* betas, const uint32_t* seeds, const uint32_t* swap_seeds,
               float tau_scale, int exp_kind, uint64_t sweeps, uint32_t swap_interval,
               uint32_t threads, const int8_t* initial, orc_pt_result* out) {
    if (!models || !betas || !seeds || n_betas == 0) return -1;
    if (n_betas > 1 && swap_interval > 0 && !swap_seeds) return -1;
    uint32_t* zero_seeds = NULL;
    if (!swap_seeds) {
        zero_seeds = (uint32_t*)calloc(n_ladders ? n_ladders : 1, sizeof(uint32_t));
        swap_seeds = zero_seeds;
    }
    pt_job job;
    memset(&job, 0, sizeof job);
    job.models = models;
    job.n_ladders = n_ladders;
    job.n_betas = n_betas;
    job.betas = betas;
    job.seeds = seeds;
    job.swap_seeds = swap_seeds;
    job.tau_scale = tau_scale;
    job.exp_kind = exp_kind;
    job.sweeps = sweeps;
    job.swap_interval = swap_interval;
    job.initial = initial;
    job.out = out;
    pthread_mutex_init(&job.lock, NULL);
    if (threads < 1) threads = 1;
    if (threads > n_ladders) threads = n_ladders ? n_ladders : 1;
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    for (uint32_t t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, pt_worker, &job);
    pt_worker(&job);
    for (uint32_t t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    free(tid);
    free(zero_seeds);
    pthread_mutex_destroy(&job.lock);
    return job.failed ? -1 : 0;
}


/* ======================================================================================
 * The coalesced schedule (ref: proj/src/sweep_coalesced.cpp).
 * ====================================================================================== */
orc_coalesced* orc_coalesced_create(const orc_model* m, uint32_t seed, float beta, float tau_scale,
                                    int exp_kind, const int8_t* initial) {
    if (m->layers < 4 || m->layers % 2 != 0 || (uint64_t)m->layers * m->per_layer != m->n_spins) return NULL;
    orc_coalesced* c = (orc_coalesced*)calloc(1, sizeof *c);
    if (!c) return NULL;
    const uint32_t n = m->n_spins, W = m->layers / 2, P = m->per_layer;
    c->n = n;
    c->lanes = W;
    c->per_layer = P;
    c->beta = beta;
    c->tau_scale = tau_scale;
    c->exp_kind = exp_kind;
    /* coalesce_permutation, model.cpp:190-215 */
    c->forward = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* inverse = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (uint32_t l = 0; l < m->layers; ++l) {
        for (uint32_t p = 0; p < P; ++p) {
            const uint32_t old_index = l * P + p, new_index = W * ((l % 2) * P + p) + l / 2;
            c->forward[old_index] = new_index;
            inverse[new_index] = old_index;
        }
    }
    /* apply_permutation, model.cpp:217-245: spin new_index takes the edge list of its old spin,
     * in the old order, with the targets renamed */
    orc_model* q = &c->permuted;
    const uint32_t edges = m->offsets[n];
    q->n_spins = n;
    q->layers = m->layers;
    q->per_layer = P;
    float* h = (float*)malloc(sizeof(float) * n);
    uint32_t* offsets = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    uint32_t* targets = (uint32_t*)malloc(sizeof(uint32_t) * (edges ? edges : 1));
    float* couplings = (float*)malloc(sizeof(float) * (edges ? edges : 1));
    uint8_t* tau_counts = (uint8_t*)malloc(n);
    uint32_t k = 0;
    for (uint32_t ni = 0; ni < n; ++ni) {
        const uint32_t oi = inverse[ni];
        h[ni] = m->h[oi];
        offsets[ni] = k;
        tau_counts[ni] = m->tau_counts ? m->tau_counts[oi] : 0;
        for (uint32_t e = m->offsets[oi]; e < m->offsets[oi + 1]; ++e) {
            targets[k] = c->forward[m->targets[e]];
            couplings[k] = m->couplings[e];
            ++k;
        }
    }
    offsets[n] = k;
    free(inverse);
    q->h = h;
    q->offsets = offsets;
    q->targets = targets;
    q->couplings = couplings;
    q->tau_counts = tau_counts;
    /* init_state on the permuted model: spins drawn / taken in the NEW order (sweep_state.cpp:218-234) */
    c->spins = (float*)malloc(sizeof(float) * 3 * (size_t)n);
    c->hs = c->spins + n;
    c->ht = c->hs + n;
    c->flags = (uint8_t*)calloc(n, 1);
    if (initial) {
        for (uint32_t i = 0; i < n; ++i) c->spins[i] = (float)initial[i];
    } else {
        int8_t* tmp = (int8_t*)malloc(n);
        orc_initial_spins(n, seed, tmp);
        for (uint32_t i = 0; i < n; ++i) c->spins[i] = (float)tmp[i];
        free(tmp);
    }
    orc_recompute_fields(q, c->spins, c->hs, c->ht);
    /* InterlacedMt::with_base_seed(seed, W): lane k is Mt19937(seed + k) (rng.cpp:144-148) */
    c->lane_rng = (orc_mt*)malloc(sizeof(orc_mt) * W);
    for (uint32_t t = 0; t < W; ++t) orc_mt_seed(&c->lane_rng[t], seed + t);
    return c;
}

void orc_coalesced_free(orc_coalesced* c) {
    if (!c) return;
    free((void*)c->permuted.h);
    free((void*)c->permuted.offsets);
    free((void*)c->permuted.targets);
    free((void*)c->permuted.couplings);
    free((void*)c->permuted.tau_counts);
    free(c->forward);
    free(c->spins);
    free(c->flags);
    free(c->lane_rng);
    free(c);
}

/* flip_phase, sweep_coalesced.cpp:45-83.  The uniform of (region, p, lane t) is output number
 * region*P + p of lane t's generator in this sweep (fill_unit_floats writes block b of all lanes
 * at [b*W, (b+1)*W), rng.hpp:51-53): drawing lane by lane in p order is the same stream. */
static void coalesced_flip_phase(orc_coalesced* c, uint32_t region_base) {
    const orc_model* q = &c->permuted;
    const uint32_t W = c->lanes, P = c->per_layer;
    for (uint32_t p = 0; p < P; ++p) {
        for (uint32_t t = 0; t < W; ++t) {
            const uint32_t i = region_base + W * p + t;
            const float u = orc_u32_to_unit(orc_mt_next(&c->lane_rng[t]));
            const float s = c->spins[i];
            const float x = -c->beta * (2.0f * s * (c->hs[i] + c->tau_scale * c->ht[i]));
            const float prob = orc_exp_kind(c->exp_kind, x);
            if (u < prob) {
                const float two_s = 2.0f * s;
                const uint32_t end = q->offsets[i + 1];
                for (uint32_t e = q->offsets[i]; e < end - 2; ++e) c->hs[q->targets[e]] -= two_s * q->couplings[e];
                c->ht[q->targets[end - 1]] -= two_s * q->couplings[end - 1]; /* previous layer now */
                c->spins[i] = -s;
                c->flags[i] = 1;
                ++c->flips;
            }
        }
    }
}

/* deferred_tau_phase, sweep_coalesced.cpp:87-104 */
static void coalesced_deferred_phase(orc_coalesced* c, uint32_t region_base) {
    const orc_model* q = &c->permuted;
    const uint32_t W = c->lanes, P = c->per_layer;
    for (uint32_t p = 0; p < P; ++p) {
        for (uint32_t t = 0; t < W; ++t) {
            const uint32_t i = region_base + W * p + t;
            if (!c->flags[i]) continue;
            const float two_s = -2.0f * c->spins[i]; /* twice the pre-flip spin */
            const uint32_t up = q->offsets[i + 1] - 2;
            c->ht[q->targets[up]] -= two_s * q->couplings[up];
        }
    }
}

void orc_coalesced_sweep(orc_coalesced* c, uint64_t sweeps) {
    const uint32_t odd_base = c->lanes * c->per_layer;
    for (uint64_t sw = 0; sw < sweeps; ++sw) {
        coalesced_flip_phase(c, 0);
        coalesced_deferred_phase(c, 0);
        coalesced_flip_phase(c, odd_base);
        coalesced_deferred_phase(c, odd_base);
        c->attempts += c->n;
        memset(c->flags, 0, c->n);
    }
}

void orc_coalesced_read_spins(const orc_coalesced* c, int8_t* out) {
    for (uint32_t i = 0; i < c->n; ++i) out[i] = c->spins[c->forward[i]] > 0.0f ? 1 : -1;
}
