// Generic-graph kernels: state lives in HBM in the replica-interleaved layout described in
// device_batch.hpp, one warp per tile of 32 chains, lane = chain.  Every chain follows the
// reference's scalar engine exactly (ref: proj/src/sweep_basic.cpp:12-56): spins in index
// order, one MT19937 draw per attempt, accept iff u < exp_kind(x) with no clamp, neighbour
// fields decremented by (2s)*J in adjacency order.
#include "device_batch.hpp"
#include "device_math.cuh"
#include "device_mt.cuh"

namespace isingb200 {

namespace {

constexpr int kWarpsPerBlock = 4;
constexpr int kThreads = kWarpsPerBlock * 32;

struct TileView {
    uint32_t tile, lane, chain;
    bool active;
    DevModel model;
    float* hs;
    float* ht;
    uint32_t* words;
    uint32_t* mt;
};

__device__ __forceinline__ bool open_tile(const DevBatch& b, TileView& t) {
    t.tile = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (t.tile >= b.n_tiles) return false;
    t.lane = threadIdx.x & 31u;
    t.active = t.lane < b.tile_count[t.tile];
    t.chain = b.tile_first[t.tile] + t.lane;
    t.model = b.models[b.tile_model[t.tile]];
    const size_t base = size_t(t.tile) * b.n_spins;
    t.hs = b.hs + base * 32 + t.lane;
    t.ht = b.ht ? b.ht + base * 32 + t.lane : nullptr;
    t.words = b.spin_bits + base;
    t.mt = b.mt + size_t(t.tile) * kMtN * 32 + t.lane;
    return true;
}

__device__ __forceinline__ float spin_of(uint32_t word, uint32_t lane) {
    return (word >> lane) & 1u ? -1.0f : 1.0f;
}

// ref: recompute_fields, sweep_state.cpp:236-255 — f32 sums in adjacency order, h_i first.
__device__ __forceinline__ void fields_of_spin(const DevModel& m, const uint32_t* words,
                                               uint32_t lane, uint32_t i, float& hs, float& ht) {
    const uint32_t end = m.offsets[i + 1], mid = end - m.tau_counts[i];
    float a = m.h[i];
    for (uint32_t e = m.offsets[i]; e < mid; ++e) {
        a = __fadd_rn(a, __fmul_rn(m.couplings[e], spin_of(words[m.targets[e]], lane)));
    }
    float c = 0.0f;
    for (uint32_t e = mid; e < end; ++e) {
        c = __fadd_rn(c, __fmul_rn(m.couplings[e], spin_of(words[m.targets[e]], lane)));
    }
    hs = a;
    ht = c;
}

// ref: total_cost, model.cpp:108-126 — f64, index order, each undirected edge once (t > i).
// The whole warp calls this for its tile: the terms come as a flat list in that order
// (DevModel::cost_terms); lane l fetches term l of each block of 32 and the two spin words it needs,
// one block ahead (terms two blocks ahead), and the block is then summed term by term from
// shuffles, every lane for its own chain.  (double(c) * s_i) * s_t is +-double(c) exactly, so a
// term is the coefficient with the sign bit of s_i * s_t.
__device__ double chain_cost(const DevModel& m, const uint4* term_list, const uint32_t* words, uint32_t lane) {
    const uint32_t blocks = m.n_cost_terms / 32;
    const uint4* terms = term_list + lane;
    const auto signs_of = [&](const uint4& term) {  // bit c: s_i * s_t < 0 in chain c
        const uint32_t wi = words[term.x];
        return term.y == kFieldTerm ? wi : wi ^ words[term.y];
    };
    double cost = 0.0;
    uint4 ahead = terms[0];
    uint32_t signs = signs_of(ahead);
    uint32_t coef = ahead.z;
    ahead = blocks > 1 ? terms[32] : ahead;
    for (uint32_t blk = 0; blk < blocks; ++blk) {
        const uint4 next = ahead;
        if (blk + 2 < blocks) ahead = terms[size_t(blk + 2) * 32];
        uint32_t next_signs = 0;
        if (blk + 1 < blocks) next_signs = signs_of(next);
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
            const uint32_t flip = (__shfl_sync(0xffffffffu, signs, k) >> lane) << 31;
            const float c = __uint_as_float(__shfl_sync(0xffffffffu, coef, k) ^ flip);
            cost = __dsub_rn(cost, double(c));
        }
        signs = next_signs;
        coef = next.z;
    }
    return cost;
}

// ref: state_checksum, sweep_state.cpp:325-336
__device__ unsigned long long chain_checksum(const uint32_t* words, uint32_t n, uint32_t lane) {
    unsigned long long h = 1469598103934665603ull;
    for (uint32_t i = 0; i < n; ++i) {
        h ^= (unsigned long long)(((words[i] >> lane) & 1u) ^ 1u);  // 1 for s > 0
        h *= 1099511628211ull;
    }
    return h;
}

// ---------------------------------------------------------------------------------------
// init_state for every chain of a tile (ref: sweep_state.cpp:160-234), in two launches: the spin
// words, generators and energies by one warp per tile, then the fields by one warp per (tile, spin).
__global__ void __launch_bounds__(kThreads) init_kernel(DevBatch b, const int8_t* initial) {
    TileView t;
    if (!open_tile(b, t)) return;
    const uint32_t n = b.n_spins;
    const uint32_t seed = t.active ? b.seeds[t.chain] : 0u;

    if (initial == nullptr) {
        // initial_spins(): a generator kept apart from the sweep stream, bit 31 -> -1
        mt_seed_lane(t.mt, 32, seed ^ kInitSpinSeedMix);
        MtLane g;
        g.open(t.mt, 32, 0);
        for (uint32_t i0 = 0; i0 < n; i0 += kChunk) {
            const uint32_t count = min(uint32_t(kChunk), n - i0);
            uint32_t raw[kChunk];
            g.next_chunk_raw(count, raw);
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                if (uint32_t(k) < count) {
                    const uint32_t word = __ballot_sync(0xffffffffu, t.active && (raw[k] >> 31));
                    if (t.lane == uint32_t(k)) t.words[i0 + k] = word;
                }
            }
        }
    } else {
        const int8_t* mine = initial + size_t(t.chain) * n;
        for (uint32_t i = 0; i < n; ++i) {
            const bool neg = t.active && mine[i] < 0;
            const uint32_t word = __ballot_sync(0xffffffffu, neg);
            if (t.lane == 0) t.words[i] = word;
        }
    }
    __syncwarp();
    mt_seed_lane(t.mt, 32, seed);
    if (t.lane == 0) b.mt_pos[t.tile] = 0;

    // the running energy of the tempering swap starts as the energy the sweeps sample (tau couplings
    // scaled by gamma: DevModel::tempering_terms)
    const double cost = chain_cost(t.model, t.model.tempering_terms, t.words, t.lane);
    if (t.active) {
        b.e_run[t.chain] = cost;
        b.flips[t.chain] = 0ull;
    }
}

__global__ void __launch_bounds__(256) init_fields_kernel(DevBatch b) {
    const size_t pair = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (pair >= size_t(b.n_tiles) * b.n_spins) return;
    const uint32_t tile = uint32_t(pair / b.n_spins), i = uint32_t(pair % b.n_spins), lane = threadIdx.x & 31u;
    float a, c;
    fields_of_spin(b.models[b.tile_model[tile]], b.spin_bits + size_t(tile) * b.n_spins, lane, i, a, c);
    b.hs[pair * 32 + lane] = a;
    if (b.ht) b.ht[pair * 32 + lane] = c;
}

// Swap generators: one thread per ladder.
__global__ void init_swap_kernel(DevBatch b) {
    const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= b.n_ladders) return;
    mt_seed_lane(b.swap_mt + l, b.n_ladders, b.swap_seeds[l] ^ kSwapSeedMix);
    b.swap_pos[l] = 0;
    for (uint32_t k = 0; k < b.n_betas; ++k) {
        b.chain_at_slot[size_t(l) * b.n_betas + k] = l * b.n_betas + k;
        b.slot_of_chain[size_t(l) * b.n_betas + k] = k;
        b.swap_acc[size_t(l) * b.n_betas + k] = 0ull;
        b.swap_att[size_t(l) * b.n_betas + k] = 0ull;
    }
}

// ---------------------------------------------------------------------------------------
// The sweep.  TAU selects models with tau edges (two field arrays); generic models keep
// h_eff_tau == +0 forever, and hs + gamma*(+0) only differs from hs in the sign of a zero,
// which no exp_kind can see, so the tau array is neither stored nor read for them.
// h[target] -= two_s * J for the edges [first, last) of a flipped spin, whose targets are distinct:
// groups of eight, loads before stores.  Every lane moves data, only accepting lanes change it.
__device__ __forceinline__ void flip_updates(float* field, const DevModel& m, uint32_t first, uint32_t last,
                                             float two_s, bool accept) {
    for (uint32_t e0 = first; e0 < last; e0 += 8) {
        size_t at[8];
        float coupling[8], value[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t e = min(e0 + q, last - 1);
            at[q] = size_t(__ldg(m.targets + e)) * 32;
            coupling[q] = __ldg(m.couplings + e);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) value[q] = field[at[q]];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (accept && e0 + q < last) field[at[q]] = __fsub_rn(value[q], __fmul_rn(two_s, coupling[q]));
        }
    }
}

template <int EXP, bool TAU>
__global__ void __launch_bounds__(kThreads) sweep_generic_kernel(DevBatch b, uint32_t sweeps) {
    TileView t;
    if (!open_tile(b, t)) return;
    const uint32_t n = b.n_spins;
    const DevModel& m = t.model;
    const float neg_beta = t.active ? -b.betas[b.slot_of_chain[t.chain]] : 0.0f;
    const float gamma = b.tau_scale;
    double e_run = t.active ? b.e_run[t.chain] : 0.0;
    // tempering definition (oracle/ising_oracle.h): the running energy receives one partial sum per
    // energy block of attempts (a layer of a layered model, else the sweep), summed from 0.0 in flip order
    double e_blk = 0.0;
    const uint32_t energy_block = t.model.energy_block;
    uint32_t blk_left = energy_block;
    unsigned long long flips = 0;
    const bool record_wait = b.wait_counts != nullptr && b.tile_count[t.tile] == 32;  // full tiles only
    uint32_t wait[6] = {0, 0, 0, 0, 0, 0};

    MtLane g;
    g.open(t.mt, 32, b.mt_pos[t.tile]);

    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t i0 = 0; i0 < n; i0 += kChunk) {
            const uint32_t count = min(uint32_t(kChunk), n - i0);
            float u[kChunk];
            uint32_t word[kChunk];
            g.next_chunk(count, u);
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                if (uint32_t(k) < count) word[k] = t.words[i0 + k];
            }
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                if (uint32_t(k) >= count) break;
                const uint32_t i = i0 + k;
                const float two_s = (word[k] >> t.lane) & 1u ? -2.0f : 2.0f;
                const float hsi = t.hs[size_t(i) * 32];
                float hti = 0.0f;
                float x;
                if constexpr (TAU) {
                    hti = t.ht[size_t(i) * 32];
                    x = flip_exponent(neg_beta, gamma, two_s, hsi, hti);
                } else {
                    x = __fmul_rn(neg_beta, __fmul_rn(two_s, hsi));
                }
                const float p = exp_kind<EXP>(x);
                const bool accept = t.active && (u[k] < p);
                const uint32_t ballot = __ballot_sync(0xffffffffu, accept);
                if (record_wait) wait_fold(ballot, wait);
                if (ballot != 0u) {
                    const uint32_t end = m.offsets[i + 1];
                    const uint32_t mid = TAU ? end - m.tau_counts[i] : end;
                    if (m.distinct_targets) {
                        // the neighbours of one spin are distinct: their fields are read together (one
                        // L2 round trip for up to eight instead of one each), then written together
                        flip_updates(t.hs, m, m.offsets[i], mid, two_s, accept);
                        if constexpr (TAU) flip_updates(t.ht, m, mid, end, two_s, accept);
                    } else {
                        for (uint32_t e = m.offsets[i]; e < mid; ++e) {
                            const size_t at = size_t(m.targets[e]) * 32;
                            const float d = __fmul_rn(two_s, m.couplings[e]);
                            if (accept) t.hs[at] = __fsub_rn(t.hs[at], d);
                        }
                        if constexpr (TAU) {
                            for (uint32_t e = mid; e < end; ++e) {
                                const size_t at = size_t(m.targets[e]) * 32;
                                const float d = __fmul_rn(two_s, m.couplings[e]);
                                if (accept) t.ht[at] = __fsub_rn(t.ht[at], d);
                            }
                        }
                    }
                    if (accept) {
                        ++flips;
                        e_blk = __dadd_rn(e_blk, double(__fmul_rn(two_s, __fadd_rn(hsi, __fmul_rn(gamma, hti)))));
                    }
                    if (t.lane == 0) t.words[i] = word[k] ^ ballot;
                }
                if (--blk_left == 0u) {
                    e_run = __dadd_rn(e_run, e_blk);
                    e_blk = 0.0;
                    blk_left = energy_block;
                }
            }
        }
        __syncwarp();  // lane 0's spin-word stores become visible to the whole warp
        if (record_wait) {  // flushed per sweep: the 32-bit partial counts cannot overflow (n < 2^27)
            unsigned long long* out = b.wait_counts + size_t(t.tile) * kWaitSlots;
#pragma unroll
            for (int w = 0; w < 6; ++w) {
                if (t.lane == 0) out[w] += wait[w];
                wait[w] = 0;
            }
            if (t.lane == 0) out[6] += n;
        }
    }

    if (t.lane == 0) b.mt_pos[t.tile] = g.pos;
    if (t.active) {
        b.e_run[t.chain] = e_run;
        b.flips[t.chain] += flips;
    }
}

// ---------------------------------------------------------------------------------------
// The same sweep for batches whose models are all DevModel::reduction_safe: a flip's updates
// h[t] -= (2s)*J go out as f32 reductions at L2 — h + (-(2s*J)) rounds exactly like the subtraction,
// reductions of one thread to one address apply in program order, and nothing has to come back, so a
// flip costs no round trip.  The fields are read past L1 (the reductions land in L2).  The chunk's
// eight own fields are requested together at the start of the chunk (DevModel::window) — every update
// of an earlier chunk precedes them in program order, and a flip inside the chunk patches the register
// copies of its in-chunk neighbours with the very subtraction its reduction performs.
__device__ __forceinline__ float ld_field(const float* p) {
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void reduce_field(float* p, float addend) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(addend) : "memory");
}
// The same under a (warp-uniform) predicate instead of a branch.
__device__ __forceinline__ void reduce_field_if(bool on, float* p, float addend) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.u32 p, %2, 0;\n"
        "@p red.global.add.f32 [%0], %1;\n"
        "}\n" ::"l"(p),
        "f"(addend), "r"(uint32_t(on))
        : "memory");
}

// ---------------------------------------------------------------------------------------
// Two warps per tile.  The PRODUCER warp runs ahead and fills a ring of
// shared-memory stages, one per chunk of eight attempts, with everything that does not depend on the
// chain's state: the eight uniform draws of every lane, and (warp-uniform) each attempt's first eight
// edges, its window couplings and its edge counts.  The SWEEP warp keeps the state: spin words, own
// fields, decisions, reductions, bookkeeping — about a third of the instructions of a one-warp
// version (2.2x slower on c3), on a path that is one in-order warp's instruction latency.  Stages change hands through a
// pair of mbarriers each (full: producer -> sweep, empty: sweep -> producer).
constexpr int kSplitStages = 4;
constexpr int kSplitThreads = 64;
struct SplitStage {
    float u[kChunk][32];
    uint32_t target[kChunk][8];
    float coupling[kChunk][8];
    float near[kChunk][8];
    uint32_t degree[kChunk];  // edges of attempt k
    uint32_t space[kChunk];   // the first `space` of them update h_eff_space, the rest h_eff_tau
    uint32_t first[kChunk];   // CSR offset of attempt k's edges (degree > 8: the tail is read from there)
    uint32_t pad[kChunk];
};

__device__ __forceinline__ uint32_t split_smem(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void split_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(split_smem(bar)) : "memory");
}
__device__ __forceinline__ void split_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done)
            : "r"(split_smem(bar)), "r"(parity)
            : "memory");
    } while (done == 0u);
}

template <bool TAU>
__device__ void split_producer(const DevBatch& b, const TileView& t, uint32_t sweeps, SplitStage* stages,
                               uint64_t* full, uint64_t* empty) {
    const uint32_t n = b.n_spins;
    const DevModel& m = t.model;
    const bool window = m.window != nullptr;
    MtLane g;
    g.open(t.mt, 32, b.mt_pos[t.tile]);
    uint32_t mt_next[kChunk], mt_far[kChunk];
    g.load_operands(min(uint32_t(kChunk), n), mt_next, mt_far);
    // lane l <= 8 keeps offsets[i0 + l] of the chunk, requested one chunk ahead
    uint32_t off_ahead = t.lane <= min(uint32_t(kChunk), n) ? __ldg(m.offsets + t.lane) : 0u;
    uint32_t chunk = 0;
    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t i0 = 0; i0 < n; i0 += kChunk, ++chunk) {
            const uint32_t count = min(uint32_t(kChunk), n - i0);
            const uint32_t i0_ahead = i0 + kChunk < n ? i0 + kChunk : 0u;
            const uint32_t st = chunk % kSplitStages;
            SplitStage& stage = stages[st];
            float u[kChunk];
            g.generate(count, mt_next, mt_far, u);
            g.load_operands(min(uint32_t(kChunk), n - i0_ahead), mt_next, mt_far);
            const uint32_t off_mine = off_ahead;
            off_ahead = t.lane <= min(uint32_t(kChunk), n - i0_ahead) ? __ldg(m.offsets + i0_ahead + t.lane) : 0u;
            // (attempt, edge) pairs: this lane fills (lane / 8, lane % 8) and (lane / 8 + 4, lane % 8)
            uint32_t tg[2];
            float cp[2], nr[2];
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const uint32_t k = (t.lane >> 3) + 4u * half, q = t.lane & 7u;
                const uint32_t lo = __shfl_sync(0xffffffffu, off_mine, k);
                const uint32_t hi = __shfl_sync(0xffffffffu, off_mine, k + 1);
                const bool have = k < count && lo + q < hi;
                tg[half] = have ? __ldg(m.targets + lo + q) : 0u;
                cp[half] = have ? __ldg(m.couplings + lo + q) : 0.0f;
                nr[half] = (window && k < count) ? __ldg(m.window + size_t(i0 + k) * 8 + q) : 0.0f;
            }
            uint32_t degree = 0, space = 0;
            {
                const uint32_t hi = __shfl_sync(0xffffffffu, off_mine, min(t.lane + 1, uint32_t(kChunk)));
                if (t.lane < count) {
                    degree = hi - off_mine;
                    space = TAU ? degree - m.tau_counts[i0 + t.lane] : degree;
                }
            }
            if (chunk >= uint32_t(kSplitStages)) split_wait(&empty[st], ((chunk / kSplitStages) - 1u) & 1u);
#pragma unroll
            for (int k = 0; k < kChunk; ++k) stage.u[k][t.lane] = u[k];
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const uint32_t k = (t.lane >> 3) + 4u * half, q = t.lane & 7u;
                stage.target[k][q] = tg[half];
                stage.coupling[k][q] = cp[half];
                stage.near[k][q] = nr[half];
            }
            if (t.lane < uint32_t(kChunk)) {
                stage.degree[t.lane] = degree;
                stage.space[t.lane] = space;
                stage.first[t.lane] = off_mine;
            }
            split_arrive(&full[st]);
        }
    }
    if (t.lane == 0) b.mt_pos[t.tile] = g.pos;
}

template <int EXP, bool TAU>
__device__ void split_sweep(const DevBatch& b, const TileView& t, uint32_t sweeps, const SplitStage* stages,
                            uint64_t* full, uint64_t* empty) {
    const uint32_t n = b.n_spins;
    const DevModel& m = t.model;
    const float neg_beta = t.active ? -b.betas[b.slot_of_chain[t.chain]] : 0.0f;
    const float gamma = b.tau_scale;
    double e_run = t.active ? b.e_run[t.chain] : 0.0;
    // tempering definition (oracle/ising_oracle.h): the running energy receives one partial sum per
    // energy block of attempts (a layer of a layered model, else the sweep), summed from 0.0 in flip order
    double e_blk = 0.0;
    const uint32_t energy_block = t.model.energy_block;
    uint32_t blk_left = energy_block;
    unsigned long long flips = 0;
    const bool record_wait = b.wait_counts != nullptr && b.tile_count[t.tile] == 32;  // full tiles only
    uint32_t wait[6] = {0, 0, 0, 0, 0, 0};
    const bool window = m.window != nullptr;
    uint32_t chunk = 0;
    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t i0 = 0; i0 < n; i0 += kChunk, ++chunk) {
            const uint32_t count = min(uint32_t(kChunk), n - i0);
            const uint32_t st = chunk % kSplitStages;
            const SplitStage& stage = stages[st];
            float own[kChunk], own_tau[kChunk], u[kChunk];
            uint32_t word[kChunk];
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                if (uint32_t(k) < count) {
                    word[k] = t.words[i0 + k];
                    if (window) {
                        own[k] = ld_field(t.hs + size_t(i0 + k) * 32);
                        if constexpr (TAU) own_tau[k] = ld_field(t.ht + size_t(i0 + k) * 32);
                    }
                }
            }
            split_wait(&full[st], (chunk / kSplitStages) & 1u);
#pragma unroll
            for (int k = 0; k < kChunk; ++k) u[k] = stage.u[k][t.lane];
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                if (uint32_t(k) >= count) break;
                const uint32_t i = i0 + k;
                // warp-uniform operands of this attempt, ahead of the decision
                const uint4 tg_lo = *reinterpret_cast<const uint4*>(&stage.target[k][0]);
                const uint4 tg_hi = *reinterpret_cast<const uint4*>(&stage.target[k][4]);
                const float4 cp_lo = *reinterpret_cast<const float4*>(&stage.coupling[k][0]);
                const float4 cp_hi = *reinterpret_cast<const float4*>(&stage.coupling[k][4]);
                const float4 nr_lo = *reinterpret_cast<const float4*>(&stage.near[k][0]);
                const float4 nr_hi = *reinterpret_cast<const float4*>(&stage.near[k][4]);
                const uint32_t degree = stage.degree[k], space = stage.space[k];
                const float two_s = (word[k] >> t.lane) & 1u ? -2.0f : 2.0f;
                const float hsi = window ? own[k] : ld_field(t.hs + size_t(i) * 32);
                float hti = 0.0f;
                float x;
                if constexpr (TAU) {
                    hti = window ? own_tau[k] : ld_field(t.ht + size_t(i) * 32);
                    x = flip_exponent(neg_beta, gamma, two_s, hsi, hti);
                } else {
                    x = __fmul_rn(neg_beta, __fmul_rn(two_s, hsi));
                }
                const float p = exp_kind<EXP>(x);
                const bool accept = t.active && (u[k] < p);
                const uint32_t ballot = __ballot_sync(0xffffffffu, accept);
                if (record_wait) wait_fold(ballot, wait);
                if (ballot != 0u) {
                    const uint32_t target[8] = {tg_lo.x, tg_lo.y, tg_lo.z, tg_lo.w, tg_hi.x, tg_hi.y, tg_hi.z, tg_hi.w};
                    const float coupling[8] = {cp_lo.x, cp_lo.y, cp_lo.z, cp_lo.w, cp_hi.x, cp_hi.y, cp_hi.z, cp_hi.w};
                    const float near[8] = {nr_lo.x, nr_lo.y, nr_lo.z, nr_lo.w, nr_hi.x, nr_hi.y, nr_hi.z, nr_hi.w};
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float* field = (!TAU || uint32_t(q) < space) ? t.hs : t.ht;
                        // every lane takes part (a lane that did not accept adds -0.0, the identity for
                        // every bit pattern), so the warp does not diverge once per edge
                        if (uint32_t(q) < degree) {
                            reduce_field(field + size_t(target[q]) * 32, accept ? __fmul_rn(-two_s, coupling[q]) : -0.0f);
                        }
                    }
                    if (degree > 8u) {
                        const uint32_t first = stage.first[k];
                        for (uint32_t e = 8; e < degree; ++e) {
                            float* field = (!TAU || e < space) ? t.hs : t.ht;
                            const size_t at = size_t(__ldg(m.targets + first + e)) * 32;
                            const float d = __fmul_rn(-two_s, __ldg(m.couplings + first + e));
                            reduce_field(field + at, accept ? d : -0.0f);
                        }
                    }
#pragma unroll
                    for (int q = 1; k + q < kChunk; ++q) {
                        own[k + q] = accept ? __fsub_rn(own[k + q], __fmul_rn(two_s, near[q])) : own[k + q];
                    }
                    if (accept) {
                        ++flips;
                        e_blk = __dadd_rn(e_blk, double(__fmul_rn(two_s, __fadd_rn(hsi, __fmul_rn(gamma, hti)))));
                    }
                    if (t.lane == 0) t.words[i] = word[k] ^ ballot;
                }
                if (--blk_left == 0u) {
                    e_run = __dadd_rn(e_run, e_blk);
                    e_blk = 0.0;
                    blk_left = energy_block;
                }
            }
            split_arrive(&empty[st]);
        }
        __syncwarp();  // lane 0's spin-word stores become visible to the whole warp
        if (record_wait) {  // flushed per sweep: the 32-bit partial counts cannot overflow (n < 2^27)
            unsigned long long* out = b.wait_counts + size_t(t.tile) * kWaitSlots;
#pragma unroll
            for (int w = 0; w < 6; ++w) {
                if (t.lane == 0) out[w] += wait[w];
                wait[w] = 0;
            }
            if (t.lane == 0) out[6] += n;
        }
    }
    if (t.active) {
        b.e_run[t.chain] = e_run;
        b.flips[t.chain] += flips;
    }
}

template <int EXP, bool TAU>
__global__ void __launch_bounds__(kSplitThreads) sweep_split_kernel(DevBatch b, uint32_t sweeps) {
    __shared__ __align__(16) SplitStage stages[kSplitStages];
    __shared__ __align__(8) uint64_t bars[2 * kSplitStages];
    TileView t;
    t.tile = blockIdx.x;
    t.lane = threadIdx.x & 31u;
    t.active = t.lane < b.tile_count[t.tile];
    t.chain = b.tile_first[t.tile] + t.lane;
    t.model = b.models[b.tile_model[t.tile]];
    const size_t base = size_t(t.tile) * b.n_spins;
    t.hs = b.hs + base * 32 + t.lane;
    t.ht = b.ht ? b.ht + base * 32 + t.lane : nullptr;
    t.words = b.spin_bits + base;
    t.mt = b.mt + size_t(t.tile) * kMtN * 32 + t.lane;
    if (threadIdx.x < 2 * kSplitStages) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(split_smem(&bars[threadIdx.x])), "r"(32) : "memory");
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        split_sweep<EXP, TAU>(b, t, sweeps, stages, bars, bars + kSplitStages);
    } else {
        split_producer<TAU>(b, t, sweeps, stages, bars, bars + kSplitStages);
    }
}

// ---------------------------------------------------------------------------------------
// Three warps per tile, for batches in which every model has an own-field window.  The reductions and
// the own-field loads are the two kinds of access whose order matters (a load must come after every
// reduction that can reach it), so both move to one thread each lane: the REDUCER warp.  The sweep
// warp publishes every decision (the ballot, and which of the accepting lanes held s = -1) through a
// 16-slot ring with one mbarrier per slot; the reducer issues that attempt's reductions, and after the
// last attempt of a chunk requests the next chunk's own fields and hands them back through shared
// memory.  The sweep warp is left with the decision, the in-chunk patches and the bookkeeping.
constexpr int kTrioThreads = 96;
struct TrioShared {
    SplitStage stages[kSplitStages];
    float own[2][kChunk][32];
    float own_tau[2][kChunk][32];
    uint2 decided[2 * kChunk];
    uint64_t full[kSplitStages], empty[kSplitStages];
    uint64_t decided_bar[2 * kChunk];
    uint64_t own_bar[2];
};

template <int EXP, bool TAU>
__device__ void trio_sweep(const DevBatch& b, const TileView& t, uint32_t sweeps, TrioShared& sh) {
    const uint32_t n = b.n_spins;
    const float neg_beta = t.active ? -b.betas[b.slot_of_chain[t.chain]] : 0.0f;
    const float gamma = b.tau_scale;
    double e_run = t.active ? b.e_run[t.chain] : 0.0;
    // tempering definition (oracle/ising_oracle.h): the running energy receives one partial sum per
    // energy block of attempts (a layer of a layered model, else the sweep), summed from 0.0 in flip order
    double e_blk = 0.0;
    const uint32_t energy_block = t.model.energy_block;
    uint32_t blk_left = energy_block;
    unsigned long long flips = 0;
    const bool record_wait = b.wait_counts != nullptr && b.tile_count[t.tile] == 32;  // full tiles only
    uint32_t wait[6] = {0, 0, 0, 0, 0, 0};
    uint32_t chunk = 0;
    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t i0 = 0; i0 < n; i0 += kChunk, ++chunk) {
            const uint32_t count = min(uint32_t(kChunk), n - i0);
            const uint32_t st = chunk % kSplitStages, half = chunk & 1u, phase = (chunk >> 1) & 1u;
            const SplitStage& stage = sh.stages[st];
            float own[kChunk], own_tau[kChunk], u[kChunk];
            uint32_t word[kChunk];
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                if (uint32_t(k) < count) word[k] = t.words[i0 + k];
            }
            split_wait(&sh.own_bar[half], phase);
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                own[k] = sh.own[half][k][t.lane];
                if constexpr (TAU) own_tau[k] = sh.own_tau[half][k][t.lane];
            }
            split_wait(&sh.full[st], (chunk / kSplitStages) & 1u);
#pragma unroll
            for (int k = 0; k < kChunk; ++k) u[k] = stage.u[k][t.lane];
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                const uint32_t slot = half * kChunk + k;
                if (uint32_t(k) >= count) {  // keep every slot's barrier in step with the chunk count
                    if (t.lane == 0) split_arrive(&sh.decided_bar[slot]);
                    continue;
                }
                const uint32_t i = i0 + k;
                const float4 nr_lo = *reinterpret_cast<const float4*>(&stage.near[k][0]);
                const float4 nr_hi = *reinterpret_cast<const float4*>(&stage.near[k][4]);
                const float two_s = (word[k] >> t.lane) & 1u ? -2.0f : 2.0f;
                const float hsi = own[k];
                float hti = 0.0f;
                float x;
                if constexpr (TAU) {
                    hti = own_tau[k];
                    x = flip_exponent(neg_beta, gamma, two_s, hsi, hti);
                } else {
                    x = __fmul_rn(neg_beta, __fmul_rn(two_s, hsi));
                }
                const float p = exp_kind<EXP>(x);
                const bool accept = t.active && (u[k] < p);
                const uint32_t ballot = __ballot_sync(0xffffffffu, accept);
                if (t.lane == 0) {
                    sh.decided[slot] = make_uint2(ballot, ballot & word[k]);
                    split_arrive(&sh.decided_bar[slot]);
                }
                if (record_wait) wait_fold(ballot, wait);
                if (ballot != 0u) {
                    const float near[8] = {nr_lo.x, nr_lo.y, nr_lo.z, nr_lo.w, nr_hi.x, nr_hi.y, nr_hi.z, nr_hi.w};
#pragma unroll
                    for (int q = 1; k + q < kChunk; ++q) {
                        own[k + q] = accept ? __fsub_rn(own[k + q], __fmul_rn(two_s, near[q])) : own[k + q];
                    }
                    if (accept) {
                        ++flips;
                        e_blk = __dadd_rn(e_blk, double(__fmul_rn(two_s, __fadd_rn(hsi, __fmul_rn(gamma, hti)))));
                    }
                    if (t.lane == 0) t.words[i] = word[k] ^ ballot;
                }
                if (--blk_left == 0u) {
                    e_run = __dadd_rn(e_run, e_blk);
                    e_blk = 0.0;
                    blk_left = energy_block;
                }
            }
            split_arrive(&sh.empty[st]);
        }
        __syncwarp();  // lane 0's spin-word stores become visible to the whole warp
        if (record_wait) {  // flushed per sweep: the 32-bit partial counts cannot overflow (n < 2^27)
            unsigned long long* out = b.wait_counts + size_t(t.tile) * kWaitSlots;
#pragma unroll
            for (int w = 0; w < 6; ++w) {
                if (t.lane == 0) out[w] += wait[w];
                wait[w] = 0;
            }
            if (t.lane == 0) out[6] += n;
        }
    }
    if (t.active) {
        b.e_run[t.chain] = e_run;
        b.flips[t.chain] += flips;
    }
}

template <bool TAU>
__device__ void trio_reducer(const DevBatch& b, const TileView& t, uint32_t sweeps, TrioShared& sh) {
    const uint32_t n = b.n_spins;
    const DevModel& m = t.model;
    const uint32_t chunks_per_sweep = (n + kChunk - 1) / kChunk;
    const uint32_t total_chunks = chunks_per_sweep * sweeps;
    // the own fields of chunk `c` (first spin `first`), requested after every reduction issued so far
    const auto hand_over = [&](uint32_t c, uint32_t first) {
        const uint32_t cnt = min(uint32_t(kChunk), n - first), half = c & 1u;
        float own[kChunk], own_tau[kChunk];
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
            own[k] = uint32_t(k) < cnt ? ld_field(t.hs + size_t(first + k) * 32) : 0.0f;
            if constexpr (TAU) own_tau[k] = uint32_t(k) < cnt ? ld_field(t.ht + size_t(first + k) * 32) : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
            sh.own[half][k][t.lane] = own[k];
            if constexpr (TAU) sh.own_tau[half][k][t.lane] = own_tau[k];
        }
        split_arrive(&sh.own_bar[half]);
    };
    if (total_chunks != 0) hand_over(0, 0);
    uint32_t chunk = 0;
    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t i0 = 0; i0 < n; i0 += kChunk, ++chunk) {
            const uint32_t count = min(uint32_t(kChunk), n - i0);
            const uint32_t st = chunk % kSplitStages, half = chunk & 1u, phase = (chunk >> 1) & 1u;
            const SplitStage& stage = sh.stages[st];
            split_wait(&sh.full[st], (chunk / kSplitStages) & 1u);
#pragma unroll 1
            for (uint32_t k = 0; k < count; ++k) {
                const uint32_t slot = half * kChunk + k;
                // the attempt's operands are in the stage already: requested before the wait for its decision
                const uint4 tg_lo = *reinterpret_cast<const uint4*>(&stage.target[k][0]);
                const uint4 tg_hi = *reinterpret_cast<const uint4*>(&stage.target[k][4]);
                const float4 cp_lo = *reinterpret_cast<const float4*>(&stage.coupling[k][0]);
                const float4 cp_hi = *reinterpret_cast<const float4*>(&stage.coupling[k][4]);
                const uint32_t degree = stage.degree[k];
                const uint32_t space = stage.space[k];
                split_wait(&sh.decided_bar[slot], phase);
                const uint2 decision = sh.decided[slot];
                if (decision.x == 0u) continue;
                const bool accept = (decision.x >> t.lane) & 1u;
                const float minus_two_s = (decision.y >> t.lane) & 1u ? 2.0f : -2.0f;
                const uint32_t target[8] = {tg_lo.x, tg_lo.y, tg_lo.z, tg_lo.w, tg_hi.x, tg_hi.y, tg_hi.z, tg_hi.w};
                const float coupling[8] = {cp_lo.x, cp_lo.y, cp_lo.z, cp_lo.w, cp_hi.x, cp_hi.y, cp_hi.z, cp_hi.w};
                // addresses and addends first, then the eight reductions back to back (a lane that did
                // not accept adds -0.0, the identity for every bit pattern: full 128-byte reductions, no
                // divergence; past the spin's last edge the reduction is predicated off)
                float* at[8];
                float addend[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    at[q] = ((!TAU || uint32_t(q) < space) ? t.hs : t.ht) + size_t(target[q]) * 32;
                    addend[q] = accept ? __fmul_rn(minus_two_s, coupling[q]) : -0.0f;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) reduce_field_if(uint32_t(q) < degree, at[q], addend[q]);
                if (degree > 8u) {
                    const uint32_t first = stage.first[k];
                    for (uint32_t e = 8; e < degree; ++e) {
                        float* field = (!TAU || e < space) ? t.hs : t.ht;
                        const size_t at = size_t(__ldg(m.targets + first + e)) * 32;
                        const float d = __fmul_rn(minus_two_s, __ldg(m.couplings + first + e));
                        reduce_field(field + at, accept ? d : -0.0f);
                    }
                }
            }
            split_arrive(&sh.empty[st]);
            if (chunk + 1 < total_chunks) hand_over(chunk + 1, i0 + kChunk < n ? i0 + kChunk : 0u);
        }
    }
}

template <int EXP, bool TAU>
__global__ void __launch_bounds__(kTrioThreads) sweep_trio_kernel(DevBatch b, uint32_t sweeps) {
    __shared__ __align__(16) TrioShared sh;
    TileView t;
    t.tile = blockIdx.x;
    t.lane = threadIdx.x & 31u;
    t.active = t.lane < b.tile_count[t.tile];
    t.chain = b.tile_first[t.tile] + t.lane;
    t.model = b.models[b.tile_model[t.tile]];
    const size_t base = size_t(t.tile) * b.n_spins;
    t.hs = b.hs + base * 32 + t.lane;
    t.ht = b.ht ? b.ht + base * 32 + t.lane : nullptr;
    t.words = b.spin_bits + base;
    t.mt = b.mt + size_t(t.tile) * kMtN * 32 + t.lane;
    const auto init = [](uint64_t* bar, uint32_t count) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(split_smem(bar)), "r"(count) : "memory");
    };
    if (threadIdx.x < kSplitStages) {
        init(&sh.full[threadIdx.x], 32);
        init(&sh.empty[threadIdx.x], 64);  // the sweep warp and the reducer both read a stage
    }
    if (threadIdx.x < 2 * kChunk) init(&sh.decided_bar[threadIdx.x], 1);
    if (threadIdx.x < 2) init(&sh.own_bar[threadIdx.x], 32);
    __syncthreads();
    const uint32_t role = threadIdx.x >> 5;
    if (role == 0) {
        trio_sweep<EXP, TAU>(b, t, sweeps, sh);
    } else if (role == 1) {
        split_producer<TAU>(b, t, sweeps, sh.stages, sh.full, sh.empty);
    } else {
        trio_reducer<TAU>(b, t, sweeps, sh);
    }
}

// ---------------------------------------------------------------------------------------
// Tempering swap round (new semantics, oracle/ising_oracle.h): pairs of
// slots (k,k+1), k = round&1, +2, ...; one draw per pair from the ladder's own generator;
// accept iff u < exp_kind(float((beta_k - beta_k1) * (E_a - E_b))); the chains exchange slots.
__global__ void swap_kernel(DevBatch b, unsigned long long round) {
    const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= b.n_ladders) return;
    const uint32_t nb = b.n_betas;
    MtLane g;
    g.open(b.swap_mt + l, b.n_ladders, b.swap_pos[l]);
    uint32_t* at_slot = b.chain_at_slot + size_t(l) * nb;
    for (uint32_t k = uint32_t(round & 1ull); k + 1 < nb; k += 2) {
        const uint32_t ca = at_slot[k], cb = at_slot[k + 1];
        const float u = u32_to_unit(g.next_raw());
        const double db = __dsub_rn(double(b.betas[k]), double(b.betas[k + 1]));
        const double de = __dsub_rn(b.e_run[ca], b.e_run[cb]);
        const float p = exp_kind_dyn(b.exp_kind, __double2float_rn(__dmul_rn(db, de)));
        ++b.swap_att[size_t(l) * nb + k];
        if (u < p) {
            at_slot[k] = cb;
            at_slot[k + 1] = ca;
            b.slot_of_chain[ca] = k + 1;
            b.slot_of_chain[cb] = k;
            ++b.swap_acc[size_t(l) * nb + k];
        }
    }
    b.swap_pos[l] = g.pos;
}

// ---------------------------------------------------------------------------------------
// Readout.
__global__ void __launch_bounds__(kThreads) energies_kernel(DevBatch b, double* out) {
    TileView t;
    if (!open_tile(b, t)) return;
    const double cost = chain_cost(t.model, t.model.cost_terms, t.words, t.lane);  // the whole warp, see chain_cost
    if (t.active) out[t.chain] = cost;
}

__global__ void __launch_bounds__(kThreads) resync_energies_kernel(DevBatch b) {
    TileView t;
    if (!open_tile(b, t)) return;
    const double cost = chain_cost(t.model, t.model.tempering_terms, t.words, t.lane);  // as init_kernel does
    if (t.active) b.e_run[t.chain] = cost;
}

__global__ void __launch_bounds__(kThreads) checksums_kernel(DevBatch b, unsigned long long* out) {
    TileView t;
    if (!open_tile(b, t) || !t.active) return;
    out[t.chain] = chain_checksum(t.words, b.n_spins, t.lane);
}

// ref: field_coherence_ulp / ulp_distance, sweep_state.cpp:338-354
__device__ __forceinline__ long long ulp_key(float v) {
    const int bits = __float_as_int(v);
    return bits < 0 ? 0x80000000ll - (long long)bits : (long long)bits;
}

__global__ void __launch_bounds__(kThreads) coherence_kernel(DevBatch b, unsigned long long* out) {
    TileView t;
    if (!open_tile(b, t) || !t.active) return;
    unsigned long long worst = 0;
    for (uint32_t i = 0; i < b.n_spins; ++i) {
        float a, c;
        fields_of_spin(t.model, t.words, t.lane, i, a, c);
        const long long d1 = llabs(ulp_key(t.hs[size_t(i) * 32]) - ulp_key(a));
        const long long d2 = t.ht ? llabs(ulp_key(t.ht[size_t(i) * 32]) - ulp_key(c)) : 0ll;
        worst = max(worst, (unsigned long long)max(d1, d2));
    }
    out[t.chain] = worst;
}

__global__ void unpack_spins_kernel(DevBatch b, uint32_t first_chain, uint32_t n_chains,
                                    int8_t* out) {
    const size_t idx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t total = size_t(n_chains) * b.n_spins;
    if (idx >= total) return;
    const uint32_t c = first_chain + uint32_t(idx / b.n_spins);
    const uint32_t i = uint32_t(idx % b.n_spins);
    const uint32_t loc = b.chain_loc[c];
    const uint32_t word = b.spin_bits[size_t(loc >> 5) * b.n_spins + i];
    out[idx] = (word >> (loc & 31u)) & 1u ? int8_t(-1) : int8_t(1);
}

__global__ void gather_fields_kernel(DevBatch b, uint32_t chain, float* hs, float* ht) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= b.n_spins) return;
    const uint32_t loc = b.chain_loc[chain];
    const size_t at = (size_t(loc >> 5) * b.n_spins + i) * 32 + (loc & 31u);
    hs[i] = b.hs[at];
    if (b.ht) {
        ht[i] = b.ht[at];
    } else {
        // not stored (generic graphs: identically zero; layered family: rebuilt exactly from spins)
        float a, c;
        fields_of_spin(b.models[b.tile_model[loc >> 5]], b.spin_bits + size_t(loc >> 5) * b.n_spins, loc & 31u,
                       i, a, c);
        ht[i] = c;
    }
}

struct ResultRecord {  // 32 bytes per chain, see ising_batch_pack_results
    double energy;
    double e_run;
    unsigned long long flips;
    unsigned long long checksum;
};

__global__ void __launch_bounds__(kThreads) pack_results_kernel(DevBatch b, ResultRecord* out) {
    TileView t;
    if (!open_tile(b, t)) return;
    ResultRecord r;
    r.energy = chain_cost(t.model, t.model.cost_terms, t.words, t.lane);  // the whole warp, see chain_cost
    if (!t.active) return;
    r.e_run = b.e_run[t.chain];
    r.flips = b.flips[t.chain];
    r.checksum = chain_checksum(t.words, b.n_spins, t.lane);
    out[t.chain] = r;
}

inline dim3 tile_grid(const DevBatch& b) { return dim3((b.n_tiles + kWarpsPerBlock - 1) / kWarpsPerBlock); }

template <int EXP>
void launch_sweep_exp(const DevBatch& b, uint32_t sweeps, cudaStream_t s) {
    if (b.generic_reduce && b.generic_windows && b.n_tiles != 0) {
        if (b.ht) sweep_trio_kernel<EXP, true><<<b.n_tiles, kTrioThreads, 0, s>>>(b, sweeps);
        else sweep_trio_kernel<EXP, false><<<b.n_tiles, kTrioThreads, 0, s>>>(b, sweeps);
    } else if (b.generic_reduce && b.n_tiles != 0) {
        if (b.ht) sweep_split_kernel<EXP, true><<<b.n_tiles, kSplitThreads, 0, s>>>(b, sweeps);
        else sweep_split_kernel<EXP, false><<<b.n_tiles, kSplitThreads, 0, s>>>(b, sweeps);
    } else if (b.ht) {
        sweep_generic_kernel<EXP, true><<<tile_grid(b), kThreads, 0, s>>>(b, sweeps);
    } else {
        sweep_generic_kernel<EXP, false><<<tile_grid(b), kThreads, 0, s>>>(b, sweeps);
    }
}

}  // namespace

cudaError_t launch_init(const DevBatch& b, const int8_t* initial, cudaStream_t s) {
    init_kernel<<<tile_grid(b), kThreads, 0, s>>>(b, initial);
    const size_t field_threads = size_t(b.n_tiles) * b.n_spins * 32;
    if (field_threads) init_fields_kernel<<<unsigned((field_threads + 255) / 256), 256, 0, s>>>(b);
    init_swap_kernel<<<(b.n_ladders + 127) / 128, 128, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t launch_sweep_generic(const DevBatch& b, uint32_t sweeps, cudaStream_t s) {
    switch (b.exp_kind) {
        case kExpExact: launch_sweep_exp<kExpExact>(b, sweeps, s); break;
        case kExpFast: launch_sweep_exp<kExpFast>(b, sweeps, s); break;
        default: launch_sweep_exp<kExpAccurate>(b, sweeps, s); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_swap(const DevBatch& b, uint64_t round, cudaStream_t s) {
    swap_kernel<<<(b.n_ladders + 127) / 128, 128, 0, s>>>(b, round);
    return cudaGetLastError();
}

cudaError_t launch_resync_energies(const DevBatch& b, cudaStream_t s) {
    resync_energies_kernel<<<tile_grid(b), kThreads, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t launch_energies(const DevBatch& b, double* out, cudaStream_t s) {
    energies_kernel<<<tile_grid(b), kThreads, 0, s>>>(b, out);
    return cudaGetLastError();
}

cudaError_t launch_checksums(const DevBatch& b, unsigned long long* out, cudaStream_t s) {
    checksums_kernel<<<tile_grid(b), kThreads, 0, s>>>(b, out);
    return cudaGetLastError();
}

cudaError_t launch_coherence(const DevBatch& b, unsigned long long* out, cudaStream_t s) {
    coherence_kernel<<<tile_grid(b), kThreads, 0, s>>>(b, out);
    return cudaGetLastError();
}

cudaError_t launch_unpack_spins(const DevBatch& b, uint32_t first_chain, uint32_t n_chains,
                                int8_t* out, cudaStream_t s) {
    const size_t total = size_t(n_chains) * b.n_spins;
    if (total == 0) return cudaSuccess;
    unpack_spins_kernel<<<unsigned((total + 255) / 256), 256, 0, s>>>(b, first_chain, n_chains, out);
    return cudaGetLastError();
}

cudaError_t launch_gather_fields(const DevBatch& b, uint32_t chain, float* hs, float* ht,
                                 cudaStream_t s) {
    if (b.n_spins == 0) return cudaSuccess;
    gather_fields_kernel<<<(b.n_spins + 255) / 256, 256, 0, s>>>(b, chain, hs, ht);
    return cudaGetLastError();
}

cudaError_t launch_pack_results(const DevBatch& b, void* out, cudaStream_t s) {
    pack_results_kernel<<<tile_grid(b), kThreads, 0, s>>>(b, static_cast<ResultRecord*>(out));
    return cudaGetLastError();
}

}  // namespace isingb200
