// Per-chain MT19937 inside a replica-interleaved state block (shared by both kernel families).
#pragma once

#include "device_math.cuh"

namespace isingb200 {

constexpr int kChunk = 8;  // attempts whose random draws are generated together

// ---------------------------------------------------------------------------------------
// One chain's MT19937 inside a replica-interleaved block: word i lives at w[i * stride].
// The state is regenerated in place one word per draw (the classic loop of
// ref: rng.cpp:89-96, unrolled in time): draw j of a block rewrites word j from the old words
// j, j+1 and word j+397 (already new once j >= 227), which is exactly what a whole-block twist
// followed by reading word j produces.
struct MtLane {
    uint32_t* w;
    uint32_t stride;
    uint32_t pos;  // next word to regenerate, 0..623
    uint32_t cur;  // old value of word `pos`

    __device__ __forceinline__ void open(uint32_t* base, uint32_t stride_, uint32_t pos_) {
        w = base;
        stride = stride_;
        pos = pos_;
        cur = w[size_t(pos) * stride];
    }

    __device__ __forceinline__ uint32_t next_raw() {
        const uint32_t jn = pos + 1 == kMtN ? 0u : pos + 1;
        const uint32_t jf = pos >= kMtN - kMtM ? pos - (kMtN - kMtM) : pos + kMtM;
        const uint32_t nxt = w[size_t(jn) * stride];
        const uint32_t far = w[size_t(jf) * stride];
        const uint32_t v = mt_recurrence(cur, nxt, far);
        w[size_t(pos) * stride] = v;
        cur = nxt;
        pos = jn;
        return mt_temper(v);
    }

    // The recurrence operands of the next `count` (<= kChunk) draws.  None of them is a word the
    // draws before them in the same or the previous chunk rewrite (the `next` words lie ahead, the
    // `far` words 227 draws behind or 397 ahead), so they may be requested a whole chunk early.
    __device__ __forceinline__ void load_operands(uint32_t count, uint32_t (&nxt)[kChunk], uint32_t (&far)[kChunk]) const {
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
            if (uint32_t(k) < count) {
                uint32_t jn = pos + k + 1;
                jn = jn >= kMtN ? jn - kMtN : jn;
                uint32_t jf = pos + k + kMtM;
                jf = jf >= kMtN ? jf - kMtN : jf;
                nxt[k] = w[size_t(jn) * stride];
                far[k] = w[size_t(jf) * stride];
            }
        }
    }

    // Regenerates `count` words in place from operands loaded by load_operands at this position.
    __device__ __forceinline__ void generate(uint32_t count, const uint32_t (&nxt)[kChunk],
                                             const uint32_t (&far)[kChunk], float (&u)[kChunk]) {
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
            if (uint32_t(k) < count) {
                const uint32_t v = mt_recurrence(cur, nxt[k], far[k]);
                uint32_t j = pos + k;
                j = j >= kMtN ? j - kMtN : j;
                w[size_t(j) * stride] = v;
                cur = nxt[k];
                u[k] = u32_to_unit(mt_temper(v));
            }
        }
        pos += count;
        pos = pos >= kMtN ? pos - kMtN : pos;
    }

    // `count` (<= kChunk) draws with every load issued before the first store, so the loads
    // overlap instead of serialising on L2 latency.
    __device__ __forceinline__ void next_chunk(uint32_t count, float (&u)[kChunk]) {
        uint32_t nxt[kChunk], far[kChunk];
        load_operands(count, nxt, far);
        generate(count, nxt, far, u);
    }

    // The same chunk as tempered 32-bit outputs (initial_spins reads bit 31 of each).
    __device__ __forceinline__ void next_chunk_raw(uint32_t count, uint32_t (&raw)[kChunk]) {
        uint32_t nxt[kChunk], far[kChunk];
        load_operands(count, nxt, far);
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
            if (uint32_t(k) < count) {
                const uint32_t v = mt_recurrence(cur, nxt[k], far[k]);
                uint32_t j = pos + k;
                j = j >= kMtN ? j - kMtN : j;
                w[size_t(j) * stride] = v;
                cur = nxt[k];
                raw[k] = mt_temper(v);
            }
        }
        pos += count;
        pos = pos >= kMtN ? pos - kMtN : pos;
    }
};

// ref: Mt19937::reseed, rng.cpp:37-44
__device__ inline void mt_seed_lane(uint32_t* w, uint32_t stride, uint32_t seed) {
    uint32_t prev = seed;
    w[0] = prev;
    for (uint32_t i = 1; i < kMtN; ++i) {
        prev = 1812433253u * (prev ^ (prev >> 30)) + i;
        w[size_t(i) * stride] = prev;
    }
}

}  // namespace isingb200
