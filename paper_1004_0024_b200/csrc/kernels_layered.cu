// Layered-model sweep kernel: the performance path for identical-layer ("QMC-style") models.
//
// One persistent CTA per SM; four SWEEP warps and four RNG warps per CTA.  Sweep warp w and RNG
// warp 4+w share a tile of 32 chains (lane = chain) and — because warp_id % 4 picks the SM
// sub-partition — the same scheduler, so the generator's integer work fills the issue slots the
// sweep's dependent floating-point chain leaves empty.
//
// A chain's working set for one layer lives ON CHIP:
//   * Tensor Memory holds the space fields of the layer being swept: column p of the warp's own
//     32-lane TMEM quarter is h_eff_space[(layer, p)] of its 32 chains (512 columns x 128 lanes x
//     4 B = the whole 256 KB TMEM of an SM for 4 warps x 512 positions).
//   * A five-entry REGISTER WINDOW slides over the columns p-2..p+2 of the position being
//     attempted.  Updates of the near ("band") neighbours are predicated register adds, so the
//     loop-carried dependency from one attempt to the next is a single FADD; only the far
//     neighbours of a flip are read-modify-written in Tensor Memory (tcgen05.ld / tcgen05.st).
//   * The tau field is NOT stored.  For these models it only takes the values {2J, +0, -2J}
//     and every incremental update of it is exact (HostModel::layered_uniform), so it is rebuilt
//     from two spin bits of the adjacent layers.  That removes 8 of the 17 bytes per attempt the
//     generic layout streams, and both tau read-modify-writes of every flip.
//   * Spins are one bit per chain: a 32-bit word per (tile, spin) holds the 32 lanes' signs.
//     Three layers of words (previous, current, next) sit in shared memory per warp.
//   * One layer's graph (band couplings + far-edge list per position) sits in shared memory.
//   * The RNG warp regenerates the chains' MT19937 states (replica-interleaved in HBM/L2) and
//     hands uniforms over through a shared-memory ring guarded by mbarriers.
//
// The attempt itself is branch-free (flips are predicated, empty band slots add -0.0), so the
// compiler can overlap the side work of attempt p with the decision chain of attempt p+1.
//
// HBM traffic per sweep is one read and one write of the f32 space fields plus the bit words
// (8.25 B per attempt) and the MT19937 state words (12 B per attempt while they miss L2).
// The trajectory is the reference's (ref: proj/src/sweep_basic.cpp:12-56) bit for bit.
#include "device_batch.hpp"
#include "device_math.cuh"
#include "device_mt.cuh"

namespace isingb200 {

namespace {

constexpr int kSweepWarps = 4;          // one TMEM lane quarter each
constexpr int kLayeredThreads = 2 * kSweepWarps * 32;
constexpr uint32_t kTmemColumns = 512;  // the whole TMEM: one CTA per SM
constexpr uint32_t kStageDraws = 64;    // uniforms per ring stage (per lane)
constexpr uint32_t kStages = 2;
constexpr uint32_t kGenBatch = 16;      // draws whose state loads are in flight together
constexpr uint32_t kUnroll = 8;         // attempts per unrolled chunk == register-window ring size

// ---- Tensor Memory access (sm_100a tcgen05).  All of these are warp-collective.
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_result, uint32_t columns) {
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(smem_result));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst), "r"(columns)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t columns) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(columns) : "memory");
}
__device__ __forceinline__ float tmem_ld(uint32_t taddr) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
    return __uint_as_float(v);
}
__device__ __forceinline__ void tmem_st(uint32_t taddr, float v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(__float_as_uint(v)));
}
// No "memory" clobbers on the Tensor Memory traffic of the inner loop: volatile asm statements keep
// their order among themselves, and ordinary shared/global accesses are free to move across them
// (TMEM is a separate address space), which lets the compiler hoist the next attempt's loads.
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;"); }

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(r[k]);
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// ---- mbarrier (shared::cta) helpers for the uniform ring
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait suspends the warp in hardware (up to the hint) instead of spinning on the issue port.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, uint32_t backoff_ns = 0) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done;
    do {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done)
            : "r"(addr), "r"(parity), "r"(100000u)
            : "memory");
        if (done == 0u) __nanosleep(backoff_ns);
    } while (done == 0u);
}

// ---- shared-memory carve-up (per CTA): [header][graph x (1 | 4)][per-pair dynamic region x 4]
struct GraphSmem {
    uint4* pos;        // P
    uint4* band_j2;    // P
    uint4* band_mask;  // P
    uint2* far;        // max_far
};
struct PairSmem {
    uint2* agree_sign;  // P : per layer, {~(up ^ dn), up} spin words
    uint32_t* words;    // 3 * P : ring of spin-bit layers
    float* ring;        // kStages * kStageDraws * 32 uniforms
};

constexpr size_t kHeaderBytes = 256;  // tmem slot + 4 pairs x (full[kStages] + empty[kStages]) barriers

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) / 16 * 16; }
__host__ __device__ inline size_t graph_bytes(uint32_t P, uint32_t max_far) {
    return size_t(P) * 48 + align16(size_t(max_far ? max_far : 1) * 8);
}
__host__ __device__ inline size_t pair_bytes(uint32_t P) {
    return align16(size_t(P) * 8) + align16(size_t(P) * 12) + size_t(kStages) * kStageDraws * 32 * 4;
}

__device__ __forceinline__ GraphSmem carve_graph(unsigned char* base, uint32_t P) {
    GraphSmem g;
    g.pos = reinterpret_cast<uint4*>(base);
    g.band_j2 = g.pos + P;
    g.band_mask = g.band_j2 + P;
    g.far = reinterpret_cast<uint2*>(g.band_mask + P);
    return g;
}
__device__ __forceinline__ PairSmem carve_pair(unsigned char* base, uint32_t P) {
    PairSmem s;
    s.agree_sign = reinterpret_cast<uint2*>(base);
    base += align16(size_t(P) * 8);
    s.words = reinterpret_cast<uint32_t*>(base);
    base += align16(size_t(P) * 12);
    s.ring = reinterpret_cast<float*>(base);
    return s;
}

__device__ __forceinline__ void load_graph(const GraphSmem& dst, const DevLayerGraph& g, uint32_t tid,
                                           uint32_t nthreads) {
    for (uint32_t k = tid; k < g.per_layer; k += nthreads) {
        dst.pos[k] = g.pos[k];
        dst.band_j2[k] = g.band_j2[k];
        dst.band_mask[k] = g.band_mask[k];
    }
    for (uint32_t k = tid; k < g.n_far; k += nthreads) dst.far[k] = g.far[k];
}

__device__ __forceinline__ void words_copy(uint32_t* dst, const uint32_t* src, uint32_t P, uint32_t lane) {
    for (uint32_t k = lane; k < P; k += 32) dst[k] = src[k];
}

// ---------------------------------------------------------------------------------------
// RNG warp: regenerates `take` words of every lane's MT19937 state in place and writes the
// tempered, truncated uniforms to out[k*32].  The state is walked in runs that do not cross
// the recurrence's wrap points (word 227: the far operand wraps; word 623: the next operand
// wraps), so inside a run all three operands advance by one row (ref: rng.cpp:89-96).
__device__ __forceinline__ void mt_generate(uint32_t* w, uint32_t& pos, uint32_t& cur, uint32_t take,
                                            float* out) {
    uint32_t done = 0;
    while (done < take) {
        const uint32_t seg_end = pos < kMtN - kMtM ? kMtN - kMtM : (pos < kMtN - 1 ? kMtN - 1 : kMtN);
        const uint32_t cnt = min(take - done, seg_end - pos);
        uint32_t* wp = w + size_t(pos) * 32;
        const uint32_t* fp = w + size_t(pos < kMtN - kMtM ? pos + kMtM : pos - (kMtN - kMtM)) * 32;
        const uint32_t* np = pos == kMtN - 1 ? w : wp + 32;
        uint32_t k = 0;
        for (; k + kGenBatch <= cnt; k += kGenBatch) {
            uint32_t nxt[kGenBatch], far[kGenBatch];
#pragma unroll
            for (int i = 0; i < int(kGenBatch); ++i) {
                nxt[i] = np[size_t(k + i) * 32];
                far[i] = fp[size_t(k + i) * 32];
            }
#pragma unroll
            for (int i = 0; i < int(kGenBatch); ++i) {
                const uint32_t v = mt_recurrence(cur, nxt[i], far[i]);
                wp[size_t(k + i) * 32] = v;
                cur = nxt[i];
                out[size_t(k + i) * 32] = u32_to_unit(mt_temper(v));
            }
        }
        for (; k < cnt; ++k) {
            const uint32_t nx = np[size_t(k) * 32];
            const uint32_t v = mt_recurrence(cur, nx, fp[size_t(k) * 32]);
            wp[size_t(k) * 32] = v;
            cur = nx;
            out[size_t(k) * 32] = u32_to_unit(mt_temper(v));
        }
        pos += cnt;
        pos = pos == kMtN ? 0u : pos;
        done += cnt;
        out += size_t(cnt) * 32;
    }
}

struct RingCursor {
    uint32_t stage = 0;
    uint32_t parity = 0;
    __device__ __forceinline__ void advance() {
        if (++stage == kStages) {
            stage = 0;
            parity ^= 1u;
        }
    }
};

__device__ void rng_warp(const DevBatch& b, uint32_t sweeps, uint32_t lane, const PairSmem& s, uint64_t* full,
                         uint64_t* empty, RingCursor& cursor, uint32_t tile) {
    uint32_t* w = b.mt + size_t(tile) * kMtN * 32 + lane;
    uint32_t pos = b.mt_pos[tile];
    uint32_t cur = w[size_t(pos) * 32];
    uint64_t remaining = uint64_t(sweeps) * b.n_spins;
    while (remaining != 0) {
        const uint32_t take = remaining < kStageDraws ? uint32_t(remaining) : kStageDraws;
        mbar_wait(&empty[cursor.stage], cursor.parity ^ 1u, 1000);
        mt_generate(w, pos, cur, take, s.ring + size_t(cursor.stage) * kStageDraws * 32 + lane);
        mbar_arrive(&full[cursor.stage]);
        cursor.advance();
        remaining -= take;
    }
    if (lane == 0) b.mt_pos[tile] = pos;
}

// ---------------------------------------------------------------------------------------
// Per-lane state of a sweep warp that lives across attempts.
struct LaneState {
    uint32_t nb2;      // bits of -2*beta
    uint32_t sh;       // 31 - lane: shift that brings this lane's bit to the sign position
    uint32_t flips;
    double e_run;
    bool active;
};

// Everything an attempt needs that does not depend on earlier flips of the same chunk; loaded one
// attempt ahead so the shared-memory latency hides behind the previous decision chain.
struct Prep {
    uint4 rec, bj, bm;
    uint2 as;
    uint32_t word;
    float u;
};
struct ChunkPtrs {  // all pre-offset to the chunk's first position
    const uint4* pos;
    const uint4* band_j2;
    const uint4* band_mask;
    const uint2* agree_sign;
    uint32_t* words;
    const float* u;
};
template <int K>
__device__ __forceinline__ Prep load_prep(const ChunkPtrs& c) {
    Prep q;
    q.rec = c.pos[K];
    q.bj = c.band_j2[K];
    q.bm = c.band_mask[K];
    q.as = c.agree_sign[K];
    q.word = c.words[K];
    q.u = c.u[K * 32];
    return q;
}

// One Metropolis attempt at position p = p0 + K of the current layer (K is the compile-time
// index inside the unrolled chunk; the register window r[] is indexed by position & 7).
template <int EXP, int K>
__device__ __forceinline__ void attempt(float (&r)[kUnroll], LaneState& st, const Prep& q, uint32_t p0, uint32_t tm,
                                        const uint2* far, uint32_t* w_chunk, uint32_t lane) {
    const uint32_t p = p0 + K;
    const uint32_t sgn_s = (q.word << st.sh) & 0x80000000u;            // sign bit set <=> s = -1
    const uint32_t sgn_up = (q.as.y << st.sh) & 0x80000000u;
    const uint32_t agree = uint32_t(int32_t(q.as.x << st.sh) >> 31);  // all ones when s_up == s_dn
    // tau field J*(s_up + s_dn) in {+2J, +0, -2J}; rec.x carries it already scaled by gamma
    const float htg = __uint_as_float((q.rec.x ^ sgn_up) & agree);
    const float h = r[K];
    // x = -beta*((2s)*(h + gamma*ht)) == (-2*beta*s)*(h + gamma*ht): doubling is exact, so both
    // forms round once and to the same value (ref: sweep_kernels.hpp:14-16)
    const float x = __fmul_rn(__uint_as_float(st.nb2 ^ sgn_s), __fadd_rn(h, htg));
    const float pr = exp_kind<EXP>(x);
    const bool accept = st.active && (q.u < pr);

    // ---- band neighbours: h -= (2s)*J  ==  h + (-(2s)*J); an empty slot adds -0.0 (identity)
    const uint32_t neg_d = sgn_s ^ 0x80000000u;
    tmem_wait_ld();  // the entry for p+2 was requested right after the previous attempt
    if (accept) {
        r[(K + 6) & 7] = __fadd_rn(r[(K + 6) & 7], __uint_as_float((q.bj.x ^ neg_d) | q.bm.x));
        r[(K + 7) & 7] = __fadd_rn(r[(K + 7) & 7], __uint_as_float((q.bj.y ^ neg_d) | q.bm.y));
        r[(K + 1) & 7] = __fadd_rn(r[(K + 1) & 7], __uint_as_float((q.bj.z ^ neg_d) | q.bm.z));
        r[(K + 2) & 7] = __fadd_rn(r[(K + 2) & 7], __uint_as_float((q.bj.w ^ neg_d) | q.bm.w));
        ++st.flips;
        const float ht = __uint_as_float((q.rec.y ^ sgn_up) & agree);
        const float two_s = __uint_as_float(0x40000000u ^ sgn_s);
        st.e_run = __dadd_rn(st.e_run, double(__fmul_rn(two_s, __fadd_rn(h, ht))));
    }
    const uint32_t ballot = __ballot_sync(0xffffffffu, accept);
    if (lane == 0) w_chunk[K] = q.word ^ ballot;

    // ---- retire column p-2: no later attempt of this layer can reach it through the band
    if (K >= 2 || p0 != 0) tmem_st(tm + p - 2, r[(K + 6) & 7]);

    // ---- far neighbours: read-modify-write in Tensor Memory (the first two with their loads batched)
    const uint32_t far_count = q.rec.z >> 24;
    if (far_count != 0u && ballot != 0u) {
        const uint2* fe = far + (q.rec.z & 0xffffffu);
        tmem_wait_st();
        const uint2 e0 = fe[0];
        const uint2 e1 = fe[far_count > 1u ? 1 : 0];
        float v0 = tmem_ld(tm + e0.x);
        float v1 = 0.0f;
        if (far_count > 1u) v1 = tmem_ld(tm + e1.x);
        tmem_wait_ld();
        if (accept) {
            v0 = __fadd_rn(v0, __uint_as_float(e0.y ^ neg_d));
            v1 = __fadd_rn(v1, __uint_as_float(e1.y ^ neg_d));
        }
        tmem_st(tm + e0.x, v0);
        if (far_count > 1u) tmem_st(tm + e1.x, v1);
        for (uint32_t e = 2; e < far_count; ++e) {
            const uint2 ed = fe[e];
            float v = tmem_ld(tm + ed.x);
            tmem_wait_ld();
            if (accept) v = __fadd_rn(v, __uint_as_float(ed.y ^ neg_d));
            tmem_st(tm + ed.x, v);
        }
        tmem_wait_st();
    }
}

// Feeds the window entry for position p+3 after attempt p (it is first needed by attempt p+1).
template <int K>
__device__ __forceinline__ void feed(float (&r)[kUnroll], uint32_t p0, uint32_t P, uint32_t tm) {
    if (K <= 4 || p0 + kUnroll < P) r[(K + 3) & 7] = tmem_ld(tm + p0 + K + 3);
}

template <int EXP>
__device__ void sweep_warp(const DevBatch& b, uint32_t sweeps, uint32_t lane, const GraphSmem& g,
                           const PairSmem& s, uint64_t* full, uint64_t* empty, RingCursor& cursor, uint32_t tile,
                           uint32_t tm, uint32_t P, uint32_t L) {
    const uint32_t n = b.n_spins;
    const uint32_t chain = b.tile_first[tile] + lane;
    LaneState st;
    st.active = lane < b.tile_count[tile];
    st.nb2 = __float_as_uint(st.active ? -2.0f * b.betas[b.slot_of_chain[chain]] : 0.0f);
    st.sh = 31u - lane;
    st.flips = 0;
    st.e_run = st.active ? b.e_run[chain] : 0.0;
    float* hs_g = b.hs + size_t(tile) * n * 32 + lane;
    uint32_t* words_g = b.spin_bits + size_t(tile) * n;

    uint32_t slot_dn = 2, slot_cur = 0, slot_up = 1;
    words_copy(s.words + slot_dn * P, words_g + size_t(L - 1) * P, P, lane);
    words_copy(s.words + slot_cur * P, words_g, P, lane);
    words_copy(s.words + slot_up * P, words_g + size_t(1) * P, P, lane);
    __syncwarp();

    uint32_t ui = 0;  // draws consumed from the current ring stage (a multiple of kUnroll)
    const float* ring = s.ring + lane;

    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t l = 0; l < L; ++l) {
            float* hs_l = hs_g + size_t(l) * P * 32;
            const float* hs_next = hs_g + size_t(l + 1 == L ? 0 : l + 1) * P * 32 - lane;
            // ---- feed: this layer's fields HBM -> TMEM (P is a multiple of 8)
            uint32_t p0 = 0;
            for (; p0 + 32 <= P; p0 += 32) {
                float v[4][8];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) v[q][k] = hs_l[size_t(p0 + q * 8 + k) * 32];
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) tmem_st8(tm + p0 + q * 8, v[q]);
            }
            for (; p0 < P; p0 += 8) {
                float v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) v[k] = hs_l[size_t(p0 + k) * 32];
                tmem_st8(tm + p0, v);
            }
            uint32_t* w_cur = s.words + slot_cur * P;
            {   // the tau field of this whole layer is fixed while it is swept: previous layer already
                // visited, next layer not yet.  agree = neighbours equal, sign = their common spin bit.
                const uint32_t* w_up = s.words + slot_up * P;
                const uint32_t* w_dn = s.words + slot_dn * P;
                for (uint32_t k = lane; k < P; k += 32) s.agree_sign[k] = make_uint2(~(w_up[k] ^ w_dn[k]), w_up[k]);
            }
            __syncwarp();
            tmem_wait_st();

            // register window: positions 0..2 (entries for -2, -1 stay unused: their band slots are empty)
            float r[kUnroll];
#pragma unroll
            for (int k = 0; k < int(kUnroll); ++k) r[k] = 0.0f;
            r[0] = tmem_ld(tm + 0);
            r[1] = tmem_ld(tm + 1);
            r[2] = tmem_ld(tm + 2);
            tmem_wait_ld();

            for (p0 = 0; p0 < P; p0 += kUnroll) {
                if (ui == 0) mbar_wait(&full[cursor.stage], cursor.parity);
                if ((p0 & 31u) == 0 && p0 + lane < P) prefetch_l2(hs_next + size_t(p0 + lane) * 32);
                ChunkPtrs c;
                c.pos = g.pos + p0;
                c.band_j2 = g.band_j2 + p0;
                c.band_mask = g.band_mask + p0;
                c.agree_sign = s.agree_sign + p0;
                c.words = w_cur + p0;
                c.u = ring + (size_t(cursor.stage) * kStageDraws + ui) * 32;
                const Prep q0 = load_prep<0>(c);
                const Prep q1 = load_prep<1>(c);
                attempt<EXP, 0>(r, st, q0, p0, tm, g.far, c.words, lane);
                feed<0>(r, p0, P, tm);
                const Prep q2 = load_prep<2>(c);
                attempt<EXP, 1>(r, st, q1, p0, tm, g.far, c.words, lane);
                feed<1>(r, p0, P, tm);
                const Prep q3 = load_prep<3>(c);
                attempt<EXP, 2>(r, st, q2, p0, tm, g.far, c.words, lane);
                feed<2>(r, p0, P, tm);
                const Prep q4 = load_prep<4>(c);
                attempt<EXP, 3>(r, st, q3, p0, tm, g.far, c.words, lane);
                feed<3>(r, p0, P, tm);
                const Prep q5 = load_prep<5>(c);
                attempt<EXP, 4>(r, st, q4, p0, tm, g.far, c.words, lane);
                feed<4>(r, p0, P, tm);
                const Prep q6 = load_prep<6>(c);
                attempt<EXP, 5>(r, st, q5, p0, tm, g.far, c.words, lane);
                feed<5>(r, p0, P, tm);
                const Prep q7 = load_prep<7>(c);
                attempt<EXP, 6>(r, st, q6, p0, tm, g.far, c.words, lane);
                feed<6>(r, p0, P, tm);
                attempt<EXP, 7>(r, st, q7, p0, tm, g.far, c.words, lane);
                feed<7>(r, p0, P, tm);
                ui += kUnroll;
                if (ui == kStageDraws) {
                    mbar_arrive(&empty[cursor.stage]);
                    cursor.advance();
                    ui = 0;
                }
            }
            // the last two columns leave the window
            tmem_st(tm + P - 2, r[6]);
            tmem_st(tm + P - 1, r[7]);
            tmem_wait_st();

            // ---- retire: TMEM -> HBM, and rotate the spin-bit ring
            for (p0 = 0; p0 < P; p0 += 8) {
                float v[8];
                tmem_ld8(tm + p0, v);
                tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < 8; ++k) hs_l[size_t(p0 + k) * 32] = v[k];
            }
            __syncwarp();
            words_copy(words_g + size_t(l) * P, w_cur, P, lane);
            // layer l-1's slot is free now: it receives layer l+2 (the `up` of the next layer)
            words_copy(s.words + slot_dn * P, words_g + size_t((l + 2) % L) * P, P, lane);
            __syncwarp();
            const uint32_t freed = slot_dn;
            slot_dn = slot_cur;
            slot_cur = slot_up;
            slot_up = freed;
        }
    }
    if (ui != 0) {  // hand a partly used last stage back
        mbar_arrive(&empty[cursor.stage]);
        cursor.advance();
    }
    if (st.active) {
        b.e_run[chain] = st.e_run;
        b.flips[chain] += st.flips;
    }
    __syncwarp();
}

template <int EXP>
__global__ void __launch_bounds__(kLayeredThreads, 1) sweep_layered_kernel(DevBatch b, uint32_t sweeps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + 16);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t pair = warp & 3u;
    const bool is_rng = warp >= kSweepWarps;
    uint64_t* full = bars + pair * 2 * kStages;
    uint64_t* empty = full + kStages;

    const uint32_t maxP = b.max_per_layer;
    const size_t gbytes = graph_bytes(maxP, b.max_far_edges);
    unsigned char* graph_base = smem_raw + kHeaderBytes + (b.graph_shared ? 0 : size_t(pair) * gbytes);
    unsigned char* pair_base =
        smem_raw + kHeaderBytes + (b.graph_shared ? 1 : kSweepWarps) * gbytes + size_t(pair) * pair_bytes(maxP);
    const GraphSmem gs = carve_graph(graph_base, maxP);
    const PairSmem s = carve_pair(pair_base, maxP);

    if (warp == 0) tmem_alloc(tmem_slot, kTmemColumns);
    if (threadIdx.x < kSweepWarps * 2 * kStages) mbar_init(&bars[threadIdx.x], 32);
    if (b.graph_shared) load_graph(gs, b.layer_graphs[0], threadIdx.x, kLayeredThreads);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = *tmem_slot;
    // this pair's lane quarter: bits 31..16 of a TMEM address are the lane, 15..0 the column
    const uint32_t tm = tmem_base + ((pair * 32u) << 16);
    RingCursor cursor;

    // tiles are dealt round-robin: CTA c, pair w, round r -> tile c + grid*(w + 4r)
    for (uint32_t tile = blockIdx.x + gridDim.x * pair; tile < b.n_tiles; tile += gridDim.x * kSweepWarps) {
        if (is_rng) {
            rng_warp(b, sweeps, lane, s, full, empty, cursor, tile);
        } else {
            const DevLayerGraph g = b.layer_graphs[b.tile_model[tile]];
            if (!b.graph_shared) {
                load_graph(gs, g, lane, 32);
                __syncwarp();
            }
            sweep_warp<EXP>(b, sweeps, lane, gs, s, full, empty, cursor, tile, tm, g.per_layer, g.layers);
        }
    }

    if (!is_rng) {
        tmem_wait_ld();
        tmem_wait_st();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, kTmemColumns);
}

}  // namespace

size_t layered_smem_bytes(uint32_t per_layer, uint32_t max_far_edges, bool graph_shared) {
    if (per_layer == 0 || per_layer > kTmemColumns || per_layer % kUnroll != 0) return 0;
    const size_t bytes = kHeaderBytes + (graph_shared ? 1 : kSweepWarps) * graph_bytes(per_layer, max_far_edges) +
                         kSweepWarps * pair_bytes(per_layer);
    return bytes <= 227 * 1024 ? bytes : 0;
}

cudaError_t prepare_layered_kernels(size_t smem_bytes) {
    cudaError_t e = cudaFuncSetAttribute(sweep_layered_kernel<kExpExact>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_bytes));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(sweep_layered_kernel<kExpFast>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem_bytes));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(sweep_layered_kernel<kExpAccurate>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_bytes));
}

cudaError_t launch_sweep_layered(const DevBatch& b, uint32_t sweeps, int sm_count, cudaStream_t stream) {
    const size_t smem = size_t(b.layered_smem);
    const uint32_t ctas = uint32_t(sm_count) < b.n_tiles ? uint32_t(sm_count) : b.n_tiles;
    const dim3 grid(ctas ? ctas : 1);
    switch (b.exp_kind) {
        case kExpExact: sweep_layered_kernel<kExpExact><<<grid, kLayeredThreads, smem, stream>>>(b, sweeps); break;
        case kExpFast: sweep_layered_kernel<kExpFast><<<grid, kLayeredThreads, smem, stream>>>(b, sweeps); break;
        default: sweep_layered_kernel<kExpAccurate><<<grid, kLayeredThreads, smem, stream>>>(b, sweeps); break;
    }
    return cudaGetLastError();
}

}  // namespace isingb200
