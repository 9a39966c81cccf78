// Layer-wavefront ("strand") sweep kernel for identical-layer models: the throughput path.
//
// A chain's sweep is sequential in the reference order (ref: proj/src/sweep_basic.cpp:12-56), but for a
// layered model the order only binds three things: within a layer, position p comes after every
// position before it; spin (l, p) comes after (l-1, p) (whose NEW value it reads) and before (l+1, p)
// (whose OLD value it reads); and layer 0 of the next sweep comes after layer L-1 of this one.  So the
// layers of one tile (32 chains, lane = chain) are swept by S concurrent warps — STRANDS — in a
// wavefront: strand j takes layers j, j+S, j+2S, ... and runs a few positions behind the strand of the
// layer below it.  Every chain still sees exactly the reference's sequence of decisions:
//
//   * space fields only ever receive updates from flips of their own layer, all issued by the one
//     strand that owns the layer, in position order — the f32 sums round exactly as in the reference;
//   * the tau field of these models takes the values {2J, +0, -2J} and is rebuilt from the two
//     neighbouring spins (HostModel::layered_uniform), read from the neighbouring strands' spin bytes
//     under the ordering above;
//   * draw (sweep, l, p) of the chain's MT19937 stream is word (sweep*L + l)*P + p of a TAPE that a
//     PRODUCER warp per tile generates in stream order (lane = chain, three coalesced row accesses per
//     word: x[k] = f(x[k-624], x[k-623], x[k-227]), ref: proj/src/rng.cpp:22-25,89-96) into a ring in
//     global memory; the strands temper and convert their own words.
//
// Nothing is staged on chip beyond registers, so a tile is not bound to an SM or to Tensor Memory:
// strands and producers are independent warps of a persistent grid that meet through per-tile
// progress counters in global memory (st.release.gpu / ld.acquire.gpu), a few thousand of them in
// flight — enough to hide every latency, which the one-warp-per-tile kernels cannot.
//
// Per strand, fields move in chunks of 8 positions: the window of positions p-2..p+2 lives in
// registers (band neighbours are predicated register adds, as in kernels_layered.cu); eight columns
// enter it from HBM and eight leave it per chunk (full 128-byte lines); far neighbours are
// read-modify-written in global memory after the chunk, in groups of distinct targets whose loads go
// out together.  All field traffic of a layer comes from one thread per chain, so program order is
// the only ordering it needs.  HBM traffic per attempt: 4 B field in, 4 B out, 1/4 B spin bytes, plus
// the tape (4 B written, 4 B read, both L2 hits while the ring fits).
#include "device_batch.hpp"
#include "device_math.cuh"

namespace isingb200 {

namespace {

constexpr uint32_t kStrandMaxWarps = 20;
constexpr uint32_t kFlagStride = 32;  // one 128-byte line per progress counter

// ---- memory access helpers -----------------------------------------------------------------
__device__ __forceinline__ float ld_cg_f32(const float* p) {
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_cg_u8(const uint8_t* p) {
    uint32_t v;
    asm volatile("ld.global.cg.u8 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double ld_cg_f64(const double* p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_f32(float* p, float v) {
    asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_u8(uint8_t* p, uint32_t v) {
    asm volatile("st.global.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Blocks until the counter at `p` has reached `need` (counters only grow; compared modulo 2^32).
// Every lane polls — one broadcast transaction — so every lane's later loads are ordered after
// the value it saw.
__device__ __forceinline__ void wait_counter(const uint32_t* p, uint32_t need, uint32_t& cached) {
    if (int32_t(need - cached) > 0) {
        uint32_t v = ld_acquire(p);
        while (int32_t(need - v) > 0) {
            __nanosleep(100);
            v = ld_acquire(p);
        }
        cached = __reduce_min_sync(0xffffffffu, v);
    }
}
// The whole warp's earlier writes, then the counter (the release is cumulative over what lane 0
// observed through the warp barrier).
__device__ __forceinline__ void publish(uint32_t* p, uint32_t value, uint32_t lane) {
    __syncwarp();
    if (lane == 0) st_release(p, value);
}

// ---- one attempt ----------------------------------------------------------------------------
// Everything an attempt needs that does not depend on the fields, per chunk of eight attempts.
struct ChunkBits {
    uint32_t cur8;    // bit k: the spin of attempt k is -1 (before the attempt)
    uint32_t up8;     // bit k: the spin above (next layer, not yet visited) is -1
    uint32_t agree8;  // bit k: the spins above and below are equal
};

// Attempt K (compile-time index in the unrolled chunk; the register window r[] is indexed by
// position & 7) of position p = p0 + K.  `tau_g` holds the bits of gamma * 2J_tau(p), `band` points
// at the band_pm pair of p.  ref: sweep_kernels.hpp:14-16, sweep_basic.cpp:36-48.
template <int EXP, int K>
__device__ __forceinline__ void strand_attempt(float (&r)[8], uint32_t raw, const ChunkBits& cb,
                                               uint32_t nb2, float u_offset, uint32_t tau_g, const uint4* band,
                                               uint32_t& acc8, double& e_blk) {
    // u32_to_unit (x * 2^-32 is exact, so is adding +0); padding lanes get u + 2 and never accept
    const float u = __fmaf_rn(__uint2float_rz(mt_temper(raw)), 0x1p-32f, u_offset);
    const uint32_t sgn = (cb.cur8 << (31 - K)) & 0x80000000u;     // set <=> s = -1
    const uint32_t sgn_up = (cb.up8 << (31 - K)) & 0x80000000u;
    const uint32_t agree = uint32_t(int32_t(cb.agree8 << (31 - K)) >> 31);
    // gamma * h_tau, h_tau = J*(s_up + s_dn) in {+2J, +0, -2J}
    const float hz = __uint_as_float((tau_g ^ sgn_up) & agree);
    // x = -beta*((2s)*v) == (-2*beta*s)*v: doubling is exact, one rounding either way
    const float v = __fadd_rn(r[K], hz);
    const float x = __fmul_rn(__uint_as_float(nb2 ^ sgn), v);
    const bool accept = u < exp_kind<EXP>(x);
    // band neighbours p-2, p-1, p+1, p+2: h -= (2s)*J == h + (-(2s)*J); entry 2p+1 is for s = +1; an
    // empty slot holds -0.0
    const uint4 op = __ldg(band + ((sgn >> 31) ^ 1u));
    if (accept) {
        r[(K + 6) & 7] = __fadd_rn(r[(K + 6) & 7], __uint_as_float(op.x));
        r[(K + 7) & 7] = __fadd_rn(r[(K + 7) & 7], __uint_as_float(op.y));
        r[(K + 1) & 7] = __fadd_rn(r[(K + 1) & 7], __uint_as_float(op.z));
        r[(K + 2) & 7] = __fadd_rn(r[(K + 2) & 7], __uint_as_float(op.w));
        // running energy of the tempering swap: (2s)*(h + gamma*h_tau), the inner factor of x
        e_blk = __dadd_rn(e_blk, double(__uint_as_float(__float_as_uint(__fmul_rn(v, 2.0f)) ^ sgn)));
        acc8 |= 1u << K;
    }
}

// What a flip of attempt e.y adds to the field at e.x: -(2s)*J, i.e. 2J (e.z) with the sign of -s.
__device__ __forceinline__ float edge_addend(const uint4 e, uint32_t cur8) {
    return __uint_as_float(e.z ^ ((((cur8 >> e.y) & 1u) ^ 1u) << 31));
}

// Far neighbours of the chunk's flips, after its last attempt: read-modify-writes in global memory,
// in groups of up to 8 edges with distinct targets (loads together, then adds and stores).  Groups
// and edges are in attempt order, so every column receives its updates in the reference's order.
__device__ __forceinline__ void apply_groups(float* hs_l, const DevStrandGraph& g, uint32_t ginfo, uint32_t acc8,
                                             uint32_t cur8) {
    const uint32_t* grp = g.groups + (ginfo & 0xffffu);
    const uint32_t n_groups = ginfo >> 16;
#pragma unroll 1
    for (uint32_t q = 0; q < n_groups; ++q) {
        const uint32_t info = __ldg(grp + q);
        const uint4* fe = g.edges + (info & 0xffffu);
        const uint32_t n = info >> 16;
        uint4 e[8];
        float v[8];
#pragma unroll
        for (uint32_t i = 0; i < 8; ++i) {
            if (i < n) e[i] = __ldg(fe + i);
        }
#pragma unroll
        for (uint32_t i = 0; i < 8; ++i) {
            if (i < n) v[i] = ld_cg_f32(hs_l + size_t(e[i].x) * 32);
        }
#pragma unroll
        for (uint32_t i = 0; i < 8; ++i) {
            if (i < n && ((acc8 >> e[i].y) & 1u)) {
                st_f32(hs_l + size_t(e[i].x) * 32, __fadd_rn(v[i], edge_addend(e[i], cur8)));
            }
        }
    }
}

// A CAREFUL chunk: some attempt has a far neighbour among the columns that have already been
// requested (p+3 .. p0+10).  The entering columns go through a per-warp shared-memory scratch
// ([8][32] floats, a lane only touches its own entries; the caller has stored them there), where
// such updates are applied before the column enters the register window.  Out of line and by value:
// the hot loop keeps its window in registers.
struct Window {
    float r[8];
};
struct RawWords {
    uint32_t v[8];
};
struct CarefulResult {
    Window w;
    uint32_t acc8;
    double e_blk;
};

template <int EXP, int K>
__device__ __forceinline__ void careful_attempt(float (&r)[8], float* scratch, uint32_t raw, const ChunkBits& cb,
                                                uint32_t nb2, float u_offset, const uint4 posrec, const uint4* band,
                                                uint32_t& acc8, double& e_blk, const uint4* edges, uint32_t p0) {
    const uint32_t before = acc8;
    strand_attempt<EXP, K>(r, raw, cb, nb2, u_offset, posrec.x, band, acc8, e_blk);
    const uint32_t near = posrec.y;
    if ((near >> 16) != 0u && acc8 != before) {
        const uint4* ne = edges + (near & 0xffffu);
        for (uint32_t i = 0; i < (near >> 16); ++i) {
            const uint4 e = __ldg(ne + i);
            float* cell = scratch + (e.x - (p0 + 3)) * 32;
            *cell = __fadd_rn(*cell, edge_addend(e, cb.cur8));
        }
    }
}

template <int EXP>
__device__ __noinline__ CarefulResult careful_chunk(Window w, RawWords raw, ChunkBits cb, uint32_t nb2, float u_offset,
                                                    const uint4* pos, const uint4* band, const uint4* edges,
                                                    uint32_t p0, float* hs_l, float* scratch, double e_blk) {
    float (&r)[8] = w.r;
    uint32_t acc8 = 0;
#define ISING_CAREFUL(K)                                                                                              \
    careful_attempt<EXP, K>(r, scratch, raw.v[K], cb, nb2, u_offset, __ldg(pos + K), band + 2 * K, acc8, e_blk, edges, \
                            p0);                                                                                      \
    if (p0 != 0 || K >= 2) st_f32(hs_l + (size_t(p0) + K - 2) * 32, r[(K + 6) & 7]);                                  \
    r[(K + 3) & 7] = scratch[K * 32];
    ISING_CAREFUL(0)
    ISING_CAREFUL(1)
    ISING_CAREFUL(2)
    ISING_CAREFUL(3)
    ISING_CAREFUL(4)
    ISING_CAREFUL(5)
    ISING_CAREFUL(6)
    ISING_CAREFUL(7)
#undef ISING_CAREFUL
    CarefulResult out;
    out.w = w;
    out.acc8 = acc8;
    out.e_blk = e_blk;
    return out;
}

// ---- a strand ---------------------------------------------------------------------------------
template <int EXP, bool WAIT>
__device__ void strand_run(const DevBatch& b, const DevStrandGraph& g, uint32_t tile, uint32_t j, uint32_t sweeps,
                           uint32_t lane, float* scratch) {
    const uint32_t P = g.per_layer, L = g.layers, C = P / 8, S = b.strands, n = b.n_spins;
    const uint32_t blocks_per_sweep = L / S;
    const uint32_t total_blocks = blocks_per_sweep * sweeps;
    const uint32_t chain = b.tile_first[tile] + lane;
    const bool active = lane < b.tile_count[tile];
    const uint32_t nb2 = __float_as_uint(active ? -2.0f * b.betas[b.slot_of_chain[chain]] : 0.0f);
    const float u_offset = active ? 0.0f : 2.0f;
    float* hs_tile = b.hs + size_t(tile) * n * 32 + lane;
    uint8_t* bytes_tile = b.spin_bytes + size_t(tile) * (n / 8) * 32 + lane;
    const uint32_t R = b.tape_rows;
    const uint32_t* tape = b.tape + size_t(tile) * R * 32 + lane;
    uint32_t* flags = b.strand_flags + size_t(tile) * (S + 1) * kFlagStride;
    uint32_t* my_flag = flags + j * kFlagStride;
    const uint32_t* pred_flag = flags + ((j + S - 1) % S) * kFlagStride;
    const uint32_t* head_flag = flags + S * kFlagStride;
    const uint32_t pub = b.strand_pub;
    uint32_t pred_cached = 0, head_cached = 0;
    uint32_t flips = 0;
    uint32_t seq = 0;  // chunks finished
    // wait statistics (ref: FlipStats::group_wait): lane k folds the ballot of attempt k of every chunk
    const bool record_wait = WAIT && b.wait_counts != nullptr && b.tile_count[tile] == 32;
    uint32_t wait[6] = {0, 0, 0, 0, 0, 0};

    for (uint32_t blk = 0; blk < total_blocks; ++blk) {
        const uint32_t sw = blk / blocks_per_sweep, m = blk - sw * blocks_per_sweep;
        const uint32_t l = j + S * m;
        const uint32_t l_up = l + 1 == L ? 0u : l + 1, l_dn = l == 0 ? L - 1 : l - 1;
        float* hs_l = hs_tile + size_t(l) * P * 32;
        uint8_t* by_cur = bytes_tile + size_t(l) * C * 32;
        const uint8_t* by_up = bytes_tile + size_t(l_up) * C * 32;
        const uint8_t* by_dn = bytes_tile + size_t(l_dn) * C * 32;
        // The strand of the layer below: its chunk c of the matching block must be finished before
        // this strand reads that layer's new spins.  For j > 0 the matching block has this block's
        // index, for j == 0 it is the block before (layer L-1 of the previous sweep when m == 0).
        const bool has_pred = S > 1 && !(j == 0 && blk == 0);
        const uint32_t pred_base = (j == 0 ? blk - 1 : blk) * C;
        // this block's draws: tape rows 624 + (sw*L + l)*P + p
        const uint32_t row0 = kMtN + (sw * L + l) * P;
        uint32_t slot = row0 % R;  // (R and row0 are multiples of 8: a chunk's rows never wrap)
        double e_blk = 0.0;

        RawWords raw_words;
        uint32_t (&raw)[8] = raw_words.v;
        wait_counter(head_flag, row0 + 8, head_cached);
#pragma unroll
        for (int k = 0; k < 8; ++k) raw[k] = ld_cg_u32(tape + size_t(slot + k) * 32);

        // register window: positions 0..2 (entries for -2, -1 stay unused: their band slots are empty)
        Window w;
        float (&r)[8] = w.r;
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = 0.0f;
        r[0] = ld_cg_f32(hs_l);
        r[1] = ld_cg_f32(hs_l + 32);
        r[2] = ld_cg_f32(hs_l + 64);

        for (uint32_t c = 0; c < C; ++c) {
            const uint32_t p0 = c * 8;
            const uint4 chunk_info = __ldg(g.chunks + c);
            if (has_pred) wait_counter(pred_flag, pred_base + c + 1, pred_cached);
            // ---- requests: the columns entering the window (p0+3 .. p0+10; the last chunk has five),
            // the spin bytes, the next chunk's tape rows; L2 prefetches one chunk ahead
            float nx[8];
            const float* enter = hs_l + (size_t(p0) + 3) * 32;
#pragma unroll
            for (int k = 0; k < 8; ++k) nx[k] = (k < 5 || c + 1 < C) ? ld_cg_f32(enter + k * 32) : 0.0f;
            ChunkBits cb;
            cb.cur8 = ld_cg_u8(by_cur + c * 32);
            cb.up8 = ld_cg_u8(by_up + c * 32);
            cb.agree8 = ~(cb.up8 ^ ld_cg_u8(by_dn + c * 32));
            uint32_t raw_next[8];
            if (c + 1 < C) {
                slot = slot + 8 == R ? 0u : slot + 8;
                wait_counter(head_flag, row0 + p0 + 16, head_cached);
#pragma unroll
                for (int k = 0; k < 8; ++k) raw_next[k] = ld_cg_u32(tape + size_t(slot + k) * 32);
                if (lane < 8 && p0 + 11 + lane < P) prefetch_l2(enter + (8 + lane) * 32);
            }
            {
                const uint32_t n_edges = chunk_info.y >> 16;
                if (lane < n_edges) prefetch_l2(hs_l + size_t(__ldg(g.edges + (chunk_info.y & 0xffffu) + lane).x) * 32);
            }

            // ---- eight attempts
            uint32_t acc8 = 0;
            if (__builtin_expect((chunk_info.z & 1u) == 0u, 1)) {
                const uint4* band = g.band_pm + 2 * size_t(p0);
                const uint4* pos = g.pos + p0;
#define ISING_STRAND_ATTEMPT(K)                                                                                   \
    strand_attempt<EXP, K>(r, raw[K], cb, nb2, u_offset, __ldg(&pos[K].x), band + 2 * K, acc8, e_blk);           \
    if (c != 0 || K >= 2) st_f32(hs_l + (size_t(p0) + K - 2) * 32, r[(K + 6) & 7]);                               \
    r[(K + 3) & 7] = nx[K];
                ISING_STRAND_ATTEMPT(0)
                ISING_STRAND_ATTEMPT(1)
                ISING_STRAND_ATTEMPT(2)
                ISING_STRAND_ATTEMPT(3)
                ISING_STRAND_ATTEMPT(4)
                ISING_STRAND_ATTEMPT(5)
                ISING_STRAND_ATTEMPT(6)
                ISING_STRAND_ATTEMPT(7)
#undef ISING_STRAND_ATTEMPT
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) scratch[k * 32] = nx[k];
                const CarefulResult res = careful_chunk<EXP>(w, raw_words, cb, nb2, u_offset, g.pos + p0,
                                                             g.band_pm + 2 * size_t(p0), g.edges, p0, hs_l, scratch, e_blk);
                w = res.w;
                acc8 = res.acc8;
                e_blk = res.e_blk;
            }

            // ---- after the chunk: spins, far neighbours, progress
            st_u8(by_cur + c * 32, cb.cur8 ^ acc8);
            flips += __popc(acc8);
            if (WAIT && record_wait) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t ballot = __ballot_sync(0xffffffffu, (acc8 >> k) & 1u);
                    if (lane == uint32_t(k)) wait_fold(ballot, wait);
                }
            }
            if ((chunk_info.x >> 16) != 0u && __any_sync(0xffffffffu, acc8 != 0u)) {
                apply_groups(hs_l, g, chunk_info.x, acc8, cb.cur8);
            }
            ++seq;
            if (c + 1 < C) {
#pragma unroll
                for (int k = 0; k < 8; ++k) raw[k] = raw_next[k];
                if (seq % pub == 0u) publish(my_flag, seq, lane);
            }
        }
        // ---- end of the layer: the last two columns leave the window; the block's partial sum joins
        // the running energy after the partial sums of all earlier blocks (tempering definition,
        // oracle/ising_oracle.h), which the strand of the layer below has published with its block
        st_f32(hs_l + (size_t(P) - 2) * 32, r[6]);
        st_f32(hs_l + (size_t(P) - 1) * 32, r[7]);
        if (has_pred) wait_counter(pred_flag, pred_base + C, pred_cached);
        if (active) {
            double* e_run = b.e_run + chain;
            const double e = ld_cg_f64(e_run);
            asm volatile("st.global.f64 [%0], %1;" ::"l"(e_run), "d"(__dadd_rn(e, e_blk)) : "memory");
        }
        publish(my_flag, seq, lane);
        if (WAIT && record_wait) {  // flushed per layer (lanes 0..7 hold partial sums of at most 64 * 32 each)
            unsigned long long* out = b.wait_counts + size_t(tile) * kWaitSlots;
#pragma unroll
            for (int w8 = 0; w8 < 6; ++w8) {
                uint32_t v = wait[w8];
                for (int off = 4; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
                if (lane == 0) atomicAdd(out + w8, static_cast<unsigned long long>(v));
                wait[w8] = 0;
            }
            if (lane == 0) atomicAdd(out + 6, static_cast<unsigned long long>(P));
        }
    }
    if (active && flips != 0u) atomicAdd(b.flips + chain, static_cast<unsigned long long>(flips));
}

// ---- the producer -------------------------------------------------------------------------------
// Stream position of strand `s` after `seq` finished chunks: the draw index of its next attempt
// (0xffffffff when it has finished).
__device__ __forceinline__ uint32_t strand_draw_index(uint32_t seq, uint32_t s, uint32_t S, uint32_t C, uint32_t L,
                                                      uint32_t P, uint32_t total_blocks) {
    const uint32_t blocks_per_sweep = L / S;
    const uint32_t blk = seq / C, c = seq - blk * C;
    if (blk >= total_blocks) return 0xffffffffu;
    const uint32_t sw = blk / blocks_per_sweep, m = blk - sw * blocks_per_sweep;
    return (sw * L + s + S * m) * P + c * 8;
}

// MT19937 as a tape: row a of the ring holds word x[a] of all 32 chains, x[0..623] being the state
// at launch in draw order, and draw q of the launch is temper(x[624 + q]).  Rows are generated in
// order, 32 at a time, never overwriting a row a strand has yet to read or the 624 rows behind the
// head; the head is published after every batch.  At the end the last 624 rows go back to the
// in-place state array the other kernel families use.
__device__ void producer_run(const DevBatch& b, const DevStrandGraph& g, uint32_t tile, uint32_t sweeps, uint32_t lane) {
    const uint32_t P = g.per_layer, L = g.layers, C = P / 8, S = b.strands, R = b.tape_rows;
    uint32_t* tape = b.tape + size_t(tile) * R * 32 + lane;
    uint32_t* state = b.mt + size_t(tile) * kMtN * 32 + lane;
    uint32_t* flags = b.strand_flags + size_t(tile) * (S + 1) * kFlagStride;
    uint32_t* head_flag = flags + S * kFlagStride;
    const uint32_t pos = b.mt_pos[tile];
    const uint32_t total = sweeps * b.n_spins;  // draws of this launch (a multiple of 8)
    const uint32_t total_blocks = (L / S) * sweeps;

    for (uint32_t i = 0; i < kMtN; ++i) {
        uint32_t w = pos + i;
        w = w >= kMtN ? w - kMtN : w;
        st_u32(tape + size_t(i) * 32, state[size_t(w) * 32]);
    }

    const uint32_t end = kMtN + total;
    uint32_t a = kMtN;      // next row to generate
    uint32_t tail = 0;      // draws known to be consumed by every strand
    uint32_t so = kMtN % R, sa = 0, sf = kMtM % R;  // slots of rows a, a-624, a-227 (624 - 227 = 397)
    uint32_t cur = ld_cg_u32(tape);                         // x[a-624]
    while (a < end) {
        const uint32_t batch = min(32u, end - a);
        // rows a .. a+batch-1 overwrite rows a-R .. : they must be consumed draws (row < 624 + tail)
        while (int32_t(a + batch - R - kMtN - tail) > 0) {
            uint32_t d = 0xffffffffu;
            if (lane < S) d = strand_draw_index(ld_acquire(flags + lane * kFlagStride), lane, S, C, L, P, total_blocks);
            d = __reduce_min_sync(0xffffffffu, d);
            if (d == 0xffffffffu) d = total;
            if (d == tail) __nanosleep(200);
            tail = d;
        }
        for (uint32_t g8 = 0; g8 < batch; g8 += 8) {
            uint32_t nxt[8], far[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                uint32_t s1 = sa + k + 1;  // (sa is a multiple of 8: only sa + 8 can wrap)
                s1 = s1 == R ? 0u : s1;
                uint32_t s2 = sf + k;
                s2 = s2 >= R ? s2 - R : s2;
                nxt[k] = ld_cg_u32(tape + size_t(s1) * 32);
                far[k] = ld_cg_u32(tape + size_t(s2) * 32);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                st_u32(tape + size_t(so + k) * 32, mt_recurrence(cur, nxt[k], far[k]));
                cur = nxt[k];
            }
            so = so + 8 == R ? 0u : so + 8;
            sa = sa + 8 == R ? 0u : sa + 8;
            sf = sf + 8 >= R ? sf + 8 - R : sf + 8;
        }
        a += batch;
        publish(head_flag, a, lane);
    }

    // the generators' state for whoever runs next: word (pos + total + i) % 624 is x[total + i]
    uint32_t w = (pos + total % kMtN) % kMtN, s = total % R;
    for (uint32_t i = 0; i < kMtN; ++i) {
        state[size_t(w) * 32] = ld_cg_u32(tape + size_t(s) * 32);
        w = w + 1 == kMtN ? 0u : w + 1;
        s = s + 1 == R ? 0u : s + 1;
    }
    if (lane == 0) b.mt_pos[tile] = (pos + total % kMtN) % kMtN;
}

// Persistent grid of independent warps.  Work items of a round: for each of `tiles_per_round` tiles
// its S strands and its producer; every item of a round is resident at once (the launcher sizes the
// rounds), so the waits above always end.
template <int EXP, bool WAIT>
__global__ void __launch_bounds__(kStrandMaxWarps * 32, 1) sweep_strand_kernel(DevBatch b, uint32_t sweeps,
                                                                                 uint32_t tiles_per_round) {
    __shared__ float scratch_all[kStrandMaxWarps][8][32];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t item = warp * gridDim.x + blockIdx.x;
    const uint32_t S = b.strands;
    for (uint32_t base = 0; base < b.n_tiles; base += tiles_per_round) {
        const uint32_t tiles = min(tiles_per_round, b.n_tiles - base);
        if (item >= tiles * (S + 1)) continue;
        // consecutive items are the same role of consecutive tiles: an SM hosts a mix of tiles
        const uint32_t role = item / tiles, tile = base + item - role * tiles;
        const DevStrandGraph& g = b.strand_graphs[b.tile_model[tile]];
        if (role == S) producer_run(b, g, tile, sweeps, lane);
        else strand_run<EXP, WAIT>(b, g, tile, role, sweeps, lane, &scratch_all[warp][0][lane]);
    }
}

// spin words [tile][spin] (bit = lane) -> spin bytes [tile][spin/8][lane] (bit = position in the chunk)
__global__ void __launch_bounds__(256) words_to_bytes_kernel(DevBatch b) {
    const size_t idx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t chunks = size_t(b.n_tiles) * (b.n_spins / 8);
    if (idx >= chunks * 32) return;
    const size_t chunk = idx >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    const uint4* w = reinterpret_cast<const uint4*>(b.spin_bits + chunk * 8);
    const uint4 lo = w[0], hi = w[1];
    const uint32_t word[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t byte = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) byte |= ((word[k] >> lane) & 1u) << k;
    b.spin_bytes[idx] = uint8_t(byte);
}

__global__ void __launch_bounds__(256) bytes_to_words_kernel(DevBatch b) {
    const size_t idx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t chunks = size_t(b.n_tiles) * (b.n_spins / 8);
    if (idx >= chunks * 32) return;  // (whole warps: the total is a multiple of 32)
    const size_t chunk = idx >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t byte = b.spin_bytes[idx];
    uint32_t mine = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t word = __ballot_sync(0xffffffffu, (byte >> k) & 1u);
        if (lane == uint32_t(k)) mine = word;
    }
    if (lane < 8) b.spin_bits[chunk * 8 + lane] = mine;
}

}  // namespace

uint32_t strand_max_warps() { return kStrandMaxWarps; }
uint32_t strand_flag_words(uint32_t n_tiles, uint32_t strands) { return n_tiles * (strands + 1) * kFlagStride; }

cudaError_t launch_sweep_strand(const DevBatch& b, uint32_t sweeps, int sm_count, uint32_t warps_per_cta,
                                cudaStream_t stream) {
    if (b.n_tiles == 0 || sweeps == 0) return cudaSuccess;
    const uint32_t capacity = uint32_t(sm_count) * warps_per_cta;
    const uint32_t per_tile = b.strands + 1;
    const uint32_t tiles_per_round = min(b.n_tiles, capacity / per_tile);
    if (tiles_per_round == 0) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaMemsetAsync(b.strand_flags, 0, size_t(strand_flag_words(b.n_tiles, b.strands)) * 4, stream);
    if (e != cudaSuccess) return e;
    const size_t cells = size_t(b.n_tiles) * (b.n_spins / 8) * 32;
    const unsigned convert_blocks = unsigned((cells + 255) / 256);
    words_to_bytes_kernel<<<convert_blocks, 256, 0, stream>>>(b);
    // no more CTAs than the first round's items need
    const uint32_t items = tiles_per_round * per_tile;
    const uint32_t ctas = min(uint32_t(sm_count), (items + warps_per_cta - 1) / warps_per_cta);
    const dim3 grid(ctas), block(warps_per_cta * 32);
    // items are dealt warp-major over the launched CTAs: recompute the round size for this grid
    const uint32_t round = min(b.n_tiles, ctas * warps_per_cta / per_tile);
    // the wait-statistics variant is a separate instantiation: the default kernel carries none of it
    const bool wait = b.wait_counts != nullptr;
#define ISING_LAUNCH_STRAND(EXP)                                                              \
    if (wait) sweep_strand_kernel<EXP, true><<<grid, block, 0, stream>>>(b, sweeps, round);   \
    else sweep_strand_kernel<EXP, false><<<grid, block, 0, stream>>>(b, sweeps, round);
    switch (b.exp_kind) {
        case kExpExact: ISING_LAUNCH_STRAND(kExpExact) break;
        case kExpFast: ISING_LAUNCH_STRAND(kExpFast) break;
        default: ISING_LAUNCH_STRAND(kExpAccurate) break;
    }
#undef ISING_LAUNCH_STRAND
    bytes_to_words_kernel<<<convert_blocks, 256, 0, stream>>>(b);
    return cudaGetLastError();
}

}  // namespace isingb200
