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
//     4 B = the whole 256 KB TMEM of an SM for 4 warps x 512 positions).  Every neighbour
//     update of a flip is a tcgen05.ld / tcgen05.st on a warp-uniform column — no HBM traffic.
//   * The tau field is NOT stored.  For these models it only takes the values {2J, +0, -2J}
//     and every incremental update of it is exact (HostModel::layered_uniform), so it is rebuilt
//     from two spin bits of the adjacent layers.  That removes 8 of the 17 bytes per attempt the
//     generic layout streams, and both tau read-modify-writes of every flip.
//   * Spins are one bit per chain: a 32-bit word per (tile, spin) holds the 32 lanes' signs.
//     Three layers of words (previous, current, next) sit in shared memory per warp.
//   * One layer's graph ({column, 2J} per half-edge) sits in shared memory.
//   * The RNG warp regenerates the chains' MT19937 states (replica-interleaved in HBM/L2) and
//     hands uniforms over through a shared-memory ring guarded by mbarriers.
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
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr) : "memory");
    return __uint_as_float(v);
}
__device__ __forceinline__ void tmem_st(uint32_t taddr, float v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(__float_as_uint(v))
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done;
    do {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
    } while (done == 0u);
}

// ---- shared-memory carve-up (per CTA): [tmem base | barriers][per-pair region x 4]
struct PairSmem {
    uint32_t* offsets;  // P + 1
    uint2* edges;       // max_edges : {TMEM column, bits of 2J}
    float2* tau;        // P : {gamma*2J_tau, 2J_tau}
    uint2* agree_sign;  // P : per layer, {~(up ^ dn), up} spin words
    uint32_t* words;    // 3 * P : ring of spin-bit layers
    float* ring;        // kStages * kStageDraws * 32 uniforms
};

constexpr size_t kHeaderBytes = 256;  // tmem slot + 4 pairs x (full[kStages] + empty[kStages]) barriers

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) / 16 * 16; }

__host__ __device__ inline size_t pair_region_bytes(uint32_t P, uint32_t max_edges) {
    return align16(size_t(P + 1) * 4) + align16(size_t(max_edges) * 8) + align16(size_t(P) * 8) +
           align16(size_t(P) * 8) + align16(size_t(P) * 12) + size_t(kStages) * kStageDraws * 32 * 4;
}

__device__ __forceinline__ PairSmem carve(unsigned char* base, uint32_t P, uint32_t max_edges) {
    PairSmem s;
    s.offsets = reinterpret_cast<uint32_t*>(base);
    base += align16(size_t(P + 1) * 4);
    s.edges = reinterpret_cast<uint2*>(base);
    base += align16(size_t(max_edges) * 8);
    s.tau = reinterpret_cast<float2*>(base);
    base += align16(size_t(P) * 8);
    s.agree_sign = reinterpret_cast<uint2*>(base);
    base += align16(size_t(P) * 8);
    s.words = reinterpret_cast<uint32_t*>(base);
    base += align16(size_t(P) * 12);
    s.ring = reinterpret_cast<float*>(base);
    return s;
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

__device__ void rng_warp(const DevBatch& b, uint32_t sweeps, uint32_t pair, uint32_t lane, const PairSmem& s,
                         uint64_t* full, uint64_t* empty, RingCursor& cursor, uint32_t tile) {
    uint32_t* w = b.mt + size_t(tile) * kMtN * 32 + lane;
    uint32_t pos = b.mt_pos[tile];
    uint32_t cur = w[size_t(pos) * 32];
    uint64_t remaining = uint64_t(sweeps) * b.n_spins;
    while (remaining != 0) {
        const uint32_t take = remaining < kStageDraws ? uint32_t(remaining) : kStageDraws;
        mbar_wait(&empty[cursor.stage], cursor.parity ^ 1u);
        mt_generate(w, pos, cur, take, s.ring + size_t(cursor.stage) * kStageDraws * 32 + lane);
        mbar_arrive(&full[cursor.stage]);
        cursor.advance();
        remaining -= take;
    }
    if (lane == 0) b.mt_pos[tile] = pos;
    (void)pair;
}

// ---------------------------------------------------------------------------------------
template <int EXP>
__device__ void sweep_warp(const DevBatch& b, uint32_t sweeps, uint32_t lane, const PairSmem& s, uint64_t* full,
                           uint64_t* empty, RingCursor& cursor, uint32_t tile, uint32_t tm,
                           const DevLayerGraph& g) {
    const uint32_t P = g.per_layer, L = g.layers, n = b.n_spins;
    const bool active = lane < b.tile_count[tile];
    const uint32_t chain = b.tile_first[tile] + lane;
    // -2*beta: x = -beta*((2s)*v) == (-2*beta*s)*v exactly (doubling is exact, one rounding each way)
    const uint32_t nb2 = __float_as_uint(active ? -2.0f * b.betas[b.slot_of_chain[chain]] : 0.0f);
    double e_run = active ? b.e_run[chain] : 0.0;
    uint32_t flips = 0;
    float* hs_g = b.hs + size_t(tile) * n * 32 + lane;
    uint32_t* words_g = b.spin_bits + size_t(tile) * n;
    const uint32_t sh = 31u - lane;  // shift that brings this lane's bit to the sign position

    uint32_t slot_dn = 2, slot_cur = 0, slot_up = 1;
    words_copy(s.words + slot_dn * P, words_g + size_t(L - 1) * P, P, lane);
    words_copy(s.words + slot_cur * P, words_g, P, lane);
    words_copy(s.words + slot_up * P, words_g + size_t(1) * P, P, lane);
    __syncwarp();

    uint32_t ui = 0;        // draws consumed from the current ring stage
    bool have_stage = false;
    const float* ring = s.ring + lane;

    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t l = 0; l < L; ++l) {
            float* hs_l = hs_g + size_t(l) * P * 32;
            const float* hs_next = hs_g + size_t(l + 1 == L ? 0 : l + 1) * P * 32 - lane;
            // ---- feed: this layer's fields HBM -> TMEM
            for (uint32_t p0 = 0; p0 < P; p0 += 32) {
                float v[4][8];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t p = p0 + q * 8 + k;
                        v[q][k] = p < P ? hs_l[size_t(p) * 32] : 0.0f;
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (p0 + q * 8 < P) tmem_st8(tm + p0 + q * 8, v[q]);
                }
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

            for (uint32_t p = 0; p < P; ++p) {
                if (!have_stage) {
                    mbar_wait(&full[cursor.stage], cursor.parity);
                    have_stage = true;
                }
                const float u = ring[(size_t(cursor.stage) * kStageDraws + ui) * 32];
                const float h = tmem_ld(tm + p);
                const uint2 as = s.agree_sign[p];
                const float2 tau = s.tau[p];
                const uint32_t word = w_cur[p];
                if ((p & 31u) == 0 && p + lane < P) prefetch_l2(hs_next + size_t(p + lane) * 32);
                const uint32_t sgn_s = (word << sh) & 0x80000000u;       // sign bit set <=> s = -1
                const uint32_t sgn_up = (as.y << sh) & 0x80000000u;
                const uint32_t agree = uint32_t(int32_t(as.x << sh) >> 31);  // all ones when s_up == s_dn
                // tau field J*(s_up + s_dn) in {+2J, +0, -2J}, scaled by gamma for the exponent
                const float htg = __uint_as_float((__float_as_uint(tau.x) ^ sgn_up) & agree);
                tmem_wait_ld();
                const float v = __fadd_rn(h, htg);
                const float x = __fmul_rn(__uint_as_float(nb2 ^ sgn_s), v);
                const float pr = exp_kind<EXP>(x);
                const bool accept = active && (u < pr);
                const uint32_t ballot = __ballot_sync(0xffffffffu, accept);
                if (ballot != 0u) {
                    const uint32_t neg_d = sgn_s ^ 0x80000000u;  // sign of -(2s): h -= (2s)*J == h + (-(2s)J)
                    const uint32_t e1 = s.offsets[p + 1];
                    for (uint32_t e = s.offsets[p]; e < e1; ++e) {
                        const uint2 ed = s.edges[e];
                        const float old = tmem_ld(tm + ed.x);
                        const float nd = __uint_as_float(ed.y ^ neg_d);
                        tmem_wait_ld();
                        tmem_st(tm + ed.x, accept ? __fadd_rn(old, nd) : old);
                    }
                    if (accept) {
                        ++flips;
                        const float ht = __uint_as_float((__float_as_uint(tau.y) ^ sgn_up) & agree);
                        const float two_s = __uint_as_float(0x40000000u ^ sgn_s);
                        e_run = __dadd_rn(e_run, double(__fmul_rn(two_s, __fadd_rn(h, ht))));
                    }
                    if (lane == 0) w_cur[p] = word ^ ballot;
                    tmem_wait_st();
                }
                if (++ui == kStageDraws) {
                    mbar_arrive(&empty[cursor.stage]);
                    cursor.advance();
                    ui = 0;
                    have_stage = false;
                }
            }

            // ---- retire: TMEM -> HBM, and rotate the spin-bit ring
            for (uint32_t p0 = 0; p0 < P; p0 += 8) {
                float v[8];
                tmem_ld8(tm + p0, v);
                tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (p0 + k < P) hs_l[size_t(p0 + k) * 32] = v[k];
                }
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
    if (active) {
        b.e_run[chain] = e_run;
        b.flips[chain] += flips;
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

    if (warp == 0) tmem_alloc(tmem_slot, kTmemColumns);
    if (threadIdx.x < kSweepWarps * 2 * kStages) mbar_init(&bars[threadIdx.x], 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = *tmem_slot;
    // this pair's lane quarter: bits 31..16 of a TMEM address are the lane, 15..0 the column
    const uint32_t tm = tmem_base + ((pair * 32u) << 16);
    const PairSmem s = carve(smem_raw + kHeaderBytes + size_t(pair) * pair_region_bytes(b.max_per_layer, b.max_layer_edges),
                             b.max_per_layer, b.max_layer_edges);
    RingCursor cursor;

    // tiles are dealt round-robin: CTA c, pair w, round r -> tile c + grid*(w + 4r)
    for (uint32_t tile = blockIdx.x + gridDim.x * pair; tile < b.n_tiles; tile += gridDim.x * kSweepWarps) {
        if (is_rng) {
            rng_warp(b, sweeps, pair, lane, s, full, empty, cursor, tile);
        } else {
            const DevLayerGraph g = b.layer_graphs[b.tile_model[tile]];
            // ---- graph of one layer into shared memory
            for (uint32_t k = lane; k <= g.per_layer; k += 32) s.offsets[k] = g.offsets[k];
            for (uint32_t k = lane; k < g.n_edges; k += 32) {
                s.edges[k] = make_uint2(uint32_t(g.targets[k]), __float_as_uint(g.j2[k]));
            }
            for (uint32_t k = lane; k < g.per_layer; k += 32) s.tau[k] = make_float2(g.tau2g[k], g.tau2[k]);
            __syncwarp();
            sweep_warp<EXP>(b, sweeps, lane, s, full, empty, cursor, tile, tm, g);
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

size_t layered_smem_bytes(uint32_t per_layer, uint32_t max_layer_edges) {
    if (per_layer == 0 || per_layer > kTmemColumns) return 0;
    const size_t bytes = kHeaderBytes + kSweepWarps * pair_region_bytes(per_layer, max_layer_edges);
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
