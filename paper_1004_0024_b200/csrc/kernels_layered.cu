// Layered-model sweep kernel: the performance path for identical-layer ("QMC-style") models.
//
// One persistent CTA per SM, four sweep warps per CTA, one warp per tile of 32 chains
// (lane = chain).  What makes it fast is that a chain's working set for one layer lives ON CHIP:
//
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
//   * One layer's graph (CSR of in-layer targets with doubled couplings) sits in shared memory.
//
// HBM traffic per sweep is therefore one read and one write of the f32 space fields plus the bit
// words: 8.25 B per attempt, streamed layer by layer with full 128-byte lines per warp access.
// The trajectory is the reference's (ref: proj/src/sweep_basic.cpp:12-56) bit for bit.
#include "device_batch.hpp"
#include "device_math.cuh"
#include "device_mt.cuh"

namespace isingb200 {

namespace {

constexpr int kSweepWarps = 4;          // one TMEM lane quarter each
constexpr int kLayeredThreads = kSweepWarps * 32;
constexpr uint32_t kTmemColumns = 512;  // the whole TMEM: one CTA per SM

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

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ---- shared-memory carve-up (per CTA): [tmem base][per-warp region x 4]
struct WarpSmem {
    uint32_t* offsets;   // P + 1
    float* j2;           // max_edges
    float* tau2;         // P
    float* tau2g;        // P
    uint32_t* words;     // 3 * P : ring of spin-bit layers
    uint16_t* targets;   // max_edges
};

__host__ __device__ inline size_t warp_region_bytes(uint32_t P, uint32_t max_edges) {
    size_t words = size_t(P + 1) + max_edges + 2 * size_t(P) + 3 * size_t(P);
    size_t bytes = words * 4 + ((size_t(max_edges) * 2 + 15) / 16) * 16;
    return (bytes + 15) / 16 * 16;
}

__device__ __forceinline__ WarpSmem carve(unsigned char* base, uint32_t P, uint32_t max_edges) {
    WarpSmem s;
    uint32_t* w = reinterpret_cast<uint32_t*>(base);
    s.offsets = w;
    w += P + 1;
    s.j2 = reinterpret_cast<float*>(w);
    w += max_edges;
    s.tau2 = reinterpret_cast<float*>(w);
    w += P;
    s.tau2g = reinterpret_cast<float*>(w);
    w += P;
    s.words = w;
    w += 3 * P;
    s.targets = reinterpret_cast<uint16_t*>(w);
    return s;
}

// Copies one layer of spin-bit words between HBM and the warp's ring (each lane its own slice).
__device__ __forceinline__ void words_load(uint32_t* dst, const uint32_t* src, uint32_t P, uint32_t lane) {
    for (uint32_t k = lane; k < P; k += 32) dst[k] = src[k];
}
__device__ __forceinline__ void words_store(uint32_t* dst, const uint32_t* src, uint32_t P, uint32_t lane) {
    for (uint32_t k = lane; k < P; k += 32) dst[k] = src[k];
}

template <int EXP>
__global__ void __launch_bounds__(kLayeredThreads, 1) sweep_layered_kernel(DevBatch b, uint32_t sweeps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t n = b.n_spins;

    if (warp == 0) tmem_alloc(tmem_slot, kTmemColumns);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = *tmem_slot;
    // this warp's lane quarter: bits 31..16 of a TMEM address are the lane, 15..0 the column
    const uint32_t tm = tmem_base + ((warp * 32u) << 16);

    // tiles are dealt round-robin: CTA c, warp w, round r -> tile c + grid*(w + 4r)
    for (uint32_t tile = blockIdx.x + gridDim.x * warp; tile < b.n_tiles; tile += gridDim.x * kSweepWarps) {
        const DevLayerGraph g = b.layer_graphs[b.tile_model[tile]];
        const uint32_t P = g.per_layer, L = g.layers;
        const WarpSmem s =
            carve(smem_raw + 16 + size_t(warp) * warp_region_bytes(b.max_per_layer, b.max_layer_edges), P,
                  b.max_layer_edges);
        // ---- graph of one layer into shared memory
        for (uint32_t k = lane; k <= P; k += 32) s.offsets[k] = g.offsets[k];
        for (uint32_t k = lane; k < g.n_edges; k += 32) {
            s.j2[k] = g.j2[k];
            s.targets[k] = g.targets[k];
        }
        for (uint32_t k = lane; k < P; k += 32) {
            s.tau2[k] = g.tau2[k];
            s.tau2g[k] = g.tau2g[k];
        }

        const bool active = lane < b.tile_count[tile];
        const uint32_t chain = b.tile_first[tile] + lane;
        const float neg_beta = active ? -b.betas[b.slot_of_chain[chain]] : 0.0f;
        double e_run = active ? b.e_run[chain] : 0.0;
        unsigned long long flips = 0;
        float* hs_g = b.hs + size_t(tile) * n * 32 + lane;
        uint32_t* words_g = b.spin_bits + size_t(tile) * n;
        MtLane rng;
        rng.open(b.mt + size_t(tile) * kMtN * 32 + lane, 32, b.mt_pos[tile]);

        // ring of three word layers (previous, current, next); slots rotate as the sweep advances
        uint32_t slot_dn = 2, slot_cur = 0, slot_up = 1;
        words_load(s.words + slot_dn * P, words_g + size_t(L - 1) * P, P, lane);
        words_load(s.words + slot_cur * P, words_g, P, lane);
        words_load(s.words + slot_up * P, words_g + size_t(1) * P, P, lane);
        __syncwarp();

        for (uint32_t sw = 0; sw < sweeps; ++sw) {
            for (uint32_t l = 0; l < L; ++l) {
                float* hs_l = hs_g + size_t(l) * P * 32;
                const float* hs_next = hs_g + size_t(l + 1 == L ? 0 : l + 1) * P * 32;
                // ---- feed: this layer's fields HBM -> TMEM, 8 columns per step
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
                tmem_wait_st();

                uint32_t* w_cur = s.words + slot_cur * P;
                const uint32_t* w_up = s.words + slot_up * P;
                const uint32_t* w_dn = s.words + slot_dn * P;

                for (uint32_t p0 = 0; p0 < P; p0 += kChunk) {
                    const uint32_t count = min(uint32_t(kChunk), P - p0);
                    float u[kChunk];
                    rng.next_chunk(count, u);
                    // pull the same positions of the next layer towards L2 while this one computes
                    if (lane < count) prefetch_l2(hs_next + size_t(p0 + lane) * 32 - lane);
#pragma unroll
                    for (int k = 0; k < kChunk; ++k) {
                        if (uint32_t(k) >= count) break;
                        const uint32_t p = p0 + k;
                        const uint32_t word = w_cur[p];
                        const uint32_t sbit = (word >> lane) & 1u;
                        const uint32_t ub = (w_up[p] >> lane) & 1u, db = (w_dn[p] >> lane) & 1u;
                        const float h = tmem_ld(tm + p);
                        // tau field J*(s_up + s_dn): +/-2J when the neighbours agree, +0 otherwise
                        const float t2g = s.tau2g[p], t2 = s.tau2[p];
                        const float htg = ub == db ? (ub ? -t2g : t2g) : 0.0f;
                        const float ht = ub == db ? (ub ? -t2 : t2) : 0.0f;
                        const float two_s = sbit ? -2.0f : 2.0f;
                        tmem_wait_ld();
                        const float x = __fmul_rn(neg_beta, __fmul_rn(two_s, __fadd_rn(h, htg)));
                        const float pr = exp_kind<EXP>(x);
                        const bool accept = active && (u[k] < pr);
                        const uint32_t ballot = __ballot_sync(0xffffffffu, accept);
                        if (ballot != 0u) {
                            const uint32_t e1 = s.offsets[p + 1];
                            for (uint32_t e = s.offsets[p]; e < e1; ++e) {
                                const uint32_t col = tm + s.targets[e];
                                const float j2 = s.j2[e];
                                const float old = tmem_ld(col);
                                const float d = sbit ? -j2 : j2;  // (2s)*J, exact
                                tmem_wait_ld();
                                tmem_st(col, accept ? __fsub_rn(old, d) : old);
                            }
                            if (accept) {
                                ++flips;
                                e_run = __dadd_rn(e_run, double(__fmul_rn(two_s, __fadd_rn(h, ht))));
                            }
                            if (lane == 0) w_cur[p] = word ^ ballot;
                            tmem_wait_st();
                        }
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
                words_store(words_g + size_t(l) * P, w_cur, P, lane);
                // layer l-1's slot is free now: it receives layer l+2 (the `up` of the next layer)
                const uint32_t l2 = (l + 2) % L;
                __syncwarp();
                words_load(s.words + slot_dn * P, words_g + size_t(l2) * P, P, lane);
                __syncwarp();
                const uint32_t freed = slot_dn;
                slot_dn = slot_cur;
                slot_cur = slot_up;
                slot_up = freed;
            }
        }

        if (lane == 0) b.mt_pos[tile] = rng.pos;
        if (active) {
            b.e_run[chain] = e_run;
            b.flips[chain] += flips;
        }
        __syncwarp();
    }

    tmem_wait_ld();
    tmem_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, kTmemColumns);
}

}  // namespace

size_t layered_smem_bytes(uint32_t per_layer, uint32_t max_layer_edges) {
    if (per_layer == 0 || per_layer > kTmemColumns) return 0;
    const size_t bytes = 16 + kSweepWarps * warp_region_bytes(per_layer, max_layer_edges);
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
    // all models of a batch share n_spins but may differ in per_layer; size for the largest region
    const size_t smem = size_t(b.layered_smem);
    const uint32_t ctas = uint32_t(sm_count) < (b.n_tiles + 0u) ? uint32_t(sm_count) : b.n_tiles;
    const dim3 grid(ctas ? ctas : 1);
    switch (b.exp_kind) {
        case kExpExact: sweep_layered_kernel<kExpExact><<<grid, kLayeredThreads, smem, stream>>>(b, sweeps); break;
        case kExpFast: sweep_layered_kernel<kExpFast><<<grid, kLayeredThreads, smem, stream>>>(b, sweeps); break;
        default: sweep_layered_kernel<kExpAccurate><<<grid, kLayeredThreads, smem, stream>>>(b, sweeps); break;
    }
    return cudaGetLastError();
}

}  // namespace isingb200
