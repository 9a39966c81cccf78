// Intra-system ("coalesced") sweep kernel: one warp per chain, W = L/2 lanes, see coalesced.hpp.
//
// The region being swept (even or odd layers: W*P spins) is staged in shared memory, so the
// strictly sequential walk over the P positions pays shared-memory latency per step, not L2:
//   hs, ht f32 [P][W], spins i8 [P][W], flip flags one bit per (p, lane).
// Lane t only ever touches column t of the staged region (space edges stay inside a layer), so a
// phase needs no synchronisation.  The two tau updates of a flip leave the region (previous layer:
// immediately; next layer: in the deferred phase, ref: sweep_coalesced.cpp:10-22): they go to the
// OTHER region's h_tau in global memory as fire-and-forget `red.global.add.f32` of the negated
// addend — h - d == h + (-d) bit for bit, every location receives at most one update per phase, and
// a fence + warp barrier between phases keeps the reference's order (immediate, then deferred).
#include "coalesced.hpp"
#include "device_math.cuh"
#include "device_mt.cuh"

namespace isingb200 {

namespace {

struct RegionSmem {
    float* hs;
    float* ht;
    int8_t* spins;
    uint32_t* flags;  // [ceil(P/32)][32]
};

__host__ __device__ inline size_t region_bytes(uint32_t lanes, uint32_t per_layer) {
    const size_t cells = size_t(lanes) * per_layer;
    return cells * 4 * 2 + (cells + 15) / 16 * 16 + size_t((per_layer + 31) / 32) * 32 * 4;
}

template <int EXP>
__global__ void __launch_bounds__(32) sweep_coalesced_kernel(CoalescedDev d, uint32_t sweeps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t chain = blockIdx.x, lane = threadIdx.x;
    const uint32_t W = d.lanes, P = d.per_layer, n = d.n_spins, cells = W * P;
    const bool active = lane < W;
    RegionSmem s;
    s.hs = reinterpret_cast<float*>(smem_raw);
    s.ht = s.hs + cells;
    s.spins = reinterpret_cast<int8_t*>(s.ht + cells);
    s.flags = reinterpret_cast<uint32_t*>(smem_raw + size_t(cells) * 8 + (size_t(cells) + 15) / 16 * 16);

    float* hs_g = d.hs + size_t(chain) * n;
    float* ht_g = d.ht + size_t(chain) * n;
    int8_t* spins_g = d.spins + size_t(chain) * n;
    const float neg_beta = -d.betas[chain];
    const float gamma = d.tau_scale;
    unsigned long long flips = 0;

    MtLane g;
    if (active) g.open(d.mt + size_t(chain) * kMtN * W + lane, W, d.mt_pos[chain]);

    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t region = 0; region < 2; ++region) {
            const uint32_t base = region * cells;
            // ---- stage the region in (the other region's tau updates of the previous phase pair
            // have been fenced below)
            for (uint32_t k = lane; k < cells; k += 32) {
                s.hs[k] = hs_g[base + k];
                s.ht[k] = ht_g[base + k];
                s.spins[k] = spins_g[base + k];
            }
            for (uint32_t k = lane; k < (P + 31) / 32 * 32; k += 32) s.flags[k] = 0u;
            __syncwarp();

            // ---- flip phase (ref: flip_phase, sweep_coalesced.cpp:45-83)
            for (uint32_t p0 = 0; p0 < P; p0 += kChunk) {
                const uint32_t count = min(uint32_t(kChunk), P - p0);
                float u[kChunk];
                if (active) g.next_chunk(count, u);
#pragma unroll
                for (int k = 0; k < kChunk; ++k) {
                    if (uint32_t(k) >= count) break;
                    const uint32_t p = p0 + k;
                    if (!active) continue;
                    const uint32_t cell = W * p + lane;
                    const float spin = float(s.spins[cell]);
                    const float two_s = __fmul_rn(2.0f, spin);
                    const float x = flip_exponent(neg_beta, gamma, two_s, s.hs[cell], s.ht[cell]);
                    if (u[k] < exp_kind<EXP>(x)) {  // no clamp (ref: sweep_coalesced.cpp:66)
                        const uint32_t i = base + cell;
                        const uint32_t end = d.offsets[i + 1];
                        for (uint32_t e = d.offsets[i]; e + 2 < end; ++e) {
                            const uint32_t t = d.targets[e] - base;  // same layer: column `lane` of this region
                            s.hs[t] = __fsub_rn(s.hs[t], __fmul_rn(two_s, d.couplings[e]));
                        }
                        // tau edge to the previous layer now; the one to the next layer waits
                        atomicAdd(ht_g + d.targets[end - 1], -__fmul_rn(two_s, d.couplings[end - 1]));
                        s.spins[cell] = int8_t(-s.spins[cell]);
                        s.flags[(p >> 5) * 32 + lane] |= 1u << (p & 31u);
                        ++flips;
                    }
                }
            }
            __threadfence();
            __syncwarp();

            // ---- deferred phase (ref: deferred_tau_phase, sweep_coalesced.cpp:87-104)
            if (active) {
                for (uint32_t p = 0; p < P; ++p) {
                    if (((s.flags[(p >> 5) * 32 + lane] >> (p & 31u)) & 1u) == 0u) continue;
                    const uint32_t cell = W * p + lane;
                    const float two_s = __fmul_rn(-2.0f, float(s.spins[cell]));  // twice the pre-flip spin
                    const uint32_t up = d.offsets[base + cell + 1] - 2;
                    atomicAdd(ht_g + d.targets[up], -__fmul_rn(two_s, d.couplings[up]));
                }
            }
            // ---- stage out
            __syncwarp();
            for (uint32_t k = lane; k < cells; k += 32) {
                hs_g[base + k] = s.hs[k];
                ht_g[base + k] = s.ht[k];
                spins_g[base + k] = s.spins[k];
            }
            __threadfence();
            __syncwarp();
        }
    }
    if (active && lane == 0) {
        d.mt_pos[chain] = g.pos;
    }
    // flips of all lanes
    for (int off = 16; off > 0; off >>= 1) flips += __shfl_down_sync(0xffffffffu, flips, off);
    if (lane == 0) d.flips[chain] += flips;
}

}  // namespace

size_t coalesced_smem_bytes(uint32_t lanes, uint32_t per_layer) {
    if (lanes == 0 || lanes > 32 || per_layer == 0) return 0;
    const size_t bytes = region_bytes(lanes, per_layer);
    return bytes <= 227 * 1024 ? bytes : 0;
}

cudaError_t prepare_coalesced_kernels(size_t smem_bytes) {
    cudaError_t e = cudaFuncSetAttribute(sweep_coalesced_kernel<kExpExact>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_bytes));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(sweep_coalesced_kernel<kExpFast>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem_bytes));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(sweep_coalesced_kernel<kExpAccurate>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(smem_bytes));
}

cudaError_t launch_sweep_coalesced(const CoalescedDev& d, uint32_t sweeps, size_t smem_bytes, cudaStream_t stream) {
    if (d.n_chains == 0) return cudaSuccess;
    switch (d.exp_kind) {
        case kExpExact: sweep_coalesced_kernel<kExpExact><<<d.n_chains, 32, smem_bytes, stream>>>(d, sweeps); break;
        case kExpFast: sweep_coalesced_kernel<kExpFast><<<d.n_chains, 32, smem_bytes, stream>>>(d, sweeps); break;
        default: sweep_coalesced_kernel<kExpAccurate><<<d.n_chains, 32, smem_bytes, stream>>>(d, sweeps); break;
    }
    return cudaGetLastError();
}

}  // namespace isingb200
