// Intra-system ("coalesced") sweep kernel: one warp per chain, W = L/2 lanes, see coalesced.hpp.
//
// The region being swept (even or odd layers: W*P spins) is staged in shared memory, so the
// strictly sequential walk over the P positions pays shared-memory latency per step, not L2:
//   hs f32 [P][W], spins i8 [P][W], and — when the copy fits (GRAPH = true) — one layer's edge list,
//   read warp-uniformly (validate_model guarantees identical layers).
// Lane t only ever touches column t of the staged region (space edges stay inside a layer), so a
// phase needs no synchronisation.  The region's h_tau is only read (it changes in the OTHER
// region's phases), so it stays in global memory; everything a step needs from there (uniforms,
// tau fields and couplings) is requested a chunk of 8 steps ahead, independent of the decisions.
//
// The two tau updates of a flip leave the region: the edge to the previous layer at once, the edge
// to the next layer in the reference's DEFERRED phase (ref: sweep_coalesced.cpp:10-22, 87-104),
// because a location of the other region can receive one of each in the same flip phase — from
// two neighbouring lanes, both at the same position p — and the immediate one must round first.
// Here the lane that owns the immediate update also applies its neighbour's deferred one: the
// neighbour's addend arrives by warp shuffle in the same step, and the lane issues two
// `red.global.add.f32` to that address in program order (same thread, same address: ordered).
// That is the reference's order per location, without a second pass and without flip flags.
// h - d == h + (-d) bit for bit, so the reductions add the negated addend.
#include "coalesced.hpp"
#include "device_math.cuh"
#include "device_mt.cuh"

namespace isingb200 {

namespace {

__host__ __device__ inline size_t region_bytes(uint32_t lanes, uint32_t per_layer, uint32_t n_layer_edges) {
    const size_t cells = size_t(lanes) * per_layer;
    size_t bytes = cells * 4 + (cells + 15) / 16 * 16;
    if (n_layer_edges != 0) bytes += (size_t(per_layer) + 1 + 3) / 4 * 16 + size_t(n_layer_edges) * 8;
    return bytes;
}

// A load the compiler may not sink into the branch that consumes it (it is issued where it stands).
__device__ __forceinline__ float ld_stream(const float* p) {
    float v;
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

// The same for data this kernel also updates with reductions in other phases: read at L2.
__device__ __forceinline__ float ld_coherent(const float* p) {
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}

template <int EXP, bool GRAPH>
__global__ void __launch_bounds__(32) sweep_coalesced_kernel(CoalescedDev d, uint32_t sweeps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t chain = blockIdx.x, lane = threadIdx.x;
    const uint32_t W = d.lanes, P = d.per_layer, n = d.n_spins, cells = W * P;
    const bool active = lane < W;
    float* hs_s = reinterpret_cast<float*>(smem_raw);
    int8_t* spins_s = reinterpret_cast<int8_t*>(hs_s + cells);
    uint32_t* graph_off = reinterpret_cast<uint32_t*>(smem_raw + size_t(cells) * 4 + (size_t(cells) + 15) / 16 * 16);
    uint2* graph_edges = reinterpret_cast<uint2*>(graph_off + (P + 1 + 3) / 4 * 4);
    if (GRAPH) {
        for (uint32_t k = lane; k <= P; k += 32) graph_off[k] = d.layer_offsets[k];
        for (uint32_t k = lane; k < d.n_layer_edges; k += 32) graph_edges[k] = d.layer_edges[k];
    }

    float* hs_g = d.hs + size_t(chain) * n;
    float* ht_g = d.ht + size_t(chain) * n;
    int8_t* spins_g = d.spins + size_t(chain) * n;
    const float neg_beta = -d.betas[chain];
    const float gamma = d.tau_scale;
    unsigned long long flips = 0;
    const uint32_t lane_c = active ? lane : 0u;  // idle lanes read column 0 and never accept

    MtLane g;
    if (active) g.open(d.mt + size_t(chain) * kMtN * W + lane, W, d.mt_pos[chain]);

    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t region = 0; region < 2; ++region) {
            const uint32_t base = region * cells, other = cells - base;
            // tau targets of (p, lane) in the other region (ref: check_engine_model, sweep_state.cpp:131-141)
            // Location (p, j) of the other region gets the immediate update of lane `j + 1` (even
            // region) or `j` (odd region) and the deferred one of lane `j` resp. `j - 1`: in both
            // regions the deferred addend this lane applies comes from lane - 1.
            const uint32_t down_lane = region == 0 ? (lane_c + W - 1) % W : lane_c;
            const uint32_t source_lane = (lane_c + W - 1) % W;

            // ---- stage the region in (tau updates it received from the other region's phases were
            // fenced before the warp barrier that ended them)
#pragma unroll 8
            for (uint32_t k = lane; k < cells; k += 32) {
                hs_s[k] = hs_g[base + k];
                spins_s[k] = spins_g[base + k];
            }
            __syncwarp();

            // ---- flip phase (ref: flip_phase, sweep_coalesced.cpp:45-83).  The global operands of a
            // chunk (tau couplings, this region's tau fields — which do not change while it is swept)
            // are requested while the chunk before it is processed.
            float j_down_next[kChunk], j_up_next[kChunk], ht_next[kChunk];
            const auto request = [&](uint32_t p0) {
#pragma unroll
                for (int k = 0; k < kChunk; ++k) {
                    const uint32_t at = base + W * min(p0 + k, P - 1) + lane_c;
                    j_down_next[k] = ld_stream(d.tau_down + at);
                    j_up_next[k] = ld_stream(d.tau_up + at);
                    ht_next[k] = ld_coherent(ht_g + at);
                }
            };
            request(0);
            uint32_t mt_next[kChunk], mt_far[kChunk];
            if (active) g.load_operands(min(uint32_t(kChunk), P), mt_next, mt_far);
            for (uint32_t p0 = 0; p0 < P; p0 += kChunk) {
                const uint32_t count = min(uint32_t(kChunk), P - p0);
                float u[kChunk], j_down[kChunk], j_up[kChunk], ht[kChunk];
#pragma unroll
                for (int k = 0; k < kChunk; ++k) {
                    j_down[k] = j_down_next[k];
                    j_up[k] = j_up_next[k];
                    ht[k] = ht_next[k];
                    u[k] = 2.0f;
                }
                if (active) g.generate(count, mt_next, mt_far, u);
                if (p0 + kChunk < P) {
                    request(p0 + kChunk);
                    if (active) g.load_operands(min(uint32_t(kChunk), P - p0 - kChunk), mt_next, mt_far);
                }
#pragma unroll
                for (int k = 0; k < kChunk; ++k) {
                    if (uint32_t(k) >= count) break;
                    const uint32_t p = p0 + k;
                    const uint32_t cell = W * p + lane_c;
                    const int8_t spin_i = spins_s[cell];
                    const float two_s = __fmul_rn(2.0f, float(spin_i));
                    const float x = flip_exponent(neg_beta, gamma, two_s, hs_s[cell], ht[k]);
                    const bool accept = active && u[k] < exp_kind<EXP>(x);  // no clamp (ref: sweep_coalesced.cpp:66)
                    if (GRAPH) {
                        if (__any_sync(0xffffffffu, accept)) {
                            // the targets of one position are distinct (validate_model rejects duplicate
                            // edges): groups of eight are read together, then written together
                            const uint32_t end = graph_off[p + 1];
                            for (uint32_t e0 = graph_off[p]; e0 < end; e0 += 8) {
                                uint2 edge[8];
                                float v[8];
#pragma unroll
                                for (int q = 0; q < 8; ++q) {
                                    edge[q] = graph_edges[min(e0 + q, end - 1)];  // warp-uniform
                                    v[q] = hs_s[W * edge[q].x + lane_c];
                                }
#pragma unroll
                                for (int q = 0; q < 8; ++q) {
                                    if (accept && e0 + q < end) {
                                        hs_s[W * edge[q].x + lane_c] = __fsub_rn(v[q], __fmul_rn(two_s, __uint_as_float(edge[q].y)));
                                    }
                                }
                            }
                        }
                    } else if (accept) {
                        const uint32_t i = base + cell, end = d.offsets[i + 1];
                        for (uint32_t e = d.offsets[i]; e + 2 < end; ++e) {
                            const uint32_t t = d.targets[e] - base;  // same layer: this lane's column
                            hs_s[t] = __fsub_rn(hs_s[t], __fmul_rn(two_s, d.couplings[e]));
                        }
                    }
                    // tau edges: previous layer (mine, first), then next layer of the lane before me
                    const uint32_t accepted = __ballot_sync(0xffffffffu, accept);
                    const float deferred = __shfl_sync(0xffffffffu, -__fmul_rn(two_s, j_up[k]), source_lane);
                    float* tau_cell = ht_g + other + W * p + down_lane;
                    if (accept) {
                        atomicAdd(tau_cell, -__fmul_rn(two_s, j_down[k]));
                        spins_s[cell] = int8_t(-spin_i);
                        ++flips;
                    }
                    if (active && ((accepted >> source_lane) & 1u)) atomicAdd(tau_cell, deferred);
                }
            }
            // ---- stage out
#pragma unroll 8
            for (uint32_t k = lane; k < cells; k += 32) {
                hs_g[base + k] = hs_s[k];
                spins_g[base + k] = spins_s[k];
            }
            __threadfence();
            __syncwarp();
        }
    }
    if (lane == 0) d.mt_pos[chain] = g.pos;
    for (int off = 16; off > 0; off >>= 1) flips += __shfl_down_sync(0xffffffffu, flips, off);
    if (lane == 0) d.flips[chain] += flips;
}

// ------------------------------------------------------------------------------------------
// REGISTER WINDOW variant (per_layer % 8 == 0, identical layers, band table in shared memory).
// As in the layered family, the fields of positions p-2 .. p+2 live in a ring of eight registers
// (indexed by position & 7 in an 8x unrolled chunk): the four band neighbours of a flip — most of
// its edges — are predicated register adds with addends from a per-sign table, an empty slot adds
// -0.0.  Only the remaining ("far") neighbours are read-modify-written in the staged region.  A
// column enters the window after attempt p-3 (after that attempt's far updates, so it is current)
// and leaves it after attempt p+2.
__host__ __device__ inline size_t window_bytes(uint32_t lanes, uint32_t per_layer, uint32_t n_far_edges) {
    const size_t cells = size_t(lanes) * per_layer;
    return cells * 4 + (cells + 15) / 16 * 16 + size_t(per_layer) * 32 + (size_t(per_layer) + 1 + 3) / 4 * 16 +
           size_t(n_far_edges ? n_far_edges : 1) * 8;
}

struct WindowSmem {
    float* hs;
    int8_t* spins;
    const uint4* band_pm;
    const uint32_t* far_off;
    const uint2* far_edges;
};

template <int EXP, int K>
__device__ __forceinline__ void window_step(float (&r)[8], const WindowSmem& s, uint32_t W, uint32_t P, uint32_t p0,
                                            uint32_t lane, uint32_t lane_c, bool active, float u, float ht, float j_up,
                                            float j_down, float neg_beta, float gamma, float* tau_row,
                                            uint32_t down_lane, uint32_t source_lane, unsigned long long& flips) {
    const uint32_t p = p0 + K;
    const uint32_t cell = W * p + lane_c;
    const int8_t spin_i = s.spins[cell];
    const float two_s = __fmul_rn(2.0f, float(spin_i));
    const float h = r[K];
    const float x = flip_exponent(neg_beta, gamma, two_s, h, ht);
    const bool accept = active && u < exp_kind<EXP>(x);  // no clamp (ref: sweep_coalesced.cpp:66)

    // band neighbours: h -= (2s)*J  ==  h + (-(2s)*J); the table entry is picked by the spin's sign
    const uint4 op = s.band_pm[2 * p + (spin_i > 0 ? 1 : 0)];
    const float a0 = __fadd_rn(r[(K + 6) & 7], __uint_as_float(op.x));
    const float a1 = __fadd_rn(r[(K + 7) & 7], __uint_as_float(op.y));
    const float a2 = __fadd_rn(r[(K + 1) & 7], __uint_as_float(op.z));
    const float a3 = __fadd_rn(r[(K + 2) & 7], __uint_as_float(op.w));
    r[(K + 6) & 7] = accept ? a0 : r[(K + 6) & 7];
    r[(K + 7) & 7] = accept ? a1 : r[(K + 7) & 7];
    r[(K + 1) & 7] = accept ? a2 : r[(K + 1) & 7];
    r[(K + 2) & 7] = accept ? a3 : r[(K + 2) & 7];
    // column p-2 leaves the window
    if (K >= 2 || p0 != 0) s.hs[W * (p - 2) + lane_c] = r[(K + 6) & 7];

    // far neighbours, in the staged region (never inside the window: |t - p| > 2)
    const uint32_t accepted = __ballot_sync(0xffffffffu, accept);
    if (accepted != 0u) {
        const uint32_t end = s.far_off[p + 1];
        for (uint32_t e = s.far_off[p]; e < end; ++e) {
            const uint2 edge = s.far_edges[e];  // warp-uniform
            const uint32_t t = W * edge.x + lane_c;
            const float v = s.hs[t];  // every lane rewrites its own cell, accepting lanes with the new value
            s.hs[t] = accept ? __fsub_rn(v, __fmul_rn(two_s, __uint_as_float(edge.y))) : v;
        }
    }
    // column p+3 enters (after the far updates above: it may have been one of their targets)
    if (K <= 4 || p0 + 8 < P) r[(K + 3) & 7] = s.hs[W * (p + 3) + lane_c];

    // tau edges: previous layer (mine, first), then next layer of the lane before me (see the file header)
    // (branch-free: a lane without an update adds -0.0, the identity for every value, when any lane has one)
    const float mine_up = accept ? -__fmul_rn(two_s, j_up) : -0.0f;
    const float deferred = __shfl_sync(0xffffffffu, mine_up, source_lane);
    if (accepted != 0u) {
        float* tau_cell = tau_row + W * p + down_lane;
        if (active) {
            atomicAdd(tau_cell, accept ? -__fmul_rn(two_s, j_down) : -0.0f);
            atomicAdd(tau_cell, deferred);
        }
        s.spins[cell] = accept ? int8_t(-spin_i) : spin_i;
        flips += accept ? 1u : 0u;
    }
}

template <int EXP>
__global__ void __launch_bounds__(32) sweep_coalesced_window_kernel(CoalescedDev d, uint32_t sweeps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t chain = blockIdx.x, lane = threadIdx.x;
    const uint32_t W = d.lanes, P = d.per_layer, n = d.n_spins, cells = W * P;
    const bool active = lane < W;
    WindowSmem s;
    s.hs = reinterpret_cast<float*>(smem_raw);
    s.spins = reinterpret_cast<int8_t*>(s.hs + cells);
    uint4* band = reinterpret_cast<uint4*>(smem_raw + size_t(cells) * 4 + (size_t(cells) + 15) / 16 * 16);
    uint32_t* far_off = reinterpret_cast<uint32_t*>(band + 2 * size_t(P));
    uint2* far_edges = reinterpret_cast<uint2*>(far_off + (P + 1 + 3) / 4 * 4);
    for (uint32_t k = lane; k < 2 * P; k += 32) band[k] = d.band_pm[k];
    for (uint32_t k = lane; k <= P; k += 32) far_off[k] = d.far_offsets[k];
    for (uint32_t k = lane; k < d.n_far_edges; k += 32) far_edges[k] = d.far_edges[k];
    s.band_pm = band;
    s.far_off = far_off;
    s.far_edges = far_edges;

    float* hs_g = d.hs + size_t(chain) * n;
    float* ht_g = d.ht + size_t(chain) * n;
    int8_t* spins_g = d.spins + size_t(chain) * n;
    const float neg_beta = -d.betas[chain];
    const float gamma = d.tau_scale;
    unsigned long long flips = 0;
    const uint32_t lane_c = active ? lane : 0u;  // idle lanes read column 0 and never accept

    MtLane g;
    if (active) g.open(d.mt + size_t(chain) * kMtN * W + lane, W, d.mt_pos[chain]);

    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t region = 0; region < 2; ++region) {
            const uint32_t base = region * cells, other = cells - base;
            const uint32_t down_lane = region == 0 ? (lane_c + W - 1) % W : lane_c;
            const uint32_t source_lane = (lane_c + W - 1) % W;
#pragma unroll 8
            for (uint32_t k = lane; k < cells; k += 32) {
                s.hs[k] = hs_g[base + k];
                s.spins[k] = spins_g[base + k];
            }
            __syncwarp();

            float r[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = 0.0f;
            r[0] = s.hs[W * 0 + lane_c];
            r[1] = s.hs[W * 1 + lane_c];
            r[2] = s.hs[W * 2 + lane_c];

            float j_down_next[kChunk], j_up_next[kChunk], ht_next[kChunk];
            const auto request = [&](uint32_t p0) {
#pragma unroll
                for (int k = 0; k < kChunk; ++k) {
                    const uint32_t at = base + W * (p0 + k) + lane_c;
                    j_down_next[k] = ld_stream(d.tau_down + at);
                    j_up_next[k] = ld_stream(d.tau_up + at);
                    ht_next[k] = ld_coherent(ht_g + at);
                }
            };
            request(0);
            uint32_t mt_next[kChunk], mt_far[kChunk];
            if (active) g.load_operands(kChunk, mt_next, mt_far);
            float* tau_row = ht_g + other;
            for (uint32_t p0 = 0; p0 < P; p0 += kChunk) {
                float u[kChunk], j_down[kChunk], j_up[kChunk], ht[kChunk];
#pragma unroll
                for (int k = 0; k < kChunk; ++k) {
                    j_down[k] = j_down_next[k];
                    j_up[k] = j_up_next[k];
                    ht[k] = ht_next[k];
                    u[k] = 2.0f;
                }
                if (active) g.generate(kChunk, mt_next, mt_far, u);
                if (p0 + kChunk < P) {
                    request(p0 + kChunk);
                    if (active) g.load_operands(kChunk, mt_next, mt_far);
                }
#define ISING_WINDOW_STEP(K)                                                                                     \
    window_step<EXP, K>(r, s, W, P, p0, lane, lane_c, active, u[K], ht[K], j_up[K], j_down[K], neg_beta, gamma, \
                        tau_row, down_lane, source_lane, flips);
                ISING_WINDOW_STEP(0)
                ISING_WINDOW_STEP(1)
                ISING_WINDOW_STEP(2)
                ISING_WINDOW_STEP(3)
                ISING_WINDOW_STEP(4)
                ISING_WINDOW_STEP(5)
                ISING_WINDOW_STEP(6)
                ISING_WINDOW_STEP(7)
#undef ISING_WINDOW_STEP
            }
            // the last two columns leave the window
            s.hs[W * (P - 2) + lane_c] = r[6];
            s.hs[W * (P - 1) + lane_c] = r[7];
            __syncwarp();
#pragma unroll 8
            for (uint32_t k = lane; k < cells; k += 32) {
                hs_g[base + k] = s.hs[k];
                spins_g[base + k] = s.spins[k];
            }
            __threadfence();
            __syncwarp();
        }
    }
    if (lane == 0) d.mt_pos[chain] = g.pos;
    for (int off = 16; off > 0; off >>= 1) flips += __shfl_down_sync(0xffffffffu, flips, off);
    if (lane == 0) d.flips[chain] += flips;
}

template <int EXP>
cudaError_t prepare_exp(size_t smem_bytes) {
    cudaError_t e = cudaFuncSetAttribute(sweep_coalesced_kernel<EXP, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_bytes));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(sweep_coalesced_window_kernel<EXP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem_bytes));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(sweep_coalesced_kernel<EXP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(smem_bytes));
}

template <int EXP>
void launch_exp(const CoalescedDev& d, uint32_t sweeps, size_t smem_bytes, cudaStream_t stream) {
    if (d.band_pm != nullptr) sweep_coalesced_window_kernel<EXP><<<d.n_chains, 32, smem_bytes, stream>>>(d, sweeps);
    else if (d.layer_edges != nullptr) sweep_coalesced_kernel<EXP, true><<<d.n_chains, 32, smem_bytes, stream>>>(d, sweeps);
    else sweep_coalesced_kernel<EXP, false><<<d.n_chains, 32, smem_bytes, stream>>>(d, sweeps);
}

}  // namespace

size_t coalesced_smem_bytes(uint32_t lanes, uint32_t per_layer, uint32_t n_layer_edges) {
    if (lanes == 0 || lanes > 32 || per_layer == 0) return 0;
    const size_t bytes = region_bytes(lanes, per_layer, n_layer_edges);
    return bytes <= 227 * 1024 ? bytes : 0;
}

size_t coalesced_window_smem_bytes(uint32_t lanes, uint32_t per_layer, uint32_t n_far_edges) {
    if (lanes == 0 || lanes > 32 || per_layer == 0 || per_layer % 8 != 0) return 0;
    const size_t bytes = window_bytes(lanes, per_layer, n_far_edges);
    return bytes <= 227 * 1024 ? bytes : 0;
}

// The attribute is per function and context, shared by every live batch: it is always set to the
// largest size any batch can ask for (227 KB, the opt-in maximum), never to one batch's own need,
// so creating a small batch cannot take shared memory away from a large one.
cudaError_t prepare_coalesced_kernels(size_t smem_bytes) {
    if (smem_bytes > 227 * 1024) return cudaErrorInvalidValue;
    smem_bytes = 227 * 1024;
    cudaError_t e = prepare_exp<kExpExact>(smem_bytes);
    if (e == cudaSuccess) e = prepare_exp<kExpFast>(smem_bytes);
    if (e == cudaSuccess) e = prepare_exp<kExpAccurate>(smem_bytes);
    return e;
}

cudaError_t launch_sweep_coalesced(const CoalescedDev& d, uint32_t sweeps, size_t smem_bytes, cudaStream_t stream) {
    if (d.n_chains == 0) return cudaSuccess;
    switch (d.exp_kind) {
        case kExpExact: launch_exp<kExpExact>(d, sweeps, smem_bytes, stream); break;
        case kExpFast: launch_exp<kExpFast>(d, sweeps, smem_bytes, stream); break;
        default: launch_exp<kExpAccurate>(d, sweeps, smem_bytes, stream); break;
    }
    return cudaGetLastError();
}

}  // namespace isingb200
