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
//     neighbouring spins (HostModel::layered_uniform), read from the neighbouring strands' versioned
//     spin words (DevBatch::spin_nbr) under the ordering above;
//   * draw (sweep, l, p) of the chain's MT19937 stream is word (sweep*L + l)*P + p of a TAPE that a
//     PRODUCER warp per tile generates in stream order (lane = chain, three coalesced row accesses per
//     word: x[k] = f(x[k-624], x[k-623], x[k-227]), ref: proj/src/rng.cpp:22-25,89-96) into a ring in
//     global memory; the strands temper and convert their own words.
//
// A tile is not bound to an SM or to Tensor Memory: strands and producers are independent warps of a
// persistent grid, a few thousand of them in flight, that meet through global memory only.  A release
// store costs a device-wide fence (MEMBAR.ALL.GPU, ~3,500 cycles), so only the tape head (every 192
// rows) and a strand's end of layer (where the running energy is handed on) are published that way.
// Inside a layer a strand's progress counter is a fence-free hint, and what the next strand reads — the
// chunk's spins — carries the chunk's sweep count in the same 16-bit word: the reader checks the
// version instead of relying on an order between counter and data.  What a warp reads more than once
// is staged in shared memory: the layer graph (per CTA), the cells of the layer being swept, and the
// landing stages of the bulk copies that bring tape rows and field columns a chunk ahead.
//
// Per strand, fields move in chunks of 8 positions: the window of positions p-2..p+2 lives in
// registers (band neighbours are predicated register adds, as in kernels_layered.cu); eight columns
// enter it from HBM and eight leave it per chunk (full 128-byte lines), each exactly once per sweep.
// A FAR neighbour's update is not sent to the field in memory (a scattered read-modify-write of a
// 32-byte sector per flip: 6 B of HBM traffic per attempt on c5, a quarter of the total, and a
// reduction instruction per edge): the TARGET pulls it when its column enters the window, from the
// source chunk's CELL — 16 bits per chain and chunk, the chunk's spins and which of them flipped in the
// chunk's latest sweep — kept in shared memory for the layer being swept (8 bytes per position and
// strand; in global memory when that does not fit).  A column's far sources after it flipped in the
// sweep before, those before it in this sweep: pulled in that order they reproduce the reference's
// order of subtractions from h[t] exactly.  Between sweeps the fields in memory therefore lack the far
// updates of the latest sweep ("pending"); settle_fields_kernel applies them when anything else wants
// the fields (Batch::settle).  All field traffic of a layer comes from one thread per chain, so
// program order is the only ordering it needs.  HBM traffic per attempt: 4 B field in, 4 B out, 3/4 B
// cells and versioned spins, plus the tape (4 B written, 4 B read).
#include "device_batch.hpp"
#include "device_math.cuh"

// -DISING_STRAND_PROFILE: per-segment cycle counters of a few strands, printed at the end of the
// launch (profiles/r02_strand_segments.md was made with it); never in the product build.
#ifdef ISING_STRAND_PROFILE
#include <cstdio>
#define ISING_TICK(acc)             \
    do {                            \
        const long long now_ = clock64(); \
        acc += now_ - t0;           \
        t0 = now_;                  \
    } while (0)
#else
#define ISING_TICK(acc) \
    do {                \
    } while (0)
#endif

namespace isingb200 {

namespace {

// registers are granted 32 per thread at a time: 20 warps x 96.  (Measured with 32 warps x 64 registers:
// the strand spills, c5 1.36e11 at 4 strands per tile and 1.22e11 at 8.)
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
__device__ __forceinline__ uint32_t ld_cg_u16(const uint16_t* p) {
    uint32_t v;
    asm volatile("{\n.reg .b16 t;\nld.global.cg.u16 t, [%1];\ncvt.u32.u16 %0, t;\n}" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_u16(uint16_t* p, uint32_t v) {
    asm volatile("{\n.reg .b16 t;\ncvt.u16.u32 t, %1;\nst.global.u16 [%0], t;\n}" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    uint32_t v;
    asm volatile("{\n.reg .b16 t;\nld.shared.u16 t, [%1];\ncvt.u32.u16 %0, t;\n}" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u16(uint32_t addr, uint32_t v) {
    asm volatile("{\n.reg .b16 t;\ncvt.u16.u32 t, %1;\nst.shared.u16 [%0], t;\n}" ::"r"(addr), "r"(v) : "memory");
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
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Blocks until the counter at `p` has reached `need` (counters only grow; compared modulo 2^32).
// Every lane polls — one broadcast transaction.  The polls are relaxed loads; the value that ends the
// wait is read once more with acquire semantics (ptxas turns every ld.acquire.gpu into a load plus an
// invalidation of the SM's whole L1, CCTL.IVALL: one per wait, not one per poll), so every lane's
// later loads are ordered after a value >= need.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u16(const uint16_t* p) {
    uint32_t v;
    asm volatile("{\n.reg .b16 t;\nld.relaxed.gpu.global.u16 t, [%1];\ncvt.u32.u16 %0, t;\n}" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u16(uint16_t* p, uint32_t v) {
    asm volatile("{\n.reg .b16 t;\ncvt.u16.u32 t, %1;\nst.relaxed.gpu.global.u16 [%0], t;\n}" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// The same wait without the acquire: a HINT that what the counter announces is probably visible — for
// data that carries its own version (DevBatch::spin_nbr), checked by the reader.
__device__ __forceinline__ void wait_hint(const uint32_t* p, uint32_t need, uint32_t& cached) {
    if (int32_t(need - cached) > 0) {
        while (int32_t(need - ld_relaxed(p)) > 0) __nanosleep(128);
        cached = __reduce_min_sync(0xffffffffu, ld_relaxed(p));
    }
}
__device__ __forceinline__ void wait_counter(const uint32_t* p, uint32_t need, uint32_t& cached) {
    if (int32_t(need - cached) > 0) {
        while (int32_t(need - ld_relaxed(p)) > 0) __nanosleep(128);
        cached = __reduce_min_sync(0xffffffffu, ld_acquire(p));
    }
}
// The whole warp's earlier writes, then the counter (the release is cumulative over what lane 0
// observed through the warp barrier).
__device__ __forceinline__ void publish(uint32_t* p, uint32_t value, uint32_t lane) {
    __syncwarp();
    if (lane == 0) st_release(p, value);
}
// A strand's progress line: word 0 its finished chunks (what the strand of the next layer waits on),
// word 1 the draw index it will need next (what the producer may not overwrite yet; 0xffffffff: done).
// Inside a layer the same line is only a hint (no fence: MEMBAR.ALL.GPU costs ~3,500 cycles): the spins
// the next strand reads carry their own version.
__device__ __forceinline__ void hint_strand(uint32_t* line, uint32_t chunks, uint32_t next_draw, uint32_t lane) {
    if (lane == 0) {
        st_relaxed(line + 1, next_draw);
        st_relaxed(line, chunks);
    }
}
__device__ __forceinline__ void publish_strand(uint32_t* line, uint32_t chunks, uint32_t next_draw, uint32_t lane) {
    __syncwarp();
    if (lane == 0) {
        st_u32(line + 1, next_draw);
        st_release(line, chunks);
    }
}

// ---- bulk (TMA) copies into a warp's landing buffers, completion on an mbarrier ------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (done == 0u);
}
// global -> shared, `bytes` a multiple of 16, both addresses 16-byte aligned (SASS: UBLKCP.S.G)
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// ---- one attempt ----------------------------------------------------------------------------
// Everything an attempt needs that does not depend on the fields, per chunk of eight attempts.
struct ChunkBits {
    uint32_t cur8;    // bit k: the spin of attempt k is -1 (before the attempt)
    uint32_t up8;     // bit k: the spin above (next layer, not yet visited) is -1
    uint32_t agree8;  // bit k: the spins above and below are equal (set by finish(), from dn8)
    uint32_t dn8;     // bit k: the spin below (previous layer, already visited) is -1
    // (kept apart from the loads, so that requesting the bytes does not wait for them)
    __device__ __forceinline__ void finish() { agree8 = ~(up8 ^ dn8); }
};

// The part of a chunk's eight attempts that does not depend on the fields — eight independent
// strings of integer work, computed together ahead of the attempts so that they overlap each other
// instead of lengthening the loop-carried chain: the uniform draws (MT19937 tempering, u32_to_unit),
// -2*beta*s, and gamma * h_tau.
struct Prepared {
    float u[8];
    uint32_t ny[8];  // bits of -2*beta*s
    float hz[8];     // gamma * h_tau, h_tau = J*(s_up + s_dn) in {+2J, +0, -2J}
};
__device__ __forceinline__ void prepare_chunk(Prepared& pr, const uint32_t (&raw)[8], const ChunkBits& cb, uint32_t nb2,
                                              float u_offset, const uint4 tau_lo, const uint4 tau_hi) {
    const uint32_t tau_g[8] = {tau_lo.x, tau_lo.y, tau_lo.z, tau_lo.w, tau_hi.x, tau_hi.y, tau_hi.z, tau_hi.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        // u32_to_unit (x * 2^-32 is exact, so is adding +0); padding lanes get u + 2 and never accept
        pr.u[k] = __fmaf_rn(__uint2float_rz(mt_temper(raw[k])), 0x1p-32f, u_offset);
        const uint32_t sgn = (cb.cur8 << (31 - k)) & 0x80000000u;  // set <=> s = -1
        const uint32_t sgn_up = (cb.up8 << (31 - k)) & 0x80000000u;
        const uint32_t agree = uint32_t(int32_t(cb.agree8 << (31 - k)) >> 31);
        pr.ny[k] = nb2 ^ sgn;
        pr.hz[k] = __uint_as_float((tau_g[k] ^ sgn_up) & agree);
    }
}
// The layer graph's tables (DevStrandGraph), read either from the CTA's staged copy in shared
// memory (STAGED: explicit ld.shared on 32-bit addresses — generic loads that resolve to shared
// memory cost several times the latency) or from global memory through the read-only cache.
template <bool STAGED>
struct Tables;
template <>
struct Tables<false> {
    const uint4 *chunks, *pos, *band, *tau, *edges, *inslots;
    __device__ __forceinline__ uint4 chunk(uint32_t c) const { return __ldg(chunks + c); }
    __device__ __forceinline__ uint4 tau4(uint32_t i) const { return __ldg(tau + i); }
    __device__ __forceinline__ uint4 posrec(uint32_t p) const { return __ldg(pos + p); }
    __device__ __forceinline__ uint4 edge(uint32_t i) const { return __ldg(edges + i); }
    __device__ __forceinline__ uint4 inslot(uint32_t p) const { return __ldg(inslots + p); }
    __device__ __forceinline__ uint4 band_at(uint32_t p, uint32_t byte_off) const {
        return __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const unsigned char*>(band + 2 * size_t(p)) + byte_off));
    }
};
__device__ __forceinline__ uint4 lds_v4(uint32_t addr) {
    uint4 v;
    // not volatile: the tables are constant while the kernel runs
    asm("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
template <>
struct Tables<true> {
    uint32_t chunks, pos, band, tau, edges, inslots;  // shared-window addresses
    __device__ __forceinline__ uint4 chunk(uint32_t c) const { return lds_v4(chunks + c * 16); }
    __device__ __forceinline__ uint4 tau4(uint32_t i) const { return lds_v4(tau + i * 16); }
    __device__ __forceinline__ uint4 posrec(uint32_t p) const { return lds_v4(pos + p * 16); }
    __device__ __forceinline__ uint4 edge(uint32_t i) const { return lds_v4(edges + i * 16); }
    __device__ __forceinline__ uint4 inslot(uint32_t p) const { return lds_v4(inslots + p * 16); }
    __device__ __forceinline__ uint4 band_at(uint32_t p, uint32_t byte_off) const {
        return lds_v4(band + p * 32 + byte_off);
    }
};

// The cells of the layer a strand is sweeping, as this lane sees them: `at(off)` is the lane's cell of
// the chunk whose row starts `off` bytes into the layer (64 bytes per chunk).  STAGED: the warp's copy
// in shared memory, which the strand keeps current itself; otherwise global memory, past L1 (the
// lane's own earlier stores, in program order).
template <bool STAGED>
struct Cells;
template <>
struct Cells<false> {
    const unsigned char* layer;
    __device__ __forceinline__ uint32_t at(uint32_t off) const { return ld_cg_u16(reinterpret_cast<const uint16_t*>(layer + off)); }
    __device__ __forceinline__ void keep(uint32_t, uint32_t) const {}
};
template <>
struct Cells<true> {
    uint32_t layer;  // shared-window address
    __device__ __forceinline__ uint32_t at(uint32_t off) const { return lds_u16(layer + off); }
    __device__ __forceinline__ void keep(uint32_t off, uint32_t cell) const { sts_u16(layer + off, cell); }
};

// One far in-edge of a column (DevStrandGraph::inslots): `cell` is the source chunk's cell, `meta`'s
// low five bits the shift that brings the source's spin bit to bit 31 and its flip bit to bit 23.
// A flip of the source from s to -s subtracted (2s)*J from h: adds 2J with the sign of the NEW spin.
// Not flipped (or a null slot, meta == kNullSlot): adds -0.0, the identity for every bit pattern.
constexpr uint32_t kNullSlot = 31u;
__device__ __forceinline__ float pull_slot(float h, uint32_t j2, uint32_t meta, uint32_t cell) {
    const uint32_t x = __funnelshift_l(0u, cell, meta);  // (the shift wraps at 32)
    const uint32_t addend = (x & 0x00800000u) != 0u ? (j2 ^ (x & 0x80000000u)) : 0x80000000u;
    return __fadd_rn(h, __uint_as_float(addend));
}
// Every far in-edge of column `col`, in application order (the two slots, then the list).
template <bool STAGED>
__device__ __forceinline__ float pull_column(float h, uint32_t col, const Tables<STAGED>& t, const Cells<STAGED>& cells) {
    const uint4 in = t.inslot(col);
    h = pull_slot(h, in.x, in.y, cells.at(in.y >> 8));
    h = pull_slot(h, in.z, in.w, cells.at(in.w >> 8));
    const uint32_t more = t.posrec(col).z;
    for (uint32_t i = 0; i < (more >> 16); ++i) {
        const uint4 e = t.edge((more & 0xffffu) + i);
        h = pull_slot(h, e.x, e.y, cells.at(e.y >> 8));
    }
    return h;
}

// The band_pm entry of the flip of position p, attempt K of its chunk: the pair's first entry is for
// s = -1, the second (16 bytes on) for s = +1.
template <int K, bool STAGED>
__device__ __forceinline__ uint4 band_entry(const Tables<STAGED>& t, uint32_t p, uint32_t cur8) {
    const uint32_t off = ((K <= 4 ? cur8 << (4 - K) : cur8 >> (K - 4)) & 16u) ^ 16u;
    return t.band_at(p, off);
}

// Attempt K (compile-time index in the unrolled chunk; the register window r[] is indexed by
// position & 7) of position p = p0 + K: the loop-carried part.  `op` is the band_pm entry of the
// flip.  ref: sweep_kernels.hpp:14-16, sweep_basic.cpp:36-48.
template <int EXP, int K>
__device__ __forceinline__ void strand_attempt(float (&r)[8], const Prepared& pr, uint32_t nb2, const uint4 op,
                                               uint32_t& acc8, double& e_blk) {
    // x = -beta*((2s)*v) == (-2*beta*s)*v: doubling is exact, one rounding either way
    const float v = __fadd_rn(r[K], pr.hz[K]);
    const float x = __fmul_rn(__uint_as_float(pr.ny[K]), v);
    const bool accept = pr.u[K] < exp_kind<EXP>(x);
    // band neighbours p-2, p-1, p+1, p+2: h -= (2s)*J == h + (-(2s)*J); an empty slot holds -0.0
    if (accept) {
        r[(K + 6) & 7] = __fadd_rn(r[(K + 6) & 7], __uint_as_float(op.x));
        r[(K + 7) & 7] = __fadd_rn(r[(K + 7) & 7], __uint_as_float(op.y));
        r[(K + 1) & 7] = __fadd_rn(r[(K + 1) & 7], __uint_as_float(op.z));
        r[(K + 2) & 7] = __fadd_rn(r[(K + 2) & 7], __uint_as_float(op.w));
        // running energy of the tempering swap: (2s)*(h + gamma*h_tau), the inner factor of x — 2v with
        // its sign flipped where s = -1 (ny ^ nb2 is that sign bit)
        e_blk = __dadd_rn(e_blk, double(__uint_as_float(__float_as_uint(__fmul_rn(v, 2.0f)) ^ pr.ny[K] ^ nb2)));
        acc8 |= 1u << K;
    }
}

// What a flip of attempt e.y adds to the field at e.x: -(2s)*J, i.e. 2J (e.z) with the sign of -s.
__device__ __forceinline__ float edge_addend(const uint4 e, uint32_t cur8) {
    return __uint_as_float(e.z ^ ((((cur8 >> e.y) & 1u) ^ 1u) << 31));
}

// A CAREFUL chunk: some attempt has a far neighbour among the columns that have already been
// requested (p+3 .. p0+10), or a column entering has more far in-edges than the two slots.  The
// entering columns go through a per-warp shared-memory scratch ([8][32] floats, a lane only touches
// its own entries; the caller has stored them there with everything pulled), where the near updates
// are applied before the column enters the register window.  Out of line and by value:
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

template <int EXP, int K, bool STAGED>
__device__ __forceinline__ void careful_attempt(float (&r)[8], float* scratch, const Prepared& pr, uint32_t nb2,
                                                uint32_t cur8, const Tables<STAGED>& t, uint32_t& acc8, double& e_blk,
                                                uint32_t p0) {
    const uint32_t before = acc8;
    strand_attempt<EXP, K>(r, pr, nb2, band_entry<K>(t, p0 + K, cur8), acc8, e_blk);
    const uint32_t near = t.posrec(p0 + K).y;
    if ((near >> 16) != 0u && acc8 != before) {
        for (uint32_t i = 0; i < (near >> 16); ++i) {
            const uint4 e = t.edge((near & 0xffffu) + i);
            float* cell = scratch + (e.x - (p0 + 3)) * 32;
            *cell = __fadd_rn(*cell, edge_addend(e, cur8));
        }
    }
}

template <int EXP, bool STAGED>
__device__ __noinline__ CarefulResult careful_chunk(Window w, RawWords raw, ChunkBits cb, uint32_t nb2, float u_offset,
                                                    const Tables<STAGED> t, uint32_t p0, float* hs_l, float* scratch,
                                                    double e_blk) {
    float (&r)[8] = w.r;
    uint32_t acc8 = 0;
    Prepared pr;
    prepare_chunk(pr, raw.v, cb, nb2, u_offset, t.tau4(p0 / 4), t.tau4(p0 / 4 + 1));
#define ISING_CAREFUL(K)                                                                  \
    careful_attempt<EXP, K>(r, scratch, pr, nb2, cb.cur8, t, acc8, e_blk, p0);             \
    if (p0 != 0 || K >= 2) st_f32(hs_l + (size_t(p0) + K - 2) * 32, r[(K + 6) & 7]);       \
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
// Per-strand shared memory: two landing stages for what the bulk copies bring (8 tape rows = 1 KB and
// the 8 field columns entering the window = 1 KB; the latter doubles as the scratch of a careful
// chunk), three mbarriers and — STAGED — the cells of the layer being swept (64 bytes per chunk).
constexpr uint32_t kStageBytes = 2048;
constexpr uint32_t kWarpSmem = 2 * kStageBytes + 32;

// Everything a chunk reads from global memory is requested one chunk ahead or more: the tape rows and
// the eight field columns entering the window by bulk (TMA) copies of one elected lane into the warp's
// landing stage (no registers held meanwhile; nobody but this strand writes those columns, and it last
// did a sweep ago), the versioned spins of the two neighbouring layers by strong loads into a register
// each (once the layer below's hint says it has finished that chunk; verified when used); the layer's
// cells arrive by one bulk copy per layer.  So the loop-carried chain of the attempts is all a strand waits
// for.
template <int EXP, bool WAIT, bool STAGED>
__device__ void strand_run(const DevBatch& b, const Tables<STAGED>& t, uint32_t P, uint32_t L, uint32_t tile, uint32_t j,
                           uint32_t sweeps, uint32_t lane, unsigned char* warp_smem) {
    const uint32_t C = P / 8, S = b.strands, n = b.n_spins;
    const uint32_t blocks_per_sweep = L / S;
    const uint32_t total_blocks = blocks_per_sweep * sweeps;
    const uint32_t chain = b.tile_first[tile] + lane;
    const bool active = lane < b.tile_count[tile];
    const uint32_t nb2 = __float_as_uint(active ? -2.0f * b.betas[b.slot_of_chain[chain]] : 0.0f);
    const float u_offset = active ? 0.0f : 2.0f;
    float* hs_tile = b.hs + size_t(tile) * n * 32 + lane;
    uint16_t* cells_tile = b.spin_cells + size_t(tile) * (n / 8) * 32 + lane;
    uint16_t* nbr_tile = b.spin_nbr + size_t(tile) * (n / 8) * 32 + lane;
    const uint32_t R = b.tape_rows;
    const uint32_t* tape = b.tape + size_t(tile) * R * 32;  // (no lane offset: rows are copied whole)
    uint32_t* flags = b.strand_flags + size_t(tile) * (S + 1) * kFlagStride;
    uint32_t* my_flag = flags + j * kFlagStride;
    const uint32_t* pred_flag = flags + ((j + S - 1) % S) * kFlagStride;
    const uint32_t* head_flag = flags + S * kFlagStride;
    const uint32_t pub = b.strand_pub;
    uint32_t pred_cached = 0, head_cached = 0;  // last values read WITH acquire
    uint32_t pred_hint = 0;                     // last value of the layer below's counter read without (wait_hint)
    uint32_t flips = 0;
    uint32_t seq = 0;  // chunks finished
    uint32_t until_pub = pub;
    // landing stages: stage s at wsm + s * kStageBytes (tape rows, then columns); then the barriers, the cells
    const uint32_t wsm = smem_u32(warp_smem);
    const uint32_t bar0 = wsm + 2 * kStageBytes, bar_cells = bar0 + 16;
    const uint32_t cells_smem = wsm + kWarpSmem;
    uint32_t stage = 0, phases = 0;  // current stage; bit s of phases = parity the next wait on stage s sees (bit 2: the cells)
    if (lane == 0) {
        mbar_init(bar0, 1);
        mbar_init(bar0 + 8, 1);
        mbar_init(bar_cells, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // wait statistics (ref: FlipStats::group_wait): lane k folds the ballot of attempt k of every chunk
    const bool record_wait = WAIT && b.wait_counts != nullptr && b.tile_count[tile] == 32;
    uint32_t wait[6] = {0, 0, 0, 0, 0, 0};

    // one elected lane requests a chunk's tape rows and entering columns (`columns` points at lane 0's
    // entry of the first one) into stage `st`
    const auto request = [&](uint32_t st, uint32_t slot, const float* columns, uint32_t column_bytes) {
        if (lane == 0) {
            const uint32_t dst = wsm + st * kStageBytes, bar = bar0 + st * 8;
            // the rows were written through the generic proxy (by the producer, acquired above; the
            // columns by this warp before the block began, fenced there): order the async-proxy reads
            // after what this lane has observed (measured: the fence is not what a request costs — issuing
            // the two copies is, about 300 cycles)
            asm volatile("fence.proxy.async.global;" ::: "memory");
            mbar_expect(bar, 1024 + column_bytes);
            bulk_load(dst, tape + size_t(slot) * 32, 1024, bar);
            bulk_load(dst + 1024, columns, column_bytes, bar);
        }
    };

#ifdef ISING_STRAND_PROFILE
    long long tA = 0, tB = 0, tC = 0, tD = 0, tE = 0, tF = 0, t0 = 0, tPred = 0, tHead = 0, tReq = 0, tStart = 0;
#define ISING_TIMED(acc, stmt)                  \
    {                                           \
        const long long before_ = clock64();    \
        stmt;                                   \
        acc += clock64() - before_;             \
    }
#else
#define ISING_TIMED(acc, stmt) stmt;
#endif
    for (uint32_t blk = 0; blk < total_blocks; ++blk) {
        const uint32_t sw = blk / blocks_per_sweep, m = blk - sw * blocks_per_sweep;
        const uint32_t l = j + S * m;
        const uint32_t l_up = l + 1 == L ? 0u : l + 1, l_dn = l == 0 ? L - 1 : l - 1;
        float* hs_l = hs_tile + size_t(l) * P * 32;
        // The strand of the layer below: its chunk c of the matching block must be finished before
        // this strand reads that layer's new spins.  For j > 0 the matching block has this block's
        // index, for j == 0 it is the block before (layer L-1 of the previous sweep when m == 0).
        const bool has_pred = S > 1 && !(j == 0 && blk == 0);
        uint32_t pred_need = (j == 0 ? blk - 1 : blk) * C + 1;  // the predecessor's count once it has finished chunk c
        // this block's draws: tape rows 624 + (sw*L + l)*P + p
        const uint32_t row0 = kMtN + (sw * L + l) * P;
        uint32_t head_need = row0 + 8;  // the head once chunk c's rows exist
        uint32_t slot = row0 % R;       // (R and row0 are multiples of 8: a chunk's rows never wrap)
        double e_blk = 0.0;

        // running pointers: the chunk being swept (…_c) is at p0 = 8c; the neighbours' spins are the
        // high bytes of their cells
        float* hs_c = hs_l;
        uint16_t* cur_c = cells_tile + size_t(l) * C * 32;
        uint16_t* out_c = nbr_tile + size_t(l) * C * 32;
        const uint16_t* up_c = nbr_tile + size_t(l_up) * C * 32;
        const uint16_t* dn_c = nbr_tile + size_t(l_dn) * C * 32;
        // Versions (DevBatch::spin_nbr): this sweep leaves `version` behind.  The layer below was swept in
        // this sweep — except below layer 0, which is the last layer of the sweep before; the layer above
        // will be swept later in this sweep — except above the last layer, which is layer 0, swept already.
        const uint32_t version = (b.strand_epoch + sw + 1u) & 0xffu, before = (b.strand_epoch + sw) & 0xffu;
        const uint32_t dn_version = l == 0u ? before : version, up_version = l_up == 0u ? version : before;
        Cells<STAGED> cells;
        // What the bulk copies of this block read — the layer's columns and cells as this warp left
        // them a sweep ago (or as the launch found them) — was stored through the generic proxy by every
        // lane, and every lane has read the shared-memory copies they replace: both come before them.
        asm volatile("fence.proxy.async.global;\n\tfence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if constexpr (STAGED) {
            if (lane == 0) {
                mbar_expect(bar_cells, C * 64);
                bulk_load(cells_smem, cur_c - lane, C * 64, bar_cells);
            }
            cells.layer = cells_smem + lane * 2;
        } else {
            cells.layer = reinterpret_cast<const unsigned char*>(cur_c);
        }

        // ---- the first chunk's operands (the only exposed round trips of the block)
        ISING_TIMED(tStart, wait_counter(head_flag, head_need, head_cached))
        __syncwarp();  // every lane has left the stage's previous contents
        request(stage, slot, hs_c - lane + 3 * 32, 1024);  // (a layer has two chunks at least)
        // The neighbour spins of a chunk are requested a chunk ahead when the layer below's counter says it
        // has probably finished it; whether they are this sweep's is read off their versions when they
        // are used (the counter is a hint: no fence orders it after the spins).  The spins above need no
        // wait — their strand is behind this one — except above the last layer: layer 0 was swept earlier
        // in this sweep, by the strand S - 1 hops ahead in the ring of waits.
        uint32_t up_next = 0, dn_next = 0;
        bool dn_ready = false;
        const auto versions_ok = [&]() {
            return __all_sync(0xffffffffu, (dn_next >> 8) == dn_version && (up_next >> 8) == up_version);
        };
        // register window: positions 0..2 (entries for -2, -1 stay unused: their band slots are empty)
        Window w;
        float (&r)[8] = w.r;
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = 0.0f;
        r[0] = ld_cg_f32(hs_c);
        r[1] = ld_cg_f32(hs_c + 32);
        r[2] = ld_cg_f32(hs_c + 64);
        if constexpr (STAGED) {
            mbar_wait(bar_cells, (phases >> 2) & 1u);
            phases ^= 4u;
        }
        r[0] = pull_column(r[0], 0u, t, cells);
        r[1] = pull_column(r[1], 1u, t, cells);
        r[2] = pull_column(r[2], 2u, t, cells);

        for (uint32_t c = 0; c < C; ++c) {
#ifdef ISING_STRAND_PROFILE
            t0 = clock64();
#endif
            const uint32_t p0 = c * 8;
            const uint4 chunk_info = t.chunk(c);
            const bool more = c + 1 < C;
            // ---- the chunk's spins: the layer below must have finished it (normally known from an earlier
            // wait, and the byte requested a chunk ago)
            if (!dn_ready || !versions_ok()) {
                if (has_pred) ISING_TIMED(tPred, wait_hint(pred_flag, pred_need, pred_hint))
                for (uint32_t polls = 0;; ++polls) {
                    dn_next = ld_relaxed_u16(dn_c);
                    up_next = ld_relaxed_u16(up_c);
                    if (versions_ok()) break;
                    // (the layer below finishes the chunk within microseconds of its counter saying so: ten
                    // seconds of polling mean the versions are inconsistent — fail loudly instead of hanging)
                    if (polls > (1u << 26)) __trap();
                    __nanosleep(128);
                }
            }
            ChunkBits cb;
            cb.cur8 = (STAGED ? cells.at(c * 64) : ld_cg_u16(cur_c)) >> 8;
            cb.up8 = up_next & 0xffu;
            cb.dn8 = dn_next & 0xffu;
            dn_ready = false;
            // ---- the next chunk's tape rows and entering columns (p0+11 .. p0+18; the last chunk has five),
            // by bulk copy; its neighbour spins
            if (more) {
                slot = slot + 8 == R ? 0u : slot + 8;
                head_need += 8;
                ++pred_need;
                if (!has_pred || int32_t(pred_hint - pred_need) >= 0) {
                    dn_next = ld_relaxed_u16(dn_c + 32);
                    up_next = ld_relaxed_u16(up_c + 32);
                    dn_ready = true;
                }
                ISING_TIMED(tHead, wait_counter(head_flag, head_need, head_cached))
                __syncwarp();  // every lane has left the other stage's previous contents
                ISING_TIMED(tReq, request(stage ^ 1u, slot, hs_c - lane + 11 * 32, c + 2 < C ? 1024u : 640u); __syncwarp())
            }
            // ---- this chunk's tape words have landed
            ISING_TICK(tA);
            mbar_wait(bar0 + stage * 8, (phases >> stage) & 1u);
            ISING_TICK(tB);
            phases ^= 1u << stage;
            // (plain loads: the compiler may put each one next to its use; the wait above keeps them behind it)
            const uint32_t* landed = reinterpret_cast<const uint32_t*>(warp_smem + stage * kStageBytes) + lane;
            float* nx = reinterpret_cast<float*>(warp_smem + stage * kStageBytes + 1024) + lane;  // column p0+3+k at nx[k * 32]
            RawWords raw_words;
            uint32_t (&raw)[8] = raw_words.v;
#pragma unroll
            for (int k = 0; k < 8; ++k) raw[k] = landed[k * 32];
            cb.finish();

            // ---- eight attempts
            uint32_t acc8 = 0;
            if (__builtin_expect((chunk_info.z & 1u) == 0u, 1)) {
                Prepared pr;
                prepare_chunk(pr, raw, cb, nb2, u_offset, t.tau4(2 * c), t.tau4(2 * c + 1));
                // the band entry of an attempt is requested during the attempt before it; the far in-edges
                // of the column that enters after the attempt, and their cells, before it (their sources
                // lie in earlier chunks or later positions: nothing this chunk decides)
                uint4 op = band_entry<0>(t, p0, cb.cur8);
#define ISING_STRAND_ATTEMPT(K, NEXT)                                                \
    {                                                                                \
        const uint4 op_next = band_entry<NEXT>(t, p0 + NEXT, cb.cur8);               \
        const uint4 in = t.inslot(p0 + 3 + K);                                       \
        const uint32_t cell_a = cells.at(in.y >> 8);                                 \
        float entering = pull_slot(nx[K * 32], in.x, in.y, cell_a);                  \
        /* (warp-uniform: most columns of a sparse layer have one far in-edge or none) */ \
        if (in.w != kNullSlot) entering = pull_slot(entering, in.z, in.w, cells.at(in.w >> 8)); \
        strand_attempt<EXP, K>(r, pr, nb2, op, acc8, e_blk);                         \
        if (c != 0 || K >= 2) st_f32(hs_c + (K - 2) * 32, r[(K + 6) & 7]);      \
        r[(K + 3) & 7] = entering;                                                   \
        op = op_next;                                                                \
    }
                ISING_STRAND_ATTEMPT(0, 1)
                ISING_STRAND_ATTEMPT(1, 2)
                ISING_STRAND_ATTEMPT(2, 3)
                ISING_STRAND_ATTEMPT(3, 4)
                ISING_STRAND_ATTEMPT(4, 5)
                ISING_STRAND_ATTEMPT(5, 6)
                ISING_STRAND_ATTEMPT(6, 7)
                ISING_STRAND_ATTEMPT(7, 7)
#undef ISING_STRAND_ATTEMPT
            } else {
                // the landed columns are the scratch: everything pulled first, in place
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (k < 5 || more) nx[k * 32] = pull_column(nx[k * 32], p0 + 3 + k, t, cells);
                }
                const CarefulResult res = careful_chunk<EXP>(w, raw_words, cb, nb2, u_offset, t, p0, hs_l, nx, e_blk);
                w = res.w;
                acc8 = res.acc8;
                e_blk = res.e_blk;
                // (this stage's next bulk copy comes after these generic writes)
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }

            // ---- after the chunk: the cell (new spins, what flipped), progress
            ISING_TICK(tC);
            const uint32_t cell = acc8 | (cb.cur8 ^ acc8) << 8;
            st_u16(cur_c, cell);
            cells.keep(c * 64, cell);
            st_relaxed_u16(out_c, (cb.cur8 ^ acc8) | version << 8);
            flips += __popc(acc8);
            if (WAIT && record_wait) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t ballot = __ballot_sync(0xffffffffu, (acc8 >> k) & 1u);
                    if (lane == uint32_t(k)) wait_fold(ballot, wait);
                }
            }
            ++seq;
            ISING_TICK(tD);
            if (more) {
                stage ^= 1u;
                hs_c += 8 * 32;
                cur_c += 32;
                out_c += 32;
                up_c += 32;
                dn_c += 32;
                if (--until_pub == 0u) {
                    hint_strand(my_flag, seq, row0 - kMtN + (c + 1) * 8, lane);
                    until_pub = pub;
                }
            }
            ISING_TICK(tE);
        }
#ifdef ISING_STRAND_PROFILE
        t0 = clock64();
#endif
        stage ^= 1u;
        // ---- end of the layer: the last two columns leave the window; the block's partial sum joins
        // the running energy after the partial sums of all earlier blocks (tempering definition,
        // oracle/ising_oracle.h), which the strand of the layer below has published with its block
        st_f32(hs_c + 6 * 32, r[6]);
        st_f32(hs_c + 7 * 32, r[7]);
        if (has_pred) wait_counter(pred_flag, pred_need, pred_cached);
        if (active) {
            double* e_run = b.e_run + chain;
            const double e = ld_cg_f64(e_run);
            asm volatile("st.global.f64 [%0], %1;" ::"l"(e_run), "d"(__dadd_rn(e, e_blk)) : "memory");
        }
        // (the draw this strand needs next is the first of its next layer, S layers on — or of layer j of
        // the next sweep: the rows in between belong to the other strands)
        const uint32_t nb = blk + 1, nsw = nb / blocks_per_sweep;
        publish_strand(my_flag, seq, nb == total_blocks ? 0xffffffffu : (nsw * L + j + S * (nb - nsw * blocks_per_sweep)) * P, lane);
        ISING_TICK(tF);
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
#ifdef ISING_STRAND_PROFILE
    if (lane == 0 && (tile % 97) == 0) printf("tile %u strand %u chunks %u: per chunk request %lld wait %lld attempts %lld cell %lld rotate %lld (in request: pred wait %lld head wait %lld bulk requests %lld); block end %lld, head wait at the start %lld per block\n", tile, j, seq, tA / seq, tB / seq, tC / seq, tD / seq, tE / seq, tPred / seq, tHead / seq, tReq / seq, tF / total_blocks, tStart / total_blocks);
#endif
}

// ---- the producer -------------------------------------------------------------------------------
// MT19937 as a tape: row a of the ring holds word x[a] of all 32 chains, x[0..623] being the state
// at launch in draw order, and draw q of the launch is temper(x[624 + q]).  Rows are generated in
// order, 32 at a time, never overwriting a row a strand has yet to read or the 624 rows behind the
// head; the head is published after every batch.  At the end the last 624 rows go back to the
// in-place state array the other kernel families use.
// `landing`: 2 stages of 8 KB (32 rows x[a-623..] and 32 rows x[a-227..]) plus two mbarriers, in shared
// memory, or nullptr: then the operands of a group are loaded into registers, one round trip per
// 32 rows (about a third of the rate).
constexpr uint32_t kProducerStage = 8192;
// Rows between two publications of the head (each costs a device-scope fence, ~3,500 cycles, a third of
// the producer's time at 64 rows — and on small batches the producer sets the pace of its tile: c4 +5 % from
// 128 to 192); at most 192, see below.
#ifndef ISING_X_PRODUCER_BATCH
#define ISING_X_PRODUCER_BATCH 192
#endif
constexpr uint32_t kProducerBatch = ISING_X_PRODUCER_BATCH;
// How far the head may run ahead of the most advanced strand's published need, in rows: 256 + 64 S.
// A strand publishes its need every strand_pub (<= 16) chunks and needs 8 rows at a time — anything
// above 136 rows cannot deadlock — and a strand starting a layer is S - 1 strand lags ahead of the most
// advanced one (measured: c5, S = 4, 512 rows 2.35e11 against 2.32e11 unbounded, DRAM reads -18 %;
// c4, S = 16, 512 rows 4.0e10, 1280 rows as unbounded).
constexpr uint32_t kProducerLeadBase = 256, kProducerLeadPerStrand = 64;
static_assert(kProducerBatch % 32 == 0 && kProducerBatch <= 192, "operands of a group must lie before its batch");
constexpr uint32_t kProducerSmem = 2 * kProducerStage + 16;
__device__ void producer_run(const DevBatch& b, uint32_t tile, uint32_t sweeps, uint32_t lane, unsigned char* landing) {
    const uint32_t S = b.strands, R = b.tape_rows;
    uint32_t* tape = b.tape + size_t(tile) * R * 32 + lane;
    uint32_t* state = b.mt + size_t(tile) * kMtN * 32 + lane;
    uint32_t* flags = b.strand_flags + size_t(tile) * (S + 1) * kFlagStride;
    uint32_t* head_flag = flags + S * kFlagStride;
    const uint32_t pos = b.mt_pos[tile];
    const uint32_t total = sweeps * b.n_spins;  // draws of this launch (a multiple of 8)

    for (uint32_t i = 0; i < kMtN; ++i) {
        uint32_t w = pos + i;
        w = w >= kMtN ? w - kMtN : w;
        st_u32(tape + size_t(i) * 32, state[size_t(w) * 32]);
    }
    // Bulk copies read the ring through the async proxy: every row they fetch must be globally
    // performed first.  The rows above are made so here; later ones by the fence of a publication —
    // a group's nearest operand is 227 rows behind the row being written, the last group of a batch starts
    // kProducerBatch - 32 rows into it: the operands of every group lie before the batch, i.e. published.
    const uint32_t lsm = landing != nullptr ? smem_u32(landing) : 0u;
    const uint32_t lbar = lsm + 2 * kProducerStage;
    uint32_t lstage = 0, lphases = 0;
    bool in_flight = false;  // the operands of the group at (sa, sf) have been requested into stage lstage
    if (landing != nullptr) {
        __threadfence();
        if (lane == 0) {
            mbar_init(lbar, 1);
            mbar_init(lbar + 8, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    const uint32_t* tape_rows = b.tape + size_t(tile) * R * 32;  // (no lane offset: rows are copied whole)
    const auto request_group = [&](uint32_t st, uint32_t slot_a, uint32_t slot_f) {
        __syncwarp();  // every lane has left the stage's previous contents
        if (lane == 0) {
            const uint32_t dst = lsm + st * kProducerStage, bar = lbar + st * 8;
            asm volatile("fence.proxy.async.global;" ::: "memory");
            mbar_expect(bar, kProducerStage);
            bulk_load(dst, tape_rows + size_t(slot_a + 1) * 32, 4096, bar);
            bulk_load(dst + 4096, tape_rows + size_t(slot_f) * 32, 4096, bar);
        }
    };

    const uint32_t end = kMtN + total;
    uint32_t a = kMtN;      // next row to generate
    uint32_t tail = 0;      // draws known to be consumed by every strand
    uint32_t front = 0;     // the largest draw index a strand has said it needs next
    const uint32_t lead = kProducerLeadBase + kProducerLeadPerStrand * S;
    uint32_t so = kMtN % R, sa = 0, sf = kMtM % R;  // slots of rows a, a-624, a-227 (624 - 227 = 397)
    uint32_t cur = ld_cg_u32(tape);                 // x[a-624]
    // A producer feeds S strands and is one in-order warp: what bounds it is the round trip of its
    // operand loads.  So rows are generated 32 at a time with all 64 operand loads in flight together
    // (x[a-623+k] and x[a-227+k], k < 32: every one of them lies behind row a).
    while (a < end) {
        const uint32_t batch = min(kProducerBatch, end - a);  // (a multiple of 8)
        // Rows a .. a+batch-1 overwrite rows a-R .. : they must be consumed draws (row < 624 + tail).  And
        // they should not be far ahead of the most advanced strand (draw `front`): rows nobody needs yet
        // only push the rows the strands are about to read out of L2 (`lead` rows per tile in flight
        // instead of up to R).  Both bounds are monotonic, so stale values only delay.
        while (int32_t(a + batch - R - kMtN - tail) > 0 || int32_t(a - kMtN - front - lead) > 0) {
            // (relaxed: a strand's draw index is published after its last read of the rows before it, and
            // the rows written next are published with a release of their own)
            const uint32_t d = lane < S ? ld_relaxed(flags + lane * kFlagStride + 1) : 0xffffffffu;
            uint32_t lo = __reduce_min_sync(0xffffffffu, d);
            uint32_t hi = __reduce_max_sync(0xffffffffu, d == 0xffffffffu ? 0u : d);
            if (lo == 0xffffffffu) lo = hi = total;  // every strand has finished
            if (lo == tail && hi == front) __nanosleep(1000);
            tail = lo;
            front = hi;
        }
        for (uint32_t done = 0; done < batch;) {
            const uint32_t rows = min(32u, batch - done);
            const bool whole = rows == 32u && sa + 32 < R && sf + 32 <= R && so + 32 <= R;  // no run crosses the end of the ring
            if (whole && landing != nullptr) {
                if (!in_flight) request_group(lstage, sa, sf);
                // the group after this one, while this one is generated (its operands lie behind row a too)
                const uint32_t sa2 = sa + 32, sf2 = sf + 32 == R ? 0u : sf + 32, so2 = so + 32 == R ? 0u : so + 32;
                const bool next_whole = a + done + 64 <= end && sa2 + 32 < R && sf2 + 32 <= R && so2 + 32 <= R;
                if (next_whole) request_group(lstage ^ 1u, sa2, sf2);
                mbar_wait(lbar + lstage * 8, (lphases >> lstage) & 1u);
                lphases ^= 1u << lstage;
                const uint32_t* in = reinterpret_cast<const uint32_t*>(landing + lstage * kProducerStage) + lane;
                uint32_t* po = tape + size_t(so) * 32;
#pragma unroll 8
                for (int k = 0; k < 32; ++k) {
                    const uint32_t nx = in[k * 32];
                    st_u32(po + k * 32, mt_recurrence(cur, nx, in[1024 + k * 32]));
                    cur = nx;
                }
                sa = sa2;
                sf = sf2;
                so = so2;
                done += 32;
                lstage ^= 1u;
                in_flight = next_whole;
            } else if (whole) {
                const uint32_t* pa = tape + size_t(sa) * 32;
                const uint32_t* pf = tape + size_t(sf) * 32;
                uint32_t* po = tape + size_t(so) * 32;
                uint32_t nxt[32], far[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    nxt[k] = ld_cg_u32(pa + (k + 1) * 32);
                    far[k] = ld_cg_u32(pf + k * 32);
                }
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    st_u32(po + k * 32, mt_recurrence(cur, nxt[k], far[k]));
                    cur = nxt[k];
                }
                sa += 32;
                sf = sf + 32 == R ? 0u : sf + 32;
                so = so + 32 == R ? 0u : so + 32;
                done += 32;
            } else {  // near the end of the ring, or a short tail: 8 rows at a time, every slot wrapped
                if (in_flight) {  // operands requested for a whole group that is not to be: let them land, unused
                    mbar_wait(lbar + lstage * 8, (lphases >> lstage) & 1u);
                    lphases ^= 1u << lstage;
                    in_flight = false;
                }
                uint32_t nxt[8], far[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    uint32_t s1 = sa + k + 1;
                    s1 = s1 >= R ? s1 - R : s1;
                    uint32_t s2 = sf + k;
                    s2 = s2 >= R ? s2 - R : s2;
                    nxt[k] = ld_cg_u32(tape + size_t(s1) * 32);
                    far[k] = ld_cg_u32(tape + size_t(s2) * 32);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    st_u32(tape + size_t(so + k) * 32, mt_recurrence(cur, nxt[k], far[k]));  // (so is a multiple of 8)
                    cur = nxt[k];
                }
                sa = sa + 8 >= R ? sa + 8 - R : sa + 8;
                sf = sf + 8 >= R ? sf + 8 - R : sf + 8;
                so = so + 8 >= R ? so + 8 - R : so + 8;
                done += 8;
                in_flight = false;
            }
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

// Which logical warp (work item dealer below) each hardware warp of a CTA is.  The four schedulers of
// an SM take the hardware warps round-robin (warp % 4), a tile advances at the pace of its slowest
// warp, and a producer costs about half a strand's issue slots: so the strands take the low
// hardware warps and each producer the next free warp of the least loaded scheduler, leaving gaps
// (c5: 14 strands + 4 producers per CTA as 4 | 4 | 3 + 2 | 3 + 2 instead of 4 + 1 | 4 + 1 | 3 + 1 | 3 + 1).
constexpr uint32_t kIdleWarp = 0xffu;
struct StrandWarpMap {
    uint8_t logical[32];
};

// Persistent grid of independent warps.  Work items of a round: for each of `tiles_per_round` tiles
// its S strands and its producer; every item of a round is resident at once (the launcher sizes the
// rounds), so the waits above always end.  Items are dealt warp-major, so a CTA's low warps are
// strands and its high warps producers.  Dynamic shared memory: `strand_regions` regions of kWarpSmem
// bytes (landing stages, scratch) plus — STAGED, single-model batches — the cells of the strand's
// layer; then a copy of the layer graph, which every strand of the CTA reads; then `producer_slots`
// landing buffers for the producers.
template <int EXP, bool WAIT, bool STAGED>
__global__ void __launch_bounds__(kStrandMaxWarps * 32, 1) sweep_strand_kernel(DevBatch b, uint32_t sweeps,
                                                                                 uint32_t tiles_per_round,
                                                                                 uint32_t strand_regions,
                                                                                 uint32_t producer_slots, uint32_t tile_local,
                                                                                 StrandWarpMap map) {
    extern __shared__ __align__(128) unsigned char strand_smem[];
    // `warp` is the LOGICAL warp index (see StrandWarpMap); kIdleWarp: a padding warp
    const uint32_t warp = map.logical[threadIdx.x >> 5], lane = threadIdx.x & 31u;
    const uint32_t region_bytes = kWarpSmem + (STAGED ? b.max_per_layer * 8u : 0u);
    unsigned char* warp_smem = strand_smem + size_t(warp) * region_bytes;  // (strands only: warp < strand_regions)
    unsigned char* graph_smem = strand_smem + size_t(strand_regions) * region_bytes;
    unsigned char* producer_smem = graph_smem + ((STAGED ? b.strand_graph_smem : 0u) + 15u) / 16u * 16u;
    Tables<STAGED> staged{};
    // STAGED with several models: the launcher has dealt the items so that every warp of this CTA works
    // on tile blockIdx.x % tiles_per_round (tile_local; one round)
    const uint32_t staged_model = STAGED && tile_local != 0u ? b.tile_model[blockIdx.x % tiles_per_round] : 0u;
    if constexpr (STAGED) {
        const DevStrandGraph g0 = b.strand_graphs[staged_model];
        const uint32_t P = g0.per_layer;
        uint4* pos = reinterpret_cast<uint4*>(graph_smem);
        uint4* band = pos + P;
        uint4* chunks = band + 2 * size_t(P);
        uint4* tau = chunks + P / 8;
        uint4* inslots = tau + P / 4;
        uint4* edges = inslots + P + 8;
        for (uint32_t k = threadIdx.x; k < P; k += blockDim.x) pos[k] = g0.pos[k];
        for (uint32_t k = threadIdx.x; k < 2 * P; k += blockDim.x) band[k] = g0.band_pm[k];
        for (uint32_t k = threadIdx.x; k < P / 8; k += blockDim.x) chunks[k] = g0.chunks[k];
        for (uint32_t k = threadIdx.x; k < P / 4; k += blockDim.x) tau[k] = g0.tau[k];
        for (uint32_t k = threadIdx.x; k < P + 8; k += blockDim.x) inslots[k] = g0.inslots[k];
        for (uint32_t k = threadIdx.x; k < g0.n_edges; k += blockDim.x) edges[k] = g0.edges[k];
        staged.pos = smem_u32(pos);
        staged.band = smem_u32(band);
        staged.chunks = smem_u32(chunks);
        staged.tau = smem_u32(tau);
        staged.inslots = smem_u32(inslots);
        staged.edges = smem_u32(edges);
        __syncthreads();
    }
    if (warp == kIdleWarp) return;
    const uint32_t item = warp * gridDim.x + blockIdx.x;
    const uint32_t S = b.strands;
    for (uint32_t base = 0; base < b.n_tiles; base += tiles_per_round) {
        const uint32_t tiles = min(tiles_per_round, b.n_tiles - base);
        if (item >= tiles * (S + 1)) continue;
        // consecutive items are the same role of consecutive tiles: an SM hosts a mix of tiles
        const uint32_t role = item / tiles, tile = base + item - role * tiles;
        if (role == S) {
            // a CTA's producers are consecutive warps, at most `producer_slots` of them: landing buffer
            // number (warp - first warp that can be a producer) mod producer_slots, when the launcher has
            // provided them
            const uint32_t first_producer_warp = tiles * S / gridDim.x;
            unsigned char* landing =
                producer_slots != 0u ? producer_smem + size_t((warp - first_producer_warp) % producer_slots) * kProducerSmem : nullptr;
            producer_run(b, tile, sweeps, lane, landing);
            continue;
        }
        const DevStrandGraph& g = b.strand_graphs[STAGED ? staged_model : b.tile_model[tile]];
        if constexpr (STAGED) {
            strand_run<EXP, WAIT, true>(b, staged, g.per_layer, g.layers, tile, role, sweeps, lane, warp_smem);
        } else {
            Tables<false> t;
            t.chunks = g.chunks;
            t.pos = g.pos;
            t.band = g.band_pm;
            t.tau = g.tau;
            t.edges = g.edges;
            t.inslots = g.inslots;
            strand_run<EXP, WAIT, false>(b, t, g.per_layer, g.layers, tile, role, sweeps, lane, warp_smem);
        }
    }
}

// spin words [tile][spin] (bit = lane) -> cells [tile][spin/8][lane] (bit 8+k = spin 8c+k is -1; nothing flipped)
__global__ void __launch_bounds__(256) words_to_cells_kernel(DevBatch b) {
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
    b.spin_cells[idx] = uint16_t(byte << 8);
    b.spin_nbr[idx] = uint16_t(byte | (b.strand_epoch & 0xffu) << 8);
}

__global__ void __launch_bounds__(256) cells_to_words_kernel(DevBatch b) {
    const size_t idx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t chunks = size_t(b.n_tiles) * (b.n_spins / 8);
    if (idx >= chunks * 32) return;  // (whole warps: the total is a multiple of 32)
    const size_t chunk = idx >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t byte = uint32_t(b.spin_cells[idx]) >> 8;
    uint32_t mine = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t word = __ballot_sync(0xffffffffu, (byte >> k) & 1u);
        if (lane == uint32_t(k)) mine = word;
    }
    if (lane < 8) b.spin_bits[chunk * 8 + lane] = mine;
}

// What the strands leave pending: the far updates of every layer's latest sweep that their targets
// have not pulled yet — for column t, its far sources AFTER t (those before it were pulled when t
// entered the window in that same sweep), in position order.  One warp per (tile, layer), lane = chain.
__global__ void __launch_bounds__(256) settle_fields_kernel(DevBatch b) {
    const uint32_t lane = threadIdx.x & 31u;
    const size_t unit = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    // (layer counts differ between models: units are dealt per tile with the largest count)
    const uint32_t tile = uint32_t(unit / b.max_layers), l = uint32_t(unit % b.max_layers);
    if (tile >= b.n_tiles) return;
    const DevStrandGraph g = b.strand_graphs[b.tile_model[tile]];
    if (l >= g.layers) return;
    const uint32_t P = g.per_layer, C = P / 8;
    float* hs_l = b.hs + (size_t(tile) * b.n_spins + size_t(l) * P) * 32 + lane;
    const uint16_t* cells_l = b.spin_cells + (size_t(tile) * (b.n_spins / 8) + size_t(l) * C) * 32 + lane;
    const auto pending = [&](float h, uint32_t t, uint32_t j2, uint32_t meta) {
        const int q = int(meta >> 8) / 64 * 8 + 23 - int(meta & 31u);  // (a null slot gives -8)
        if (q <= int(t)) return h;
        return pull_slot(h, j2, meta, cells_l[(meta >> 8) / 2]);
    };
    for (uint32_t t = 0; t < P; ++t) {
        const uint4 in = __ldg(g.inslots + t);
        const uint32_t more = __ldg(g.pos + t).z;
        const int q0 = int(in.y >> 8) / 64 * 8 + 23 - int(in.y & 31u);
        if (q0 <= int(t)) continue;  // in application order the sources after t come first: none
        float h = hs_l[size_t(t) * 32];
        h = pending(h, t, in.x, in.y);
        h = pending(h, t, in.z, in.w);
        for (uint32_t i = 0; i < (more >> 16); ++i) {
            const uint4 e = __ldg(g.edges + (more & 0xffffu) + i);
            h = pending(h, t, e.x, e.y);
        }
        hs_l[size_t(t) * 32] = h;
    }
}

}  // namespace

uint32_t strand_max_warps() { return kStrandMaxWarps; }
uint32_t strand_warp_smem() { return kWarpSmem; }
uint32_t strand_flag_words(uint32_t n_tiles, uint32_t strands) { return n_tiles * (strands + 1) * kFlagStride; }
// Shared-memory bytes of a staged layer graph (see sweep_strand_kernel).
size_t strand_graph_bytes(uint32_t per_layer, uint32_t n_edges) {
    return (size_t(per_layer) * 4 + 8 + per_layer / 8 + per_layer / 4 + n_edges) * sizeof(uint4);
}

namespace {
constexpr size_t kStrandSmemLimit = 227 * 1024;

struct StrandLaunch {
    dim3 grid, block;
    uint32_t round, regions, tiles_over_ctas;
    bool tile_local;  // every CTA hosts warps of one tile only
    StrandWarpMap map;
};

// Hardware warps for `logical_warps` logical ones, the first `strands` of them strands (see
// StrandWarpMap); returns the hardware warps per CTA.
uint32_t place_warps(uint32_t logical_warps, uint32_t strands, StrandWarpMap& map) {
    for (uint8_t& w : map.logical) w = uint8_t(kIdleWarp);
    float load[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    uint32_t used = 0;
    for (uint32_t w = 0; w < strands; ++w) {
        map.logical[w] = uint8_t(w);
        load[w % 4] += 1.0f;
        used = w + 1;
    }
    for (uint32_t w = strands; w < logical_warps; ++w) {
        uint32_t best = 0;
        for (uint32_t sch = 1; sch < 4; ++sch) {
            if (load[sch] < load[best]) best = sch;
        }
        uint32_t hw = strands;
        while (hw < kStrandMaxWarps && (map.logical[hw] != kIdleWarp || hw % 4 != best)) ++hw;
        if (hw >= kStrandMaxWarps) {  // no room on that scheduler: the first free warp
            hw = strands;
            while (map.logical[hw] != kIdleWarp) ++hw;
        }
        map.logical[hw] = uint8_t(w);
        load[hw % 4] += 0.55f;
        used = max(used, hw + 1);
    }
    return used;
}

template <int EXP, bool WAIT, bool STAGED>
cudaError_t launch_strand_variant(const DevBatch& b, uint32_t sweeps, const StrandLaunch& geo, cudaStream_t stream) {
    // the attribute is per function and context: always the opt-in maximum, never one batch's own need
    static bool prepared = false;
    if (!prepared) {
        const cudaError_t e = cudaFuncSetAttribute(sweep_strand_kernel<EXP, WAIT, STAGED>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, int(kStrandSmemLimit));
        if (e != cudaSuccess) return e;
        prepared = true;
    }
    const size_t region = kWarpSmem + (STAGED ? size_t(b.max_per_layer) * 8 : 0);
    const size_t base = (size_t(geo.regions) * region + (STAGED ? b.strand_graph_smem : 0u) + 15) / 16 * 16;
    // landing buffers for the producers a CTA can host, when they fit; else the producers load their
    // operands into registers
    uint32_t slots = geo.tiles_over_ctas;
    if (base + size_t(slots) * kProducerSmem > kStrandSmemLimit) slots = 0;
    const size_t total_smem = base + size_t(slots) * kProducerSmem;
    sweep_strand_kernel<EXP, WAIT, STAGED><<<geo.grid, geo.block, total_smem, stream>>>(b, sweeps, geo.round, geo.regions, slots,
                                                                                        geo.tile_local ? 1u : 0u, geo.map);
    return cudaGetLastError();
}
template <int EXP>
cudaError_t launch_strand_exp(const DevBatch& b, uint32_t sweeps, const StrandLaunch& geo, cudaStream_t stream) {
    // Separate instantiations: the wait-statistics variant is the only one that carries them (and reads
    // the graph and the cells from global memory); the default stages the graph and the strands' cells
    // in shared memory when the batch has one model and they fit.
    const bool wait = b.wait_counts != nullptr;
    const size_t staged_bytes = size_t(geo.regions) * (kWarpSmem + size_t(b.max_per_layer) * 8) + b.strand_graph_smem;
    const bool staged = !wait && (b.strand_single_model != 0u || geo.tile_local) && staged_bytes <= kStrandSmemLimit;
    if (wait) return launch_strand_variant<EXP, true, false>(b, sweeps, geo, stream);
    if (staged) return launch_strand_variant<EXP, false, true>(b, sweeps, geo, stream);
    return launch_strand_variant<EXP, false, false>(b, sweeps, geo, stream);
}
}  // namespace

cudaError_t launch_sweep_strand(const DevBatch& b, uint32_t sweeps, int sm_count, uint32_t warps_per_cta, bool from_words,
                                cudaStream_t stream) {
    if (b.n_tiles == 0 || sweeps == 0) return cudaSuccess;
    const uint32_t capacity = uint32_t(sm_count) * warps_per_cta;
    const uint32_t per_tile = b.strands + 1;
    const uint32_t most_tiles = min(b.n_tiles, capacity / per_tile);
    if (most_tiles == 0) return cudaErrorInvalidConfiguration;
    // rounds of equal size, and every SM in use: the items of a round (S + 1 warps per tile) are dealt
    // over all `sm_count` CTAs, each just wide enough (c5: 2560 items = 148 CTAs of 18 warps, not 128 of 20)
    const uint32_t rounds = (b.n_tiles + most_tiles - 1) / most_tiles;
    const uint32_t tiles_per_round = (b.n_tiles + rounds - 1) / rounds;
    cudaError_t e = cudaMemsetAsync(b.strand_flags, 0, size_t(strand_flag_words(b.n_tiles, b.strands)) * 4, stream);
    if (e != cudaSuccess) return e;
    if (from_words) {
        const size_t cells = size_t(b.n_tiles) * (b.n_spins / 8) * 32;
        words_to_cells_kernel<<<unsigned((cells + 255) / 256), 256, 0, stream>>>(b);
    }
    const uint32_t items = tiles_per_round * per_tile;
    uint32_t ctas = min(uint32_t(sm_count), items);
    // Batches of several models with no more tiles than SMs, in one round: a whole number of CTAs per
    // tile.  Items are dealt warp-major over the grid (item = warp * ctas + block, tile = item % tiles),
    // so with ctas a multiple of the tile count every warp of a CTA works on tile block % tiles — and the
    // CTA can stage that tile's graph and cells in shared memory like a single-model batch.
    const bool tile_local = b.strand_single_model == 0u && rounds == 1 && b.n_tiles <= uint32_t(sm_count) && b.wait_counts == nullptr;
    if (tile_local) ctas = min(uint32_t(sm_count) / b.n_tiles, per_tile) * b.n_tiles;
    warps_per_cta = (items + ctas - 1) / ctas;  // <= the caller's bound, since items <= capacity
    StrandLaunch geo;
    geo.tile_local = tile_local;
    geo.grid = dim3(ctas);
    geo.round = tiles_per_round;
    geo.regions = min(warps_per_cta, (tiles_per_round * b.strands + ctas - 1) / ctas);  // warps that can be strands
    geo.block = dim3(place_warps(warps_per_cta, geo.regions, geo.map) * 32);
    geo.tiles_over_ctas = (tiles_per_round + ctas - 1) / ctas;                          // producers a CTA can host
    switch (b.exp_kind) {
        case kExpExact: return launch_strand_exp<kExpExact>(b, sweeps, geo, stream);
        case kExpFast: return launch_strand_exp<kExpFast>(b, sweeps, geo, stream);
        default: return launch_strand_exp<kExpAccurate>(b, sweeps, geo, stream);
    }
}

cudaError_t launch_strand_settle(const DevBatch& b, cudaStream_t stream) {
    if (b.n_tiles == 0) return cudaSuccess;
    // one warp per (tile, layer), then the spin words from the cells
    const size_t threads = size_t(b.n_tiles) * b.max_layers * 32;
    settle_fields_kernel<<<unsigned((threads + 255) / 256), 256, 0, stream>>>(b);
    const size_t cells = size_t(b.n_tiles) * (b.n_spins / 8) * 32;
    cells_to_words_kernel<<<unsigned((cells + 255) / 256), 256, 0, stream>>>(b);
    return cudaGetLastError();
}

}  // namespace isingb200
