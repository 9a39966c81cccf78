// Layered-model sweep kernel: the performance path for identical-layer ("QMC-style") models.
//
// One persistent CTA per SM, 16 warps = 4 tiles x 4 roles.  A TILE is 32 chains (lane = chain); its
// four warps share warp_id % 4, hence one SM sub-partition (scheduler, register file slice, TMEM lane
// quarter).  A chain's sweep is strictly sequential (attempt p+1 needs the flips of attempt p), so
// the SWEEP warp is latency bound; everything that is not on that loop-carried chain runs in the
// other three warps, whose instructions fill the issue slots the chain leaves empty:
//
//   producer (ahead)   MT19937 regeneration in place (replica-interleaved state, HBM/L2 resident),
//                      tempering, u32 -> unit float, and per attempt the PREP RECORD
//                      {u, -2*beta*s, gamma*h_tau, h_tau} plus one sign word per chunk
//   sweep              decision, band-neighbour updates in registers, ballot; moves the register
//                      window through Tensor Memory eight columns at a time
//   post (behind)      accept counts, running energy (f64), spin-word flips
//   far (behind)       far-neighbour field updates as batched Tensor Memory read-modify-writes
//
// Work moves in CHUNKS of 8 attempts through a shared-memory ring of stages: `full` mbarriers
// (producer -> sweep), one named hardware barrier per tile (sweep -> post, far: they sleep in it, and
// the sweep warp is never more than one chunk ahead of them), `empty` mbarriers (post + far -> producer).
//
// A chain's working set for one layer lives ON CHIP:
//   * Tensor Memory holds the space fields of the layer being swept: column p of the tile's 32-lane
//     quarter is h_eff_space[(layer, p)] of its 32 chains (512 columns x 128 lanes x 4 B = the whole
//     256 KB TMEM of an SM for 4 tiles x 512 positions).  All three TMEM roles of a tile change
//     layers together (layer_transition: a third of the columns each, HBM <-> TMEM, streaming hints).
//   * A REGISTER WINDOW of the sweep warp slides over the columns p-2..p+2 of the position being
//     attempted.  Updates of these band neighbours are predicated register adds.  In a LEAN chunk
//     (97 % of them) the eight columns that enter the window are loaded with one tcgen05.ld.x8 and
//     the eight that leave it stored with one tcgen05.st.x8; the attempts themselves touch no TMEM.
//   * Far (non-band) neighbours of a flip are updated in Tensor Memory by whoever can do it without
//     stalling the sweep: the FAR warp for every target the sweep warp is not about to load
//     (backward targets, forward targets two or more chunks ahead), in groups of 8 edges with
//     distinct targets whose loads go out together; the sweep warp itself for the few NEAR forward
//     targets — after the chunk for targets the next chunk will load, per attempt (CAREFUL chunk,
//     out of line) for targets inside the columns already loaded.  See build_layer_graph (batch.cpp)
//     for the split and the ordering argument.
//   * The tau field is NOT stored.  For these models it only takes the values {2J, +0, -2J}
//     and every incremental update of it is exact (HostModel::layered_uniform), so it is rebuilt
//     from two spin bits of the adjacent layers.  That removes 8 of the 17 bytes per attempt the
//     generic layout streams, and both tau read-modify-writes of every flip.
//   * Spins are one bit per chain: a 32-bit word per (tile, spin) holds the 32 lanes' signs.
//     Three layers of words (previous, current, next) sit in shared memory per tile.
//   * One layer's graph (band addends per sign, edge groups per chunk) sits in shared memory.
//
// HBM traffic per sweep is one read and one write of the f32 space fields plus the bit words
// (8.25 B per attempt); the MT19937 state (12 B per attempt if it missed) is pinned in L2.
// The trajectory is the reference's (ref: proj/src/sweep_basic.cpp:12-56) bit for bit.
#include "device_batch.hpp"
#include "device_math.cuh"
#include "device_mt.cuh"

namespace isingb200 {

namespace {

constexpr int kSweepWarps = 4;          // one TMEM lane quarter each
constexpr int kRolesPerPair = 4;        // sweep, producer, post, far
constexpr int kLayeredThreads = kRolesPerPair * kSweepWarps * 32;
constexpr uint32_t kTmemColumns = 512;  // the whole TMEM: one CTA per SM
constexpr uint32_t kUnroll = 8;         // attempts per ring stage == unrolled chunk == window ring size
constexpr uint32_t kMaxStages = 8;

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
// No "memory" clobbers on the Tensor Memory traffic of the inner loop: volatile asm statements keep
// their order among themselves, and ordinary shared/global accesses are free to move across them
// (TMEM is a separate address space), which lets the compiler hoist the next attempt's loads.
__device__ __forceinline__ float tmem_ld(uint32_t taddr) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
    return __uint_as_float(v);
}
__device__ __forceinline__ void tmem_st(uint32_t taddr, float v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(__float_as_uint(v)));
}
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
// wait::ld tied to the registers of a tmem_ld8, so that no use of them can be scheduled before it
__device__ __forceinline__ void tmem_wait_ld8(float (&v)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]), "+f"(v[7]));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// ---- mbarrier (shared::cta) helpers for the stage ring
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    // not volatile: only used on the layer graph, which is constant while a tile is swept
    asm("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
// the volatile flavour, for data other warps write (prep records)
__device__ __forceinline__ float4 lds_rec(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, uint32_t backoff_ns) {
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
        if (done == 0u && backoff_ns != 0u) __nanosleep(backoff_ns);
    } while (done == 0u);
}

// Hardware-blocking rendezvous of a tile's sweep, post and far warps (named barrier, 96 threads):
// the sweep warp calls it when it has finished a chunk, the trailing two when they are ready to
// start that chunk, so they sleep in the barrier instead of polling, and the sweep warp can never
// be more than one chunk ahead of them.
__device__ __forceinline__ void chunk_barrier(uint32_t id) {
    asm volatile("bar.sync %0, 96;" ::"r"(id) : "memory");
}

// ---- shared-memory carve-up (per CTA): [header][graph x (1 | 4)][per-pair dynamic region x 4]
struct GraphSmem {
    uint4* pos;      // P : DevLayerGraph::pos
    uint4* band_pm;  // 2P : DevLayerGraph::band_pm (32-byte aligned: the entry pair of a position)
    uint4* chunks;   // P/8 : DevLayerGraph::chunks
    uint4* far;      // max_far edges
    uint32_t* groups;  // max_far groups at most
};
struct PairSmem {
    uint2* agree_sign;  // P : per layer, {~(up ^ dn), up} spin words
    uint32_t* words;    // 3 * P : ring of spin-bit layers
    float4* recs;       // stages * 8 * 32 prep records {u | h, -2*beta*s, gamma*h_tau, h_tau}
    uint32_t* ballots;  // stages * 8
    uint32_t* signs;    // stages * 32 : per lane, bit 7-k set <=> the spin of the stage's attempt k was -1
};

// header: tmem slot (16 B) + per tile full[8], (unused)[8], empty[8] mbarriers (192 B) x 4
constexpr size_t kRingBarriers = kSweepWarps * 3 * kMaxStages;
constexpr size_t kHeaderBytes = 16 + kRingBarriers * 8 + 16;  // + one far-warp progress counter per tile

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) / 16 * 16; }
__host__ __device__ inline size_t graph_bytes(uint32_t P, uint32_t max_far, uint32_t max_groups) {
    // pos + band_pm + chunks + far edges + groups; a multiple of 32 keeps band_pm pairs 32-byte aligned
    return (size_t(P) * 48 + size_t(P) * 2 + size_t(max_far ? max_far : 1) * 16 +
            size_t(max_groups ? max_groups : 1) * 4 + 31) / 32 * 32;
}
__host__ __device__ inline size_t pair_bytes(uint32_t P, uint32_t stages) {
    return align16(size_t(P) * 8) + align16(size_t(P) * 12) + size_t(stages) * kUnroll * 32 * 16 +
           align16(size_t(stages) * kUnroll * 4) + size_t(stages) * 32 * 4;
}

__device__ __forceinline__ GraphSmem carve_graph(unsigned char* base, uint32_t P) {
    GraphSmem g;
    g.pos = reinterpret_cast<uint4*>(base);
    g.band_pm = g.pos + P;
    g.chunks = g.band_pm + 2 * size_t(P);
    g.far = g.chunks + P / 8;
    g.groups = nullptr;  // set by the caller: it follows the far edges (max_far of them)
    return g;
}
__device__ __forceinline__ PairSmem carve_pair(unsigned char* base, uint32_t P, uint32_t stages) {
    PairSmem s;
    s.agree_sign = reinterpret_cast<uint2*>(base);
    base += align16(size_t(P) * 8);
    s.words = reinterpret_cast<uint32_t*>(base);
    base += align16(size_t(P) * 12);
    s.recs = reinterpret_cast<float4*>(base);
    base += size_t(stages) * kUnroll * 32 * 16;
    s.ballots = reinterpret_cast<uint32_t*>(base);
    base += align16(size_t(stages) * kUnroll * 4);
    s.signs = reinterpret_cast<uint32_t*>(base);
    return s;
}

__device__ __forceinline__ void load_graph(const GraphSmem& dst, const DevLayerGraph& g, uint32_t tid,
                                           uint32_t nthreads) {
    for (uint32_t k = tid; k < g.per_layer; k += nthreads) {
        dst.pos[k] = g.pos[k];
        dst.band_pm[2 * k] = g.band_pm[2 * k];
        dst.band_pm[2 * k + 1] = g.band_pm[2 * k + 1];
    }
    for (uint32_t k = tid; k < g.per_layer / 8; k += nthreads) dst.chunks[k] = g.chunks[k];
    for (uint32_t k = tid; k < g.n_far; k += nthreads) dst.far[k] = g.far[k];
    for (uint32_t k = tid; k < g.n_groups; k += nthreads) dst.groups[k] = g.groups[k];
}

__device__ __forceinline__ void words_copy(uint32_t* dst, const uint32_t* src, uint32_t P, uint32_t lane) {
    for (uint32_t k = lane; k < P; k += 32) dst[k] = src[k];
}

// Position of a pair in its stage ring.  Both warps of a pair walk the same sequence of stages;
// a stage's barrier phase parity is the number of times it has been waited on, kept as one bit
// per stage.
struct RingCursor {
    uint32_t stage = 0;
    uint32_t parity_bits = 0;  // next parity to wait for, per stage
    __device__ __forceinline__ uint32_t parity() const { return (parity_bits >> stage) & 1u; }
    __device__ __forceinline__ void waited() { parity_bits ^= 1u << stage; }
    __device__ __forceinline__ void advance(uint32_t stages) { stage = stage + 1 == stages ? 0u : stage + 1; }
};

// =======================================================================================
// Producer warp (ahead of the sweep), post and far warps (behind it)
// =======================================================================================
struct ProducerState {
    uint32_t* mt;      // this lane's MT19937 state column
    uint32_t pos, cur;
    uint32_t nxt[kUnroll], far[kUnroll];  // operands of the next 8 draws, loaded one chunk ahead
    uint32_t nb2, sh;
    bool active;
};

// Loads the recurrence operands of draws pos..pos+7 (ref: rng.cpp:22-25).  Fast path: the run does
// not cross a wrap point (word 227: far operand wraps, 623: next operand wraps).
__device__ __forceinline__ void mt_load_operands(ProducerState& h) {
    const uint32_t pos = h.pos;
    const bool straight = pos + kUnroll <= kMtN - kMtM || (pos >= kMtN - kMtM && pos + kUnroll <= kMtN - 1);
    if (straight) {
        const uint32_t* np = h.mt + size_t(pos + 1) * 32;
        const uint32_t* fp = h.mt + size_t(pos < kMtN - kMtM ? pos + kMtM : pos - (kMtN - kMtM)) * 32;
#pragma unroll
        for (int k = 0; k < int(kUnroll); ++k) {
            h.nxt[k] = np[size_t(k) * 32];
            h.far[k] = fp[size_t(k) * 32];
        }
    } else {
#pragma unroll
        for (int k = 0; k < int(kUnroll); ++k) {
            uint32_t jn = pos + k + 1, jf = pos + k + kMtM;
            jn = jn >= kMtN ? jn - kMtN : jn;
            jf = jf >= kMtN ? jf - kMtN : jf;
            h.nxt[k] = h.mt[size_t(jn) * 32];
            h.far[k] = h.mt[size_t(jf) * 32];
        }
    }
}

// Regenerates words pos..pos+7 in place from the preloaded operands and returns the raw outputs.
// None of the operands of a chunk is a word the chunk before it rewrote (the `next` words lie
// ahead of it, the `far` words 227 draws behind or 397 ahead), so loading them a chunk early
// reads exactly what the in-place loop of ref: rng.cpp:89-96 reads.
__device__ __forceinline__ void mt_generate8(ProducerState& h, uint32_t (&raw)[kUnroll]) {
    const uint32_t pos = h.pos;
    const bool wraps = pos + kUnroll > kMtN;
#pragma unroll
    for (int k = 0; k < int(kUnroll); ++k) {
        uint32_t j = pos + k;
        if (wraps) j = j >= kMtN ? j - kMtN : j;
        const uint32_t nx = h.nxt[k];
        const uint32_t v = mt_recurrence(h.cur, nx, h.far[k]);
        h.mt[size_t(j) * 32] = v;
        h.cur = nx;
        raw[k] = mt_temper(v);
    }
    h.pos = pos + kUnroll >= kMtN ? pos + kUnroll - kMtN : pos + kUnroll;
}

// Producer: MT19937, uniforms and the prep records of every attempt; owns the spin-word ring.
__device__ void producer_warp(const DevBatch& b, uint32_t sweeps, uint32_t lane, const GraphSmem& g,
                              const PairSmem& s, uint64_t* full, uint64_t* empty, RingCursor& cursor,
                              uint32_t stages, uint32_t tile, uint32_t P, uint32_t L) {
    const uint32_t n = b.n_spins;
    const uint32_t chain = b.tile_first[tile] + lane;
    ProducerState h;
    h.active = lane < b.tile_count[tile];
    h.nb2 = __float_as_uint(h.active ? -2.0f * b.betas[b.slot_of_chain[chain]] : 0.0f);
    h.sh = 1u << (31u - lane);  // word * sh moves this lane's bit to bit 31 (a multiply: FMA pipe, not ALU)
    const float u_offset = h.active ? 0.0f : 2.0f;  // padding lanes draw u >= 2: they never accept
    h.mt = b.mt + size_t(tile) * kMtN * 32 + lane;
    h.pos = b.mt_pos[tile];
    h.cur = h.mt[size_t(h.pos) * 32];
    mt_load_operands(h);

    uint32_t* words_g = b.spin_bits + size_t(tile) * n;
    uint32_t slot_dn = 2, slot_cur = 0, slot_up = 1;
    words_copy(s.words + slot_dn * P, words_g + size_t(L - 1) * P, P, lane);
    words_copy(s.words + slot_cur * P, words_g, P, lane);
    words_copy(s.words + slot_up * P, words_g + size_t(1) * P, P, lane);
    __syncwarp();

    uint32_t in_flight = 0;  // bit s set: stage s was filled and its `empty` has not been waited for yet

    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t l = 0; l < L; ++l) {
            const uint32_t* w_cur = s.words + slot_cur * P;
            // the words of layer l+2 are read at the end of this layer: have them in L2 by then
            if (lane * 32 < P) prefetch_l2(words_g + size_t((l + 2) % L) * P + lane * 32);
            {   // the tau field of this whole layer is fixed while it is swept: previous layer already
                // visited, next layer not yet.  agree = neighbours equal, sign = their common spin bit.
                const uint32_t* w_up = s.words + slot_up * P;
                const uint32_t* w_dn = s.words + slot_dn * P;
                for (uint32_t k = lane; k < P; k += 32) s.agree_sign[k] = make_uint2(~(w_up[k] ^ w_dn[k]), w_up[k]);
            }
            __syncwarp();

            for (uint32_t p0 = 0; p0 < P; p0 += kUnroll) {
                const uint32_t st = cursor.stage;
                float4* recs = s.recs + size_t(st) * kUnroll * 32 + lane;
                if ((in_flight >> st) & 1u) {  // recycle: the post and far warps must be done with it
                    mbar_wait(&empty[st], cursor.parity(), 400);
                    cursor.waited();
                }
                uint32_t raw[kUnroll];
                uint32_t signs = 0;
                mt_generate8(h, raw);
                mt_load_operands(h);  // operands of the next chunk: in flight while this one is prepared
#pragma unroll
                for (int k = 0; k < int(kUnroll); ++k) {
                    const uint32_t p = p0 + k;
                    const uint32_t word = w_cur[p];
                    const uint2 as = s.agree_sign[p];
                    const uint32_t tau_g = *reinterpret_cast<const uint32_t*>(g.pos + p);  // bits of gamma * 2J_tau
                    const uint32_t spin_top = word * h.sh;  // bit 31 set <=> s = -1 (lower bits: other lanes)
                    const uint32_t sgn_up = (as.y * h.sh) & 0x80000000u;
                    const uint32_t agree = uint32_t(int32_t(as.x * h.sh) >> 31);  // ones when s_up == s_dn
                    float4 rec;
                    // u32_to_unit (x * 2^-32 is exact, so is adding +0); padding lanes get u + 2
                    rec.x = __fmaf_rn(__uint2float_rz(raw[k]), 0x1p-32f, u_offset);
                    // x = -beta*((2s)*v) == (-2*beta*s)*v: doubling is exact, one rounding either way
                    rec.y = __uint_as_float(h.nb2 ^ (spin_top & 0x80000000u));
                    signs = __funnelshift_l(spin_top, signs, 1);  // attempt k ends up at bit 7-k
                    // tau field J*(s_up + s_dn) in {+2J, +0, -2J}, scaled by gamma
                    rec.z = __uint_as_float((tau_g ^ sgn_up) & agree);
                    rec.w = 0.0f;
                    recs[k * 32] = rec;
                }
                s.signs[st * 32 + lane] = signs;
                in_flight |= 1u << st;
                mbar_arrive(&full[st]);
                cursor.advance(stages);
            }

            // ---- end of layer: every stage must have been post-processed (the spin words of this
            // layer are final) before the ring rotates and the next layer's tau words are formed
            {
                uint32_t st = cursor.stage;  // oldest stage first
                for (uint32_t k = 0; k < stages; ++k) {
                    if ((in_flight >> st) & 1u) {
                        mbar_wait(&empty[st], (cursor.parity_bits >> st) & 1u, 100);
                        cursor.parity_bits ^= 1u << st;
                        in_flight &= ~(1u << st);
                    }
                    st = st + 1 == stages ? 0u : st + 1;
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
    if (lane == 0) b.mt_pos[tile] = h.pos;
    __syncwarp();
}

// Layer change, shared by the tile's sweep, post and far warps (part 0, 1, 2 of 3): each retires
// its third of the finished layer's columns TMEM -> HBM and feeds the same columns with the next
// layer HBM -> TMEM (full 128-byte lines, streaming hints), so the sweep warp pays a third of the
// transfer.  A warp only reuses columns it has read out itself, so no rendezvous is needed between
// the two halves; the caller closes the transition with one (chunk_barrier) before the sweep resumes.
__device__ __forceinline__ void layer_transition(uint32_t part, uint32_t tm, float* hs_old, const float* hs_new,
                                                 uint32_t P) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (hs_old != nullptr) {
        for (uint32_t p0 = part * 8; p0 < P; p0 += 24) {
            float v[8];
            tmem_ld8(tm + p0, v);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 8; ++k) __stcs(hs_old + size_t(p0 + k) * 32, v[k]);
        }
    }
    if (hs_new != nullptr) {
        // this warp's 8-column groups sit 24 columns apart; four of them (32 loads) are requested
        // before the previous four are stored, so two batches are always in flight
        uint32_t p0 = part * 8;
        float v[4][8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[q][k] = p0 + q * 24 < P ? __ldcs(hs_new + size_t(p0 + q * 24 + k) * 32) : 0.0f;
        }
        for (; p0 < P; p0 += 96) {
            float nv[4][8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    nv[q][k] = p0 + 96 + q * 24 < P ? __ldcs(hs_new + size_t(p0 + 96 + q * 24 + k) * 32) : 0.0f;
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (p0 + q * 24 < P) tmem_st8(tm + p0 + q * 24, v[q]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
#pragma unroll
                for (int k = 0; k < 8; ++k) v[q][k] = nv[q][k];
            }
        }
    }
    tmem_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// Post: accept counts, running energy and spin words of every consumed stage (ref:
// sweep_basic.cpp:47-48; the energy bookkeeping is the tempering definition of
// oracle/ising_oracle.h).
template <bool WAIT>
__device__ void post_warp(const DevBatch& b, uint32_t sweeps, uint32_t lane, const PairSmem& s,
                          uint32_t bar_id, uint64_t* empty, RingCursor& cursor, uint32_t stages,
                          uint32_t tile, uint32_t tm, uint32_t P, uint32_t L) {
    float* hs_g = b.hs + size_t(tile) * b.n_spins * 32 + lane;
    float* hs_prev = nullptr;
    const uint32_t chain = b.tile_first[tile] + lane;
    const bool active = lane < b.tile_count[tile];
    double e_run = active ? b.e_run[chain] : 0.0;
    uint32_t flips = 0;
    const uint32_t lane_top = 1u << (31u - lane);
    // wait statistics: lane k folds the ballot of attempt k of every chunk (full tiles only)
    const bool record_wait = WAIT && b.wait_counts != nullptr && b.tile_count[tile] == 32;
    uint32_t wait[6] = {0, 0, 0, 0, 0, 0};
    uint32_t slot_cur = 0;  // follows the producer's ring rotation: layer l lives in slot l % 3 of the visit order
    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t l = 0; l < L; ++l) {
            uint32_t* w_cur = s.words + slot_cur * P;
            double e_blk = 0.0;  // one partial sum per layer (tempering definition, oracle/ising_oracle.h)
            layer_transition(1, tm, hs_prev, hs_g + size_t(l) * P * 32, P);
            chunk_barrier(bar_id);
            hs_prev = hs_g + size_t(l) * P * 32;
            for (uint32_t p0 = 0; p0 < P; p0 += kUnroll) {
                const uint32_t st = cursor.stage;
                chunk_barrier(bar_id);  // the sweep warp has finished this chunk
                const float4* recs = s.recs + size_t(st) * kUnroll * 32 + lane;
                const uint32_t* ballots = s.ballots + st * kUnroll;
                // spin words: lane k flips the bits of attempt k's accepting chains
                if (lane < kUnroll) {
                    const uint32_t mine_ballot = ballots[lane];
                    w_cur[p0 + lane] ^= mine_ballot;
                    if (WAIT && record_wait) wait_fold(mine_ballot, wait);
                }
#pragma unroll
                for (int k = 0; k < int(kUnroll); ++k) {
                    const uint32_t ballot = ballots[k];
                    const float4 rec = recs[k * 32];
                    // (2s)*(h + gamma*h_tau), the inner factor of the flip exponent: doubling is exact, and
                    // rec.y = -2*beta*s carries the opposite of the spin's sign, so the product is
                    // 2*(h + gamma*h_tau) with its sign flipped where s = -1
                    const float twice = __fmul_rn(__fadd_rn(rec.x, rec.z), 2.0f);
                    const float de = __uint_as_float(__float_as_uint(twice) ^ (~__float_as_uint(rec.y) & 0x80000000u));
                    const bool mine = int32_t(ballot * lane_top) < 0;  // bit `lane` of the ballot, moved to the sign
                    flips += mine ? 1u : 0u;
                    e_blk = __dadd_rn(e_blk, double(mine ? de : -0.0f));  // -0.0: the identity for every value
                }
                mbar_arrive(&empty[st]);
                cursor.advance(stages);
            }
            e_run = __dadd_rn(e_run, e_blk);
            chunk_barrier(bar_id);  // layer rendezvous (the sweep warp waits for the far warp here)
            slot_cur = slot_cur == 2 ? 0u : slot_cur + 1;
            if (WAIT && record_wait) {  // flushed per layer (lanes 0..7 hold partial sums of at most 64 * 32 each)
                unsigned long long* out = b.wait_counts + size_t(tile) * kWaitSlots;
#pragma unroll
                for (int w = 0; w < 6; ++w) {
                    uint32_t v = wait[w];
                    for (int off = 4; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
                    if (lane == 0) out[w] += v;
                    wait[w] = 0;
                }
                if (lane == 0) out[6] += P;
            }
        }
    }
    layer_transition(1, tm, hs_prev, nullptr, P);
    chunk_barrier(bar_id);
    if (active) {
        b.e_run[chain] = e_run;
        b.flips[chain] += flips;
    }
    __syncwarp();
}

// Applies the edge groups `ginfo` (begin | count << 16) of one finished chunk: h[t] -= (2s)*J for
// every lane that accepted attempt k of the chunk, as Tensor Memory read-modify-writes on column t.
// The targets of a group are distinct, so its loads go out together; all 32 lanes move data, a lane
// that did not accept adds -0.0.  Groups are normally padded to 8 edges (the padding targets a
// column nobody else writes meanwhile and belongs to no attempt that can accept: see batch.cpp).
// `signs_addr`/`ballots_addr` are the chunk's stage (this lane's sign word, the 8 ballots).
__device__ __forceinline__ uint32_t edge_addend(uint4 e, uint32_t acc_neg) {
    // e = {column, 7 - attempt index, bits of 2J, 0}.  acc_neg: bit 7-k = this lane accepted attempt
    // k; bit 16+7-k = sign bit of rec.y = -2*beta*s, the sign of the addend -(2s)*J relative to 2J
    const uint32_t t = acc_neg >> e.y;
    const uint32_t add = ((t << 15) & 0x80000000u) ^ e.z;
    return (t & 1u) ? add : 0x80000000u;
}
__device__ __forceinline__ void apply_groups(uint32_t tm, const GraphSmem& g, uint32_t ginfo, uint32_t signs_addr,
                                             uint32_t ballots_addr, uint32_t lane) {
    uint32_t acc_neg;
    {
        uint4 b0, b1;
        uint32_t spins;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b0.x), "=r"(b0.y), "=r"(b0.z), "=r"(b0.w) : "r"(ballots_addr) : "memory");
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b1.x), "=r"(b1.y), "=r"(b1.z), "=r"(b1.w) : "r"(ballots_addr + 16) : "memory");
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(spins) : "r"(signs_addr) : "memory");
        const uint32_t bl[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        // rec.y = -2*beta*s is negative for s = +1, i.e. where the spin bit is clear (an accepting
        // lane is never a padding lane, whose -2*beta is +0)
        acc_neg = (~spins & 0xffu) << 16;
#pragma unroll
        for (uint32_t k = 0; k < kUnroll; ++k) acc_neg |= ((bl[k] >> lane) & 1u) << (7u - k);
    }
    const uint32_t* grp = g.groups + (ginfo & 0xffffu);
    const uint32_t n_groups = ginfo >> 16;
#pragma unroll 1
    for (uint32_t q = 0; q < n_groups; ++q) {
        const uint32_t info = grp[q];
        const uint4* fe = g.far + (info & 0xffffu);
        const uint32_t n = info >> 16;
        if (n == kUnroll) {
            uint4 e[kUnroll];
            float v[kUnroll];
#pragma unroll
            for (uint32_t i = 0; i < kUnroll; ++i) e[i] = fe[i];
#pragma unroll
            for (uint32_t i = 0; i < kUnroll; ++i) v[i] = tmem_ld(tm + e[i].x);
            tmem_wait_ld();
#pragma unroll
            for (uint32_t i = 0; i < kUnroll; ++i) {
                tmem_st(tm + e[i].x, __fadd_rn(v[i], __uint_as_float(edge_addend(e[i], acc_neg))));
            }
        } else {  // unpadded group (near groups; layers too short to find padding columns): one edge at a time
#pragma unroll 1
            for (uint32_t i = 0; i < n; ++i) {
                const uint4 e = fe[i];
                const float v = tmem_ld(tm + e.x);
                tmem_wait_ld();
                tmem_st(tm + e.x, __fadd_rn(v, __uint_as_float(edge_addend(e, acc_neg))));
            }
        }
        tmem_wait_st();  // the next group may hit one of these columns again
    }
}

// Far: applies the far-neighbour updates the sweep warp does not need soon — every BACKWARD target
// (its column left the register window before the flipping attempt ran) and every FORWARD target
// that enters the window at least two chunks later.  It trails the sweep warp by whole chunks,
// shares its TMEM lane quarter, and publishes how many chunks it has finished; the sweep warp
// waits on that count before it reads a column this warp may still owe an update.  Per column the
// updates stay in attempt order: this warp walks attempts in order, and the sweep warp touches a
// column (near forward update, window entry) only after the chunks that could still target it here.
__device__ void far_warp(float* hs_g, uint32_t sweeps, uint32_t lane, const GraphSmem& g, const PairSmem& s,
                         uint32_t bar_id, uint64_t* empty, uint32_t* far_done, uint32_t& chunks_done,
                         RingCursor& cursor, uint32_t stages, uint32_t tm, uint32_t P, uint32_t L) {
    float* hs_prev = nullptr;
    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t l = 0; l < L; ++l) {
            layer_transition(2, tm, hs_prev, hs_g + size_t(l) * P * 32, P);
            chunk_barrier(bar_id);
            hs_prev = hs_g + size_t(l) * P * 32;
            for (uint32_t p0 = 0; p0 < P; p0 += kUnroll) {
                const uint32_t st = cursor.stage;
                const uint32_t ginfo = g.chunks[p0 / kUnroll].x;  // (static: requested before the rendezvous)
                chunk_barrier(bar_id);  // the sweep warp has finished this chunk
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if ((ginfo >> 16) != 0u) {
                    apply_groups(tm, g, ginfo, smem_u32(s.signs + st * 32 + lane), smem_u32(s.ballots + st * kUnroll),
                                 lane);
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&empty[st]);
                cursor.advance(stages);
                // publish progress: the sweep warp orders its own reads of the updated columns on it
                ++chunks_done;
                __syncwarp();
                if (lane == 0) {
                    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(far_done)), "r"(chunks_done)
                                 : "memory");
                }
            }
            chunk_barrier(bar_id);  // layer rendezvous: every update of this layer has landed
        }
    }
    layer_transition(2, tm, hs_prev, nullptr, P);
    chunk_barrier(bar_id);
    __syncwarp();
}

// =======================================================================================
// Sweep warp
// =======================================================================================
// Far neighbours of a flipped spin: h[t] -= (2s)*J as a Tensor Memory read-modify-write on column t
// (the first two with their loads batched).  All 32 lanes move data; only accepting lanes change it.
__device__ __noinline__ void far_update(uint32_t tm, const uint4* fe, uint32_t far_count, uint32_t neg_d,
                                        bool accept) {
    tmem_wait_st();  // a column retired by an earlier attempt may be a target
    const uint4 e0 = fe[0];
    const uint4 e1 = fe[far_count > 1u ? 1 : 0];
    const uint32_t c0 = tm + e0.x, c1 = tm + e1.x;
    const float v0 = tmem_ld(c0);
    float v1 = 0.0f;
    if (far_count > 1u) v1 = tmem_ld(c1);
    tmem_wait_ld();
    const float n0 = __fadd_rn(v0, __uint_as_float(e0.z ^ neg_d));
    const float n1 = __fadd_rn(v1, __uint_as_float(e1.z ^ neg_d));
    tmem_st(c0, accept ? n0 : v0);
    if (far_count > 1u) tmem_st(c1, accept ? n1 : v1);
#pragma unroll 1
    for (uint32_t e = 2; e < far_count; ++e) {
        const uint4 ed = fe[e];
        const uint32_t c = tm + ed.x;
        const float v = tmem_ld(c);
        tmem_wait_ld();
        const float nv = __fadd_rn(v, __uint_as_float(ed.z ^ neg_d));
        tmem_st(c, accept ? nv : v);
    }
    tmem_wait_st();  // a target may be the next column to enter the window
}

// Progress of the FAR warp as seen by the sweep warp.  Chunks are counted over the whole kernel
// (both warps walk the same sequence), `cached` is the last value read.
struct FarProgress {
    uint32_t addr;        // shared-memory address of the pair's counter
    uint32_t cached;
    uint32_t layer_base;  // chunks finished before this layer began
};
// Blocks until the far warp has finished `need_abs` chunks; then its Tensor Memory updates of
// those chunks are ordered before whatever this warp does next.
__device__ __forceinline__ void wait_far(FarProgress& ps, uint32_t need_abs) {
    if (int32_t(need_abs - ps.cached) > 0) {
        uint32_t v;
        do {
            asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(ps.addr) : "memory");
        } while (int32_t(need_abs - v) > 0);
        ps.cached = v;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
}

// The Metropolis decision of one attempt (ref: sweep_kernels.hpp:14-16, sweep_basic.cpp:36-37: no clamp).
template <int EXP>
__device__ __forceinline__ bool decide(float h, const float4 rec) {
    const float x = __fmul_rn(rec.y, __fadd_rn(h, rec.z));
    return rec.x < exp_kind<EXP>(x);
}

// Band neighbours of a flip: h -= (2s)*J  ==  h + (-(2s)*J), predicated register adds on the window
// entries p-2, p-1, p+1, p+2.  The addend comes from the band_pm entry of the flipped spin's sign
// (the sign bit of rec.y = -2*beta*s picks it); an empty slot adds -0.0.
template <int K>
__device__ __forceinline__ void band_update(float (&r)[kUnroll], bool accept, uint32_t band_addr, float rec_y) {
    const uint32_t sel = ((__float_as_uint(rec_y) >> 27) & 16u) | band_addr;  // band_addr is 32-byte aligned
    const uint4 op = lds128(sel + K * 32);
    const float a0 = __fadd_rn(r[(K + 6) & 7], __uint_as_float(op.x));
    const float a1 = __fadd_rn(r[(K + 7) & 7], __uint_as_float(op.y));
    const float a2 = __fadd_rn(r[(K + 1) & 7], __uint_as_float(op.z));
    const float a3 = __fadd_rn(r[(K + 2) & 7], __uint_as_float(op.w));
    r[(K + 6) & 7] = accept ? a0 : r[(K + 6) & 7];
    r[(K + 7) & 7] = accept ? a1 : r[(K + 7) & 7];
    r[(K + 1) & 7] = accept ? a2 : r[(K + 1) & 7];
    r[(K + 2) & 7] = accept ? a3 : r[(K + 2) & 7];
}

// Addresses of the stage the sweep warp is consuming (shared-memory window addresses).
struct StageAddr {
    uint32_t rec_x;    // this lane's rec.x of attempt 0 (attempts are 512 B apart)
    uint32_t ballots;  // ballot of attempt 0
    uint32_t band;     // band_pm pair of position p0
};

// One attempt at position p = p0 + K of a CAREFUL chunk (K is the compile-time index inside the
// unrolled chunk; the register window r[] is indexed by position & 7): the window moves one column
// per attempt, and near forward far targets are updated in Tensor Memory before they enter it.
template <int EXP, int K>
__device__ __forceinline__ void attempt(float (&r)[kUnroll], const float4 rec, const StageAddr& sa, uint32_t far_info,
                                        FarProgress& ps, uint32_t chunks_before, uint32_t p0, uint32_t P, uint32_t tm,
                                        const uint4* far, uint32_t lane) {
    const float h = r[K];
    const bool accept = decide<EXP>(h, rec);
    tmem_wait_ld();  // the entry for p+2 was requested right after the previous attempt
    band_update<K>(r, accept, sa.band, rec.y);
    const uint32_t ballot = __ballot_sync(0xffffffffu, accept);
    sts32(sa.rec_x + K * 512, __float_as_uint(h));  // the post warp needs the field this decision saw
    if (lane == 0) sts32(sa.ballots + K * 4, ballot);

    // ---- retire column p-2: no later attempt of this layer can reach it through the band
    if (K >= 2 || p0 != 0) tmem_st(tm + p0 + K - 2, r[(K + 6) & 7]);

    // ---- near forward far neighbours: read-modify-write in Tensor Memory, out of line (a near
    // target may also have updates pending in the far warp, all from earlier chunks: they land first)
    const uint32_t near_count = (far_info >> 16) & 15u;
    if (near_count != 0u && ballot != 0u) {
        wait_far(ps, chunks_before);
        far_update(tm, far + (far_info & 0xffffu), near_count, __float_as_uint(rec.y) & 0x80000000u, accept);
    }
    // ---- the window entry for p+3 (first needed by attempt p+1)
    if (K <= 4 || p0 + kUnroll < P) r[(K + 3) & 7] = tmem_ld(tm + p0 + K + 3);
}

// One attempt of a LEAN chunk (no near forward far targets, not the first or last chunk of the
// layer): the eight columns entering the window were loaded together (nx), the eight leaving it
// are collected (out) and stored together, so the attempt touches no Tensor Memory at all.
template <int EXP, int K>
__device__ __forceinline__ void attempt_lean(float (&r)[kUnroll], float (&out)[kUnroll], float (&nx)[kUnroll],
                                             const float4 rec, const StageAddr& sa, uint32_t lane) {
    const float h = r[K];
    const bool accept = decide<EXP>(h, rec);
    if (K == 0) tmem_wait_ld8(nx);  // in flight during the first decision
    band_update<K>(r, accept, sa.band, rec.y);
    const uint32_t ballot = __ballot_sync(0xffffffffu, accept);
    sts32(sa.rec_x + K * 512, __float_as_uint(h));
    if (lane == 0) sts32(sa.ballots + K * 4, ballot);
    out[K] = r[(K + 6) & 7];  // column p-2 is final
    r[(K + 3) & 7] = nx[K];   // column p+3 enters
}

#define ISING_ATTEMPT(K) \
    attempt<EXP, K>(r, rec##K, sa, g.pos[p0 + K].z, ps, chunk_seq, p0, P, tm, g.far, lane);
#define ISING_ATTEMPT_LEAN(K) attempt_lean<EXP, K>(r, out, nx, rec##K, sa, lane);

// Near groups of a lean chunk (columns 8c+11 .. 8c+18, not loaded yet): the far warp may still owe
// them updates from the chunk before this one, which must land first.
__device__ __noinline__ void apply_near_groups(uint32_t tm, const GraphSmem& g, uint32_t ginfo, uint32_t signs_addr,
                                               uint32_t ballots_addr, uint32_t far_done_addr, uint32_t chunk_seq,
                                               uint32_t lane) {
    FarProgress ps{far_done_addr, 0u, 0u};
    __syncwarp();
    wait_far(ps, chunk_seq);
    apply_groups(tm, g, ginfo, signs_addr, ballots_addr, lane);
}

// The register window of the sweep warp, passed by value to the out-of-line chunk below.
struct Window {
    float r[kUnroll];
};

// A chunk that is not plain lean: careful (per-attempt window traffic and near updates), or lean
// but first / last of its layer.  Out of line, so that the sweep
// warp's hot loop (plain lean chunks, ~97 % of them) stays a few KB of straight code.
template <int EXP>
__device__ __noinline__ Window special_chunk(Window w, const GraphSmem g, const PairSmem s, uint32_t far_done_addr,
                                             uint32_t chunk_seq, uint32_t st, uint32_t p0, uint32_t P, uint32_t tm,
                                             uint32_t band_base, uint32_t lane) {
    float (&r)[kUnroll] = w.r;
    FarProgress ps{far_done_addr, 0u, 0u};
    const float4* recs = s.recs + size_t(st) * kUnroll * 32 + lane;
    StageAddr sa;
    sa.rec_x = smem_u32(recs);
    sa.ballots = smem_u32(s.ballots + st * kUnroll);
    sa.band = band_base + p0 * 32;
    const uint4 chunk_info = g.chunks[p0 / kUnroll];
    const float4 rec0 = recs[0 * 32], rec1 = recs[1 * 32], rec2 = recs[2 * 32], rec3 = recs[3 * 32];
    const float4 rec4 = recs[4 * 32], rec5 = recs[5 * 32], rec6 = recs[6 * 32], rec7 = recs[7 * 32];
    if ((chunk_info.z & 1u) == 0u) {
        float nx[kUnroll], out[kUnroll];
        // columns p0+3 .. p0+10 enter; the last chunk of a layer has only five left
        if (p0 + kUnroll < P) {
            tmem_ld8(tm + p0 + 3, nx);
        } else {
#pragma unroll
            for (int k = 0; k < int(kUnroll); ++k) nx[k] = k < 5 ? tmem_ld(tm + p0 + 3 + k) : 0.0f;
        }
        ISING_ATTEMPT_LEAN(0)
        ISING_ATTEMPT_LEAN(1)
        ISING_ATTEMPT_LEAN(2)
        ISING_ATTEMPT_LEAN(3)
        ISING_ATTEMPT_LEAN(4)
        ISING_ATTEMPT_LEAN(5)
        ISING_ATTEMPT_LEAN(6)
        ISING_ATTEMPT_LEAN(7)
        if ((chunk_info.y >> 16) != 0u) {
            apply_near_groups(tm, g, chunk_info.y, smem_u32(s.signs + st * 32 + lane), sa.ballots, far_done_addr,
                              chunk_seq, lane);
        }
        // columns p0-2 .. p0+5 leave the window (the first chunk has no p0-2, p0-1)
        if (p0 != 0) {
            tmem_st8(tm + p0 - 2, out);
        } else {
#pragma unroll
            for (int k = 2; k < int(kUnroll); ++k) tmem_st(tm + k - 2, out[k]);
        }
    } else {
        ISING_ATTEMPT(0)
        ISING_ATTEMPT(1)
        ISING_ATTEMPT(2)
        ISING_ATTEMPT(3)
        ISING_ATTEMPT(4)
        ISING_ATTEMPT(5)
        ISING_ATTEMPT(6)
        ISING_ATTEMPT(7)
        tmem_wait_ld();  // entries requested by the last attempts
    }
    return w;
}

template <int EXP>
__device__ void sweep_warp(const DevBatch& b, uint32_t sweeps, uint32_t lane, const GraphSmem& g,
                           const PairSmem& s, uint64_t* full, uint32_t bar_id, uint32_t far_done_addr,
                           uint32_t& chunk_seq, RingCursor& cursor, uint32_t stages, uint32_t tile,
                           uint32_t tm, uint32_t P, uint32_t L) {
    const uint32_t n = b.n_spins;
    float* hs_g = b.hs + size_t(tile) * n * 32 + lane;
    float* hs_prev = nullptr;
    uint32_t p0 = 0;
    const uint32_t band_base = smem_u32(g.band_pm);
    const uint32_t recs_u32 = smem_u32(s.recs + lane), ballots_u32 = smem_u32(s.ballots);
    const uint32_t signs_u32 = smem_u32(s.signs + lane);

    for (uint32_t sw = 0; sw < sweeps; ++sw) {
        for (uint32_t l = 0; l < L; ++l) {
            float* hs_l = hs_g + size_t(l) * P * 32;
            const float* hs_next = hs_g + size_t(l + 1 == L ? 0 : l + 1) * P * 32 - lane;
            // ---- layer change: retire the previous layer, feed this one (a third each with the
            // post and far warps), then rendezvous
            layer_transition(0, tm, hs_prev, hs_l, P);
            chunk_barrier(bar_id);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            hs_prev = hs_l;

            // register window: positions 0..2 (entries for -2, -1 stay unused: their band slots are empty)
            Window w;
            float (&r)[kUnroll] = w.r;
#pragma unroll
            for (int k = 0; k < int(kUnroll); ++k) r[k] = 0.0f;
            r[0] = tmem_ld(tm + 0);
            r[1] = tmem_ld(tm + 1);
            r[2] = tmem_ld(tm + 2);
            tmem_wait_ld();

            for (p0 = 0; p0 < P; p0 += kUnroll) {
                const uint32_t st = cursor.stage;
                const uint4 chunk_info = g.chunks[p0 / kUnroll];  // (static: requested before the wait)
                mbar_wait(&full[st], cursor.parity(), 0);
                cursor.waited();
                // columns entering the window during this chunk may be owed updates by the far warp from
                // attempts at least two chunks back: the chunk rendezvous below guarantees it has
                // finished those (it cannot be more than one chunk behind)
                if ((p0 & 31u) == 0 && p0 + lane < P) prefetch_l2(hs_next + size_t(p0 + lane) * 32);
                const uint32_t special = chunk_info.z;
                StageAddr sa;
                sa.rec_x = recs_u32 + st * (kUnroll * 32 * 16);
                sa.ballots = ballots_u32 + st * (kUnroll * 4);
                sa.band = band_base + p0 * 32;
                // (requested before the branch on `special`, whose own load is still in flight)
                const float4 rec0 = lds_rec(sa.rec_x + 0 * 512), rec1 = lds_rec(sa.rec_x + 1 * 512);
                const float4 rec2 = lds_rec(sa.rec_x + 2 * 512), rec3 = lds_rec(sa.rec_x + 3 * 512);
                const float4 rec4 = lds_rec(sa.rec_x + 4 * 512), rec5 = lds_rec(sa.rec_x + 5 * 512);
                const float4 rec6 = lds_rec(sa.rec_x + 6 * 512), rec7 = lds_rec(sa.rec_x + 7 * 512);
                if (__builtin_expect(special == 0u, 1)) {
                    // plain lean chunk: eight columns in, eight attempts, eight columns out
                    float nx[kUnroll], out[kUnroll];
                    tmem_ld8(tm + p0 + 3, nx);  // columns p0+3 .. p0+10: final by now (see delegated() in batch.cpp)
                    ISING_ATTEMPT_LEAN(0)
                    ISING_ATTEMPT_LEAN(1)
                    ISING_ATTEMPT_LEAN(2)
                    ISING_ATTEMPT_LEAN(3)
                    ISING_ATTEMPT_LEAN(4)
                    ISING_ATTEMPT_LEAN(5)
                    ISING_ATTEMPT_LEAN(6)
                    ISING_ATTEMPT_LEAN(7)
                    if (__builtin_expect((chunk_info.y >> 16) != 0u, 0)) {
                        apply_near_groups(tm, g, chunk_info.y, signs_u32 + st * 128, sa.ballots, far_done_addr,
                                          chunk_seq, lane);
                    }
                    tmem_st8(tm + p0 - 2, out);  // columns p0-2 .. p0+5 leave the window
                } else {
                    w = special_chunk<EXP>(w, g, s, far_done_addr, chunk_seq, st, p0, P, tm, band_base, lane);
                }
                // the far warp may now update columns this chunk retired: they must have landed
                tmem_wait_st();
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                chunk_barrier(bar_id);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                cursor.advance(stages);
                ++chunk_seq;
            }
            // the last two columns leave the window
            tmem_st(tm + P - 2, r[6]);
            tmem_st(tm + P - 1, r[7]);
            tmem_wait_st();
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            // layer rendezvous: the far warp's updates of this layer are in, and the three warps may
            // now read the layer out together
            chunk_barrier(bar_id);
        }
    }
    layer_transition(0, tm, hs_prev, nullptr, P);
    chunk_barrier(bar_id);
    __syncwarp();
}
#undef ISING_ATTEMPT
#undef ISING_ATTEMPT_LEAN

template <int EXP, bool WAIT, bool SPREAD>
__global__ void __launch_bounds__(kLayeredThreads, 1) sweep_layered_kernel(DevBatch b, uint32_t sweeps) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + 16);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t role = warp >> 2;  // 0 sweep, 1 producer, 2 post, 3 far
    // A tile's sweep, post and far warps must sit on scheduler `pair` (it is also the TMEM lane quarter
    // they may touch); the producer touches no Tensor Memory.  SPREAD (the host picks it when a CTA has
    // at most two tiles, pairs 0 and 1): their producers run on the two schedulers that would otherwise
    // idle — a tile is 14 % faster without its producer's 43 instructions per attempt in its issue port.
    const uint32_t pair = (SPREAD && role == 1) ? (warp + 2u) & 3u : warp & 3u;  // 0 sweep, 1 producer, 2 post, 3 far — all four on scheduler `pair`
    uint64_t* full = bars + pair * 3 * kMaxStages;   // producer -> sweep
    uint64_t* empty = full + 2 * kMaxStages;         // post + far -> producer
    const uint32_t bar_id = 5 + pair;                // named barrier of the tile's sweep/post/far rendezvous
    uint32_t* far_done = reinterpret_cast<uint32_t*>(bars + kRingBarriers) + pair;  // far -> sweep progress

    const uint32_t maxP = b.max_per_layer;
    const uint32_t stages = b.layered_stages;
    const size_t gbytes = graph_bytes(maxP, b.max_far_edges, b.max_groups);
    unsigned char* graph_base = smem_raw + kHeaderBytes + (b.graph_shared ? 0 : size_t(pair) * gbytes);
    unsigned char* pair_base = smem_raw + kHeaderBytes + (b.graph_shared ? 1 : kSweepWarps) * gbytes +
                               size_t(pair) * pair_bytes(maxP, stages);
    GraphSmem gs = carve_graph(graph_base, maxP);
    gs.groups = reinterpret_cast<uint32_t*>(gs.far + (b.max_far_edges ? b.max_far_edges : 1));
    const PairSmem s = carve_pair(pair_base, maxP, stages);

    if (warp == 0) tmem_alloc(tmem_slot, kTmemColumns);
    // `empty` collects both trailing roles (post and far): 64 arrivals; the others 32
    if (threadIdx.x < kRingBarriers) mbar_init(&bars[threadIdx.x], (threadIdx.x % (3 * kMaxStages)) >= 2 * kMaxStages ? 64 : 32);
    if (threadIdx.x < kSweepWarps) reinterpret_cast<uint32_t*>(bars + kRingBarriers)[threadIdx.x] = 0u;
    if (b.graph_shared) load_graph(gs, b.layer_graphs[0], threadIdx.x, kLayeredThreads);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = *tmem_slot;
    // this pair's lane quarter: bits 31..16 of a TMEM address are the lane, 15..0 the column
    const uint32_t tm = tmem_base + ((pair * 32u) << 16);
    RingCursor cursor;
    uint32_t chunk_seq = 0;  // chunks this role has finished, over the whole kernel

    // tiles are dealt round-robin: CTA c, pair w, round r -> tile c + grid*(w + 4r)
    for (uint32_t tile = blockIdx.x + gridDim.x * pair; tile < b.n_tiles; tile += gridDim.x * kSweepWarps) {
        const DevLayerGraph g = b.layer_graphs[b.tile_model[tile]];
        if (!b.graph_shared) {
            // the three warps of the pair use the pair's graph copy: the sweep warp loads it
            if (role == 0) load_graph(gs, g, lane, 32);
            asm volatile("bar.sync %0, 128;" ::"r"(pair + 1) : "memory");
        }
        if (role == 1) {
            producer_warp(b, sweeps, lane, gs, s, full, empty, cursor, stages, tile, g.per_layer, g.layers);
        } else if (role == 2) {
            post_warp<WAIT>(b, sweeps, lane, s, bar_id, empty, cursor, stages, tile, tm, g.per_layer, g.layers);
        } else if (role == 3) {
            far_warp(b.hs + size_t(tile) * b.n_spins * 32 + lane, sweeps, lane, gs, s, bar_id, empty, far_done, chunk_seq,
                     cursor, stages, tm, g.per_layer,
                     g.layers);
        } else {
            sweep_warp<EXP>(b, sweeps, lane, gs, s, full, bar_id, smem_u32(far_done), chunk_seq, cursor, stages, tile, tm,
                            g.per_layer, g.layers);
        }
        if (!b.graph_shared) asm volatile("bar.sync %0, 128;" ::"r"(pair + 1) : "memory");
    }

    if (role != 1) {  // the roles that touch Tensor Memory
        tmem_wait_ld();
        tmem_wait_st();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, kTmemColumns);
}

}  // namespace

// Ring depth: 8 stages when they fit, otherwise 4 (multi-model batches keep a graph copy per pair).
static uint32_t pick_stages(uint32_t per_layer, uint32_t max_far_edges, uint32_t max_groups, bool graph_shared,
                            size_t* bytes_out) {
    for (uint32_t stages : {8u, 4u, 2u}) {
        const size_t bytes = kHeaderBytes + (graph_shared ? 1 : kSweepWarps) * graph_bytes(per_layer, max_far_edges, max_groups) +
                             kSweepWarps * pair_bytes(per_layer, stages);
        if (bytes <= 227 * 1024) {
            *bytes_out = bytes;
            return stages;
        }
    }
    *bytes_out = 0;
    return 0;
}

size_t layered_smem_bytes(uint32_t per_layer, uint32_t max_far_edges, uint32_t max_groups, bool graph_shared) {
    if (per_layer == 0 || per_layer > kTmemColumns || per_layer % kUnroll != 0) return 0;
    size_t bytes = 0;
    pick_stages(per_layer, max_far_edges, max_groups, graph_shared, &bytes);
    return bytes;
}

uint32_t layered_stage_count(uint32_t per_layer, uint32_t max_far_edges, uint32_t max_groups, bool graph_shared) {
    size_t bytes = 0;
    return pick_stages(per_layer, max_far_edges, max_groups, graph_shared, &bytes);
}

namespace {
template <int EXP, bool WAIT>
cudaError_t prepare_one(size_t smem_bytes) {
    cudaError_t e = cudaFuncSetAttribute(sweep_layered_kernel<EXP, WAIT, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_bytes));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(sweep_layered_kernel<EXP, WAIT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(smem_bytes));
}
template <int EXP, bool SPREAD>
void launch_one(const DevBatch& b, uint32_t sweeps, dim3 grid, size_t smem, cudaStream_t stream) {
    // the wait-statistics variant is a separate instantiation: the default kernel carries none of it
    if (b.wait_counts != nullptr) {
        sweep_layered_kernel<EXP, true, SPREAD><<<grid, kLayeredThreads, smem, stream>>>(b, sweeps);
    } else {
        sweep_layered_kernel<EXP, false, SPREAD><<<grid, kLayeredThreads, smem, stream>>>(b, sweeps);
    }
}
template <int EXP>
void launch_either(const DevBatch& b, uint32_t sweeps, dim3 grid, size_t smem, cudaStream_t stream) {
    // at most two tiles per CTA: the producers move to the idle schedulers (see the kernel)
    if (b.n_tiles <= 2u * grid.x) launch_one<EXP, true>(b, sweeps, grid, smem, stream);
    else launch_one<EXP, false>(b, sweeps, grid, smem, stream);
}
}  // namespace

// The attribute is per function and context, shared by every live batch: it is always set to the
// largest size any batch can ask for (227 KB, the opt-in maximum), never to one batch's own need,
// so creating a batch with a small layer graph cannot take shared memory away from a large one.
cudaError_t prepare_layered_kernels(size_t smem_bytes) {
    if (smem_bytes > 227 * 1024) return cudaErrorInvalidValue;
    smem_bytes = 227 * 1024;
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = prepare_one<kExpExact, false>(smem_bytes);
    if (e == cudaSuccess) e = prepare_one<kExpExact, true>(smem_bytes);
    if (e == cudaSuccess) e = prepare_one<kExpFast, false>(smem_bytes);
    if (e == cudaSuccess) e = prepare_one<kExpFast, true>(smem_bytes);
    if (e == cudaSuccess) e = prepare_one<kExpAccurate, false>(smem_bytes);
    if (e == cudaSuccess) e = prepare_one<kExpAccurate, true>(smem_bytes);
    return e;
}

cudaError_t launch_sweep_layered(const DevBatch& b, uint32_t sweeps, int sm_count, cudaStream_t stream) {
    const size_t smem = size_t(b.layered_smem);
    const uint32_t ctas = uint32_t(sm_count) < b.n_tiles ? uint32_t(sm_count) : b.n_tiles;
    const dim3 grid(ctas ? ctas : 1);
    switch (b.exp_kind) {
        case kExpExact: launch_either<kExpExact>(b, sweeps, grid, smem, stream); break;
        case kExpFast: launch_either<kExpFast>(b, sweeps, grid, smem, stream); break;
        default: launch_either<kExpAccurate>(b, sweeps, grid, smem, stream); break;
    }
    return cudaGetLastError();
}

}  // namespace isingb200
