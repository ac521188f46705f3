// compact_sliced.cuh — up to 8 CA steps per pass over the compact state, 32 tiles per warp
// bit-sliced ACROSS tiles.
//
// The reference steps the whole grid once per call (run_ca, dispatch.cpp:517-557: step i reads
// buffer i & 1, writes the other). One step over the compact state is one HBM pass (8 B read +
// 8 B write per member), so the pass is temporally blocked (as in compact_pass.cuh) — and the
// blocking is cheap enough here to go to K = 8 steps per pass:
//
// A warp takes a BATCH of up to 32 ρ = 32 tiles and holds the state as 32-bit words, one per
// cell position of the tile (and of its halo), bit t = that cell in tile t of the batch. Every
// tile has the same member pattern (x ⊆ y), so one word operation advances the same cell of 32
// tiles: a CA step of the batch is one bit-sliced adder tree per member position (243 tile
// cells + the halo slots still needed), with the 8 neighbours read from a per-warp "box" of
// words in shared memory (the 32 x 32 tile plus a K-cell frame, 48 x 48 words; non-member
// positions stay 0). 1024 cells advance per warp instruction, all of them members — the row
// bit-slicing of compact_pass.cuh spends 3/4 of its lanes on the empty half of the tile box.
//
// Words in and out: lane l owns the tile cells li = 32k + l (k = 0..7; the tile's 9 x 27
// compact sub-block read in its own row-major order, so a warp's loads of one tile are
// coalesced). λ batches are consecutive tile ordinals inside one tile row — adjacent compact
// sub-blocks — so tile t of the batch is 216 B after tile t-1 and every load and store is a
// register + immediate address. Halo: the member cells outside a tile that reach it within K
// steps, 8 / 22 / 36 / 58 / 76 / 104 / 128 / 166 positions for K = 1..8 (nbbhost::slice_slots,
// grouped by the neighbouring tile they lie in); lane t gathers tile t's halo cell, one ballot
// makes the slot's word. Step j advances the tile cells and the halo slots of layer <= K - j
// (a slot is needed only while its layer in THIS tile's neighbourhood is <= K - j; slots
// computed beyond that may be stale but feed nothing that is needed — DESIGN.md §4).
//
// Walks: λ (batches of the orthotope's tile order, this shard's range), BB (every warp scans a
// contiguous range of the (n/32)^2 box tiles, culls non-member tiles and batches the members,
// each addressed through λ⁻¹ of its block coordinates) and P2P (the λ walk whose halo cells in
// other ranks' tiles are read from their buffers over NVLink; the flag barrier of
// compact_kernels.cuh orders the passes).
#pragma once

#include "compact_kernels.cuh"
#include "nbb_host.hpp"

namespace nbbgpu {

using nbbhost::kSliceMaxK;
using nbbhost::kSliceSlots;
using nbbhost::SliceSlots;
__constant__ SliceSlots c_sslots;

constexpr int kSlicePipes = 2;                    // loader/stepper pipelines per CTA
constexpr int kSliceWarps = 2 * kSlicePipes;      // warps per CTA
constexpr int kBoxH = 32 + 2 * kSliceMaxK;        // box rows: the tile and a K-cell frame
constexpr int kBoxW = kBoxH + 1;                  // odd row pitch: rows fall on different banks
constexpr int kBoxWords = kBoxW * kBoxH;
constexpr int kSliceChunk = 16;                   // halo loads in flight per lane
constexpr int kSliceLag = 1;                      // tiles of loads in flight ahead of their use
constexpr int kSliceMaxM = 4;                     // halo slots a lane advances per step (<= 128 / 32)
constexpr int kSliceDirMax = 30;                  // slots per neighbouring tile (host-checked)

// The λ walk's batches: up to 32 consecutive tile ordinals inside one tile row of the shard
// [tile_begin, tile_end): the first (possibly partial) row, whole rows, a last partial row.
struct SliceBatches {
    uint32_t row0, col0, cols0, nb0;  // first row: columns [col0, col0 + cols0), nb0 batches
    uint32_t mid_rows, nb_row;        // whole rows after it, batches per whole row
    FastDiv div_nb_row;
    uint32_t last_cols;               // then columns [0, last_cols) of one more row
    uint32_t total;                   // batches
    int K;                            // steps per pass, 1..8
    RuleTab rule;                     // the rule's mux-tree constants (generic-rule instantiation)
};

// One step of a cell position of 32 tiles: its word and the 8 neighbouring words of the box
// (B3/S23 constant-folded; any other rule through its RuleTab, a kernel parameter).
template <bool CONWAY, int BW = kBoxW>
__device__ __forceinline__ uint32_t sliced_cell_step(const uint32_t* c, const RuleTab& rt) {
    if constexpr (CONWAY)
        return life_rule(c[-BW - 1], c[-BW], c[-BW + 1], c[-1], c[1], c[BW - 1], c[BW], c[BW + 1], c[0], 1u << 3,
                         (1u << 2) | (1u << 3));
    else
        return life_rule_tab(c[-BW - 1], c[-BW], c[-BW + 1], c[-1], c[1], c[BW - 1], c[BW], c[BW + 1], c[0], rt);
}

// K steps of a batch in its box: the tile's member positions (lane: members 32k + lane in
// row-major order, box index table cb) and the halo slots of layer <= K - j at step j (slot
// lane + 32m, box index table bidx, existence mask hmask); then the lane's tile words (cells
// li = 32k + lane, box index table tb) into w.
template <bool CONWAY>
__device__ __forceinline__ void sliced_steps(uint32_t* box, const uint32_t* hmask, int K, const uint16_t* cb,
                                             const uint16_t* bidx, const uint16_t* tb, const RuleTab& rt,
                                             uint32_t (&w)[8]) {
    const int lane = threadIdx.x & 31;
    const bool k7 = lane < 19;  // member / cell 32 * 7 + lane < 243
    __syncwarp();
    for (int j = 1; j <= K; ++j) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < 7 || k7) w[k] = sliced_cell_step<CONWAY>(box + cb[32 * k + lane], rt);
        const int ns = c_sslots.upto[K - j];
        uint32_t hn[kSliceMaxM];
#pragma unroll
        for (int m = 0; m < kSliceMaxM; ++m) {
            const int s = lane + 32 * m;
            hn[m] = 0u;
            if (s < ns) hn[m] = sliced_cell_step<CONWAY>(box + bidx[s], rt) & hmask[s];
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < 7 || k7) box[cb[32 * k + lane]] = w[k];
#pragma unroll
        for (int m = 0; m < kSliceMaxM; ++m) {
            const int s = lane + 32 * m;
            if (s < ns) box[bidx[s]] = hn[m];
        }
        __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = (k < 7 || k7) ? box[tb[32 * k + lane]] : 0u;
}

// Named barriers of the loader / stepper hand-off (64 threads: the pipeline's two warps). Stage b
// (b = batch index & 1) is FULL once the loader stored the batch's tile words, EMPTY once the
// stepper copied them into its box. Compile-time ids (ptxas then reserves 9 barriers per CTA; a
// runtime id reserves all 16 and the SM's barrier pool caps the resident CTAs): pipeline p uses
// FULL 1 + 4p + b and EMPTY 3 + 4p + b.
template <int ID>
__device__ __forceinline__ void nb_sync() { asm volatile("bar.sync %0, 64;" ::"n"(ID) : "memory"); }
template <int ID>
__device__ __forceinline__ void nb_arrive() { asm volatile("bar.arrive %0, 64;" ::"n"(ID) : "memory"); }
template <bool SYNC>
__device__ __forceinline__ void nb_op(int id) {
    switch (id) {
#define NBB_NB_CASE(I) \
    case I:            \
        if (SYNC) nb_sync<I>(); else nb_arrive<I>(); break;
        NBB_NB_CASE(1) NBB_NB_CASE(2) NBB_NB_CASE(3) NBB_NB_CASE(4)
        NBB_NB_CASE(5) NBB_NB_CASE(6) NBB_NB_CASE(7) NBB_NB_CASE(8)
#undef NBB_NB_CASE
        default: break;
    }
}
__device__ __forceinline__ int nb_full(int pipe, int b) { return 1 + 4 * pipe + b; }
__device__ __forceinline__ int nb_empty(int pipe, int b) { return 3 + 4 * pipe + b; }
static_assert(kSlicePipes * 4 + 1 <= 16, "named barriers");

// Bulk (TMA) copies for the λ loader: a group of kTmaTiles consecutive tiles of a batch is nine
// contiguous runs of 27·kTmaTiles values (one per compact row of the tiles' sub-blocks), each
// fetched by one cp.async.bulk into shared memory (16-byte aligned: the run starts one value
// early when its first value sits at an odd index), completion counted on an mbarrier.
#ifndef NBB_SLICE_TMA  // λ loader: bulk copies (1) or register-staged loads (0; tuning builds)
#define NBB_SLICE_TMA 1
#endif
constexpr bool kSliceTma = NBB_SLICE_TMA != 0;
constexpr int kTmaTiles = 4;
constexpr int kTmaRowBytes = ((8 * (27 * kTmaTiles + 1)) + 15) / 16 * 16;  // 880
// dynamic shared memory of a launch: the λ loaders' staging buffers (BB and P2P-free BB: none)
constexpr size_t kSliceDynSmem = kSliceTma ? (size_t)kSlicePipes * 2 * 9 * kTmaRowBytes : 0;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* mb, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mb, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(mb)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mb) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(mb))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

#ifndef NBB_SLICE_MINB  // resident CTAs per SM the register budget is cut for (tuning builds)
#define NBB_SLICE_MINB 5
#endif
constexpr int kStageWords = 256;  // a batch's 243 tile words (loader -> stepper)
// CTA = kSlicePipes pipelines of two warps. The LOADER streams each batch's tile values from HBM
// (8 loads per lane per tile, one tile of loads in flight ahead of the folding) into the words of
// stage (i & 1); the STEPPER gathers the batch's halo words into its box, copies the stage's tile
// words in, frees the stage, advances K steps in place and stores the results, while the loader
// already fills the other stage. The pipelines walk the batches with a grid stride.
template <bool CONWAY, bool P2P, bool BB>
__global__ void __launch_bounds__(32 * kSliceWarps, NBB_SLICE_MINB)
    ca_compact_sliced_kernel(CompactCaArgs a, SliceBatches sb, FastDiv div_hb, const int32_t* __restrict__ nbr_tab,
                             P2PArgs p) {
    static_assert(!(P2P && BB), "the multi-GPU pass walks the λ orthotope");
    __shared__ uint32_t s_box[kSlicePipes][kBoxWords];
    __shared__ uint32_t s_stage[kSlicePipes][2][kStageWords]; // loader -> stepper tile words
    __shared__ uint32_t s_hmask[kSlicePipes][kSliceSlots];   // slot s exists in tile t: bit t
    __shared__ uint2 s_dir[8][kSliceDirMax];                 // per neighbouring tile: (offset in it, slot)
    __shared__ uint16_t s_bidx[kSliceSlots];                 // box index of every slot
    __shared__ uint16_t s_tb[256];                           // box index of tile cell li
    __shared__ uint16_t s_cb[256];                           // box index of the c-th member, row-major
    __shared__ uint32_t s_list[kSliceWarps][32];             // BB: [warp] the batch's tile ordinals
    __shared__ unsigned long long s_hp[kSlicePipes][6][33];  // stepper: halo tile pointers [direction][tile]
    __shared__ uint32_t s_hdm[kSlicePipes][6];               // stepper: halo tiles present [direction]
    __shared__ const long long* s_peer[kMaxP2P];
    extern __shared__ __align__(16) unsigned char s_dyn[];  // λ loader staging [pipe][2][9][kTmaRowBytes]
    auto s_tma = reinterpret_cast<unsigned char (*)[2][9][kTmaRowBytes]>(s_dyn);
    __shared__ __align__(8) uint64_t s_mbar[kSlicePipes][2];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int pipe = wib >> 1;
    const bool loader = (wib & 1) == 0;
    const int K = sb.K;
    pdl_trigger();
    if (P2P && threadIdx.x < (unsigned)p.world) s_peer[threadIdx.x] = p.peer_src[threadIdx.x];
    for (int s = threadIdx.x; s < c_sslots.count; s += blockDim.x)
        s_bidx[s] = (uint16_t)((c_sslots.y[s] + kSliceMaxK) * kBoxW + c_sslots.x[s] + kSliceMaxK);
    for (int i = threadIdx.x; i < 8 * kSliceDirMax; i += blockDim.x) {
        const int d = i / kSliceDirMax, j = i % kSliceDirMax;
        uint2 e = make_uint2(0u, 0u);
        if (j < c_sslots.dir_upto[d][kSliceMaxK]) {
            const uint32_t s = c_sslots.by_dir[d][j], li = c_sslots.li[s];
            e = make_uint2(8u * ((li / 27u) * a.W + li % 27u), s);
        }
        s_dir[d][j] = e;
    }
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        const uint32_t pos = i < 243 ? c_local_pos[i] : 0u;
        s_tb[i] = (uint16_t)(((pos >> 5) + kSliceMaxK) * kBoxW + (pos & 31u) + kSliceMaxK);
    }
    for (int i = threadIdx.x; i < kSlicePipes * kBoxWords; i += blockDim.x) (&s_box[0][0])[i] = 0u;
    if (!BB && threadIdx.x < 2 * kSlicePipes) mbar_init(&s_mbar[threadIdx.x >> 1][threadIdx.x & 1], 1u);
    if (!BB) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (P2P && p.wait_target != 0u) {
        // the arrival wait (this rank's own previous pass is among the arrivals); the first pass
        // of every call also waits for its predecessor grid (whatever last wrote the state)
        if (threadIdx.x == 0) p2p_wait(p);
        if (p.first_pass) pdl_wait();
    } else {
        pdl_wait();
    }
    __syncthreads();
    // every thread (not only the poller) orders its peer reads after the arrivals it waited for:
    // the poller's ld.acquire.sys synchronises with the peers' fence.acq_rel.sys + red.relaxed.sys,
    // bar.sync carries that to the CTA, and this fence makes each thread's own later ld.relaxed.sys
    // of peer memory observe it at system scope
    if (P2P && p.wait_target != 0u) {
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");  // before the λ loader's bulk copies
    }
    // the lane's tile cells li = 32k + lane (loads, stores): byte offset in a tile's sub-block
    // (recomputed per batch: short register lifetimes); the cells it advances in the steps: the
    // (32k + lane)-th member in row-major order, so the 32 lanes' box words of one access fall on
    // (nearly) distinct banks (box index table s_cb, built once)
    {
        uint32_t y = 0, seen = 0;
        for (uint32_t c = threadIdx.x; c < 243u; c += blockDim.x) {
            while (seen + (1u << __popc(y)) <= c) seen += 1u << __popc(y++);
            s_cb[c] = (uint16_t)((y + kSliceMaxK) * kBoxW + pdep32(c - seen, y) + kSliceMaxK);
        }
    }
    __syncthreads();
    auto tile_offsets = [&](uint32_t* off) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t li = min(32u * k + lane, 242u);
            off[k] = 8u * ((li / 27u) * a.W + li % 27u);
        }
    };
    const bool k7 = lane < 19;  // slot k = 7 holds li < 243 for lanes 0..18
    auto tile_base = [&](uint32_t t) -> uint32_t {  // element offset of tile t's sub-block
        const uint32_t wxb = fastdiv(t, div_hb), wyb = t - wxb * a.Hb;
        return 9u * wxb * a.W + 27u * wyb;
    };

    // ---- loader: tile words of a batch into a stage (word li = cell li of the 32 tiles) --------
    // lane t < cnt holds tile ordinal u; base0 = element offset of tile 0 (λ: tile t at +27 t).
    auto load_batch = [&](uint32_t u, uint32_t cnt, uint32_t base0, uint32_t* stage) {
        uint32_t off[8];
        tile_offsets(off);
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = 0u;
        const uint64_t tbase = (BB && lane < (int)cnt) ? 8ull * tile_base(u) : 0ull;
        const char* P0 = reinterpret_cast<const char*>(a.src) + 8ull * base0;
        long long ring[kSliceLag + 1][8];
#pragma unroll
        for (int t = 0; t < 32 + kSliceLag; ++t) {
            if (t >= (int)cnt + kSliceLag) break;
            if (t < 32 && t < (int)cnt) {
                const char* P = P0 + 216u * t;  // λ: tile t of the batch follows tile t - 1
                if constexpr (BB) P = reinterpret_cast<const char*>(a.src) + __shfl_sync(0xFFFFFFFFu, tbase, t);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    ring[t % (kSliceLag + 1)][k] =
                        (k < 7 || k7) ? __ldg(reinterpret_cast<const long long*>(P + off[k])) : 0ll;
            }
            if (t >= kSliceLag) {
                const int tc = t - kSliceLag;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const long long v = ring[tc % (kSliceLag + 1)][k];
                    const uint32_t nz = (uint32_t)v | (uint32_t)((unsigned long long)v >> 32);
                    w[k] |= min(nz, 1u) << tc;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < 7 || k7) stage[32 * k + lane] = w[k];
    };

    // ---- stepper: halo words, K steps, stores ---------------------------------------------------
    // Halo words, one neighbouring tile direction at a time (the 6 directions that hold halo
    // cells: 0,1,3,4,6,7): lane j owns slot j of the direction's list; for each of the 32 tiles of
    // the batch it loads that slot's value from the tile's neighbour (all 32 loads in flight, then
    // folded into the slot's word, bit t). A warp load thus reads the slots of ONE neighbour tile —
    // a few sectors of its sub-block — instead of one scattered value per tile.
    auto halo_batch = [&](uint32_t u, uint32_t cnt, uint32_t* box, uint32_t* hmask) {
#ifdef NBB_EXP_NOHALO
        return;
#endif
        // lane t: the neighbouring tiles of tile t -> base pointers (0: no member tile there; bit 0:
        // another rank's buffer)
        {
            int4 n0 = make_int4(-1, -1, -1, -1), n1 = n0;
            if (lane < (int)cnt) {
                n0 = __ldg(reinterpret_cast<const int4*>(nbr_tab + 8ull * u));
                n1 = __ldg(reinterpret_cast<const int4*>(nbr_tab + 8ull * u) + 1);
            }
            const int32_t nbr6[6] = {n0.x, n0.y, n0.w, n1.x, n1.z, n1.w};  // directions 0,1,3,4,6,7
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                const bool ex = nbr6[q] >= 0;
                unsigned long long ptr = 0ull;
                if (ex) {
                    const uint32_t own = P2P ? fastdiv((uint32_t)nbr6[q], p.div_chunk) : 0u;
                    const long long* src = P2P ? s_peer[own] : a.src;
                    ptr = reinterpret_cast<unsigned long long>(src) + 8ull * tile_base((uint32_t)nbr6[q]);
                    if (P2P && own != (uint32_t)p.rank) ptr |= 1ull;
                }
                s_hp[pipe][q][lane] = ptr;
                const uint32_t dm = __ballot_sync(0xFFFFFFFFu, ex);
                if (lane == 0) s_hdm[pipe][q] = dm;
            }
        }
        __syncwarp();
#pragma unroll 1
        for (int q = 0; q < 6; ++q) {
            const int d = q < 2 ? q : q < 4 ? q + 1 : q + 2;
            const int ns = c_sslots.dir_upto[d][K];
            if (ns == 0) continue;
            const bool mine = lane < ns;
            const uint2 e = mine ? s_dir[d][lane] : make_uint2(0u, 0u);
            long long v[32];
#pragma unroll
            for (int t = 0; t < 32; ++t) {
                v[t] = 0;
                const unsigned long long P = s_hp[pipe][q][t];  // broadcast
                if (mine && P != 0ull) {
                    const long long* qp = reinterpret_cast<const long long*>((P & ~1ull) + e.x);
                    if (P2P && (P & 1ull))  // a cell of another rank's tile: its buffer over NVLink
                        asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v[t]) : "l"(qp));
                    else
                        v[t] = __ldg(qp);
                }
            }
            uint32_t hw = 0u;
#pragma unroll
            for (int t = 0; t < 32; ++t) {
                const uint32_t nz = (uint32_t)v[t] | (uint32_t)((unsigned long long)v[t] >> 32);
                hw |= min(nz, 1u) << t;
            }
            if (mine) {
                const uint32_t dm = s_hdm[pipe][q];
                box[s_bidx[e.y]] = hw & dm;
                hmask[e.y] = dm;
            }
        }
    };
    auto step_batch = [&](uint32_t u, uint32_t cnt, uint32_t base0, uint32_t* box, const uint32_t* hmask) {
        uint32_t w[8];
        sliced_steps<CONWAY>(box, hmask, K, s_cb, s_bidx, s_tb, sb.rule, w);
        // cell li of tile t = bit t of w[k]
#ifdef NBB_EXP_NOSTORE
        if (w[0] != 0x12345u) return;
#endif
        uint32_t off[8];
        tile_offsets(off);
        const uint64_t tbase = (BB && lane < (int)cnt) ? 8ull * tile_base(u) : 0ull;
        char* Q0 = reinterpret_cast<char*>(a.dst) + 8ull * base0;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            if (t >= (int)cnt) break;
            char* Q = Q0 + 216u * t;
            if constexpr (BB) Q = reinterpret_cast<char*>(a.dst) + __shfl_sync(0xFFFFFFFFu, tbase, t);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < 7 || k7) *reinterpret_cast<long long*>(Q + off[k]) = (long long)((w[k] >> t) & 1u);
        }
    };

    // ---- the walk: batch i of a pipeline uses stage i & 1 --------------------------------------
    // Both warps of a pipeline enumerate the same batches. The loader waits for EMPTY before
    // refilling a stage (not for its first two batches) and arrives FULL; the stepper writes the
    // halo words of batch i into its box, waits for FULL, copies the tile words in and arrives
    // EMPTY only when the loader will wait for it (batch i + 2 exists).
    uint32_t* box = s_box[pipe];
    auto run = [&](uint32_t i, bool more2, uint32_t u, uint32_t cnt, uint32_t base0) {
        const int b = (int)(i & 1u);
        uint32_t* stage = s_stage[pipe][b];
        if (loader) {
            if (i >= 2) nb_op<true>(nb_empty(pipe, b));
            load_batch(u, cnt, base0, stage);
            __syncwarp();
            nb_op<false>(nb_full(pipe, b));
        } else {
            halo_batch(u, cnt, box, s_hmask[pipe]);
            nb_op<true>(nb_full(pipe, b));
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < 7 || k7) box[s_tb[32 * k + lane]] = stage[32 * k + lane];
            __syncwarp();
            if (more2) nb_op<false>(nb_empty(pipe, b));
            step_batch(u, cnt, base0, box, s_hmask[pipe]);
        }
    };
    const uint32_t pipe_global = blockIdx.x * kSlicePipes + (uint32_t)pipe;
    const uint32_t npipes = gridDim.x * kSlicePipes;
    if constexpr (!BB) {
        auto decode = [&](uint32_t bt, uint32_t& row, uint32_t& c0, uint32_t& cnt) {
            if (bt < sb.nb0) {
                row = sb.row0;
                c0 = sb.col0 + 32u * bt;
                cnt = min(32u, sb.col0 + sb.cols0 - c0);
            } else {
                const uint32_t b2 = bt - sb.nb0, q = fastdiv(b2, sb.div_nb_row);
                if (q < sb.mid_rows) {
                    row = sb.row0 + 1u + q;
                    c0 = 32u * (b2 - q * sb.nb_row);
                    cnt = min(32u, a.Hb - c0);
                } else {
                    row = sb.row0 + 1u + sb.mid_rows;
                    c0 = 32u * (b2 - sb.mid_rows * sb.nb_row);
                    cnt = min(32u, sb.last_cols - c0);
                }
            }
        };
        if (!loader || !kSliceTma) {
            uint32_t i = 0;
            for (uint32_t bt = pipe_global; bt < sb.total; bt += npipes, ++i) {
                uint32_t row, c0, cnt;
                decode(bt, row, c0, cnt);
                run(i, bt + 2u * npipes < sb.total, row * a.Hb + c0 + (uint32_t)lane, cnt, 9u * row * a.W + 27u * c0);
            }
        } else {
            // The λ loader: its batches as a stream of groups of kTmaTiles tiles; group g + 1 is
            // fetched by bulk copies (lane 0) into staging buffer (g + 1) & 1 while group g is folded
            // into the words, so a group (15.6 KB) is always in flight without holding registers.
            unsigned char (*tma)[9][kTmaRowBytes] = s_tma[pipe];
            uint64_t* mbar = s_mbar[pipe];
            const uint64_t total_elems = (uint64_t)a.W * (uint64_t)(a.tiles / a.Hb) * 9u;  // 3^r
            struct Group {
                uint32_t bt, q, base0, cnt;  // batch, group in batch, batch's element base, batch tiles
            };
            auto first_group = [&](uint32_t bt, Group& gr) -> bool {
                if (bt >= sb.total) return false;
                uint32_t row, c0, cnt;
                decode(bt, row, c0, cnt);
                gr = Group{bt, 0u, 9u * row * a.W + 27u * c0, cnt};
                return true;
            };
            // lane-0 work: the nine runs of group gr into staging buffer sbuf
            auto issue = [&](const Group& gr, int sbuf) {
                if (lane == 0) {
                    const uint32_t t0 = kTmaTiles * gr.q, nt = min((uint32_t)kTmaTiles, gr.cnt - t0);
                    uint32_t bytes[9], total = 0;
                    for (int r = 0; r < 9; ++r) {
                        const uint64_t e0 = (uint64_t)gr.base0 + (uint64_t)r * a.W + 27u * t0, sh = e0 & 1u;
                        uint64_t nb = (8u * (27u * nt + sh) + 15u) & ~15ull;
                        const uint64_t room = (8u * (total_elems - (e0 - sh))) & ~15ull;  // never past the array
                        bytes[r] = (uint32_t)(nb < room ? nb : room);
                        total += bytes[r];
                    }
                    mbar_expect_tx(&mbar[sbuf], total);
                    for (int r = 0; r < 9; ++r) {
                        const uint64_t e0 = (uint64_t)gr.base0 + (uint64_t)r * a.W + 27u * t0, sh = e0 & 1u;
                        bulk_g2s(tma[sbuf][r], a.src + (e0 - sh), bytes[r], &mbar[sbuf]);
                    }
                }
            };
            uint32_t g = 0;  // groups consumed so far (staging buffer g & 1, its use count g >> 1)
            Group cur;
            if (first_group(pipe_global, cur)) issue(cur, 0);
            uint32_t i = 0;
            for (uint32_t bt = pipe_global; bt < sb.total; bt += npipes, ++i) {
                const int b = (int)(i & 1u);
                if (i >= 2) nb_op<true>(nb_empty(pipe, b));
                uint32_t w[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) w[k] = 0u;
                const uint32_t ngroups = (cur.cnt + kTmaTiles - 1) / kTmaTiles;
                for (uint32_t q = 0; q < ngroups; ++q, ++g) {
                    Group nxt;
                    bool more;
                    if (q + 1 < ngroups) {
                        nxt = cur;
                        nxt.q = q + 1;
                        more = true;
                    } else {
                        more = first_group(bt + npipes, nxt);
                    }
                    if (more) issue(nxt, (int)((g + 1) & 1u));
                    const int sb_ = (int)(g & 1u);
                    mbar_wait(&mbar[sb_], (g >> 1) & 1u);
                    const uint32_t t0 = kTmaTiles * q, nt = min((uint32_t)kTmaTiles, cur.cnt - t0);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        if (k == 7 && !k7) continue;
                        const uint32_t li = 32u * k + lane, row = li / 27u, col = li % 27u;
                        const uint64_t e0 = (uint64_t)cur.base0 + (uint64_t)row * a.W + 27u * t0;
                        const uint32_t sh = (uint32_t)(e0 & 1u);
                        const uint64_t want = (uint64_t)(((8u * (27u * nt + sh) + 15u) & ~15u) / 8u);
                        const uint64_t room = (total_elems - (e0 - sh)) & ~1ull;
                        const uint32_t copied = (uint32_t)(want < room ? want : room);
                        const long long* rowp = reinterpret_cast<const long long*>(tma[sb_][row]);
#pragma unroll
                        for (int t = 0; t < kTmaTiles; ++t) {
                            if (t < (int)nt) {
                                const uint32_t idx = sh + 27u * t + col;
                                const long long v = idx < copied ? rowp[idx] : __ldg(a.src + e0 + 27u * t + col);
                                const uint32_t nz = (uint32_t)v | (uint32_t)((unsigned long long)v >> 32);
                                w[k] |= min(nz, 1u) << (t0 + t);
                            }
                        }
                    }
                    __syncwarp();
                    fence_proxy_async();  // the reads of this buffer before the next bulk copy into it
                    if (more && q + 1 == ngroups) cur = nxt;
                }
                uint32_t* stage = s_stage[pipe][b];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (k < 7 || k7) stage[32 * k + lane] = w[k];
                __syncwarp();
                nb_op<false>(nb_full(pipe, b));
            }
        }
    } else {
        // both warps scan the (n/32)^2 box tiles in windows of 32, window j by CTA j mod grid
        // (interleaved: box rows hold 2^popc(by) member tiles, so contiguous ranges would not
        // balance), and batch the member tiles in the same order; a box tile holds members iff
        // bx ⊆ by — the reference's threads of the other tiles all fail their membership test
        const uint32_t nbox = (uint32_t)(a.n >> 5), lg = 31u - __clz(nbox), boxes = nbox * nbox;
        auto tile_of_box = [&](uint32_t bi) -> uint32_t {  // λ⁻¹ at block level
            const uint32_t bx = bi & (nbox - 1u), by = bi >> lg;
            const uint32_t wx = bits_base3(even_bits(bx)) + bits_base3(even_bits(by));
            const uint32_t wy = bits_base3(even_bits(bx >> 1)) + bits_base3(even_bits(by >> 1));
            return wx * a.Hb + wy;
        };
        // the batches of this CTA: counted first (the stepper must know whether batch i + 2 exists)
        uint32_t members = 0;
        for (uint32_t bw = 32u * pipe_global; bw < boxes; bw += 32u * npipes) {
            const uint32_t bi = bw + (uint32_t)lane;
            members += __popc(__ballot_sync(0xFFFFFFFFu, bi < boxes && ((bi & (nbox - 1u)) & ~(bi >> lg)) == 0u));
        }
        const uint32_t nbatch = (members + 31u) / 32u;
        uint32_t filled = 0, i = 0;
        uint32_t* list = s_list[wib];
        for (uint32_t bw = 32u * pipe_global; bw < boxes; bw += 32u * npipes) {
            const uint32_t bi = bw + (uint32_t)lane;
            const bool m = bi < boxes && ((bi & (nbox - 1u)) & ~(bi >> lg)) == 0u;
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m), nm = __popc(bal);
            const uint32_t rank = __popc(bal & ((1u << lane) - 1u));
            if (m && filled + rank < 32u) list[filled + rank] = tile_of_box(bi);
            if (filled + nm >= 32u) {
                __syncwarp();
                run(i, i + 2u < nbatch, list[lane], 32u, 0u);
                ++i;
                __syncwarp();
                if (m && filled + rank >= 32u) list[filled + rank - 32u] = tile_of_box(bi);
                filled = filled + nm - 32u;
            } else {
                filled += nm;
            }
        }
        __syncwarp();
        if (filled) run(i, false, lane < (int)filled ? list[lane] : 0u, filled, 0u);
    }
    if (P2P) p2p_arrive(p);
}

}  // namespace nbbgpu
