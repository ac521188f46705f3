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

constexpr int kSliceWarps = 4;                    // warps per CTA (one batch each)
constexpr int kBoxH = 32 + 2 * kSliceMaxK;        // box rows: the tile and a K-cell frame
constexpr int kBoxW = kBoxH + 1;                  // odd row pitch: rows fall on different banks
constexpr int kBoxWords = kBoxW * kBoxH;
constexpr int kSliceChunk = 16;                   // halo loads in flight per lane
constexpr int kSliceLag = 2;                      // tiles of loads in flight ahead of their use
constexpr int kSliceMaxM = 4;                     // halo slots a lane advances per step (<= 128 / 32)
constexpr int kSliceDirMax = 32;                  // slots per neighbouring tile (host-checked)

// The λ walk's batches: up to 32 consecutive tile ordinals inside one tile row of the shard
// [tile_begin, tile_end): the first (possibly partial) row, whole rows, a last partial row.
struct SliceBatches {
    uint32_t row0, col0, cols0, nb0;  // first row: columns [col0, col0 + cols0), nb0 batches
    uint32_t mid_rows, nb_row;        // whole rows after it, batches per whole row
    FastDiv div_nb_row;
    uint32_t last_cols;               // then columns [0, last_cols) of one more row
    uint32_t total;                   // batches
    int K;                            // steps per pass, 1..8
};

// One step of a cell position of 32 tiles: its word and the 8 neighbouring words of the box.
template <bool CONWAY>
__device__ __forceinline__ uint32_t sliced_cell_step(const uint32_t* c, uint32_t birth, uint32_t survive) {
    return life_rule(c[-kBoxW - 1], c[-kBoxW], c[-kBoxW + 1], c[-1], c[1], c[kBoxW - 1], c[kBoxW], c[kBoxW + 1],
                     c[0], CONWAY ? (1u << 3) : birth, CONWAY ? (1u << 2) | (1u << 3) : survive);
}

#ifndef NBB_SLICE_MINB  // resident CTAs per SM the register budget is cut for (tuning builds)
#define NBB_SLICE_MINB 4
#endif
template <bool CONWAY, bool P2P, bool BB>
__global__ void __launch_bounds__(32 * kSliceWarps, NBB_SLICE_MINB) ca_compact_sliced_kernel(CompactCaArgs a, SliceBatches sb,
                                                                              FastDiv div_hb,
                                                                              const int32_t* __restrict__ nbr_tab,
                                                                              P2PArgs p) {
    static_assert(!(P2P && BB), "the multi-GPU pass walks the λ orthotope");
    const uint32_t birth = a.birth, survive = a.survive;
    __shared__ uint32_t s_box[kSliceWarps][kBoxWords];
    __shared__ uint32_t s_hmask[kSliceWarps][kSliceSlots];  // slot s exists in tile t: bit t
    __shared__ uint2 s_dir[8][kSliceDirMax];                 // per neighbouring tile: (offset in it, slot)
    __shared__ uint16_t s_bidx[kSliceSlots];                 // box index of every slot
    __shared__ uint16_t s_pos[256];
    __shared__ uint16_t s_tb[256];                           // box index of tile cell li
    __shared__ uint32_t s_list[kSliceWarps][32];             // BB: the batch's tile ordinals
    __shared__ const long long* s_peer[kMaxP2P];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t* box = s_box[wib];
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
        s_pos[i] = (uint16_t)pos;
        s_tb[i] = (uint16_t)(((pos >> 5) + kSliceMaxK) * kBoxW + (pos & 31u) + kSliceMaxK);
    }
    for (int i = lane; i < kBoxWords; i += 32) box[i] = 0u;
    if (P2P && p.wait_target != 0u) {
        // the arrival wait (this rank's own previous pass is among the arrivals); the first pass
        // of every call also waits for its predecessor grid (whatever last wrote the state)
        if (threadIdx.x == 0) p2p_wait(p);
        if (p.first_pass) pdl_wait();
    } else {
        pdl_wait();
    }
    __syncthreads();
    // the lane's tile cells li = 32k + lane (loads, stores): byte offset in a tile's sub-block;
    // the cells it advances in the steps: the (32k + lane)-th member in row-major order, so the
    // 32 lanes' box words of one access fall on (nearly) distinct banks
    uint32_t off[8], cb[8];
    {
        uint32_t y = 0, seen = 0;  // walk the rows to the lane's first member
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t li = 32u * k + lane;
            const bool ok = li < 243u;
            const uint32_t row = ok ? li / 27u : 0u, col = ok ? li % 27u : 0u;
            off[k] = 8u * (row * a.W + col);
            const uint32_t c = ok ? li : 0u;  // the c-th member, row-major
            while (seen + (1u << __popc(y)) <= c) seen += 1u << __popc(y++);
            const uint32_t x = pdep32(c - seen, y);
            cb[k] = (y + kSliceMaxK) * kBoxW + x + kSliceMaxK;
        }
    }
    const bool k7 = lane < 19;  // slot k = 7 holds li < 243 for lanes 0..18
    const uint32_t nwarps = gridDim.x * kSliceWarps, warp_global = blockIdx.x * kSliceWarps + wib;
    auto tile_base = [&](uint32_t t) -> uint32_t {  // element offset of tile t's sub-block
        const uint32_t wxb = fastdiv(t, div_hb), wyb = t - wxb * a.Hb;
        return 9u * wxb * a.W + 27u * wyb;
    };

    // One batch: lane t < cnt holds tile ordinal u; base0 = element offset of tile 0 (λ walk:
    // tile t at base0 + 27 t).
    auto batch = [&](uint32_t u, uint32_t cnt, uint32_t base0) {
        // ---- tile words: w[k] bit t = cell li = 32k + lane of tile t is alive ----------------
        // Software-pipelined over the batch's tiles: tile t's 8 loads are issued kSliceLag tiles
        // before they are folded into the words (bits of tiles >= cnt are never stored).
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = 0u;
        const uint64_t tbase = (BB && lane < cnt) ? 8ull * tile_base(u) : 0ull;  // BB: per tile
        {
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
        }
        // ---- halo words: lane t gathers tile t's halo cell of each slot, a ballot makes the word
        int32_t nbr[8];
        {
            int4 n0 = make_int4(-1, -1, -1, -1), n1 = n0;
            if (lane < cnt) {
                n0 = __ldg(reinterpret_cast<const int4*>(nbr_tab + 8ull * u));
                n1 = __ldg(reinterpret_cast<const int4*>(nbr_tab + 8ull * u) + 1);
            }
            nbr[0] = n0.x; nbr[1] = n0.y; nbr[2] = n0.z; nbr[3] = n0.w;
            nbr[4] = n1.x; nbr[5] = n1.y; nbr[6] = n1.z; nbr[7] = n1.w;
        }
#pragma unroll
        for (int d = 0; d < 8; ++d) {
            if (d == 2 || d == 5) continue;  // the (+1,-1) and (-1,+1) tiles hold no halo cell
            const bool ex = nbr[d] >= 0;
            const long long* src = a.src;
            uint32_t nb = 0;
            if (ex) {
                nb = tile_base((uint32_t)nbr[d]);
                if (P2P) src = s_peer[fastdiv((uint32_t)nbr[d], p.div_chunk)];
            }
            const char* P = reinterpret_cast<const char*>(src) + 8ull * nb;
            const uint32_t dm = __ballot_sync(0xFFFFFFFFu, ex);
            const int ns = c_sslots.dir_upto[d][K];
            for (int j0 = 0; j0 < ns; j0 += kSliceChunk) {  // kSliceChunk loads in flight, then ballots
                long long v[kSliceChunk];
#pragma unroll
                for (int c = 0; c < kSliceChunk; ++c) {
                    v[c] = 0;
                    if (ex && j0 + c < ns) {
                        const long long* q = reinterpret_cast<const long long*>(P + s_dir[d][j0 + c].x);
                        if (P2P)
                            asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v[c]) : "l"(q));
                        else
                            v[c] = __ldg(q);
                    }
                }
#pragma unroll
                for (int c = 0; c < kSliceChunk; ++c) {
                    if (j0 + c < ns) {
                        const uint32_t hw = __ballot_sync(0xFFFFFFFFu, v[c] != 0ll) & dm;
                        if (lane == 0) {
                            const uint32_t sl = s_dir[d][j0 + c].y;
                            box[s_bidx[sl]] = hw;
                            s_hmask[wib][sl] = dm;
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < 7 || k7) box[s_tb[32 * k + lane]] = w[k];
        __syncwarp();
        // ---- K steps: tile cells and the halo slots of layer <= K - j ------------------------
        for (int j = 1; j <= K; ++j) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < 7 || k7) w[k] = sliced_cell_step<CONWAY>(box + cb[k], birth, survive);
            const int ns = c_sslots.upto[K - j];
            uint32_t hn[kSliceMaxM];
#pragma unroll
            for (int m = 0; m < kSliceMaxM; ++m) {
                const int s = lane + 32 * m;
                hn[m] = 0u;
                if (s < ns) hn[m] = sliced_cell_step<CONWAY>(box + s_bidx[s], birth, survive) & s_hmask[wib][s];
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < 7 || k7) box[cb[k]] = w[k];
#pragma unroll
            for (int m = 0; m < kSliceMaxM; ++m) {
                const int s = lane + 32 * m;
                if (s < ns) box[s_bidx[s]] = hn[m];
            }
            __syncwarp();
        }
        // the lane's cells in load order again
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = (k < 7 || k7) ? box[s_tb[32 * k + lane]] : 0u;
        // ---- store: cell li of tile t = bit t of w[k] --------------------------------------
        {
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
        }
    };

    if constexpr (!BB) {
        for (uint32_t b = warp_global; b < sb.total; b += nwarps) {
            uint32_t row, c0, cnt;
            if (b < sb.nb0) {
                row = sb.row0;
                c0 = sb.col0 + 32u * b;
                cnt = min(32u, sb.col0 + sb.cols0 - c0);
            } else {
                const uint32_t b2 = b - sb.nb0, q = fastdiv(b2, sb.div_nb_row);
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
            batch(row * a.Hb + c0 + (uint32_t)lane, cnt, 9u * row * a.W + 27u * c0);
        }
    } else {
        // the warps scan the (n/32)^2 box tiles in windows of 32, window i by warp i mod nwarps
        // (interleaved: box rows hold 2^popc(by) member tiles, so contiguous ranges would not
        // balance); a box tile holds members iff bx ⊆ by — the reference's threads of the other
        // tiles all fail their membership test
        const uint32_t nbox = (uint32_t)(a.n >> 5), lg = 31u - __clz(nbox), boxes = nbox * nbox;
        uint32_t* list = s_list[wib];
        auto tile_of_box = [&](uint32_t bi) -> uint32_t {  // λ⁻¹ at block level
            const uint32_t bx = bi & (nbox - 1u), by = bi >> lg;
            const uint32_t wx = bits_base3(even_bits(bx)) + bits_base3(even_bits(by));
            const uint32_t wy = bits_base3(even_bits(bx >> 1)) + bits_base3(even_bits(by >> 1));
            return wx * a.Hb + wy;
        };
        uint32_t filled = 0;
        for (uint32_t b = 32u * warp_global; b < boxes; b += 32u * nwarps) {
            const uint32_t bi = b + (uint32_t)lane;
            const bool m = bi < boxes && ((bi & (nbox - 1u)) & ~(bi >> lg)) == 0u;
            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, m), nm = __popc(bal);
            const uint32_t rank = __popc(bal & ((1u << lane) - 1u));
            if (m && filled + rank < 32u) list[filled + rank] = tile_of_box(bi);
            if (filled + nm >= 32u) {
                __syncwarp();
                batch(list[lane], 32u, 0u);
                __syncwarp();
                if (m && filled + rank >= 32u) list[filled + rank - 32u] = tile_of_box(bi);
                filled = filled + nm - 32u;
            } else {
                filled += nm;
            }
        }
        __syncwarp();
        if (filled) batch(lane < (int)filled ? list[lane] : 0u, filled, 0u);
    }
    if (P2P) p2p_arrive(p);
}

}  // namespace nbbgpu
