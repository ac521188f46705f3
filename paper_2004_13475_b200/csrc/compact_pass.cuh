// compact_pass.cuh — K CA steps per pass over the compact (λ-ordered) state, K = 1..4.
//
// The reference steps the whole grid once per call of its kernel (run_ca, dispatch.cpp:517-557:
// step i reads buffer i & 1 and writes the other). On B200 one step over the compact state is
// one HBM pass (8 B read + 8 B write per member), so the pass is temporally blocked: a warp
// loads its ρ = 32 tile (243 values, a 9 x 27 compact sub-block) and the tile's radius-K halo
// once, advances the tile K steps on chip and stores only step t+K. The result is the same
// state the reference's K single steps produce (bit-exact; tests/test_gpu_*).
//
// Halo: the gasket's tiles touch only at their corners, so the member cells within chain
// distance K of a tile's members are few — 8 / 22 / 36 / 58 positions for K = 1..4, the
// prefix of the slot table built on the host (nbbhost::halo_slots: positions sorted by their
// layer d, d = 1 the one-step halo). Every slot lies in one of the tile's 8 neighbouring tiles
// at a fixed local position, so the per-level table holds just the 8 neighbour TILE ordinals
// per tile (-1: not a member tile), 32 B per tile; a slot's compact offset is that tile's base
// plus a per-slot constant. Lane l holds slots l and 32 + l.
//
// Per pass and tile: the tile's values -> bytes in a per-warp 32 x 32 tile -> row bit masks
// (lane = row); the halo values -> a 64-bit alive mask. Step j = 1..K: the tile advances one
// bit-sliced step (compact_rows_step, H_1 bits from the mask); the slots of layer <= K - j
// advance one scalar step (popcount of the adjacent slots' bits + the in-tile neighbours of
// H_1 cells, read from tile rows 0, 30, 31 by shuffles). A slot's value is needed only while
// its layer in THIS tile's neighbourhood is <= K - j; slots computed beyond that may be stale
// but feed nothing that is needed.
//
// One kernel serves the λ launch (the warps walk the orthotope's tile order, consecutive
// warps on adjacent compact sub-blocks), the bounding-box launch (BB: the warps walk all
// (n/32)^2 box tiles, cull the non-member ones and find a member tile's storage through λ⁻¹
// of its block coordinates) and the multi-GPU pass (P2P: halo values of other ranks' tiles
// read from their buffers over NVLink, a flag barrier in peer memory orders the passes).
#pragma once

#include "compact_kernels.cuh"
#include "nbb_host.hpp"

namespace nbbgpu {

using nbbhost::HaloSlots;
using nbbhost::kPassMaxK;
__constant__ HaloSlots c_slots;

// slots of a K-step pass (layers <= K); host-checked against nbbhost::halo_slots
__host__ __device__ constexpr int pass_slots(int k) { return k <= 0 ? 0 : k == 1 ? 8 : k == 2 ? 22 : k == 3 ? 36 : 58; }

// [tile u][8] the ordinals of the 8 neighbouring tiles (dy, dx) ∈ {-1,0,1}², centre skipped,
// -1 where the neighbour lies outside the grid or holds no member (bx' ⊄ by')
__global__ void compact_nbr_table_kernel(CompactCaArgs a, FastDiv div_hb, int32_t* tab) {
    const uint32_t nb = (uint32_t)(a.n >> 5);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (uint64_t)a.tiles * 8u;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = (uint32_t)(i >> 3), d = (uint32_t)i & 7u, d9 = d < 4u ? d : d + 1u;
        const uint32_t wxb = fastdiv(u, div_hb), wyb = u - wxb * a.Hb;
        uint32_t bx, by;
        lambda_arith(wxb, wyb, bx, by);
        const uint32_t qx = bx + d9 % 3u - 1u, qy = by + d9 / 3u - 1u;  // wraps below 0
        int32_t t = -1;
        if (qx < nb && qy < nb && (qx & qy) == qx) {
            const uint32_t wx = bits_base3(even_bits(qx)) + bits_base3(even_bits(qy));
            const uint32_t wy = bits_base3(even_bits(qx >> 1)) + bits_base3(even_bits(qy >> 1));
            t = (int32_t)(wx * a.Hb + wy);
        }
        tab[i] = t;
    }
}

// Tile cells the H_1 slots neighbour, gathered into one word: bit 0 = (0, 0), bit 30 = (0, 30),
// bit 31 = (0, 31) (column 0 of the row masks), bit 1 = (31, 31), bit 2 = (1, 31)
__device__ __forceinline__ uint32_t compact_edge_word(uint32_t R) {
    const uint32_t c0 = __ballot_sync(0xFFFFFFFFu, R & 1u);
    const uint32_t r31 = __shfl_sync(0xFFFFFFFFu, R, 31);
    return (c0 & 0xC0000001u) | ((r31 >> 30) & 2u) | ((r31 << 1) & 4u);
}

#ifndef NBB_PASS_MINB  // resident CTAs per SM the register budget is cut for (tuning builds)
#define NBB_PASS_MINB 3
#endif
template <int K, bool CONWAY, bool P2P, bool BB>
__global__ void __launch_bounds__(256, NBB_PASS_MINB) ca_compact_pass_kernel(CompactCaArgs a, FastDiv div_hb,
                                                                 const int32_t* __restrict__ nbr_tab,
                                                                 P2PArgs p) {
    static_assert(K >= 1 && K <= kPassMaxK, "1 <= K <= 4 steps per pass");
    static_assert(!(P2P && BB), "the multi-GPU pass walks the λ orthotope");
    constexpr int NS = pass_slots(K);
    constexpr int NR = (NS + 31) / 32;
    const uint32_t birth = CONWAY ? (1u << 3) : a.birth;
    const uint32_t survive = CONWAY ? (1u << 2) | (1u << 3) : a.survive;
    __shared__ __align__(16) uint8_t s_cell[8][32 * 32];
    __shared__ uint32_t s_new[8][32];
    __shared__ uint16_t s_pos[256];
    __shared__ const long long* s_peer[kMaxP2P];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint8_t* cell = s_cell[wib];
    pdl_trigger();
    if (P2P && threadIdx.x < (unsigned)p.world) s_peer[threadIdx.x] = p.peer_src[threadIdx.x];
    s_pos[threadIdx.x] = threadIdx.x < 243 ? c_local_pos[threadIdx.x] : 0;
    // per-lane slot constants: neighbour direction << 29 | offset inside that tile's sub-block
    // (0xFFFFFFFF: no slot) and, for the first 32 slots, the adjacent slots; the masks of slots
    // 32.. are needed once per tile (K = 4) and live in shared memory
    __shared__ uint2 s_nbm[32];
    uint32_t sdl[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const int s = 32 * r + lane;
        const uint32_t li = s < NS ? c_slots.li[s] : 0u;
        sdl[r] = s < NS ? (uint32_t)c_slots.dir[s] << 29 | ((li / 27u) * a.W + li % 27u) : 0xFFFFFFFFu;
    }
    const uint32_t nbl = lane < NS ? c_slots.nb_lo[lane] : 0u, nbh = lane < NS ? c_slots.nb_hi[lane] : 0u;
    if (NR > 1 && threadIdx.x < 32) {
        const int s = 32 + threadIdx.x;
        s_nbm[threadIdx.x] = s < NS ? make_uint2(c_slots.nb_lo[s], c_slots.nb_hi[s]) : make_uint2(0u, 0u);
    }
    // H_1 slots: in-tile neighbours as a mask over the edge word of compact_edge_word
    const uint32_t medge = lane < 8 ? (c_slots.m0[lane] & 1u) | (c_slots.m30[lane] & 1u) << 30 |
                                          (c_slots.m31[lane] & 1u) << 31 | (c_slots.m31[lane] >> 31) << 1 |
                                          ((c_slots.m31[lane] >> 1) & 1u) << 2
                                    : 0u;
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
    if (P2P && p.wait_target != 0u) asm volatile("fence.acq_rel.sys;" ::: "memory");
    // slot k of lane l = local index 32k + l: byte offset in the tile's sub-block | byte index
    // x | y << 5 in the 32 x 32 tile << 21 (offsets < 2^21 for W <= 3^9, i.e. r <= 18)
    uint32_t sl[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t li = 32u * k + lane;
        const bool ok = li < 243u;
        const uint32_t row = ok ? li / 27u : 0u, col = ok ? li % 27u : 0u;
        sl[k] = (row * a.W + col) * 8u | (uint32_t)s_pos[li] << 21;
    }
    const bool k7 = lane < 19;
#pragma unroll
    for (int i = 0; i < 8; ++i) reinterpret_cast<uint32_t*>(cell)[32 * i + lane] = 0u;
    const uint32_t warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t warp_stride = (gridDim.x * blockDim.x) >> 5;
    const char* src0 = reinterpret_cast<const char*>(a.src);
    char* dst0 = reinterpret_cast<char*>(a.dst);
    __syncwarp();

    // ---- the tile walk: t0 (computed now), t1 (loads in flight), t2 (table entry in flight)
    constexpr uint32_t kNone = 0xFFFFFFFFu;
    uint32_t wpos = 0;
    const uint32_t nbox = (uint32_t)(a.n >> 5), lg = 31u - __clz(nbox), boxes = nbox * nbox;
    const uint32_t ustride = (warp_stride | 1u) - ((warp_stride & 1u) ? 0u : 2u);  // odd (BB)
    auto next_member = [&](uint32_t bi) -> uint32_t {  // BB: first member box tile >= bi on the stride
        while (bi < boxes && ((bi & (nbox - 1u)) & (nbox - 1u - (bi >> lg))) != 0u) bi += ustride;
        return bi;
    };
    auto tile_of_box = [&](uint32_t bi) -> uint32_t {  // λ⁻¹ at block level
        const uint32_t bx = bi & (nbox - 1u), by = bi >> lg;
        const uint32_t wx = bits_base3(even_bits(bx)) + bits_base3(even_bits(by));
        const uint32_t wy = bits_base3(even_bits(bx >> 1)) + bits_base3(even_bits(by >> 1));
        return wx * a.Hb + wy;
    };
    auto advance = [&]() -> uint32_t {
        if constexpr (!BB) {
            wpos += warp_stride;
            return wpos < a.tile_end ? wpos : kNone;
        } else {
            wpos = next_member(wpos + ustride);
            return wpos < boxes ? tile_of_box(wpos) : kNone;
        }
    };
    uint32_t t0, t1, t2;
    if constexpr (!BB) {
        wpos = a.tile_begin + warp_global;
        t0 = wpos < a.tile_end ? wpos : kNone;
    } else {
        wpos = next_member(warp_global < ustride ? warp_global : boxes);
        t0 = wpos < boxes ? tile_of_box(wpos) : kNone;
    }
    t1 = t0 != kNone ? advance() : kNone;
    t2 = t1 != kNone ? advance() : kNone;

    auto tile_base = [&](uint32_t t) -> uint32_t {  // element offset of the tile's sub-block
        const uint32_t wxb = fastdiv(t, div_hb), wyb = t - wxb * a.Hb;
        return 9u * wxb * a.W + 27u * wyb;
    };
    long long v[8];
    long long hv[NR];
    auto load_tile = [&](uint32_t b) {
        const char* src = src0 + 8ull * b;
#pragma unroll
        for (int k = 0; k < 7; ++k) v[k] = __ldg(reinterpret_cast<const long long*>(src + (sl[k] & 0x1FFFFFu)));
        v[7] = k7 ? __ldg(reinterpret_cast<const long long*>(src + (sl[7] & 0x1FFFFFu))) : 0ll;
    };
    auto nbr_entry = [&](uint32_t t) -> int32_t {
        return (t != kNone && lane < 8) ? __ldg(nbr_tab + 8ull * t + lane) : -1;
    };
    // issue tile t's value loads and its halo loads (neighbour entries `ent` on lanes 0..7);
    // returns the halo membership mask (bit s: slot s is a member cell)
    auto load_all = [&](uint32_t t, int32_t ent, uint32_t& base) -> uint64_t {
        base = tile_base(t);
        load_tile(base);
        int32_t nbase = -1;
        uint32_t own = 0;
        if (ent >= 0) {
            nbase = (int32_t)tile_base((uint32_t)ent);
            if (P2P) own = fastdiv((uint32_t)ent, p.div_chunk);
        }
        uint64_t hmem = 0;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const int32_t b = __shfl_sync(0xFFFFFFFFu, nbase, (int)(sdl[r] >> 29));
            const uint32_t o = P2P ? __shfl_sync(0xFFFFFFFFu, own, (int)(sdl[r] >> 29)) : 0u;
            const bool ok = b >= 0 && sdl[r] != 0xFFFFFFFFu;
            long long h = 0;
            if (ok) {
                const uint32_t off = (uint32_t)b + (sdl[r] & 0x1FFFFFFFu);
                if (!P2P || o == (uint32_t)p.rank)
                    h = __ldg(a.src + off);
                else  // a cell of another rank's tile: its buffer over NVLink
                    asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(h) : "l"(s_peer[o] + off));
            }
            hv[r] = h;
            hmem |= (uint64_t)__ballot_sync(0xFFFFFFFFu, ok) << (32 * r);
        }
        return hmem;
    };

    uint32_t base = 0;
    uint64_t hmem = 0;
    int32_t ent_n = -1;
    if (t0 != kNone) {
        hmem = load_all(t0, nbr_entry(t0), base);
        ent_n = nbr_entry(t1);
    }
    while (t0 != kNone) {
#pragma unroll
        for (int k = 0; k < 7; ++k) cell[sl[k] >> 21] = v[k] != 0ll;
        if (k7) cell[sl[7] >> 21] = v[7] != 0ll;
        uint64_t hm = 0;
#pragma unroll
        for (int r = 0; r < NR; ++r) hm |= (uint64_t)__ballot_sync(0xFFFFFFFFu, hv[r] != 0ll) << (32 * r);
        hm &= hmem;
        const uint64_t hmem_cur = hmem;
        uint32_t base_n = 0;
        if (t1 != kNone) {  // warp-uniform: the next tile's loads fly during this tile's steps
            hmem = load_all(t1, ent_n, base_n);
            ent_n = nbr_entry(t2);
        }
        __syncwarp();
        uint32_t R;
        {   // 0/1 bytes -> bits: per 8 cells (w0 + w1 << 4) * 0x01020408 gathers cell j into bit
            // 24 + j without carries; the four top bytes are then merged with byte permutes
            const uint4 q0 = reinterpret_cast<const uint4*>(cell + 32 * lane)[0];
            const uint4 q1 = reinterpret_cast<const uint4*>(cell + 32 * lane)[1];
            const uint32_t p0 = (q0.x + (q0.y << 4)) * 0x01020408u, p1 = (q0.z + (q0.w << 4)) * 0x01020408u;
            const uint32_t p2 = (q1.x + (q1.y << 4)) * 0x01020408u, p3 = (q1.z + (q1.w << 4)) * 0x01020408u;
            R = __byte_perm(__byte_perm(p0, p1, 0x0073u), __byte_perm(p2, p3, 0x0073u), 0x5410u);
        }
#pragma unroll
        for (int j = 1; j <= K; ++j) {
            const uint32_t Rn = compact_rows_step(R, (uint32_t)hm & 0xFFu, lane, birth, survive);
            if (j < K) {  // the halo slots of layer <= K - j, one scalar step
                const uint32_t e = compact_edge_word(R);
                const uint32_t lo = (uint32_t)hm, hi = (uint32_t)(hm >> 32);
                uint64_t nh;
                {
                    const uint32_t live = __popc(lo & nbl) + __popc(hi & nbh) + __popc(e & medge);
                    const uint32_t alive = (lo >> lane) & 1u;
                    const bool nx = CONWAY ? (live | alive) == 3u : ((((alive ? survive : birth) >> live) & 1u) != 0u);
                    nh = __ballot_sync(0xFFFFFFFFu, nx);
                }
                if constexpr (NR > 1) {
                    if (pass_slots(K - j) > 32) {
                        const uint2 m = s_nbm[lane];
                        const uint32_t live = __popc(lo & m.x) + __popc(hi & m.y);
                        const uint32_t alive = (hi >> lane) & 1u;
                        const bool nx = CONWAY ? (live | alive) == 3u
                                               : ((((alive ? survive : birth) >> live) & 1u) != 0u);
                        nh |= (uint64_t)__ballot_sync(0xFFFFFFFFu, nx) << 32;
                    }
                }
                hm = nh & hmem_cur;
            }
            R = Rn;
        }
        s_new[wib][lane] = R;
        __syncwarp();
        char* dst = dst0 + 8ull * base;
        base = base_n;
#pragma unroll
        for (int k = 0; k < 7; ++k)
            *reinterpret_cast<long long*>(dst + (sl[k] & 0x1FFFFFu)) =
                (long long)((s_new[wib][sl[k] >> 26] >> ((sl[k] >> 21) & 31u)) & 1u);
        if (k7)
            *reinterpret_cast<long long*>(dst + (sl[7] & 0x1FFFFFu)) =
                (long long)((s_new[wib][sl[7] >> 26] >> ((sl[7] >> 21) & 31u)) & 1u);
        __syncwarp();
        t0 = t1;
        t1 = t2;
        t2 = t2 != kNone ? advance() : kNone;
    }
    if (P2P) p2p_arrive(p);
}

}  // namespace nbbgpu
