// compact_cluster.cuh — the λ walk of the tile-sliced pass (compact_sliced.cuh) with each batch a
// level-3 CLUSTER of tiles: the 27 ρ = 32 tiles of one 8 x 8-tile sub-gasket.
//
// In the sliced pass a warp advances 32 tiles at once, bit t of a word = one cell of tile t, and
// every tile needs its radius-K halo (166 cells at K = 8) from its neighbouring tiles. A batch
// of 32 consecutive tile ordinals holds no pair of neighbours (consecutive ωy change tile
// coordinate bit 1 and up: the tiles are 2 apart), so the old λ walk gathers all 32 x 166 halo
// cells from HBM, one 8-byte value each — the largest cost of the pass after the state stream
// itself (compact_pass_tuning: 0.10 of 0.26 ms per 8-step pass).
//
// Tile coordinate bit 0 comes from digit 0 of ωx, bit 1 from digit 0 of ωy, bit 2 from digit 1
// of ωx (the closed-form λ, at block level). The 27 tiles with
// ωx = 9 cx + i (i < 9) and ωy = 3 cy + j (j < 3) are therefore the member tiles of one 8 x 8-tile
// box: a level-3 sub-gasket. Bit t = 3 i + j of the batch's words is tile (i, j). A tile's
// neighbour in direction d is then, for all but a handful of tiles, ANOTHER TILE OF THE BATCH:
// its halo word is a bit permutation of the batch's own tile words, built in shared memory with
// one broadcast load + one ballot per halo slot (lane t picks bit π_d(t)). Sub-gaskets touch their
// neighbours only at corners, so at most 6 (tile, direction) pairs per cluster reach outside it
// (measured at r_b = 11: mean 5.0, max 6): those few halo cells come from HBM as before. The halo
// reads drop from 27 x 166 scattered values per batch to ~150.
//
// Memory: tile (i, j) is the 9 x 27 compact sub-block at 9 (9 cx + i) W + 27 (3 cy + j), so a
// cluster is 9 groups (one per i) of three consecutive tiles = nine 81-value (648 B) runs of
// compact rows per group; the loader fetches a group with nine bulk (TMA) copies into a
// double-buffered staging area and folds it into the stage words, as in the sliced λ loader.
// The steps and stores are the sliced pass's (sliced_steps). Needs r_b >= 3 (ωx has two digits,
// ωy one) and the whole orthotope in one launch (the single-device λ walk); shards, the BB walk
// and the multi-GPU pass keep the 32-ordinal batches of compact_sliced.cuh.
#pragma once

#include "compact_sliced.cuh"

namespace nbbgpu {

constexpr int kClPipes = 2;                                         // loader/stepper pipelines per CTA
constexpr int kClWarps = 2 * kClPipes;
constexpr int kClRunBytes = ((8 * (81 + 1)) + 15) / 16 * 16;        // 656: one 81-value run (+1 for alignment)
constexpr size_t kClDynSmem = (size_t)kClPipes * 2 * 9 * kClRunBytes;  // staging [pipe][2][9 runs]
constexpr int kClExtMax = 27 * 6;                                   // (tile, direction) pairs, any cluster

struct ClusterWalk {
    uint32_t ncy;     // clusters per orthotope column: Hb / 3
    FastDiv div_ncy;
    uint32_t total;   // clusters: (Wb / 9) (Hb / 3)
    int K;            // steps per pass, 1..8
};

#ifndef NBB_CLUSTER_MINB  // resident CTAs per SM the register budget is cut for (tuning builds)
#define NBB_CLUSTER_MINB 4
#endif

template <bool CONWAY>
__global__ void __launch_bounds__(32 * kClWarps, NBB_CLUSTER_MINB)
    ca_compact_cluster_kernel(CompactCaArgs a, ClusterWalk cw, FastDiv div_hb, const int32_t* __restrict__ nbr_tab) {
    const uint32_t birth = a.birth, survive = a.survive;
    __shared__ uint32_t s_box[kClPipes][kBoxWords];
    __shared__ uint32_t s_stage[kClPipes][2][kStageWords];
    __shared__ uint32_t s_hmask[kClPipes][kSliceSlots];
    __shared__ uint32_t s_dofs[8][kSliceDirMax];           // per direction, slot j: offset in the neighbour tile (B)
    __shared__ uint32_t s_dslot[8][kSliceDirMax];          // ... slot | box index of its cell in the neighbour << 16
    __shared__ uint16_t s_bidx[kSliceSlots];
    __shared__ uint16_t s_tb[256];
    __shared__ uint16_t s_cb[256];
    __shared__ uint32_t s_extw[kClPipes][6][32];             // HBM halo bits: [direction q][slot j], bit t
    __shared__ uint32_t s_exist[kClPipes][6];                // neighbouring tile present: bit t
    __shared__ unsigned long long s_ext[kClPipes][kClExtMax];  // HBM (tile, direction) pairs: ptr | q << 56 | t << 59
    __shared__ __align__(8) uint64_t s_mbar[kClPipes][2];
    extern __shared__ __align__(16) unsigned char s_dyn[];
    auto s_tma = reinterpret_cast<unsigned char (*)[2][9][kClRunBytes]>(s_dyn);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int pipe = wib >> 1;
    const bool loader = (wib & 1) == 0;
    const int K = cw.K;
    const bool k7 = lane < 19;
    pdl_trigger();
    for (int s = threadIdx.x; s < c_sslots.count; s += blockDim.x)
        s_bidx[s] = (uint16_t)((c_sslots.y[s] + kSliceMaxK) * kBoxW + c_sslots.x[s] + kSliceMaxK);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        const uint32_t pos = i < 243 ? c_local_pos[i] : 0u;
        s_tb[i] = (uint16_t)(((pos >> 5) + kSliceMaxK) * kBoxW + (pos & 31u) + kSliceMaxK);
    }
    for (int i = threadIdx.x; i < kClPipes * kBoxWords; i += blockDim.x) (&s_box[0][0])[i] = 0u;
    if (threadIdx.x < 2 * kClPipes) mbar_init(&s_mbar[threadIdx.x >> 1][threadIdx.x & 1], 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    {
        uint32_t y = 0, seen = 0;
        for (uint32_t c = threadIdx.x; c < 243u; c += blockDim.x) {
            while (seen + (1u << __popc(y)) <= c) seen += 1u << __popc(y++);
            s_cb[c] = (uint16_t)((y + kSliceMaxK) * kBoxW + pdep32(c - seen, y) + kSliceMaxK);
        }
    }
    __syncthreads();  // s_tb before s_dslot
    for (int i = threadIdx.x; i < 8 * kSliceDirMax; i += blockDim.x) {
        const int d = i / kSliceDirMax, j = i % kSliceDirMax;
        uint32_t o = 0u, sl = 0u;
        if (j < c_sslots.dir_upto[d][kSliceMaxK]) {
            const uint32_t s = c_sslots.by_dir[d][j], li = c_sslots.li[s];
            o = 8u * ((li / 27u) * a.W + li % 27u);
            sl = s | ((uint32_t)s_tb[li] << 16);
        }
        s_dofs[d][j] = o;
        s_dslot[d][j] = sl;
    }
    pdl_wait();
    __syncthreads();

    uint32_t* box = s_box[pipe];
    uint32_t* hmask = s_hmask[pipe];
    const uint32_t pipe_global = blockIdx.x * kClPipes + (uint32_t)pipe;
    const uint32_t npipes = gridDim.x * kClPipes;
    const uint64_t total_elems = (uint64_t)a.W * (uint64_t)(a.tiles / a.Hb) * 9u;  // 3^r
    auto cluster_base = [&](uint32_t bt) -> uint32_t {  // element offset of tile (0, 0) of cluster bt
        const uint32_t cx = fastdiv(bt, cw.div_ncy), cy = bt - cx * cw.ncy;
        return 81u * cx * a.W + 81u * cy;
    };

    if (loader) {
        // ---- loader: group g of a cluster = tiles (g, 0..2) = nine runs of 81 values ------------
        unsigned char (*tma)[9][kClRunBytes] = s_tma[pipe];
        uint64_t* mbar = s_mbar[pipe];
        auto issue = [&](uint32_t base0, uint32_t g, int sbuf) {
            if (lane == 0) {
                uint32_t bytes[9], total = 0;
#pragma unroll
                for (int r = 0; r < 9; ++r) {
                    const uint64_t e0 = (uint64_t)base0 + (uint64_t)(9u * g + r) * a.W, sh = e0 & 1u;
                    const uint64_t nb = (8u * (81u + sh) + 15u) & ~15ull;
                    const uint64_t room = (8u * (total_elems - (e0 - sh))) & ~15ull;  // never past the array
                    bytes[r] = (uint32_t)(nb < room ? nb : room);
                    total += bytes[r];
                }
                mbar_expect_tx(&mbar[sbuf], total);
#pragma unroll
                for (int r = 0; r < 9; ++r) {
                    const uint64_t e0 = (uint64_t)base0 + (uint64_t)(9u * g + r) * a.W, sh = e0 & 1u;
                    bulk_g2s(tma[sbuf][r], a.src + (e0 - sh), bytes[r], &mbar[sbuf]);
                }
            }
        };
        uint32_t gc = 0;  // groups consumed (staging buffer gc & 1, use count gc >> 1)
        if (pipe_global < cw.total) issue(cluster_base(pipe_global), 0u, 0);
        uint32_t i = 0;
        for (uint32_t bt = pipe_global; bt < cw.total; bt += npipes, ++i) {
            const int b = (int)(i & 1u);
            if (i >= 2) nb_op<true>(nb_empty(pipe, b));
            const uint32_t base0 = cluster_base(bt);
            const uint32_t nbase = bt + npipes < cw.total ? cluster_base(bt + npipes) : 0u;
            uint32_t w[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) w[k] = 0u;
#pragma unroll 1
            for (uint32_t g = 0; g < 9u; ++g, ++gc) {
                if (g + 1 < 9u) issue(base0, g + 1, (int)((gc + 1) & 1u));
                else if (bt + npipes < cw.total) issue(nbase, 0u, (int)((gc + 1) & 1u));
                const int sb_ = (int)(gc & 1u);
                mbar_wait(&mbar[sb_], (gc >> 1) & 1u);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (k == 7 && !k7) continue;
                    const uint32_t li = 32u * k + lane, row = li / 27u, col = li % 27u;
                    const uint64_t e0 = (uint64_t)base0 + (uint64_t)(9u * g + row) * a.W;
                    const uint32_t sh = (uint32_t)(e0 & 1u);
                    const uint64_t want = (uint64_t)(((8u * (81u + sh) + 15u) & ~15u) / 8u);
                    const uint64_t room = (total_elems - (e0 - sh)) & ~1ull;
                    const uint32_t copied = (uint32_t)(want < room ? want : room);
                    const long long* rowp = reinterpret_cast<const long long*>(tma[sb_][row]);
#pragma unroll
                    for (int t = 0; t < 3; ++t) {
                        const uint32_t idx = sh + 27u * t + col;
                        const long long v = idx < copied ? rowp[idx] : __ldg(a.src + e0 + 27u * t + col);
                        const uint32_t nz = (uint32_t)v | (uint32_t)((unsigned long long)v >> 32);
                        w[k] |= min(nz, 1u) << (3u * g + t);
                    }
                }
                __syncwarp();
                fence_proxy_async();  // the reads of this buffer before the next bulk copy into it
            }
            uint32_t* stage = s_stage[pipe][b];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < 7 || k7) stage[32 * k + lane] = w[k];
            __syncwarp();
            nb_op<false>(nb_full(pipe, b));
        }
        return;
    }

    // ---- stepper --------------------------------------------------------------------------------
    // lane t < 27 is tile (i, j) = (t / 3, t % 3) of the cluster
    const uint32_t ti = (uint32_t)lane / 3u, tj = (uint32_t)lane % 3u;
    const bool tv = lane < 27;
    uint32_t i = 0;
    for (uint32_t bt = pipe_global; bt < cw.total; bt += npipes, ++i) {
        const int b = (int)(i & 1u);
        const bool more2 = bt + 2u * npipes < cw.total;
        const uint32_t cx = fastdiv(bt, cw.div_ncy), cy = bt - cx * cw.ncy;
        const uint32_t wx0 = 9u * cx, wy0 = 3u * cy;
        // the neighbouring tiles of tile t: in the cluster (π_q = its bit) or in HBM (ext pair)
        int4 n0 = make_int4(-1, -1, -1, -1), n1 = n0;
        if (tv) {
            const uint32_t u = (wx0 + ti) * a.Hb + wy0 + tj;
            n0 = __ldg(reinterpret_cast<const int4*>(nbr_tab + 8ull * u));
            n1 = __ldg(reinterpret_cast<const int4*>(nbr_tab + 8ull * u) + 1);
        }
        const int32_t nbr6[6] = {n0.x, n0.y, n0.w, n1.x, n1.z, n1.w};  // directions 0,1,3,4,6,7
        uint32_t pi_pack = 0u;
        uint32_t next = 0;  // ext pairs listed
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            s_extw[pipe][q][lane] = 0u;
            const int32_t nq = nbr6[q];
            uint32_t pi = 31u;  // bit 31 of a tile word is 0: no in-cluster neighbour
            bool ext = false;
            unsigned long long ptr = 0ull;
            if (nq >= 0) {
                const uint32_t wxn = fastdiv((uint32_t)nq, div_hb), wyn = (uint32_t)nq - wxn * a.Hb;
                const uint32_t di = wxn - wx0, dj = wyn - wy0;
                if (di < 9u && dj < 3u) {
                    pi = 3u * di + dj;
                } else {
                    ext = true;
                    ptr = reinterpret_cast<unsigned long long>(a.src) + 8ull * (9ull * wxn * a.W + 27ull * wyn);
                }
            }
            pi_pack |= pi << (5 * q);
            const uint32_t ex = __ballot_sync(0xFFFFFFFFu, nq >= 0);
            if (lane == 0) s_exist[pipe][q] = ex;
            const uint32_t em = __ballot_sync(0xFFFFFFFFu, ext);
            if (ext) s_ext[pipe][next + __popc(em & ((1u << lane) - 1u))] = ptr | ((unsigned long long)q << 56) |
                                                                         ((unsigned long long)lane << 59);
            next += __popc(em);
        }
        __syncwarp();
        // the HBM halo cells: pair p = (tile t, direction q); lane j loads the pair's slot j
        for (uint32_t p0 = 0; p0 < next; p0 += 8) {
            long long v[8];
            uint32_t meta[8];
#pragma unroll
            for (int p = 0; p < 8; ++p) {
                v[p] = 0;
                meta[p] = 0xFFFFFFFFu;
                if (p0 + p < next) {
                    const unsigned long long e = s_ext[pipe][p0 + p];
                    const uint32_t q = (uint32_t)(e >> 56) & 7u, t = (uint32_t)(e >> 59);
                    const int d = q < 2 ? (int)q : q < 4 ? (int)q + 1 : (int)q + 2;
                    if (lane < c_sslots.dir_upto[d][K]) {
                        const unsigned long long ptr = e & ((1ull << 56) - 1ull);
                        v[p] = __ldg(reinterpret_cast<const long long*>(ptr + s_dofs[d][lane]));
                        meta[p] = q | (t << 8);
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < 8; ++p)
                if (meta[p] != 0xFFFFFFFFu) {
                    const uint32_t nz = (uint32_t)v[p] | (uint32_t)((unsigned long long)v[p] >> 32);
                    s_extw[pipe][meta[p] & 7u][lane] |= min(nz, 1u) << (meta[p] >> 8);
                }
        }
        // the batch's tile words into the box
        nb_op<true>(nb_full(pipe, b));
        {
            const uint32_t* stage = s_stage[pipe][b];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < 7 || k7) box[s_tb[32 * k + lane]] = stage[32 * k + lane];
        }
        __syncwarp();
        if (more2) nb_op<false>(nb_empty(pipe, b));
        // halo words: slot j of direction q, bit t = bit π_q(t) of the neighbour cell's tile word
        // (one broadcast load + one ballot) | its HBM bit
#pragma unroll 1
        for (int q = 0; q < 6; ++q) {
            const int d = q < 2 ? q : q < 4 ? q + 1 : q + 2;
            const int ns = c_sslots.dir_upto[d][K];
            if (ns == 0) continue;
            const uint32_t pi = (pi_pack >> (5 * q)) & 31u;
            uint32_t mine = 0u;
            for (int j = 0; j < ns; ++j) {
                const uint32_t word = box[s_dslot[d][j] >> 16];
                const uint32_t hw = __ballot_sync(0xFFFFFFFFu, (word >> pi) & 1u);
                if (lane == j) mine = hw;
            }
            if (lane < ns) {
                const uint32_t slot = s_dslot[d][lane] & 0xFFFFu, ex = s_exist[pipe][q];
                box[s_bidx[slot]] = (mine | s_extw[pipe][q][lane]) & ex;
                hmask[slot] = ex;
            }
        }
        // K steps, then the 27 tiles' values out
        uint32_t w[8];
        sliced_steps<CONWAY>(box, hmask, K, s_cb, s_bidx, s_tb, birth, survive, w);
        uint32_t off[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t li = min(32u * k + lane, 242u);
            off[k] = 8u * ((li / 27u) * a.W + li % 27u);
        }
        char* Q0 = reinterpret_cast<char*>(a.dst) + 8ull * (81ull * cx * a.W + 81ull * cy);
        const uint64_t gstride = 72ull * a.W;  // bytes between tile groups i and i + 1
#pragma unroll
        for (int t = 0; t < 27; ++t) {
            char* Q = Q0 + (uint64_t)(t / 3) * gstride + 216u * (t % 3);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < 7 || k7) *reinterpret_cast<long long*>(Q + off[k]) = (long long)((w[k] >> t) & 1u);
        }
    }
}

}  // namespace nbbgpu
