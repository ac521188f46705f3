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
// neighbour in direction q is then, for all but a handful of tiles, ANOTHER TILE OF THE BATCH,
// and the same one in every cluster: a halo slot's word is a fixed bit permutation of the batch's
// own word at the slot's cell (cl_perm<q>, masked shifts with compile-time constants). Sub-gaskets
// touch their neighbours only at corners, so at most 6 (tile, direction) pairs per cluster reach
// outside it (measured at r_b = 11: mean 5.0, max 6): those few halo cells come from HBM (in a
// multi-GPU pass from the owning rank's buffer). The halo reads drop from 27 x 166 scattered
// values per batch to ~150.
//
// Memory: tile (i, j) is the 9 x 27 compact sub-block at 9 (9 cx + i) W + 27 (3 cy + j), so a
// cluster is 9 groups (one per i) of three consecutive tiles = nine 81-value (648 B) runs of
// compact rows per group; the loader fetches a group with nine bulk (TMA) copies into a
// double-buffered staging area, folds it into the stage words and stores the stepper's previous
// results; the stepper builds the halo words and runs the K steps (cluster_steps / _steps2,
// radius up to 12). Needs r_b >= 3 (ωx has two digits, ωy one) and a launch range of whole
// cluster columns (9 Hb tiles: the whole orthotope, or a multi-GPU shard of
// nbbhost::compact_shard_chunk); the BB walk and r < 8 keep the 32-ordinal batches of
// compact_sliced.cuh.
#pragma once

#include <type_traits>

#include "compact_sliced.cuh"

namespace nbbgpu {

using nbbhost::ClusterSlots;
using nbbhost::kClDirSlots;
using nbbhost::kClMaxK;
using nbbhost::kClSlots;
__constant__ ClusterSlots c_cslots;  // the radius-12 halo slots (nbbhost::cluster_slots)
// The box of a pass of up to F steps: the tile and an F-cell frame (odd row pitch). Two
// instantiations: F = 8 with two boxes per stepper (cluster_steps2), F = 12 with one.
template <int F>
struct ClBox {
    static constexpr int kH = 32 + 2 * F, kW = kH + 1, kWords = kW * kH;
    static constexpr int kBoxes = F <= 8 ? 2 : 1;
    static constexpr int kM = F <= 8 ? 4 : 8;  // halo slots a lane advances per step: upto[F - 1] <= 32 kM
    static_assert(F <= kClMaxK && kWords <= 4096, "box index: 12 bits");
};

constexpr int kClPipes = 2;                                         // loader/stepper pipelines per CTA
constexpr int kClWarps = 2 * kClPipes;
constexpr int kClRunBytes = ((8 * (81 + 1)) + 15) / 16 * 16;        // 656: one 81-value run (+1 for alignment)
constexpr size_t kClTmaBytes = (size_t)kClPipes * 2 * 9 * kClRunBytes;  // staging [pipe][2][9 runs]
constexpr int kClExtMax = 32;  // HBM (tile, direction) pairs per cluster (<= 6 at every level measured)

struct ClusterWalk {
    uint32_t ncy;         // clusters per orthotope column: Hb / 3
    FastDiv div_ncy;
    uint32_t total;       // clusters: (Wb / 9) (Hb / 3)
    uint32_t begin, end;  // this launch's clusters (a shard: whole cluster columns)
    int K;                // steps per pass, 1..12
    RuleTab rule;         // the rule's mux-tree constants (the generic-rule instantiation)
};

// The in-cluster neighbour of tile t = 3 i + j in halo direction q (q = 0..5: directions
// 0, 1, 3, 4, 6, 7 of compact_nbr_table_kernel, d9 = (dy + 1) * 3 + dx + 1 with the centre
// skipped), or -1. Cluster-local tile coordinates: bit 0 from digit 0 of ωx (i % 3), bit 1 from
// digit 0 of ωy (j), bit 2 from digit 1 of ωx (i / 3); digit v -> x bit (v == 2), y bit (v >= 1).
// The same for every cluster: the halo word of a slot is a FIXED bit permutation of the tile
// word its cell lies in (plus the few bits from other clusters).
__host__ __device__ constexpr int cl_src(int q, int t) {
    const int d = q < 2 ? q : q < 4 ? q + 1 : q + 2, d9 = d < 4 ? d : d + 1;
    const int dx = d9 % 3 - 1, dy = d9 / 3 - 1;
    const int i = t / 3, j = t % 3, d0 = i % 3, d1 = i / 3;
    const int lx = (d0 == 2) | ((j == 2) << 1) | ((d1 == 2) << 2);
    const int ly = (d0 >= 1) | ((j >= 1) << 1) | ((d1 >= 1) << 2);
    const int nx = lx + dx, ny = ly + dy;
    if (nx < 0 || ny < 0 || nx > 7 || ny > 7 || (nx & ~ny) != 0) return -1;
    auto dig = [](int x, int y, int b) { return ((x >> b) & 1) ? 2 : ((y >> b) & 1); };
    return (3 * dig(nx, ny, 2) + dig(nx, ny, 0)) * 3 + dig(nx, ny, 1);
}
// source bits s whose target bit is s + delta, for direction q
__host__ __device__ constexpr uint32_t cl_mask(int q, int delta) {
    uint32_t m = 0;
    for (int t = 0; t < 27; ++t) {
        const int s = cl_src(q, t);
        if (s >= 0 && t - s == delta) m |= 1u << s;
    }
    return m;
}
// the permutation: bit t of the result = bit cl_src(q, t) of x (0 where there is none), as one
// masked shift per distinct distance
template <int Q, int D = -26>
__device__ __forceinline__ uint32_t cl_perm(uint32_t x) {
    constexpr uint32_t m = cl_mask(Q, D);
    uint32_t r = 0u;
    if constexpr (m != 0u) r = D >= 0 ? (x & m) << (D >= 0 ? D : 0) : (x & m) >> (D < 0 ? -D : 0);
    if constexpr (D < 26) return r | cl_perm<Q, D + 1>(x);
    else return r;
}

#ifndef NBB_CL_LSTORE  // the loader warp stores the stepper's results (1) or the stepper does (0)
#define NBB_CL_LSTORE 1
#endif
constexpr bool kClLoaderStores = NBB_CL_LSTORE != 0;

// K steps of a batch in its box (sliced_steps of compact_sliced.cuh with the box pitch BW, up to
// 32 M halo slots, and the lane's box indices and halo masks held in registers across the steps:
// shared memory is written between the steps, so the compiler would reload them every step)
template <bool CONWAY, int BW, int M>
__device__ __forceinline__ void cluster_steps(uint32_t* box, const uint32_t* exist, const uint8_t* sq, int K,
                                              const uint16_t* cb,
                                              const uint16_t* bidx, const uint16_t* tb, const RuleTab& rt,
                                              uint32_t (&w)[8]) {
    const int lane = threadIdx.x & 31;
    const bool k7 = lane < 19;
    __syncwarp();
    uint32_t ci[8], hi[M], hm[M];
#pragma unroll
    for (int k = 0; k < 8; ++k) ci[k] = (k < 7 || k7) ? cb[32 * k + lane] : 0u;
    const int n0 = c_cslots.upto[K - 1];
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int s = lane + 32 * m;
        hi[m] = s < n0 ? bidx[s] : 0u;
        hm[m] = s < n0 ? exist[sq[s]] : 0u;  // the slot's neighbouring tile is present: bit t
    }
    for (int j = 1; j <= K; ++j) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < 7 || k7) w[k] = sliced_cell_step<CONWAY, BW>(box + ci[k], rt);
        const int ns = c_cslots.upto[K - j];
        uint32_t hn[M];
#pragma unroll
        for (int m = 0; m < M; ++m) {
            hn[m] = 0u;
            if (lane + 32 * m < ns) hn[m] = sliced_cell_step<CONWAY, BW>(box + hi[m], rt) & hm[m];
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < 7 || k7) box[ci[k]] = w[k];
#pragma unroll
        for (int m = 0; m < M; ++m)
            if (lane + 32 * m < ns) box[hi[m]] = hn[m];
        __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = (k < 7 || k7) ? box[tb[32 * k + lane]] : 0u;
}

// The same with two boxes: step j reads box[(j - 1) & 1] and writes box[j & 1], so each step
// needs one warp barrier and no result is held across it. A halo slot not advanced at step j
// (layer > K - j) keeps a stale value in the written box, read only by cells that are not needed
// either; the non-member frame is zero in both boxes.
template <bool CONWAY, int BW, int M>
__device__ __forceinline__ void cluster_steps2(uint32_t* box0, uint32_t* box1, const uint32_t* exist,
                                               const uint8_t* sq, int K,
                                               const uint16_t* cb, const uint16_t* bidx, const uint16_t* tb,
                                               const RuleTab& rt, uint32_t (&w)[8]) {
    const int lane = threadIdx.x & 31;
    const bool k7 = lane < 19;
    __syncwarp();
    uint32_t ci[8], hi[M], hm[M];
#pragma unroll
    for (int k = 0; k < 8; ++k) ci[k] = (k < 7 || k7) ? cb[32 * k + lane] : 0u;
    const int n0 = c_cslots.upto[K - 1];
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int s = lane + 32 * m;
        hi[m] = s < n0 ? bidx[s] : 0u;
        hm[m] = s < n0 ? exist[sq[s]] : 0u;  // the slot's neighbouring tile is present: bit t
    }
    for (int j = 1; j <= K; ++j) {
        const uint32_t* src = (j & 1) ? box0 : box1;
        uint32_t* dst = (j & 1) ? box1 : box0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < 7 || k7) dst[ci[k]] = sliced_cell_step<CONWAY, BW>(src + ci[k], rt);
        const int ns = c_cslots.upto[K - j];
#pragma unroll
        for (int m = 0; m < M; ++m)
            if (lane + 32 * m < ns) dst[hi[m]] = sliced_cell_step<CONWAY, BW>(src + hi[m], rt) & hm[m];
        __syncwarp();
    }
    const uint32_t* fin = (K & 1) ? box1 : box0;
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = (k < 7 || k7) ? fin[tb[32 * k + lane]] : 0u;
}

template <int F>
constexpr size_t cl_dyn_smem() { return kClTmaBytes + (size_t)kClPipes * ClBox<F>::kBoxes * ClBox<F>::kWords * 4; }

#ifndef NBB_CLUSTER_MINB  // resident CTAs per SM the register budget is cut for (tuning builds)
#define NBB_CLUSTER_MINB 3
#endif

// P2P: one rank's pass of the multi-GPU CA (its shard is whole cluster columns, so every tile of a
// cluster is its own; the halo cells of neighbouring clusters owned by other ranks are read from
// their buffers over NVLink; the flag barrier of compact_kernels.cuh orders the passes).
template <bool CONWAY, bool P2P, int F>
__global__ void __launch_bounds__(32 * kClWarps, NBB_CLUSTER_MINB)
    ca_compact_cluster_kernel(CompactCaArgs a, ClusterWalk cw, FastDiv div_hb, const int32_t* __restrict__ nbr_tab,
                              P2PArgs p) {
    constexpr int kClBoxW = ClBox<F>::kW, kClBoxWords = ClBox<F>::kWords, kClBoxes = ClBox<F>::kBoxes;
    __shared__ uint32_t s_stage[kClPipes][2][kStageWords];
    __shared__ uint8_t s_sq[kClSlots];                     // halo direction q of every slot
    __shared__ uint32_t s_dofs[8][kClDirSlots];           // per direction, slot j: offset in the neighbour tile (B)
    __shared__ uint16_t s_bidx[kClSlots];
    __shared__ uint16_t s_tb[256];
    __shared__ uint16_t s_cb[256];
    __shared__ uint32_t s_hflat[kClSlots];                // halo slots of this K, direction-major:
                                                             // box index of the cell in the neighbour
                                                             // | slot << 12
    __shared__ int s_qstart[7];                              // first flat entry of direction q
    __shared__ uint32_t s_extw[kClPipes][kClSlots];       // HBM halo bits of flat entry m, bit t
    __shared__ uint32_t s_exist[kClPipes][6];                // neighbouring tile present: bit t
    __shared__ unsigned long long s_ext[kClPipes][kClExtMax];  // HBM (tile, direction) pairs: ptr | remote << 55
                                                               // | q << 56 | t << 59
    __shared__ __align__(8) uint64_t s_mbar[kClPipes][2];
    __shared__ uint32_t s_out[kClPipes][kStageWords];         // stepper -> loader: a batch's result words
    __shared__ __align__(8) uint64_t s_obar[kClPipes][2];     // [0] out full, [1] out empty (32 arrivals)
    __shared__ const long long* s_peer[kMaxP2P];
    extern __shared__ __align__(16) unsigned char s_dyn[];
    auto s_tma = reinterpret_cast<unsigned char (*)[2][9][kClRunBytes]>(s_dyn);
    auto s_box = reinterpret_cast<uint32_t (*)[kClBoxes][kClBoxWords]>(s_dyn + kClTmaBytes);
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int pipe = wib >> 1;
    const bool loader = (wib & 1) == 0;
    const int K = cw.K;
    const bool k7 = lane < 19;
    pdl_trigger();
    if (P2P && threadIdx.x < (unsigned)p.world) s_peer[threadIdx.x] = p.peer_src[threadIdx.x];
    for (int s = threadIdx.x; s < c_cslots.count; s += blockDim.x)
        s_bidx[s] = (uint16_t)((c_cslots.y[s] + F) * kClBoxW + c_cslots.x[s] + F);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        const uint32_t pos = i < 243 ? c_local_pos[i] : 0u;
        s_tb[i] = (uint16_t)(((pos >> 5) + F) * kClBoxW + (pos & 31u) + F);
    }
    for (int i = threadIdx.x; i < kClPipes * kClBoxes * kClBoxWords; i += blockDim.x) (&s_box[0][0][0])[i] = 0u;
    if (threadIdx.x < 2 * kClPipes) {
        mbar_init(&s_mbar[threadIdx.x >> 1][threadIdx.x & 1], 1u);
        mbar_init(&s_obar[threadIdx.x >> 1][threadIdx.x & 1], 32u);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    {
        uint32_t y = 0, seen = 0;
        for (uint32_t c = threadIdx.x; c < 243u; c += blockDim.x) {
            while (seen + (1u << __popc(y)) <= c) seen += 1u << __popc(y++);
            s_cb[c] = (uint16_t)((y + F) * kClBoxW + pdep32(c - seen, y) + F);
        }
    }
    __syncthreads();  // s_tb before s_hflat
    for (int i = threadIdx.x; i < 8 * kClDirSlots; i += blockDim.x) {
        const int d = i / kClDirSlots, j = i % kClDirSlots;
        uint32_t o = 0u;
        if (j < c_cslots.dir_upto[d][kClMaxK]) {
            const uint32_t li = c_cslots.li[c_cslots.by_dir[d][j]];
            o = 8u * ((li / 27u) * a.W + li % 27u);
        }
        s_dofs[d][j] = o;
    }
    if (threadIdx.x == 0) {
        int m = 0;
        for (int q = 0; q < 6; ++q) {
            const int d = q < 2 ? q : q < 4 ? q + 1 : q + 2;
            s_qstart[q] = m;
            for (int j = 0; j < c_cslots.dir_upto[d][K]; ++j, ++m) {
                const uint32_t sl = c_cslots.by_dir[d][j];
                s_sq[sl] = (uint8_t)q;
                s_hflat[m] = (uint32_t)s_tb[c_cslots.li[sl]] | (sl << 12);
            }
        }
        s_qstart[6] = m;
    }
    if (P2P && p.wait_target != 0u) {
        // the arrival wait (this rank's own previous pass is among the arrivals); the first pass
        // of every call also waits for its predecessor grid (whatever last wrote the state)
        if (threadIdx.x == 0) p2p_wait(p);
        if (p.first_pass) pdl_wait();
    } else {
        pdl_wait();
    }
    __syncthreads();
    // every thread orders its peer reads after the arrivals waited for; the proxy
    // fence orders the generic-proxy stores it acquired (this rank's previous pass) before the
    // loader's bulk copies (async proxy) of the same buffer
    if (P2P && p.wait_target != 0u) {
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }

    uint32_t* box = s_box[pipe][0];
    const uint32_t pipe_global = blockIdx.x * kClPipes + (uint32_t)pipe;
    const uint32_t npipes = gridDim.x * kClPipes;
    const uint64_t total_elems = (uint64_t)a.W * (uint64_t)(a.tiles / a.Hb) * 9u;  // 3^r
    auto cluster_base = [&](uint32_t bt) -> uint32_t {  // element offset of tile (0, 0) of cluster bt
        const uint32_t cx = fastdiv(bt, cw.div_ncy), cy = bt - cx * cw.ncy;
        return 81u * cx * a.W + 81u * cy;
    };

    if (loader) {
        // ---- loader: group g of a cluster = tiles (g, 0..2) = nine runs of 81 values ------------
        // A run starts one value early when its first value sits at an odd element (16-byte
        // aligned bulk copies): 82 values = 656 B, except at the end of the array (the last
        // cluster: byte counts clamped, its values past the copy read directly).
        unsigned char (*tma)[9][kClRunBytes] = s_tma[pipe];
        uint64_t* mbar = s_mbar[pipe];
        const uint64_t row_bytes = 8ull * a.W;
        auto issue = [&](uint32_t base0, uint32_t g, int sbuf, bool last) {
            if (lane == 0) {
                const char* p0 = reinterpret_cast<const char*>(a.src) + 8ull * ((uint64_t)base0 + 9ull * g * a.W);
                if (!last) {
                    mbar_expect_tx(&mbar[sbuf], 9u * kClRunBytes);
#pragma unroll
                    for (int r = 0; r < 9; ++r)
                        bulk_g2s(tma[sbuf][r], reinterpret_cast<const void*>(
                                     reinterpret_cast<uintptr_t>(p0 + r * row_bytes) & ~(uintptr_t)15),
                                 kClRunBytes, &mbar[sbuf]);
                } else {
                    uint32_t bytes[9], total = 0;
#pragma unroll
                    for (int r = 0; r < 9; ++r) {
                        const uint64_t e0 = (uint64_t)base0 + (uint64_t)(9u * g + r) * a.W, sh = e0 & 1u;
                        const uint64_t room = (8u * (total_elems - (e0 - sh))) & ~15ull;  // never past the array
                        bytes[r] = (uint32_t)(kClRunBytes < room ? kClRunBytes : room);
                        total += bytes[r];
                    }
                    mbar_expect_tx(&mbar[sbuf], total);
#pragma unroll
                    for (int r = 0; r < 9; ++r) {
                        const uint64_t e0 = (uint64_t)base0 + (uint64_t)(9u * g + r) * a.W, sh = e0 & 1u;
                        bulk_g2s(tma[sbuf][r], a.src + (e0 - sh), bytes[r], &mbar[sbuf]);
                    }
                }
            }
        };
        // the lane's cells li = 32 k + lane: compact row and column inside a tile
        uint32_t rowk[8], colk[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t li = min(32u * k + lane, 242u);
            rowk[k] = li / 27u;
            colk[k] = li % 27u;
        }
        // the stepper's results: batch bo's words ow (taken from s_out as soon as they are there),
        // stored group by group while the loader folds a later batch
        uint32_t ow[8];
        uint32_t nout = 0;  // results taken so far
        auto take_out = [&]() {
            mbar_wait(&s_obar[pipe][0], nout & 1u);
#pragma unroll
            for (int k = 0; k < 8; ++k) ow[k] = (k < 7 || k7) ? s_out[pipe][32 * k + lane] : 0u;
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&s_obar[pipe][1])) : "memory");
            ++nout;
        };
        auto store_group = [&](uint32_t obase, uint32_t g) {  // tiles (g, 0..2) of the taken batch
            char* Q0 = reinterpret_cast<char*>(a.dst) + 8ull * ((uint64_t)obase + 9ull * g * a.W);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (k < 7 || k7)
                        *reinterpret_cast<long long*>(Q0 + 216u * j + 8ull * (rowk[k] * a.W + colk[k])) =
                            (long long)((ow[k] >> (3u * g + j)) & 1u);
            }
        };
        uint32_t gc = 0;  // groups consumed (staging buffer gc & 1, use count gc >> 1)
        if (cw.begin + pipe_global < cw.end)
            issue(cluster_base(cw.begin + pipe_global), 0u, 0, cw.begin + pipe_global + 1 == cw.total);
        uint32_t i = 0;
        for (uint32_t bt = cw.begin + pipe_global; bt < cw.end; bt += npipes, ++i) {
            const int b = (int)(i & 1u);
            if (i >= 2) nb_op<true>(nb_empty(pipe, b));
            const uint32_t base0 = cluster_base(bt);
            const bool last = bt + 1 == cw.total;
            const uint32_t nbase = bt + npipes < cw.end ? cluster_base(bt + npipes) : 0u;
            const bool st = kClLoaderStores && i >= 2;  // stores the result of batch i - 2 meanwhile
            const uint32_t obase = st ? cluster_base(bt - 2u * npipes) : 0u;
            uint32_t w[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) w[k] = 0u;
#pragma unroll 1
            for (uint32_t g = 0; g < 9u; ++g, ++gc) {
                if (g + 1 < 9u) issue(base0, g + 1, (int)((gc + 1) & 1u), last);
                else if (bt + npipes < cw.end) issue(nbase, 0u, (int)((gc + 1) & 1u), bt + npipes + 1 == cw.total);
                const int sb_ = (int)(gc & 1u);
                mbar_wait(&mbar[sb_], (gc >> 1) & 1u);
                // parity of a run's first element: base0 + (9 g + row) W with W odd
                const uint32_t par = (base0 ^ g) & 1u;
                if (!last) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        if (k == 7 && !k7) continue;
                        const long long* rowp = reinterpret_cast<const long long*>(tma[sb_][rowk[k]]) +
                                                ((par ^ rowk[k]) & 1u) + colk[k];
#pragma unroll
                        for (int t = 0; t < 3; ++t) {
                            const long long v = rowp[27 * t];
                            const uint32_t nz = (uint32_t)v | (uint32_t)((unsigned long long)v >> 32);
                            w[k] |= min(nz, 1u) << (3u * g + t);
                        }
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        if (k == 7 && !k7) continue;
                        const uint32_t row = rowk[k], col = colk[k];
                        const uint64_t e0 = (uint64_t)base0 + (uint64_t)(9u * g + row) * a.W;
                        const uint32_t sh = (uint32_t)(e0 & 1u);
                        const uint64_t want = kClRunBytes / 8u;
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
                }
                __syncwarp();
                fence_proxy_async();  // the reads of this buffer before the next bulk copy into it
                if (st) {
                    if (g == 0) take_out();
                    store_group(obase, g);
                }
            }
            uint32_t* stage = s_stage[pipe][b];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < 7 || k7) stage[32 * k + lane] = w[k];
            __syncwarp();
            nb_op<false>(nb_full(pipe, b));
        }
        if (kClLoaderStores) {  // the last two results
            const uint32_t nb = i;  // batches of this pipeline
            for (uint32_t o = nb >= 2 ? nb - 2 : 0; o < nb; ++o) {
                const uint32_t obase = cluster_base(cw.begin + pipe_global + o * npipes);
                take_out();
#pragma unroll 1
                for (uint32_t g = 0; g < 9u; ++g) store_group(obase, g);
            }
        }
    } else {
    // ---- stepper --------------------------------------------------------------------------------
    // lane t < 27 is tile (i, j) = (t / 3, t % 3) of the cluster
    const uint32_t ti = (uint32_t)lane / 3u, tj = (uint32_t)lane % 3u;
    const bool tv = lane < 27;
    uint32_t i = 0;
    for (uint32_t bt = cw.begin + pipe_global; bt < cw.end; bt += npipes, ++i) {
        const int b = (int)(i & 1u);
        const bool more2 = bt + 2u * npipes < cw.end;
        const uint32_t cx = fastdiv(bt, cw.div_ncy), cy = bt - cx * cw.ncy;
        const uint32_t wx0 = 9u * cx, wy0 = 3u * cy;
        // the neighbouring tiles of tile t: in the cluster (cl_src) or in HBM (an ext pair)
        int4 n0 = make_int4(-1, -1, -1, -1), n1 = n0;
        if (tv) {
            const uint32_t u = (wx0 + ti) * a.Hb + wy0 + tj;
            n0 = __ldg(reinterpret_cast<const int4*>(nbr_tab + 8ull * u));
            n1 = __ldg(reinterpret_cast<const int4*>(nbr_tab + 8ull * u) + 1);
        }
        const int32_t nbr6[6] = {n0.x, n0.y, n0.w, n1.x, n1.z, n1.w};  // directions 0,1,3,4,6,7
        uint32_t next = 0;  // ext pairs listed
        for (int m = lane; m < kClSlots; m += 32) s_extw[pipe][m] = 0u;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            const int32_t nq = nbr6[q];
            bool ext = false;
            unsigned long long ptr = 0ull;
            if (nq >= 0) {
                const uint32_t wxn = fastdiv((uint32_t)nq, div_hb), wyn = (uint32_t)nq - wxn * a.Hb;
                const uint32_t di = wxn - wx0, dj = wyn - wy0;
                if (di < 9u && dj < 3u) {
#ifdef NBB_CL_CHECK  // the compile-time permutation agrees with the neighbour table
                    if ((int)(3u * di + dj) != cl_src(q, lane)) __trap();
#endif
                } else {
                    ext = true;
                    const uint32_t own = P2P ? fastdiv((uint32_t)nq, p.div_chunk) : 0u;
                    const long long* src = P2P ? s_peer[own] : a.src;
                    ptr = reinterpret_cast<unsigned long long>(src) + 8ull * (9ull * wxn * a.W + 27ull * wyn);
                    if (P2P && own != (uint32_t)p.rank) ptr |= 1ull << 55;  // another rank's buffer
                }
            }
            const uint32_t ex = __ballot_sync(0xFFFFFFFFu, nq >= 0);
            if (lane == 0) s_exist[pipe][q] = ex;
            const uint32_t em = __ballot_sync(0xFFFFFFFFu, ext);
            if (next + __popc(em) > (uint32_t)kClExtMax) __trap();  // fail loudly, never overrun s_ext
            if (ext) s_ext[pipe][next + __popc(em & ((1u << lane) - 1u))] = ptr | ((unsigned long long)q << 56) |
                                                                         ((unsigned long long)lane << 59);
            next += __popc(em);
        }
        __syncwarp();
        // the HBM halo cells: pair p = (tile t, direction q); load unit (p, h): lane j loads the
        // pair's slot j = lane + 32 h (a direction holds up to kClDirSlots slots)
        for (uint32_t u0 = 0; u0 < 2u * next; u0 += 8) {
            long long v[8];
            uint32_t meta[8];
#pragma unroll
            for (int uu = 0; uu < 8; ++uu) {
                v[uu] = 0;
                meta[uu] = 0xFFFFFFFFu;
                const uint32_t u = u0 + uu;
                if (u < 2u * next) {
                    const unsigned long long e = s_ext[pipe][u >> 1];
                    const uint32_t q = (uint32_t)(e >> 56) & 7u, t = (uint32_t)(e >> 59);
                    const int d = q < 2 ? (int)q : q < 4 ? (int)q + 1 : (int)q + 2;
                    const int j = lane + 32 * (int)(u & 1u);
                    if (j < c_cslots.dir_upto[d][K]) {
                        const unsigned long long ptr = e & ((1ull << 55) - 1ull);
                        const long long* qp = reinterpret_cast<const long long*>(ptr + s_dofs[d][j]);
                        if (P2P && ((e >> 55) & 1ull))  // a cell of another rank's tile: over NVLink
                            asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v[uu]) : "l"(qp));
                        else
                            v[uu] = __ldg(qp);
                        meta[uu] = (uint32_t)(s_qstart[q] + j) | (t << 16);
                    }
                }
            }
#pragma unroll
            for (int uu = 0; uu < 8; ++uu)
                if (meta[uu] != 0xFFFFFFFFu) {
                    const uint32_t nz = (uint32_t)v[uu] | (uint32_t)((unsigned long long)v[uu] >> 32);
                    s_extw[pipe][meta[uu] & 0xFFFFu] |= min(nz, 1u) << (meta[uu] >> 16);
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
        // halo words: slot j (lane) of direction q = the fixed bit permutation π_q of the word of
        // its cell's tile position (cl_perm) | its HBM bits
        auto halo_dir = [&](auto qc) {
            constexpr int q = decltype(qc)::value;
            const uint32_t ex = s_exist[pipe][q];
            for (int m = s_qstart[q] + lane; m < s_qstart[q + 1]; m += 32) {
                const uint32_t e = s_hflat[m], slot = e >> 12;
                box[s_bidx[slot]] = (cl_perm<q>(box[e & 0xFFFu]) | s_extw[pipe][m]) & ex;
            }
        };
        halo_dir(std::integral_constant<int, 0>{});
        halo_dir(std::integral_constant<int, 1>{});
        halo_dir(std::integral_constant<int, 2>{});
        halo_dir(std::integral_constant<int, 3>{});
        halo_dir(std::integral_constant<int, 4>{});
        halo_dir(std::integral_constant<int, 5>{});
        // K steps, then the 27 tiles' values out
        uint32_t w[8];
        if constexpr (kClBoxes == 2)
            cluster_steps2<CONWAY, kClBoxW, ClBox<F>::kM>(box, s_box[pipe][1], s_exist[pipe], s_sq, K, s_cb, s_bidx, s_tb,
                                                          cw.rule, w);
        else
            cluster_steps<CONWAY, kClBoxW, ClBox<F>::kM>(box, s_exist[pipe], s_sq, K, s_cb, s_bidx, s_tb, cw.rule, w);
        if (kClLoaderStores) {  // to the loader: wait until it took the previous result
            if (i >= 1) mbar_wait(&s_obar[pipe][1], (i - 1u) & 1u);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < 7 || k7) s_out[pipe][32 * k + lane] = w[k];
            asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&s_obar[pipe][0])) : "memory");
            continue;
        }
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
    }  // stepper
    if (P2P) p2p_arrive(p);  // after the CTA's last store (the loader's)
}

}  // namespace nbbgpu
