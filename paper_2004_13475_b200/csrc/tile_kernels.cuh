// tile_kernels.cuh — the hot path: one warp per rho x rho tile, 32-byte sectors.
//
// Replaces the two launch loops of nbb::launch_impl (dispatch.cpp:209-467) for
// the three reference workloads (run_single_write / run_reduction / run_ca,
// dispatch.cpp:481-557) with the (subbox strategy, direct backend) semantics:
//
//   λ mode : tile t of the compact orthotope (W x H = 3^ceil(r_b/2) x 3^floor(r_b/2),
//            ordinal t = ωy*W + ωx, dispatch.cpp:262-263) sits at ρ·λ(ω)
//            (dispatch.cpp:309,355); its member cells are the local bit test
//            tx & (ρ-1-ty) == 0, i.e. tx ⊆ ty.
//   BB mode: tile t of the (n/ρ)^2 bounding box at ρ·(t % (n/ρ), t / (n/ρ)); every
//            sector tests its own membership (dispatch.cpp:278-300 semantics).
//
// Data layout (HBM): the reference's dense row-major embedded grid
// (dispatch.hpp:74-79), int64 (drop-in) or uint8 cells. A 32-byte sector holds
// CPS = 32/sizeof(cell) cells; only sectors that contain a member are read or
// written (the layout minimum). Whole sectors are written, with 0
// in co-resident non-member cells: value-identical because non-member cells are
// 0 in every SW/CA output (dispatch.cpp:530) and it avoids partial-sector RMW.
//
// Work decomposition: a warp owns TPW = 32/ρ consecutive tiles ("unit"); its
// lanes hold a fixed list of (row, sector) slots, identical for every λ tile and
// precomputed once (consecutive lanes on consecutive sectors of a row, so each
// 128-byte line is one L1 wavefront). CA gathers alive bits into one 32-bit word
// per row (lane = row), evaluates the rule bit-sliced (life_rule) with the 8
// possible halo cells of the tile, and scatters the new rows back as sectors.
// Warps are persistent and stride over units so that co-resident warps work on
// neighbouring ordinals (their halos hit in L2).
#pragma once

#include "common.cuh"

namespace nbbgpu {

enum TileOp { OP_SW = 0, OP_RD = 1, OP_CA = 2 };

struct TileArgs {
    const void* src;               // RD/CA source grid
    void* dst;                     // SW/CA destination grid
    unsigned long long* sum;       // RD accumulator (device, pre-zeroed)
    int64_t n;                     // embedding side 2^r
    uint32_t tile_begin;           // first tile ordinal (multi-device shard)
    uint32_t tiles;                // tiles in this launch
    uint32_t gw;                   // W (λ) or n/ρ (BB)
    FastDiv div_gw;                // ordinal -> (x, y)
    uint32_t birth, survive;       // CA rule masks (dispatch.hpp:131-134)
};

template <typename Cell, int RHO>
struct TileShape {
    static constexpr int CPS = 32 / (int)sizeof(Cell);          // cells per sector
    static constexpr int LOGC = (CPS == 4) ? 2 : 5;
    static constexpr int SPR = RHO / CPS;                        // sectors per tile row
    static constexpr int TPW = 32 / RHO;                         // tiles per warp
    static constexpr int popc(unsigned v) { return v == 0u ? 0 : (int)(v & 1u) + popc(v >> 1); }
    static constexpr int member_sectors() {
        int c = 0;
        for (int y = 0; y < RHO; ++y) c += 1 << popc((unsigned)(y >> LOGC));
        return c;
    }
    static constexpr int MS = member_sectors();
    static constexpr int SLOTS_L = (TPW * MS + 31) / 32;         // λ slots per lane
    static constexpr int SLOTS_B = SPR;                          // BB slots per lane
    static_assert(SPR >= 1, "tile narrower than a sector");
};

// k-th submask (increasing order) of m, i.e. pdep(k, m) for small masks.
__device__ __forceinline__ uint32_t kth_submask(uint32_t k, uint32_t m) {
    uint32_t r = 0;
    for (uint32_t bit = 1; m != 0u; m &= m - 1u) {
        const uint32_t low = m & (0u - m);
        if (k & bit) r |= low;
        bit <<= 1;
    }
    return r;
}

template <typename Cell, int RHO, int OP, bool BB>
__global__ void __launch_bounds__(256) tile_kernel(TileArgs a) {
    using S = TileShape<Cell, RHO>;
    constexpr int CPS = S::CPS, LOGC = S::LOGC, SPR = S::SPR, TPW = S::TPW;
    constexpr int SLOTS = BB ? S::SLOTS_B : S::SLOTS_L;
    constexpr int WARPS = 8;
    constexpr bool BYTE_STAGE = (CPS == 4);  // int64: nibbles staged through smem

    __shared__ uint8_t s_nib[WARPS][BYTE_STAGE ? 32 * SPR : 1];
    __shared__ uint32_t s_row[WARPS][BYTE_STAGE ? 32 : 1];

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t n = a.n;
    const uint32_t nm1 = (uint32_t)(n - 1);  // n <= 2^17 on this path

    // ---- per-lane static slot table ---------------------------------------
    uint32_t sl_rw[SLOTS];   // row in the warp's 32-row space (tile*RHO + y)
    uint32_t sl_s[SLOTS];    // sector within the row
    uint32_t sl_nib[SLOTS];  // λ: member cells of the sector
    int64_t sl_off[SLOTS];   // byte offset within the tile
    uint32_t valid = 0;
#pragma unroll
    for (int k = 0; k < SLOTS; ++k) {
        const uint32_t e = (uint32_t)(k * 32 + lane);
        uint32_t j = 0, y = 0, s = 0;
        bool ok;
        if (BB) {
            ok = e < (uint32_t)(32 * SPR);
            j = e / (RHO * SPR);
            const uint32_t rem = e % (RHO * SPR);
            y = rem / SPR;
            s = rem % SPR;
        } else {
            ok = e < (uint32_t)(TPW * S::MS);
            j = e / S::MS;
            uint32_t f = e % S::MS;
            for (y = 0; y < (uint32_t)RHO; ++y) {
                const uint32_t cnt = 1u << __popc(y >> LOGC);
                if (f < cnt) break;
                f -= cnt;
            }
            if (ok) s = kth_submask(f, y >> LOGC);
        }
        if (!ok) j = y = s = 0;
        sl_rw[k] = j * RHO + y;
        sl_s[k] = s;
        sl_nib[k] = ok ? (submask_bits(y & (CPS - 1)) & (CPS == 32 ? 0xFFFFFFFFu : ((1u << CPS) - 1u))) : 0u;
        sl_off[k] = ((int64_t)y * n + (int64_t)s * CPS) * (int64_t)sizeof(Cell);
        valid |= (ok ? 1u : 0u) << k;
    }
    if (BYTE_STAGE && !BB) {
        for (int i = lane; i < 32 * SPR; i += 32) s_nib[wib][i] = 0;  // non-member sectors stay 0
    }
    __syncwarp();

    // compute-stage identity of this lane
    const uint32_t my_j = (uint32_t)lane / RHO;
    const uint32_t my_y = (uint32_t)lane % RHO;
    const uint32_t rowmask = (RHO == 32) ? 0xFFFFFFFFu : ((1u << RHO) - 1u);

    unsigned long long acc = 0;
    const uint32_t units = (a.tiles + TPW - 1) / TPW;
    const uint32_t warp_global = (blockIdx.x * (blockDim.x >> 5)) + (uint32_t)wib;
    const uint32_t warp_stride = gridDim.x * (blockDim.x >> 5);

    const char* src = static_cast<const char*>(a.src);
    char* dst = static_cast<char*>(a.dst);

    // BB: an odd warp stride (one warp idles when the grid's warp count is even). The bounding
    // box's member tiles are bx ⊆ (n/ρ - 1 - by); with an even stride (a multiple of a large
    // power of two) a warp would always see the same low bits of bx and the members would
    // pile onto a few warps (ncu: 11-15% warps active); an odd stride cycles every residue.
    const uint32_t ustride = BB ? (warp_stride | 1u) - ((warp_stride & 1u) ? 0u : 2u) : warp_stride;
    const uint32_t ustart = (BB && warp_global >= ustride) ? units : warp_global;
    for (uint32_t u = ustart; u < units; u += ustride) {
        // ---- tile origins (lane computes its own tile j = lane / RHO) ----------
        const uint32_t t_local = u * TPW + my_j;
        const bool my_tile_ok = t_local < a.tiles;
        const uint32_t t = a.tile_begin + (my_tile_ok ? t_local : 0u);
        const uint32_t gy = fastdiv(t, a.div_gw);
        const uint32_t gx = t - gy * a.gw;
        uint32_t bx, by;
        if (BB) {
            bx = gx;
            by = gy;
        } else {
            lambda_const(gx, gy, bx, by);
        }
        const uint32_t X0 = bx * RHO, Y0 = by * RHO;
        const int64_t my_base = ((int64_t)Y0 * n + X0) * (int64_t)sizeof(Cell);
        // BB: a tile of the bounding box holds a member iff bx ⊆ (n/ρ - 1 - by) (its cell
        // (X0, Y0 + ρ - 1) is then one); the reference's threads of such a block all fail
        // their membership test and return, so the warp skips the tile outright
        const bool has_member = !BB || (bx & ((nm1 >> (31 - __clz(RHO))) - by)) == 0u;
        const uint32_t tiles_ok = __ballot_sync(0xFFFFFFFFu, my_tile_ok && has_member && my_y == 0);
        if (BB && tiles_ok == 0u) continue;

        // ---- stage 1: loads / stores of the slots ----------------------------
        uint32_t slot_nib[SLOTS];
        int64_t slot_base[SLOTS];
#pragma unroll
        for (int k = 0; k < SLOTS; ++k) {
            const uint32_t jk = sl_rw[k] / RHO;
            slot_base[k] = __shfl_sync(0xFFFFFFFFu, my_base, (int)(jk * RHO));
            uint32_t nib = sl_nib[k];
            if (BB) {
                const uint32_t X0k = __shfl_sync(0xFFFFFFFFu, X0, (int)(jk * RHO));
                const uint32_t Y0k = __shfl_sync(0xFFFFFFFFu, Y0, (int)(jk * RHO));
                const uint32_t Y = Y0k + (sl_rw[k] % RHO);
                const uint32_t Yc = nm1 - Y;  // n-1-Y
                const uint32_t X = X0k + sl_s[k] * CPS;
                const uint32_t cm = (CPS == 32) ? 0xFFFFFFFFu : ((1u << CPS) - 1u);
                nib = (((X & Yc) == 0u) ? (submask_bits((~Yc) & (CPS - 1)) & cm) : 0u);
            }
            const bool act = ((valid >> k) & 1u) && ((tiles_ok >> (jk * RHO)) & 1u) && nib != 0u;
            slot_nib[k] = act ? nib : 0u;
        }

        if (OP == OP_SW) {
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) {
                if (slot_nib[k]) {
                    const Sector v = (CPS == 4) ? expand4_i64(slot_nib[k]) : expand32_u8(slot_nib[k]);
                    stg_sector(dst + slot_base[k] + sl_off[k], v);
                }
            }
            continue;
        }
        if (OP == OP_RD) {
            // all of the unit's loads in flight before the first add (the predicated
            // load-add pairs would otherwise serialise one DRAM round trip per slot)
            Sector v[SLOTS];
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) {
                if (slot_nib[k]) v[k] = ldg_sector(src + slot_base[k] + sl_off[k]);
            }
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) {
                if (slot_nib[k]) acc += masked_sum4(v[k], slot_nib[k]);
            }
            continue;
        }

        // ---- OP_CA ---------------------------------------------------------------
        // stage 1a: gather alive bits
        uint32_t alive_row = 0;  // CPS == 32: this lane's row (slot 0 is row = lane)
        {
            Sector v[SLOTS];
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) {
                if (slot_nib[k]) v[k] = ldg_sector(src + slot_base[k] + sl_off[k]);
            }
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) {
                if (BYTE_STAGE) {
                    const uint32_t bits = slot_nib[k] ? (alive4_i64(v[k]) & slot_nib[k]) : 0u;
                    if (BB || ((valid >> k) & 1u)) s_nib[wib][sl_rw[k] * SPR + sl_s[k]] = (uint8_t)bits;
                } else {
                    alive_row = slot_nib[k] ? (alive32_u8(v[k]) & slot_nib[k]) : 0u;
                }
            }
        }
        // stage 1b: the 8 halo cells of each tile
        uint32_t hbit = 0;
        {
            // every lane participates in the shuffles; lanes >= 8*TPW ignore the result
            const uint32_t hj = ((uint32_t)lane >> 3) % TPW;
            const uint32_t X0h = __shfl_sync(0xFFFFFFFFu, X0, (int)(hj * RHO));
            const uint32_t Y0h = __shfl_sync(0xFFFFFFFFu, Y0, (int)(hj * RHO));
            const bool tile_h_ok = (tiles_ok >> (hj * RHO)) & 1u;
            if (lane < 8 * TPW && tile_h_ok) {
                const uint32_t hk = (uint32_t)lane & 7u;
                const int hx = (hk == 0 || hk == 3) ? -1 : (hk == 1 || hk == 7) ? 0 : (hk == 2) ? 1 : RHO;
                const int hy = (hk <= 2) ? -1 : (hk == 3 || hk == 5) ? RHO - 1 : (hk == 4) ? RHO - 2 : RHO;
                const int64_t gxh = (int64_t)X0h + hx, gyh = (int64_t)Y0h + hy;
                if (gasket_member(gxh, gyh, n)) {
                    const Cell* p = reinterpret_cast<const Cell*>(src) + gyh * n + gxh;
                    hbit = (__ldg(p) != (Cell)0) ? 1u : 0u;
                }
            }
        }
        const uint32_t hmask = __ballot_sync(0xFFFFFFFFu, hbit != 0u);
        __syncwarp();

        // stage 2: bit-sliced rule, lane = row my_y of tile my_j
        uint32_t R;
        if (BYTE_STAGE) {
            if (SPR == 8) {
                uint64_t x = *reinterpret_cast<const uint64_t*>(&s_nib[wib][lane * 8]);
                x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
                x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
                x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
                R = (uint32_t)x;
            } else if (SPR == 4) {
                uint32_t x = *reinterpret_cast<const uint32_t*>(&s_nib[wib][lane * 4]);
                x = (x | (x >> 4)) & 0x00FF00FFu;
                x = (x | (x >> 8)) & 0x0000FFFFu;
                R = x;
            } else {
                uint32_t x = *reinterpret_cast<const uint16_t*>(&s_nib[wib][lane * 2]);
                x = (x | (x >> 4)) & 0xFFu;
                R = x;
            }
        } else {
            R = alive_row;
        }
        const uint32_t hb = (hmask >> (my_j * 8)) & 0xFFu;
        const uint64_t h = hb;
        uint64_t E = (uint64_t)R << 1;
        if (my_y == RHO - 1) E |= (h >> 3) & 1u;                       // (-1, ρ-1)
        if (my_y == RHO - 2) E |= ((h >> 4) & 1u) << (RHO + 1);        // (ρ, ρ-2)
        if (my_y == RHO - 1) E |= ((h >> 5) & 1u) << (RHO + 1);        // (ρ, ρ-1)
        const uint64_t top = (h & 1u) | (((h >> 1) & 1u) << 1) | (((h >> 2) & 1u) << 2);
        const uint64_t bottom = (((h >> 7) & 1u) << 1) | (((h >> 6) & 1u) << (RHO + 1));
        const uint64_t Eu = __shfl_up_sync(0xFFFFFFFFu, E, 1);
        const uint64_t Ed = __shfl_down_sync(0xFFFFFFFFu, E, 1);
        const uint64_t U = (my_y == 0) ? top : Eu;
        const uint64_t D = (my_y == RHO - 1) ? bottom : Ed;
        uint32_t memb;
        if (BB) {
            const uint32_t Yc = nm1 - (Y0 + my_y);
            memb = ((X0 & Yc) == 0u) ? (submask_bits((~Yc) & (RHO - 1)) & rowmask) : 0u;
        } else {
            memb = submask_bits(my_y) & rowmask;
        }
        if (!my_tile_ok) memb = 0;
        uint32_t nrow = 0;
        if (memb != 0u) {
            nrow = life_rule((uint32_t)U, (uint32_t)(U >> 1), (uint32_t)(U >> 2), (uint32_t)E,
                             (uint32_t)(E >> 2), (uint32_t)D, (uint32_t)(D >> 1), (uint32_t)(D >> 2),
                             (uint32_t)(E >> 1), a.birth, a.survive) &
                   memb;
        }

        // stage 3: scatter new rows as sectors
        if (BYTE_STAGE) {
            s_row[wib][lane] = nrow;
            __syncwarp();
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) {
                if (slot_nib[k]) {
                    const uint32_t w = s_row[wib][sl_rw[k]];
                    const uint32_t nib = (w >> (sl_s[k] * CPS)) & 0xFu;
                    stg_sector(dst + slot_base[k] + sl_off[k], expand4_i64(nib));
                }
            }
            __syncwarp();
        } else {
            if (slot_nib[0]) stg_sector(dst + slot_base[0] + sl_off[0], expand32_u8(nrow));
        }
    }

    if (OP == OP_RD) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
        if (lane == 0 && acc != 0ull) atomicAdd(a.sum, acc);
    }
}

}  // namespace nbbgpu
