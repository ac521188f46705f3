// ca_pipe_kernel.cuh — the CA step as a warp-private cp.async pipeline.
//
// Same decomposition and arithmetic as the CA path of tile_kernel
// (tile_kernels.cuh): a warp owns TPW = 32/ρ tiles per unit, lanes hold a fixed
// slot list of member sectors, the rule is evaluated bit-sliced with lane = row.
// The difference is latency hiding: loads no longer land in registers. Each
// warp streams its units through a STAGES-deep ring in shared memory with
// cp.async (16-byte .cg copies, zero-filled when the slot is inactive, 8/4-byte
// .ca copies for the ≤ 8 halo cells), so STAGES-1 units are in flight while one
// is computed and stored. Measured motivation: the
// register-staged kernel was latency-bound (25% occupancy, 80% L1TEX stalls).
#pragma once

#include "common.cuh"
#include "tile_kernels.cuh"

namespace nbbgpu {

__device__ __forceinline__ void cp_async16(uint32_t smem, const void* gmem, bool pred) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem), "l"(gmem),
                 "r"(pred ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t smem, const void* gmem, bool pred) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem), "l"(gmem),
                 "r"(pred ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t smem, const void* gmem, bool pred) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem), "l"(gmem),
                 "r"(pred ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename Cell, int RHO, bool BB, int STAGES, int WARPS>
struct CaPipeShape {
    using S = TileShape<Cell, RHO>;
    static constexpr int SLOTS = BB ? S::SLOTS_B : S::SLOTS_L;
    static constexpr int SECTOR_BYTES = STAGES * SLOTS * 32 * 32;  // per warp
    static constexpr int HALO_BYTES = STAGES * 32 * 8;
    static constexpr int NIB_BYTES = (S::CPS == 4) ? 32 * S::SPR : 0;
    static constexpr int ROW_BYTES = (S::CPS == 4) ? 32 * 4 : 0;
    static constexpr int WARP_BYTES = SECTOR_BYTES + HALO_BYTES + NIB_BYTES + ROW_BYTES;
    static constexpr int SMEM = WARPS * WARP_BYTES;
};

template <typename Cell, int RHO, bool BB, int STAGES, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) ca_pipe_kernel(TileArgs a) {
    using S = TileShape<Cell, RHO>;
    using P = CaPipeShape<Cell, RHO, BB, STAGES, WARPS>;
    constexpr int CPS = S::CPS, LOGC = S::LOGC, SPR = S::SPR, TPW = S::TPW;
    constexpr int SLOTS = P::SLOTS;
    constexpr bool BYTE_STAGE = (CPS == 4);
    constexpr uint32_t CM = CPS == 32 ? 0xFFFFFFFFu : ((1u << CPS) - 1u);

    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    uint8_t* wbase = smem_raw + wib * P::WARP_BYTES;
    uint8_t* s_sec = wbase;                                   // [STAGES][SLOTS][32 lanes][32 B]
    uint8_t* s_halo = wbase + P::SECTOR_BYTES;                // [STAGES][32 lanes][8 B]
    uint8_t* s_nib = s_halo + P::HALO_BYTES;                  // [32 rows][SPR]
    uint32_t* s_row = reinterpret_cast<uint32_t*>(s_nib + P::NIB_BYTES);  // [32]
    const uint32_t s_sec_u = (uint32_t)__cvta_generic_to_shared(s_sec);
    const uint32_t s_halo_u = (uint32_t)__cvta_generic_to_shared(s_halo);

    const int64_t n = a.n;
    const uint32_t nm1 = (uint32_t)(n - 1);

    // ---- static slot table (identical for every λ tile) ----------------------
    uint32_t sl_pack[SLOTS];  // rw | s << 5
    uint32_t sl_nib[SLOTS];
    uint32_t sl_off[SLOTS];   // byte offset within the tile (< 2^25 for n <= 2^17)
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
        sl_pack[k] = (j * RHO + y) | (s << 5);
        sl_nib[k] = ok ? (submask_bits(y & (CPS - 1)) & CM) : 0u;
        sl_off[k] = (uint32_t)(((int64_t)y * n + (int64_t)s * CPS) * (int64_t)sizeof(Cell));
        valid |= (ok ? 1u : 0u) << k;
    }
    if (BYTE_STAGE) {
        for (int i = lane; i < 32 * SPR; i += 32) s_nib[i] = 0;  // non-member sectors stay 0
    }
    __syncwarp();

    const uint32_t my_j = (uint32_t)lane / RHO;
    const uint32_t my_y = (uint32_t)lane % RHO;
    const uint32_t rowmask = (RHO == 32) ? 0xFFFFFFFFu : ((1u << RHO) - 1u);
    const uint32_t units = (a.tiles + TPW - 1) / TPW;
    const uint32_t warp_global = blockIdx.x * WARPS + (uint32_t)wib;
    const uint32_t warp_stride = gridDim.x * WARPS;
    const char* src = static_cast<const char*>(a.src);
    char* dst = static_cast<char*>(a.dst);

    // halo cell of this lane (lanes < 8*TPW): tile j = lane/8, position lane%8
    const uint32_t hk = (uint32_t)lane & 7u;
    const int hx = (hk == 0 || hk == 3) ? -1 : (hk == 1 || hk == 7) ? 0 : (hk == 2) ? 1 : RHO;
    const int hy = (hk <= 2) ? -1 : (hk == 3 || hk == 5) ? RHO - 1 : (hk == 4) ? RHO - 2 : RHO;
    const uint32_t hj = ((uint32_t)lane >> 3) % TPW;

    // tile origin of this lane's tile for unit u
    auto origin = [&](uint32_t u, uint32_t& X0, uint32_t& Y0, bool& ok) {
        const uint32_t t_local = u * TPW + my_j;
        ok = t_local < a.tiles;
        const uint32_t t = a.tile_begin + (ok ? t_local : 0u);
        const uint32_t gy = fastdiv(t, a.div_gw);
        const uint32_t gx = t - gy * a.gw;
        uint32_t bx, by;
        if (BB) {
            bx = gx;
            by = gy;
        } else {
            lambda_const(gx, gy, bx, by);
        }
        X0 = bx * RHO;
        Y0 = by * RHO;
    };
    // active-sector nibble of slot k for the tile origin (X0k, Y0k)
    auto slot_nib = [&](int k, uint32_t X0k, uint32_t Y0k, bool tile_ok) -> uint32_t {
        uint32_t nib = sl_nib[k];
        if (BB) {
            const uint32_t Y = Y0k + ((sl_pack[k] & 31u) % RHO);
            const uint32_t Yc = nm1 - Y;
            const uint32_t X = X0k + (sl_pack[k] >> 5) * CPS;
            nib = ((X & Yc) == 0u) ? (submask_bits((~Yc) & (CPS - 1)) & CM) : 0u;
        }
        return (((valid >> k) & 1u) && tile_ok) ? nib : 0u;
    };

    auto issue = [&](uint32_t u, int st) {
        uint32_t X0, Y0;
        bool ok;
        origin(u, X0, Y0, ok);
        const int64_t my_base = ((int64_t)Y0 * n + X0) * (int64_t)sizeof(Cell);
#pragma unroll
        for (int k = 0; k < SLOTS; ++k) {
            const uint32_t jk = (sl_pack[k] & 31u) / RHO;
            const int64_t base = __shfl_sync(0xFFFFFFFFu, my_base, (int)(jk * RHO));
            const uint32_t X0k = __shfl_sync(0xFFFFFFFFu, X0, (int)(jk * RHO));
            const uint32_t Y0k = __shfl_sync(0xFFFFFFFFu, Y0, (int)(jk * RHO));
            const bool okk = __shfl_sync(0xFFFFFFFFu, ok, (int)(jk * RHO));
            const bool act = slot_nib(k, X0k, Y0k, okk) != 0u;
            const char* g = src + base + sl_off[k];
            const uint32_t sp = s_sec_u + (uint32_t)(((st * SLOTS + k) * 32 + lane) * 32);
            cp_async16(sp, act ? g : src, act);
            cp_async16(sp + 16, act ? g + 16 : src, act);
        }
        {
            const uint32_t X0h = __shfl_sync(0xFFFFFFFFu, X0, (int)(hj * RHO));
            const uint32_t Y0h = __shfl_sync(0xFFFFFFFFu, Y0, (int)(hj * RHO));
            const bool okh = __shfl_sync(0xFFFFFFFFu, ok, (int)(hj * RHO));
            const int64_t gx = (int64_t)X0h + hx, gy = (int64_t)Y0h + hy;
            const bool act = lane < 8 * TPW && okh && gasket_member(gx, gy, n);
            const uint32_t hp = s_halo_u + (uint32_t)((st * 32 + lane) * 8);
            if (sizeof(Cell) == 8) {
                const char* g = act ? src + (gy * n + gx) * 8 : src;
                cp_async8(hp, g, act);
            } else {
                const int64_t idx = act ? gy * n + gx : 0;
                cp_async4(hp, src + (idx & ~(int64_t)3), act);
            }
        }
    };

    // prologue: STAGES-1 units in flight
    uint32_t u_issue = warp_global;
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (u_issue < units) issue(u_issue, st);
        cp_async_commit();
        u_issue += warp_stride;
    }

    int st = 0;
    for (uint32_t u = warp_global; u < units; u += warp_stride) {
        // keep the ring full: issue unit u + (STAGES-1)*stride into the slot freed last round
        {
            const int st_issue = (st + STAGES - 1) % STAGES;
            if (u_issue < units) issue(u_issue, st_issue);
            cp_async_commit();
            u_issue += warp_stride;
        }
        cp_async_wait<STAGES - 1>();
        __syncwarp();

        uint32_t X0, Y0;
        bool my_ok;
        origin(u, X0, Y0, my_ok);
        const int64_t my_base = ((int64_t)Y0 * n + X0) * (int64_t)sizeof(Cell);
        const uint32_t tiles_ok = __ballot_sync(0xFFFFFFFFu, my_ok && my_y == 0);

        // stage A: alive bits of the slots
        uint32_t alive_row = 0;
        uint32_t act_nib[SLOTS];
        int64_t slot_base[SLOTS];
#pragma unroll
        for (int k = 0; k < SLOTS; ++k) {
            const uint32_t jk = (sl_pack[k] & 31u) / RHO;
            slot_base[k] = __shfl_sync(0xFFFFFFFFu, my_base, (int)(jk * RHO));
            const uint32_t X0k = __shfl_sync(0xFFFFFFFFu, X0, (int)(jk * RHO));
            const uint32_t Y0k = __shfl_sync(0xFFFFFFFFu, Y0, (int)(jk * RHO));
            act_nib[k] = slot_nib(k, X0k, Y0k, (tiles_ok >> (jk * RHO)) & 1u);
            const uint4* p = reinterpret_cast<const uint4*>(s_sec + ((st * SLOTS + k) * 32 + lane) * 32);
            const uint4 lo = p[0], hi = p[1];
            Sector v;
            v.w[0] = lo.x; v.w[1] = lo.y; v.w[2] = lo.z; v.w[3] = lo.w;
            v.w[4] = hi.x; v.w[5] = hi.y; v.w[6] = hi.z; v.w[7] = hi.w;
            if (BYTE_STAGE) {
                const uint32_t bits = act_nib[k] ? (alive4_i64(v) & act_nib[k]) : 0u;
                if (BB || ((valid >> k) & 1u))
                    s_nib[(sl_pack[k] & 31u) * SPR + (sl_pack[k] >> 5)] = (uint8_t)bits;
            } else {
                alive_row = act_nib[k] ? (alive32_u8(v) & act_nib[k]) : 0u;
            }
        }
        // halo bit of this lane
        uint32_t hbit = 0;
        if (sizeof(Cell) == 8 && lane < 8 * TPW) {
            const uint2 hv = *reinterpret_cast<const uint2*>(s_halo + (st * 32 + lane) * 8);
            hbit = (hv.x | hv.y) != 0u;
        }
        if (sizeof(Cell) == 1) {  // the 4-byte word holding the cell: pick its byte lane
            const uint32_t X0h = __shfl_sync(0xFFFFFFFFu, X0, (int)(hj * RHO));
            const uint32_t Y0h = __shfl_sync(0xFFFFFFFFu, Y0, (int)(hj * RHO));
            if (lane < 8 * TPW) {
                const int64_t gx = (int64_t)X0h + hx, gy = (int64_t)Y0h + hy;
                const bool act = gasket_member(gx, gy, n);
                const uint32_t w = *reinterpret_cast<const uint32_t*>(s_halo + (st * 32 + lane) * 8);
                const uint32_t bytelane = act ? (uint32_t)((gy * n + gx) & 3) : 0u;
                hbit = act && ((w >> (8 * bytelane)) & 0xFFu) != 0u;
            }
        }
        const uint32_t hmask = __ballot_sync(0xFFFFFFFFu, hbit != 0u);
        __syncwarp();

        // stage B: bit-sliced rule, lane = row my_y of tile my_j
        uint32_t R;
        if (BYTE_STAGE) {
            if (SPR == 8) {
                uint64_t x = *reinterpret_cast<const uint64_t*>(&s_nib[lane * 8]);
                x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
                x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
                x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
                R = (uint32_t)x;
            } else if (SPR == 4) {
                uint32_t x = *reinterpret_cast<const uint32_t*>(&s_nib[lane * 4]);
                x = (x | (x >> 4)) & 0x00FF00FFu;
                x = (x | (x >> 8)) & 0x0000FFFFu;
                R = x;
            } else {
                uint32_t x = *reinterpret_cast<const uint16_t*>(&s_nib[lane * 2]);
                x = (x | (x >> 4)) & 0xFFu;
                R = x;
            }
        } else {
            R = alive_row;
        }
        const uint64_t h = (hmask >> (my_j * 8)) & 0xFFu;
        uint64_t E = (uint64_t)R << 1;
        if (my_y == RHO - 1) E |= (h >> 3) & 1u;
        if (my_y == RHO - 2) E |= ((h >> 4) & 1u) << (RHO + 1);
        if (my_y == RHO - 1) E |= ((h >> 5) & 1u) << (RHO + 1);
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
        if (!my_ok) memb = 0;
        uint32_t nrow = 0;
        if (memb != 0u) {
            nrow = life_rule((uint32_t)U, (uint32_t)(U >> 1), (uint32_t)(U >> 2), (uint32_t)E,
                             (uint32_t)(E >> 2), (uint32_t)D, (uint32_t)(D >> 1), (uint32_t)(D >> 2),
                             (uint32_t)(E >> 1), a.birth, a.survive) &
                   memb;
        }

        // stage C: stores
        if (BYTE_STAGE) {
            s_row[lane] = nrow;
            __syncwarp();
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) {
                if (act_nib[k]) {
                    const uint32_t w = s_row[sl_pack[k] & 31u];
                    const uint32_t nib = (w >> ((sl_pack[k] >> 5) * CPS)) & 0xFu;
                    stg_sector(dst + slot_base[k] + sl_off[k], expand4_i64(nib));
                }
            }
        } else {
            if (act_nib[0]) stg_sector(dst + slot_base[0] + sl_off[0], expand32_u8(nrow));
        }
        __syncwarp();
        st = (st + 1) % STAGES;
    }
    cp_async_wait<0>();
}

}  // namespace nbbgpu
