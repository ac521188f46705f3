// bits_kernels.cuh — CA on a bit-packed embedded alive grid (cell_width = 0).
//
// The reference CA reads only `cell != 0` and writes 0/1 (dispatch.cpp:542,
// 548-549), so one bit per cell of the same row-major n x n embedding (word
// index y*(n/32) + x/32, bit x%32) is an exact device-side state. A ρ = 32 tile
// row is exactly one 32-bit word, so the λ(ω) tile kernel becomes: lane = row,
// one LDG.32 + one STG.32 per lane, the ≤ 8 halo cells, and the bit-sliced rule
// of common.cuh. The touched set of one step at n = 2^16 is 95.6 MB of 128-byte
// lines (read) + 53.7 MB of sectors (write), so consecutive steps run largely
// out of the 126 MB L2. Conversions to/from the int64 Grid happen once per
// run_ca call (pack / unpack below).
#pragma once

#include "common.cuh"
#include "tile_kernels.cuh"

namespace nbbgpu {

// ILP tiles per warp iteration (loads of all issued before any compute)
template <bool BB, int ILP>
__global__ void __launch_bounds__(256) ca_bits_kernel(TileArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t n = a.n;
    const uint32_t nm1 = (uint32_t)(n - 1);
    const uint32_t wpr = (uint32_t)(n >> 5);  // words per row
    const uint32_t* src = static_cast<const uint32_t*>(a.src);
    uint32_t* dst = static_cast<uint32_t*>(a.dst);
    const uint32_t warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t warp_stride = (gridDim.x * blockDim.x) >> 5;
    const uint32_t units = (a.tiles + ILP - 1) / ILP;

    // halo cell handled by this lane (lanes 0..7): tile-local offsets
    const uint32_t hk = (uint32_t)lane & 7u;
    const int hx = (hk == 0 || hk == 3) ? -1 : (hk == 1 || hk == 7) ? 0 : (hk == 2) ? 1 : 32;
    const int hy = (hk <= 2) ? -1 : (hk == 3 || hk == 5) ? 31 : (hk == 4) ? 30 : 32;

    // BB: odd warp stride (see tile_kernel) and whole-tile culling: a bounding-box tile holds a
    // member iff bx ⊆ (n/32 - 1 - by); a unit without one is skipped (warp-uniform)
    const uint32_t ustride = BB ? (warp_stride | 1u) - ((warp_stride & 1u) ? 0u : 2u) : warp_stride;
    const uint32_t ustart = (BB && warp_global >= ustride) ? units : warp_global;
    for (uint32_t u = ustart; u < units; u += ustride) {
        if (BB) {
            bool any = false;
#pragma unroll
            for (int i = 0; i < ILP; ++i) {
                const uint32_t tl = u * ILP + i;
                const uint32_t t = a.tile_begin + tl;
                const uint32_t gy = fastdiv(t, a.div_gw), gx = t - gy * a.gw;
                any |= tl < a.tiles && (gx & ((nm1 >> 5) - gy)) == 0u;
            }
            if (!any) continue;
        }
        uint32_t X0[ILP], Y0[ILP], memb[ILP], R[ILP], hw[ILP];
        bool ok[ILP], hact[ILP];
        uint32_t hbitpos[ILP];
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            const uint32_t tl = u * ILP + i;
            ok[i] = tl < a.tiles;
            const uint32_t t = a.tile_begin + (ok[i] ? tl : 0u);
            const uint32_t gy = fastdiv(t, a.div_gw);
            const uint32_t gx = t - gy * a.gw;
            uint32_t bx, by;
            if (BB) {
                bx = gx;
                by = gy;
            } else {
                lambda_const(gx, gy, bx, by);
            }
            X0[i] = bx * 32;
            Y0[i] = by * 32;
            if (BB) {
                const uint32_t Yc = nm1 - (Y0[i] + lane);
                memb[i] = ((X0[i] & Yc) == 0u) ? submask_bits((~Yc) & 31u) : 0u;
            } else {
                memb[i] = submask_bits((uint32_t)lane);
            }
            if (!ok[i]) memb[i] = 0;
            R[i] = memb[i] ? __ldg(src + (size_t)(Y0[i] + lane) * wpr + bx) : 0u;
            // halo
            const int64_t gxh = (int64_t)X0[i] + hx, gyh = (int64_t)Y0[i] + hy;
            hact[i] = lane < 8 && ok[i] && gasket_member(gxh, gyh, n);
            hbitpos[i] = hact[i] ? (uint32_t)(gxh & 31) : 0u;
            hw[i] = hact[i] ? __ldg(src + (size_t)gyh * wpr + (uint32_t)(gxh >> 5)) : 0u;
        }
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            const uint32_t row = R[i] & memb[i];
            const uint32_t hbit = hact[i] ? ((hw[i] >> hbitpos[i]) & 1u) : 0u;
            const uint64_t h = __ballot_sync(0xFFFFFFFFu, hbit != 0u) & 0xFFu;
            uint64_t E = (uint64_t)row << 1;
            if (lane == 31) E |= ((h >> 3) & 1u) | (((h >> 5) & 1u) << 33);
            if (lane == 30) E |= ((h >> 4) & 1u) << 33;
            const uint64_t top = (h & 1u) | (((h >> 1) & 1u) << 1) | (((h >> 2) & 1u) << 2);
            const uint64_t bottom = (((h >> 7) & 1u) << 1) | (((h >> 6) & 1u) << 33);
            const uint64_t Eu = __shfl_up_sync(0xFFFFFFFFu, E, 1);
            const uint64_t Ed = __shfl_down_sync(0xFFFFFFFFu, E, 1);
            const uint64_t U = lane == 0 ? top : Eu;
            const uint64_t D = lane == 31 ? bottom : Ed;
            if (memb[i]) {
                const uint32_t nrow =
                    life_rule((uint32_t)U, (uint32_t)(U >> 1), (uint32_t)(U >> 2), (uint32_t)E,
                              (uint32_t)(E >> 2), (uint32_t)D, (uint32_t)(D >> 1), (uint32_t)(D >> 2),
                              (uint32_t)(E >> 1), a.birth, a.survive) &
                    memb[i];
                dst[(size_t)(Y0[i] + lane) * wpr + (X0[i] >> 5)] = nrow;
            }
        }
    }
}

// clear the non-member bits of a bit grid
__global__ void sanitize_bits_kernel(uint32_t* bits, int64_t n) {
    const uint64_t wpr = (uint64_t)(n >= 32 ? n / 32 : 1);
    const uint64_t total = (uint64_t)n * wpr;
    const uint32_t nm1 = (uint32_t)(n - 1);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t Y = (uint32_t)(i / wpr);
        const uint32_t X = (uint32_t)(i % wpr) * 32u;
        const uint32_t Yc = nm1 - Y;
        uint32_t memb = ((X & Yc) == 0u) ? submask_bits((~Yc) & 31u) : 0u;
        if (n < 32) memb &= (1u << n) - 1u;
        const uint32_t w = bits[i];
        if (w & ~memb) bits[i] = w & memb;
    }
}

// int64 grid -> bit grid (every word written; non-member bits 0). One thread per word.
__global__ void pack_bits_kernel(const long long* g64, uint32_t* bits, int64_t n) {
    const uint64_t wpr = (uint64_t)(n >= 32 ? n / 32 : 1);
    const uint64_t total = (uint64_t)n * wpr;
    const uint32_t nm1 = (uint32_t)(n - 1);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t Y = (uint32_t)(i / wpr);
        const uint32_t X = (uint32_t)(i % wpr) * 32u;
        uint32_t w = 0;
        if (n < 32) {
            for (int64_t x = 0; x < n; ++x)
                if (gasket_member(x, Y, n) && g64[(int64_t)Y * n + x] != 0) w |= 1u << x;
        } else {
            const uint32_t Yc = nm1 - Y;
            const uint32_t memb = ((X & Yc) == 0u) ? submask_bits((~Yc) & 31u) : 0u;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t nib = (memb >> (4 * q)) & 0xFu;
                if (nib) w |= (alive4_i64(ld_sector(g64 + (int64_t)Y * n + X + 4 * q)) & nib) << (4 * q);
            }
        }
        bits[i] = w;
    }
}

// bit grid -> member sectors of an int64 grid whose non-member cells are already 0.
__global__ void unpack_bits_kernel(const uint32_t* bits, long long* g64, int64_t n) {
    const uint64_t wpr = (uint64_t)(n >= 32 ? n / 32 : 1);
    const uint64_t total = (uint64_t)n * wpr;
    const uint32_t nm1 = (uint32_t)(n - 1);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t Y = (uint32_t)(i / wpr);
        const uint32_t X = (uint32_t)(i % wpr) * 32u;
        if (n < 32) {
            const uint32_t w = bits[i];
            for (int64_t x = 0; x < n; ++x)
                if (gasket_member(x, Y, n)) g64[(int64_t)Y * n + x] = (w >> x) & 1u;
            continue;
        }
        const uint32_t Yc = nm1 - Y;
        const uint32_t memb = ((X & Yc) == 0u) ? submask_bits((~Yc) & 31u) : 0u;
        if (!memb) continue;
        const uint32_t w = bits[i] & memb;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if ((memb >> (4 * q)) & 0xFu)
                stg_sector(g64 + (int64_t)Y * n + X + 4 * q, expand4_i64((w >> (4 * q)) & 0xFu));
        }
    }
}

}  // namespace nbbgpu
