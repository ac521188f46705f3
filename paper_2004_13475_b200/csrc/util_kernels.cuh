// util_kernels.cuh — grid preparation kernels and the λ map-only kernels.
//
//  sanitize       : zero every non-member cell (establishes the invariant the CA
//                   step relies on: non-member cells of both buffers are 0).
//  pack / unpack  : int64 grid <-> uint8 alive grid (CA only reads cell != 0 and
//                   writes 0/1, dispatch.cpp:542,548-549, so this is exact).
//  scatter        : member values in row-major member order -> embedded grid, the
//                   order random_member_grid fills (dispatch.cpp:141-147).
//  lambda_map     : K0, λ(ω) of a whole orthotope (block_map.cpp:77-111), scalar
//                   closed form with a shared-memory digit table, and K0-TC, the
//                   paper's tensor-core encoding (§6.3, mma.cpp:49-77)
//                   with ω along M so one m16n8k16 yields 16 coordinate pairs.
#pragma once

#include "common.cuh"
#include "percell_kernels.cuh"

#include <cuda_bf16.h>

namespace nbbgpu {

// ---- sanitize ---------------------------------------------------------------
template <typename Cell>
__global__ void sanitize_kernel(Cell* grid, int64_t n, int logn) {
    constexpr int CPS = 32 / (int)sizeof(Cell);
    const uint64_t spr = (uint64_t)n / CPS > 0 ? (uint64_t)n / CPS : 1;  // sectors per row
    const uint64_t total = (uint64_t)n * spr;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t nm1 = (uint32_t)(n - 1);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const uint32_t Y = (uint32_t)(i / spr);
        const uint32_t X = (uint32_t)(i % spr) * CPS;
        const uint32_t Yc = nm1 - Y;
        if (n < CPS) {  // tiny grids: cell by cell
            for (int64_t x = 0; x < n; ++x)
                if (!gasket_member(x, Y, n)) grid[(int64_t)Y * n + x] = (Cell)0;
            continue;
        }
        const uint32_t cm = CPS == 32 ? 0xFFFFFFFFu : ((1u << CPS) - 1u);
        const uint32_t memb = ((X & Yc) == 0u) ? (submask_bits((~Yc) & (CPS - 1)) & cm) : 0u;
        Cell* p = grid + (int64_t)Y * n + X;
        if (memb == cm) continue;
        Sector v;
        if (memb == 0u) {
#pragma unroll
            for (int k = 0; k < 8; ++k) v.w[k] = 0u;
        } else {
            v = ld_sector(p);
            if (CPS == 4) {
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (!((memb >> c) & 1u)) v.w[2 * c] = v.w[2 * c + 1] = 0u;
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t nib = (memb >> (4 * k)) & 0xFu;
                    v.w[k] &= (nib * 0x00204081u & 0x01010101u) * 0xFFu;
                }
            }
        }
        stg_sector(p, v);
    }
    (void)logn;
}

// ---- int64 <-> uint8 --------------------------------------------------------
// one thread per 32-cell run (one uint8 sector, eight int64 sectors)
__global__ void pack_alive_kernel(const long long* g64, unsigned char* g8, int64_t n) {
    const uint64_t runs_per_row = (uint64_t)(n >= 32 ? n / 32 : 1);
    const uint64_t total = (uint64_t)n * runs_per_row;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t nm1 = (uint32_t)(n - 1);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const uint32_t Y = (uint32_t)(i / runs_per_row);
        const uint32_t X = (uint32_t)(i % runs_per_row) * 32u;
        if (n < 32) {
            for (int64_t x = 0; x < n; ++x) {
                const int64_t idx = (int64_t)Y * n + x;
                g8[idx] = (gasket_member(x, Y, n) && g64[idx] != 0) ? 1 : 0;
            }
            continue;
        }
        const uint32_t Yc = nm1 - Y;
        const uint32_t memb = ((X & Yc) == 0u) ? submask_bits((~Yc) & 31u) : 0u;
        uint32_t bits = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t nib = (memb >> (4 * q)) & 0xFu;
            if (nib) bits |= (alive4_i64(ld_sector(g64 + (int64_t)Y * n + X + 4 * q)) & nib) << (4 * q);
        }
        stg_sector(g8 + (int64_t)Y * n + X, expand32_u8(bits));
    }
}

// members_only: skip 32-cell runs without members (their int64 cells must already be 0)
__global__ void unpack_alive_kernel(const unsigned char* g8, long long* g64, int64_t n,
                                    int members_only = 0) {
    const uint64_t runs_per_row = (uint64_t)(n >= 32 ? n / 32 : 1);
    const uint64_t total = (uint64_t)n * runs_per_row;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t nm1 = (uint32_t)(n - 1);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const uint32_t Y = (uint32_t)(i / runs_per_row);
        const uint32_t X = (uint32_t)(i % runs_per_row) * 32u;
        if (n < 32) {
            for (int64_t x = 0; x < n; ++x) {
                const int64_t idx = (int64_t)Y * n + x;
                g64[idx] = (gasket_member(x, Y, n) && g8[idx] != 0) ? 1 : 0;
            }
            continue;
        }
        const uint32_t Yc = nm1 - Y;
        const uint32_t memb = ((X & Yc) == 0u) ? submask_bits((~Yc) & 31u) : 0u;
        if (members_only && !memb) continue;
        const uint32_t bits = memb ? (alive32_u8(ldg_sector(g8 + (int64_t)Y * n + X)) & memb) : 0u;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (!members_only || ((memb >> (4 * q)) & 0xFu))
                stg_sector(g64 + (int64_t)Y * n + X + 4 * q, expand4_i64((bits >> (4 * q)) & 0xFu));
    }
}

// ---- member-sector copy (zero-copy host transfers) -------------------------------
// Copy the member sectors of an int64 grid, one warp per row: row y's member sectors
// are s ⊆ (y >> 2), its member cells inside a sector are i ⊆ (y & 3). `mask` zeroes
// the non-member cells of each copied sector (sanitizes an arbitrary source). Either
// side may be mapped pinned host memory: only 2^popc(y>>2) sectors per row cross PCIe.
__device__ __forceinline__ uint32_t pdep32(uint32_t j, uint32_t m);
__global__ void copy_member_sectors_kernel(const long long* src, long long* dst, int64_t n, int mask) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (n < 4) {  // tiny grids: cell by cell
        if (warp == 0 && lane == 0)
            for (int64_t y = 0; y < n; ++y)
                for (int64_t x = 0; x < n; ++x)
                    if (gasket_member(x, y, n)) dst[y * n + x] = src[y * n + x];
        return;
    }
    for (uint32_t y = warp; y < (uint32_t)n; y += nwarps) {
        const uint32_t m = y >> 2, cnt = 1u << __popc(m);
        const uint32_t nib = submask_bits(y & 3u) & 0xFu;
        for (uint32_t j = (uint32_t)lane; j < cnt; j += 32u) {
            const int64_t off = (int64_t)y * n + 4 * (int64_t)pdep32(j, m);
            Sector v = ld_sector(src + off);
            if (mask) {
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (!((nib >> c) & 1u)) v.w[2 * c] = v.w[2 * c + 1] = 0u;
            }
            stg_sector(dst + off, v);
        }
    }
}

// ---- member scatter ---------------------------------------------------------
// Row y of the gasket holds 2^popc(y) members, x = pdep(j, y). The number of
// members in rows < y is sum over set bits b of y of 2^popc(y >> (b+1)) * 3^b.
__device__ __forceinline__ uint64_t members_before_row(uint32_t y) {
    uint64_t s = 0, p3 = 1;
    for (int b = 0; b < 32; ++b) {
        if ((y >> b) & 1u) s += ((uint64_t)1 << __popc(y >> (b + 1))) * p3;
        p3 *= 3u;
        if ((y >> b) == 0u) break;
    }
    return s;
}

__device__ __forceinline__ uint32_t pdep32(uint32_t j, uint32_t m) {
    uint32_t r = 0;
    for (uint32_t bit = 1; m != 0u; m &= m - 1u, bit <<= 1)
        if (j & bit) r |= m & (0u - m);
    return r;
}

// one warp per row
__global__ void scatter_members_kernel(const long long* values, long long* grid, int64_t n) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (uint32_t y = warp; y < (uint32_t)n; y += nwarps) {
        const uint64_t start = members_before_row(y);
        const uint32_t cnt = 1u << __popc(y);
        for (uint32_t j = (uint32_t)lane; j < cnt; j += 32u)
            grid[(int64_t)y * n + pdep32(j, y)] = values[start + j];
    }
}

// ---- generic specs -------------------------------------------------------------
// zero the non-member cells (any NBB spec; one thread per cell)
__global__ void sanitize_generic_kernel(DevSpec sp, long long* grid, int64_t n, int r) {
    const uint64_t total = (uint64_t)n * (uint64_t)n;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!member_spec(sp, (int64_t)(i % (uint64_t)n), (int64_t)(i / (uint64_t)n), r)) grid[i] = 0;
    }
}

// λ map of a whole orthotope for any spec (table-driven digit loop)
template <typename Coord>
__global__ void lambda_map_generic_kernel(DevSpec sp, Coord* xy, uint64_t total, uint64_t gw, int level) {
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (uint64_t)gridDim.x * blockDim.x) {
        int64_t x, y;
        lambda_spec(sp, o % gw, o / gw, level, x, y);
        xy[2 * o] = (Coord)x;
        xy[2 * o + 1] = (Coord)y;
    }
}

// ---- halo pack / unpack (K4) for sharded CA -----------------------------------
template <typename Cell>
__global__ void gather_cells_kernel(const Cell* grid, const long long* idx, long long count, Cell* out) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = grid[idx[i]];
}

template <typename Cell>
__global__ void scatter_cells_kernel(Cell* grid, const long long* idx, long long count, const Cell* vals) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        grid[idx[i]] = vals[i];
}

// ---- K0: λ map of a whole orthotope (scalar closed form) ----------------------
// 4 consecutive ordinals per thread (consecutive lanes -> consecutive 32-byte sectors);
// int32 pairs -> one 32-byte store, int64 pairs -> two. λ is separable:
// λx = X(ωx) | X(ωy) << 1, λy = Y(ωx) | Y(ωy) << 1, and X/Y of ωx = its low 6 base-3 digits
// (table entry lo = ωx mod 729) OR its high digits (entry ωx / 729) << 12. Per quad the
// ωy part and the high digits are folded into two constants, so each ω costs one shared-
// memory lookup and two logic ops; the rare carries (lo reaching 729, ωx reaching the row
// end) recompute the constants.
__device__ __forceinline__ void k0_consts(const uint32_t* s_tab, uint32_t hi, uint32_t oy, uint32_t& kx,
                                          uint32_t& ky) {
    uint32_t Xy, Yy;
    xy_from_table(s_tab, oy, Xy, Yy);
    const uint32_t b = s_tab[hi];
    kx = ((b & 0xFFFFu) << 12) | (Xy << 1);
    ky = ((b >> 16) << 12) | (Yy << 1);
}

template <typename Coord>
__global__ void __launch_bounds__(256) lambda_map_kernel(Coord* xy, uint64_t total, uint32_t gw,
                                                         FastDiv div_gw) {
    __shared__ uint32_t s_tab[729];
    for (int i = threadIdx.x; i < 729; i += blockDim.x) s_tab[i] = c_xy729[i];
    __syncthreads();
    const uint64_t quads = (total + 3) / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < quads; q += stride) {
        const uint64_t o0 = q * 4;
        uint32_t oy = fastdiv((uint32_t)o0, div_gw);
        uint32_t ox = (uint32_t)o0 - oy * gw;
        uint32_t hi = __umulhi(ox, 0x59E60383u) >> 8;  // ωx / 729
        uint32_t lo = ox - hi * 729u;
        uint32_t kx, ky;
        k0_consts(s_tab, hi, oy, kx, ky);
        uint32_t lxs[4], lys[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (ox == gw) {  // carry into the next orthotope row
                ox = 0;
                lo = 0;
                hi = 0;
                ++oy;
                k0_consts(s_tab, 0, oy, kx, ky);
            } else if (lo == 729u) {
                lo = 0;
                ++hi;
                k0_consts(s_tab, hi, oy, kx, ky);
            }
            const uint32_t a = s_tab[lo];
            lxs[i] = (a & 0xFFFFu) | kx;
            lys[i] = (a >> 16) | ky;
            ++ox;
            ++lo;
        }
        if (o0 + 4 <= total) {
            if (sizeof(Coord) == 4) {
                Sector v;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    v.w[2 * i] = lxs[i];
                    v.w[2 * i + 1] = lys[i];
                }
                stg_sector(xy + 2 * o0, v);
            } else {
                Sector v0, v1;
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    v0.w[4 * i] = lxs[i];
                    v0.w[4 * i + 1] = 0u;
                    v0.w[4 * i + 2] = lys[i];
                    v0.w[4 * i + 3] = 0u;
                    v1.w[4 * i] = lxs[i + 2];
                    v1.w[4 * i + 1] = 0u;
                    v1.w[4 * i + 2] = lys[i + 2];
                    v1.w[4 * i + 3] = 0u;
                }
                stg_sector(xy + 2 * o0, v0);
                stg_sector(xy + 2 * o0 + 4, v1);
            }
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)  // fixed indices: keeps lxs/lys in registers
                if (o0 + i < total) {
                    xy[2 * (o0 + i)] = (Coord)lxs[i];
                    xy[2 * (o0 + i) + 1] = (Coord)lys[i];
                }
        }
    }
}

// ---- K0-TC: tensor-core λ map --------------------------------------------------
// D(16 ω x 8) += A_g(16 ω x 16) * B_g(16 x 8) over level groups g of 8 levels:
// A_g[i][c] = τx(β_{8g+c+1}(ω_i)) for c < 8 and τy(β_{8g+c-7}(ω_i)) for c >= 8;
// B_g[c][0] = 2^(8g+c) (c < 8), B_g[c][1] = 2^(8g+c-8) (c >= 8). D[i][0..1] = λ(ω_i).
// All operands are 0/1 or powers of two <= 2^16 (exact in bf16) and the sums are
// < 2^24 (exact in fp32), so the result is bit-identical to the scalar map.
template <typename Coord>
__global__ void lambda_map_tc_kernel(Coord* xy, uint64_t total, uint32_t gw, FastDiv div_gw,
                                     int levels) {
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int groups = (levels + 7) / 8;
    // per-lane divisors 3^(4G+t) for the digits this lane encodes
    uint32_t pw[3];
#pragma unroll
    for (int G = 0; G < 3; ++G) {
        uint32_t p = 1;
        for (int i = 0; i < 4 * G + t; ++i) p *= 3u;
        pw[G] = p;
    }
    const uint64_t chunks = (total + 15) / 16;
    for (uint64_t ch = warp; ch < chunks; ch += nwarps) {
        const uint64_t base = ch * 16;
        uint32_t ox[2], oy[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint64_t o = base + g + 8 * h;
            if (o >= total) o = total - 1;
            oy[h] = fastdiv((uint32_t)o, div_gw);
            ox[h] = (uint32_t)o - oy[h] * gw;
        }
        float d[4] = {0.f, 0.f, 0.f, 0.f};
        for (int G = 0; G < groups; ++G) {
            const int mu1 = 8 * G + 2 * t + 1, mu2 = mu1 + 1;  // odd level -> ωx digit, even -> ωy
            uint32_t a[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t bx = (mu1 <= levels) ? (ox[h] / pw[G]) % 3u : 0u;
                const uint32_t by = (mu2 <= levels) ? (oy[h] / pw[G]) % 3u : 0u;
                // cols 2t, 2t+1: τx of levels mu1, mu2; cols 2t+8, 2t+9: τy of levels mu1, mu2
                a[h] = pack_bf16((float)(bx / 2u), (float)(by / 2u));
                a[h + 2] = pack_bf16((float)(bx - bx / 2u), (float)(by - by / 2u));
            }
            uint32_t b[2];
            {
                const int r0 = 2 * t, r1 = 2 * t + 1;  // rows of B held by this lane (k)
                const float v0 = (g == 0) ? (float)(1u << (8 * G + r0)) : 0.f;
                const float v1 = (g == 0) ? (float)(1u << (8 * G + r1)) : 0.f;
                const float w0 = (g == 1) ? (float)(1u << (8 * G + r0)) : 0.f;
                const float w1 = (g == 1) ? (float)(1u << (8 * G + r1)) : 0.f;
                b[0] = pack_bf16(v0, v1);  // rows 2t, 2t+1 (τx part), column g
                b[1] = pack_bf16(w0, w1);  // rows 2t+8, 2t+9 (τy part), column g
            }
            mma_bf16_16816(d, a, b, d);
        }
        if (t == 0) {  // lanes holding columns 0 and 1
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint64_t o = base + g + 8 * h;
                if (o < total) {
                    xy[2 * o] = (Coord)d[2 * h];
                    xy[2 * o + 1] = (Coord)d[2 * h + 1];
                }
            }
        }
    }
}

// ---- K0-TC on the 5th-generation tensor core (tcgen05 + TMEM) ----------------------
// The paper's MMA λ (mma.cpp:34-118, variant 1) as three tcgen05.mma per 128 ordinals and up to
// 24 levels: D[128 ω x 16] (fp32, TMEM) = A[128 x 48] (bf16, smem) · B[48 x 16] (bf16, smem) with
// A[i][k] = τx(β_{k+1}(ω_i)) for k < 24 and τy(β_{k-23}(ω_i)) for k >= 24, B[k][0] = 2^k (k < 24),
// B[k][1] = 2^(k-24) (k >= 24), other columns 0, so D[i][0..1] = λ(ω_i). τx(β) = [β == 2] and
// τy(β) = [β >= 1] of the level's base-3 digit are bit μ-1 of X(ωx) | X(ωy) << 1 and
// Y(ωx) | Y(ωy) << 1, read from the 729-entry digit table. Exact: 0/1 and
// powers of two <= 2^23 are exact in bf16, sums < 2^24 in fp32 (the map covers levels <= 17).
//
// One CTA = 4 warps = 128 ordinals per tile (thread i builds A row i), persistent over tiles:
// build A -> fence.proxy.async -> one elected thread issues 3 x tcgen05.mma (M=128, N=16,
// K=16) and commits to an mbarrier -> every warp tcgen05.ld's its 32 TMEM lanes (2 columns)
// -> 8-byte stores. Operands in the canonical no-swizzle K-major layout: 8-row x 16-byte core
// matrices, K-adjacent core matrices 128 B apart (LBO), 8-row groups 768 B apart (SBO).
__device__ __forceinline__ uint64_t umma_smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100)
    return d;                // base offset 0, legacy LBO mode, layout SWIZZLE_NONE (0)
}

template <typename Coord>
__global__ void __launch_bounds__(128) lambda_map_tc5_kernel(Coord* xy, uint64_t total, uint32_t gw,
                                                             FastDiv div_gw) {
    constexpr uint32_t IDESC = (1u << 4)      // D format f32
                             | (1u << 7)      // A format bf16
                             | (1u << 10)     // B format bf16
                             | (2u << 17)     // N = 16 (>> 3)
                             | (8u << 24);    // M = 128 (>> 4); A, B K-major
    constexpr uint32_t KC = 6;                // 16-byte k chunks per row (K = 48)
    constexpr uint32_t SBO = KC * 128;        // bytes between 8-row groups
    constexpr uint32_t A_BYTES = 128 * KC * 16;
    __shared__ __align__(128) uint8_t s_a[2][A_BYTES];  // two stages of [16 row groups][KC][8 rows][16 B]
    __shared__ __align__(128) uint8_t s_b[16 * KC * 16];  // [2 col groups][KC][8 cols][16 B]
    __shared__ uint32_t s_tab[729];
    __shared__ uint4 s_bits[256];  // byte b -> its 8 bits as 8 bf16 values (1.0 or 0), K-chunk ready
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ uint32_t s_tmem;
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    for (uint32_t i = tid; i < 729; i += 128) s_tab[i] = c_xy729[i];
    for (uint32_t bb = tid; bb < 256; bb += 128) {
        uint32_t w[4];
#pragma unroll
        for (int h = 0; h < 4; ++h)
            w[h] = (((bb >> (2 * h)) & 1u) ? 0x3F80u : 0u) | (((bb >> (2 * h + 1)) & 1u) ? 0x3F800000u : 0u);
        s_bits[bb] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    // B: column n (= "row" of the K-major B), k chunk c holds k = 8c..8c+7
    for (uint32_t e = tid; e < 16 * 48; e += 128) {
        const uint32_t n = e / 48, k = e % 48;
        float v = 0.f;
        if (n == 0 && k < 24) v = (float)(1u << k);
        if (n == 1 && k >= 24) v = (float)(1u << (k - 24));
        const uint32_t off = (n >> 3) * SBO + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2;
        *reinterpret_cast<__nv_bfloat16*>(s_b + off) = __float2bfloat16_rn(v);
    }
    if (warp == 0) {  // two 16-column accumulators (stages) in one 32-column allocation
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&s_tmem);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(dst));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&s_bar[0]);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    const uint32_t a_base0 = (uint32_t)__cvta_generic_to_shared(s_a[0]);
    const uint32_t b_base = (uint32_t)__cvta_generic_to_shared(s_b);
    const uint32_t row_off = (tid >> 3) * SBO + (tid & 7) * 16;  // this thread's A row
    uint32_t phase[2] = {0u, 0u};

    // wait for tile (stage st)'s MMAs, read its accumulator lanes, store the λ pairs
    auto drain = [&](uint32_t st, uint64_t o) {
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}\n"
                : "=r"(done) : "r"(bar0 + 8u * st), "r"(phase[st]) : "memory");
        phase[st] ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint32_t d0, d1;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                     : "=r"(d0), "=r"(d1) : "r"(tmem + ((warp * 32u) << 16) + 16u * st));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (o < total) {
            xy[2 * o] = (Coord)__float2uint_rn(__uint_as_float(d0));
            xy[2 * o + 1] = (Coord)__float2uint_rn(__uint_as_float(d1));
        }
    };

    // two-stage pipeline: build tile i's A while the tensor core runs tile i-1, then drain i-1
    const uint64_t tiles = (total + 127) / 128;
    uint64_t o_prev = 0;
    uint32_t i = 0;
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const uint32_t st = i & 1u;
        const uint64_t o = t * 128 + tid;
        uint32_t lx = 0, ly = 0;
        if (o < total) {
            const uint32_t oy = fastdiv((uint32_t)o, div_gw), ox = (uint32_t)o - oy * gw;
            uint32_t Xx, Yx, Xy, Yy;
            xy_from_table(s_tab, ox, Xx, Yx);
            xy_from_table(s_tab, oy, Xy, Yy);
            lambda_from_xy(Xx, Yx, Xy, Yy, lx, ly);  // bit μ-1: τx / τy of level μ
        }
        // A row (stage st; its previous MMA, tile i-2, was drained last iteration): chunks 0-2 ->
        // τx bits 0-23, chunks 3-5 -> τy bits 0-23, one byte of λ per chunk via s_bits
        uint8_t* my_row = s_a[st] + row_off;
#pragma unroll
        for (int c = 0; c < (int)KC; ++c) {
            const uint32_t byte = ((c < 3 ? lx : ly) >> (8 * (c % 3))) & 0xFFu;
            *reinterpret_cast<uint4*>(my_row + c * 128) = s_bits[byte];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();  // A[st] complete; every thread has drained tile i-2's accumulator
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int ks = 0; ks < (int)KC / 2; ++ks) {
                const uint64_t da = umma_smem_desc(a_base0 + st * A_BYTES + ks * 256, 128, SBO);
                const uint64_t db = umma_smem_desc(b_base + ks * 256, 128, SBO);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + 16u * st),
                    "l"(da), "l"(db), "r"(IDESC), "r"(ks));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         ::"r"(bar0 + 8u * st) : "memory");
        }
        if (i > 0) drain(st ^ 1u, o_prev);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        o_prev = o;
    }
    if (i > 0) drain((i - 1) & 1u, o_prev);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

}  // namespace nbbgpu
