// compact_kernels.cuh — the compact (λ-ordered) codec and a CA step on compact state.
//
// CompactGrid (block_map.hpp:82-110): the k^r member values laid out row-major over
// the packing orthotope, value(ω) = embedded(λ(ω)). compact_store / compact_load
// (block_map.cpp:245-282) become a gather / scatter through the device λ, and
// λ⁻¹ (block_map.cpp:113-148) a per-point descent.
//
// CA on compact state (gasket): the cells of the ρ = 32 tile ω_b = (ωx_b, ωy_b) at
// block level r_b = r − 5 form the contiguous sub-block
//     rows 9·ωx_b .. 9·ωx_b+8,  columns 27·ωy_b .. 27·ωy_b+26
// of the W × H compact array (level parities shift by 5: block level μ_b sits at cell
// level μ_b + 5, so block ωx digits become cell ωy digits above position 2 and block ωy
// digits cell ωx digits above position 3). Consecutive tiles of a row block are
// adjacent, so a CTA streams whole compact rows: every byte moved is a member value
// (the embedded layout moves 128-byte lines for 14.2 bytes of members per cell).
#pragma once

#include "common.cuh"
#include "tile_kernels.cuh"

namespace nbbgpu {

// local λ at level 5 (ρ = 32 tile): packed x | y << 5 for local index li = ωy_l*27 + ωx_l
__constant__ uint16_t c_local_pos[243];
// inverse: local (x, y) -> li, or 0xFFFF for non-members
__constant__ uint16_t c_local_idx[1024];

__device__ __forceinline__ void lambda_point(const DevSpec& sp, uint64_t ox, uint64_t oy, int level,
                                             int64_t& x, int64_t& y) {
    if (sp.gasket) {
        uint32_t lx, ly;
        lambda_arith((uint32_t)ox, (uint32_t)oy, lx, ly);
        x = lx;
        y = ly;
    } else {
        lambda_spec(sp, ox, oy, level, x, y);
    }
}

// compact[c] = embedded[λ(ω_c)], one thread per compact cell
__global__ void compact_store_kernel(DevSpec sp, const long long* emb, long long* comp, int64_t n,
                                     uint64_t W, uint64_t total, int level) {
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < total;
         c += (uint64_t)gridDim.x * blockDim.x) {
        int64_t x, y;
        lambda_point(sp, c % W, c / W, level, x, y);
        comp[c] = emb[y * n + x];
    }
}

// embedded[λ(ω_c)] = compact[c] (the non-member fill happens before)
__global__ void compact_load_kernel(DevSpec sp, const long long* comp, long long* emb, int64_t n,
                                    uint64_t W, uint64_t total, int level) {
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < total;
         c += (uint64_t)gridDim.x * blockDim.x) {
        int64_t x, y;
        lambda_point(sp, c % W, c / W, level, x, y);
        emb[y * n + x] = comp[c];
    }
}

// Σ of a dense int64 array (every compact value is a member), wrap-around like int64 +
__global__ void __launch_bounds__(256) dense_sum_kernel(const long long* p, uint64_t count,
                                                        unsigned long long* out) {
    unsigned long long acc = 0;
    const uint64_t vec = count / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < vec; i += stride) {
        const Sector s = ldg_sector(p + 4 * i);
        acc += masked_sum4(s, 0xFu);
    }
    for (uint64_t i = 4 * vec + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
        acc += (unsigned long long)p[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    __shared__ unsigned long long s[8];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
        if (t) atomicAdd(out, t);
    }
}

__global__ void fill_kernel(long long* p, uint64_t count, long long v) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// λ⁻¹ of points (block_map.cpp:113-148); status: 0 ok, 2 out_of_range, 6 domain_error
__global__ void lambda_inverse_kernel(DevSpec sp, const long long* xy, long long* omega, int* status,
                                      uint64_t count, int level) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        int64_t x = xy[2 * i], y = xy[2 * i + 1];
        int64_t n = 1;
        for (int l = 0; l < level; ++l) n *= sp.s;
        int st = 0;
        int64_t ox = 0, oy = 0;
        if (x < 0 || y < 0 || x >= n || y >= n) {
            st = NBB_ERR_OUT_OF_RANGE;
        } else {
            int64_t scale = n / sp.s;
            for (int mu = level; mu >= 1 && st == 0; --mu) {
                const int cx = (int)(x / scale), cy = (int)(y / scale);
                const int beta = sp.replica_at[cy * sp.s + cx];
                if (beta < 0) {
                    st = NBB_ERR_DOMAIN;
                    break;
                }
                int64_t d = 1;
                for (int j = 0; j < (mu + 1) / 2 - 1; ++j) d *= sp.k;
                if (mu & 1) ox += beta * d; else oy += beta * d;
                x -= cx * scale;
                y -= cy * scale;
                scale /= sp.s;
            }
        }
        omega[2 * i] = st ? 0 : ox;
        omega[2 * i + 1] = st ? 0 : oy;
        status[i] = st;
    }
}

// block-level λ⁻¹ of a member block (bx, by) of the gasket: ordinal digits from the bits
__device__ __forceinline__ void gasket_block_inverse(uint32_t bx, uint32_t by, int rb, uint32_t& ox,
                                                     uint32_t& oy) {
    ox = 0;
    oy = 0;
    uint32_t px = 1, py = 1;
    for (int mu = 1; mu <= rb; ++mu) {
        const uint32_t beta = ((bx >> (mu - 1)) & 1u) + ((by >> (mu - 1)) & 1u);
        if (mu & 1) {
            ox += beta * px;
            px *= 3u;
        } else {
            oy += beta * py;
            py *= 3u;
        }
    }
}

struct CompactCaArgs {
    const long long* src;
    long long* dst;
    uint32_t W;        // compact width 3^ceil(r/2)
    uint32_t Wb;       // block orthotope width 3^ceil(rb/2)
    uint32_t Hb;       // block orthotope height 3^floor(rb/2)
    int rb;            // block level r - 5
    int64_t n;         // embedding side
    uint32_t tiles;    // Wb * Hb
    uint32_t birth, survive;
};

// One warp per tile; tile u -> (ωx_b = u / Hb, ωy_b = u % Hb) so consecutive warps walk along a
// compact row block. 243 values per tile = slots k = 0..7 of lane l: li = 32k + l.
__global__ void __launch_bounds__(256, 3) ca_compact_kernel(CompactCaArgs a) {
    __shared__ uint32_t s_rows[8][32];
    __shared__ uint32_t s_new[8][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t sl_off[8], sl_pos[8];
    uint32_t valid = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t li = 32u * k + lane;
        const bool ok = li < 243u;
        const uint32_t row = ok ? li / 27u : 0u, col = ok ? li % 27u : 0u;
        sl_off[k] = row * a.W + col;               // element offset inside the tile's sub-block
        sl_pos[k] = ok ? c_local_pos[li] : 0u;
        valid |= (ok ? 1u : 0u) << k;
    }
    const uint32_t hk = (uint32_t)lane & 7u;
    const int hx = (hk == 0 || hk == 3) ? -1 : (hk == 1 || hk == 7) ? 0 : (hk == 2) ? 1 : 32;
    const int hy = (hk <= 2) ? -1 : (hk == 3 || hk == 5) ? 31 : (hk == 4) ? 30 : 32;
    const uint32_t warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t warp_stride = (gridDim.x * blockDim.x) >> 5;

    for (uint32_t u = warp_global; u < a.tiles; u += warp_stride) {
        const uint32_t wxb = u / a.Hb, wyb = u - (u / a.Hb) * a.Hb;
        const uint64_t base = (uint64_t)(9u * wxb) * a.W + 27u * wyb;
        // loads (all 8 slots in flight)
        long long v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = ((valid >> k) & 1u) ? __ldg(a.src + base + sl_off[k]) : 0ll;
        // tile origin (λ of the block ordinal: block ordinal = ωy_b * Wb + ωx_b)
        uint32_t bx, by;
        lambda_const(wxb, wyb, bx, by);
        const int64_t X0 = (int64_t)bx * 32, Y0 = (int64_t)by * 32;
        // halo cell of lanes 0..7
        uint32_t hbit = 0;
        if (lane < 8) {
            const int64_t gx = X0 + hx, gy = Y0 + hy;
            if (gasket_member(gx, gy, a.n)) {
                uint32_t ox, oy;
                gasket_block_inverse((uint32_t)(gx >> 5), (uint32_t)(gy >> 5), a.rb, ox, oy);
                const uint32_t li = c_local_idx[((uint32_t)gy & 31u) * 32u + ((uint32_t)gx & 31u)];
                const uint32_t row = li / 27u, col = li % 27u;
                const uint64_t off = (uint64_t)(9u * ox + row) * a.W + 27u * oy + col;
                hbit = __ldg(a.src + off) != 0ll;
            }
        }
        const uint32_t hmask = __ballot_sync(0xFFFFFFFFu, hbit != 0u);
        s_rows[wib][lane] = 0u;
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (((valid >> k) & 1u) && v[k] != 0ll)
                atomicOr(&s_rows[wib][sl_pos[k] >> 5], 1u << (sl_pos[k] & 31u));
        }
        __syncwarp();
        const uint32_t R = s_rows[wib][lane];
        const uint64_t h = hmask & 0xFFu;
        uint64_t E = (uint64_t)R << 1;
        if (lane == 31) E |= ((h >> 3) & 1u) | (((h >> 5) & 1u) << 33);
        if (lane == 30) E |= ((h >> 4) & 1u) << 33;
        const uint64_t top = (h & 1u) | (((h >> 1) & 1u) << 1) | (((h >> 2) & 1u) << 2);
        const uint64_t bottom = (((h >> 7) & 1u) << 1) | (((h >> 6) & 1u) << 33);
        const uint64_t Eu = __shfl_up_sync(0xFFFFFFFFu, E, 1);
        const uint64_t Ed = __shfl_down_sync(0xFFFFFFFFu, E, 1);
        const uint64_t U = lane == 0 ? top : Eu;
        const uint64_t D = lane == 31 ? bottom : Ed;
        const uint32_t memb = submask_bits((uint32_t)lane);
        s_new[wib][lane] = life_rule((uint32_t)U, (uint32_t)(U >> 1), (uint32_t)(U >> 2), (uint32_t)E,
                                     (uint32_t)(E >> 2), (uint32_t)D, (uint32_t)(D >> 1), (uint32_t)(D >> 2),
                                     (uint32_t)(E >> 1), a.birth, a.survive) & memb;
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if ((valid >> k) & 1u) {
                const uint32_t bit = (s_new[wib][sl_pos[k] >> 5] >> (sl_pos[k] & 31u)) & 1u;
                a.dst[base + sl_off[k]] = (long long)bit;
            }
        }
        __syncwarp();
    }
}

}  // namespace nbbgpu
