// percell_kernels.cuh — the paper's launch shapes: one thread per cell.
//
// BB    : (n/ρ)^2 blocks of ρ x ρ threads, identity map, per-thread membership
//         test, payload on members (dispatch.cpp:278-300).
// λ(ω)  : the reference's full configuration matrix (dispatch.cpp:302-411):
//         backend  direct | mma1 | mma2 | mma3  -> block origin
//         strategy subbox | unroll | lut        -> thread's cell
//         with the tensor-core encodings of mma.cpp:34-118 run on the tensor
//         pipe (mma.sync m16n8k16 bf16 -> fp32, exact: see DESIGN.md §MMA).
// These kernels are the parity surface for every (mode, strategy, backend)
// combination and the paper-faithful baseline; the tile kernels
// (tile_kernels.cuh) are the fast path for subbox/direct.
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"
#include "tile_kernels.cuh"

namespace nbbgpu {

struct PercellArgs {
    const void* src;
    void* dst;
    unsigned long long* partials;  // RD: 4096 slots, pre-zeroed
    int64_t n;
    uint64_t total_blocks;         // blocks of the whole plan (incl. mma2 padding)
    uint64_t ordinal_base;         // first ordinal of this launch (shard)
    uint64_t launch_count;         // ordinals in this launch
    uint64_t gw;                   // launch grid width (blocks)
    int edge;                      // thread-block edge (ρ, or ρ/2 for mma2)
    int map_level;                 // levels per block origin
    int local_level;               // intra-block fractal level
    int local_w;                   // local orthotope width (unroll)
    int local_members;             // 3^local_level
    int64_t sub_w, sub_h;          // mma2 in-range sub-orthotope
    const int16_t* lut;            // lut strategy: edge*edge (x, y) pairs, -1 = spare
    uint32_t birth, survive;
    int r;                         // scale level of the embedding
    DevSpec spec;                  // fractal descriptor (gasket fast paths when spec.gasket)
};

// D(8x8) = A(8x4) * B(4x8) + C on the FP64 tensor pipe (DMMA), exact for integers < 2^53
__device__ __forceinline__ void mma_f64_884(double (&d)[2], double a, double b, const double (&c)[2]) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
                 : "=d"(d[0]), "=d"(d[1])
                 : "d"(a), "d"(b), "d"(c[0]), "d"(c[1]));
}

// β_μ(ω) for any k (block_map.cpp:57-65)
__device__ __forceinline__ uint32_t beta_digit_k(uint64_t ox, uint64_t oy, int mu, uint32_t k) {
    uint64_t v = (mu & 1) ? ox : oy;
    for (int i = 0; i < (mu + 1) / 2 - 1; ++i) v /= k;
    return (uint32_t)(v % k);
}

__device__ __forceinline__ uint64_t flat_block() {
    return ((uint64_t)blockIdx.z * gridDim.y + blockIdx.y) * (uint64_t)gridDim.x + blockIdx.x;
}

// ---- mma.sync m16n8k16 (bf16 inputs, fp32 accumulate) ----------------------
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    const __nv_bfloat16 a = __float2bfloat16_rn(lo), b = __float2bfloat16_rn(hi);
    return (uint32_t)__bfloat16_as_ushort(a) | ((uint32_t)__bfloat16_as_ushort(b) << 16);
}

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4],
                                               const uint32_t (&b)[2], const float (&c)[4]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%10,%11,%12,%13};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "f"(c[0]), "f"(c[1]),
          "f"(c[2]), "f"(c[3]));
}

// D(16x16) = A(16x16) * B(16x16) + C(16x16), fragments staged row-major in
// shared memory as float; executed by one full warp as two m16n8k16 MMAs.
__device__ void warp_mma_16x16(const float* A, const float* B, const float* C, float* D) {
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    uint32_t a[4];
    a[0] = pack_bf16(A[g * 16 + 2 * t], A[g * 16 + 2 * t + 1]);
    a[1] = pack_bf16(A[(g + 8) * 16 + 2 * t], A[(g + 8) * 16 + 2 * t + 1]);
    a[2] = pack_bf16(A[g * 16 + 2 * t + 8], A[g * 16 + 2 * t + 9]);
    a[3] = pack_bf16(A[(g + 8) * 16 + 2 * t + 8], A[(g + 8) * 16 + 2 * t + 9]);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        const int col = half * 8 + g;
        uint32_t b[2];
        b[0] = pack_bf16(B[(2 * t) * 16 + col], B[(2 * t + 1) * 16 + col]);
        b[1] = pack_bf16(B[(2 * t + 8) * 16 + col], B[(2 * t + 9) * 16 + col]);
        const int c0 = half * 8 + 2 * t;
        float c[4] = {C ? C[g * 16 + c0] : 0.f, C ? C[g * 16 + c0 + 1] : 0.f,
                      C ? C[(g + 8) * 16 + c0] : 0.f, C ? C[(g + 8) * 16 + c0 + 1] : 0.f};
        float d[4];
        mma_bf16_16816(d, a, b, c);
        D[g * 16 + c0] = d[0];
        D[g * 16 + c0 + 1] = d[1];
        D[(g + 8) * 16 + c0] = d[2];
        D[(g + 8) * 16 + c0 + 1] = d[3];
    }
}

// β_μ(ω) for the gasket (block_map.cpp:57-65): digit ceil(μ/2)-1 of ωx (odd μ)
// or ωy (even μ); τ = H[β] with H = {(0,0),(0,1),(1,1)} (fractal.cpp:81), i.e.
// the arithmetic hash τ = (β/2, β - β/2) (block_map.cpp:150-155).
__device__ __forceinline__ uint32_t beta_digit(uint64_t ox, uint64_t oy, int mu) {
    uint64_t v = (mu & 1) ? ox : oy;
    for (int i = 0; i < (mu + 1) / 2 - 1; ++i) v /= 3u;
    return (uint32_t)(v % 3u);
}

template <typename Cell, int OP, bool BB, int STRATEGY, int BACKEND, bool GEN>
__global__ void percell_kernel(PercellArgs a) {
    __shared__ float sA[256], sB[256], sC[256], sD[256], sE[256];
    __shared__ int64_t s_origin[2];
    __shared__ unsigned long long s_red[32];

    const uint64_t flat = flat_block();
    if (flat >= a.launch_count) return;
    const uint64_t ordinal = a.ordinal_base + flat;
    const int edge = a.edge;
    const int tid = threadIdx.x;
    const bool real = tid < edge * edge;
    const int64_t tx = real ? tid % edge : 0, ty = real ? tid / edge : 0;
    const int64_t n = a.n;
    const uint64_t gx = ordinal % a.gw, gy = ordinal / a.gw;

    bool active = false;
    int64_t cx = 0, cy = 0;
    if (BB) {
        cx = (int64_t)gx * edge + tx;
        cy = (int64_t)gy * edge + ty;
        active = real && (!GEN ? gasket_member(cx, cy, n) : member_spec(a.spec, cx, cy, a.r));
    } else {
        if (BACKEND == NBB_BACKEND_MMA2 && ((int64_t)gx >= a.sub_w || (int64_t)gy >= a.sub_h)) {
            return;  // padding slot of the even-rounded cover: all spare (dispatch.cpp:321-325)
        }
        int64_t ox = 0, oy = 0;
        if (BACKEND == NBB_BACKEND_DIRECT) {
            // λ(ω) once per block, as launch_impl resolves the origin once per ordinal
            // (dispatch.cpp:307-311), broadcast through shared memory: per-thread evaluation
            // made this path issue-bound (1.44 -> 0.70 ms for SW at n = 2^16, ρ = 16)
            if (tid == 0) {
                if (!GEN) {
                    uint32_t lx, ly;
                    lambda_arith((uint32_t)gx, (uint32_t)gy, lx, ly);
                    s_origin[0] = lx;
                    s_origin[1] = ly;
                } else {
                    lambda_spec(a.spec, gx, gy, a.map_level, s_origin[0], s_origin[1]);
                }
            }
            __syncthreads();
            ox = s_origin[0];
            oy = s_origin[1];
        } else if (BACKEND == NBB_BACKEND_MMA1 && GEN) {
            // s = 3: powers 3^(μ-1) are not bf16-exact beyond 3^5 — variant 1 on the FP64
            // tensor pipe (DMMA m8n8k4): A row 0 = s^(μ-1), B cols 0/1 = τx/τy; K = 16 in 4 steps
            if (tid < 32) {
                const int g = tid >> 2, t = tid & 3;
                double d[2] = {0.0, 0.0};
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const int kk = 4 * ks + t;  // level μ = kk + 1
                    double av = 0.0, bv = 0.0;
                    if (kk < a.map_level) {
                        double p = 1.0;
                        for (int i = 0; i < kk; ++i) p *= a.spec.s;
                        if (g == 0) av = p;
                        const uint32_t beta = beta_digit_k(gx, gy, kk + 1, (uint32_t)a.spec.k);
                        if (g == 0) bv = a.spec.ox[beta];
                        if (g == 1) bv = a.spec.oy[beta];
                    }
                    mma_f64_884(d, av, bv, d);
                }
                if (tid == 0) {
                    s_origin[0] = (int64_t)d[0];
                    s_origin[1] = (int64_t)d[1];
                }
            }
            __syncthreads();
            ox = s_origin[0];
            oy = s_origin[1];
        } else {
            // warp 0 evaluates the encoding (mma.cpp:34-118) on the tensor pipe
            const int L = a.map_level;
            if (tid < 32) {
                for (int i = tid; i < 256; i += 32) {
                    sA[i] = 0.f;
                    sB[i] = 0.f;
                    sC[i] = 0.f;
                    sE[i] = 0.f;
                }
                __syncwarp();
                if (BACKEND == NBB_BACKEND_MMA1) {
                    if (tid < L) {
                        const int mu = tid + 1;
                        sA[mu - 1] = (float)(1u << (mu - 1));
                        const uint32_t beta = beta_digit(gx, gy, mu);
                        sB[(mu - 1) * 16 + 0] = (float)(beta / 2u);
                        sB[(mu - 1) * 16 + 1] = (float)(beta - beta / 2u);
                    }
                } else if (BACKEND == NBB_BACKEND_MMA2) {
                    const uint64_t first = (ordinal / 8u) * 8u;
                    if (tid < L) sA[tid] = (float)(1u << tid);
                    for (int e = tid; e < 8 * L; e += 32) {
                        const int i = e / L, mu = e % L + 1;
                        const uint64_t o = first + (uint64_t)i;
                        if (o >= a.total_blocks) continue;
                        const uint64_t wx = o % a.gw, wy = o / a.gw;
                        if ((int64_t)wx >= a.sub_w || (int64_t)wy >= a.sub_h) continue;  // inactive
                        const uint32_t beta = beta_digit(wx, wy, mu);
                        sB[(mu - 1) * 16 + 2 * i] = (float)(beta / 2u);
                        sB[(mu - 1) * 16 + 2 * i + 1] = (float)(beta - beta / 2u);
                    }
                } else {  // MMA3: rows of A = ρ·2^(μ-1); Bx/By constant rows; C = thread offsets
                    for (int e = tid; e < 16 * L; e += 32) {
                        const int i = e / L, mu = e % L + 1;
                        sA[i * 16 + mu - 1] = (float)(edge << (mu - 1));
                    }
                    for (int e = tid; e < 16 * L; e += 32) {
                        const int j = e / L, mu = e % L + 1;
                        const uint32_t beta = beta_digit(gx, gy, mu);
                        sB[(mu - 1) * 16 + j] = (float)(beta / 2u);
                        sE[(mu - 1) * 16 + j] = (float)(beta - beta / 2u);
                    }
                    for (int i = tid; i < 256; i += 32) sC[i] = (float)(i / 16);  // Cx[i][j] = i
                }
                __syncwarp();
                warp_mma_16x16(sA, sB, BACKEND == NBB_BACKEND_MMA3 ? sC : nullptr, sD);
                if (BACKEND == NBB_BACKEND_MMA3) {
                    // Dy = A * By + Cy into sB (Bx is dead once Dx is in sD)
                    __syncwarp();
                    for (int i = tid; i < 256; i += 32) sC[i] = (float)(i % 16);  // Cy[i][j] = j
                    __syncwarp();
                    warp_mma_16x16(sA, sE, sC, sB);
                }
                __syncwarp();
                if (tid == 0 && BACKEND != NBB_BACKEND_MMA3) {
                    const int slot = BACKEND == NBB_BACKEND_MMA2 ? (int)(ordinal % 8u) : 0;
                    s_origin[0] = (int64_t)sD[2 * slot];
                    s_origin[1] = (int64_t)sD[2 * slot + 1];
                }
            }
            __syncthreads();
            if (BACKEND != NBB_BACKEND_MMA3) {
                ox = s_origin[0];
                oy = s_origin[1];
            }
        }
        // intra-block strategy (dispatch.cpp:357-398)
        if (real) {
            if (STRATEGY == NBB_STRATEGY_SUBBOX) {
                active = !GEN ? (tx & (edge - 1 - ty)) == 0
                                       : member_spec(a.spec, tx, ty, a.local_level);
                if (BACKEND == NBB_BACKEND_MMA3) {
                    cx = (int64_t)sD[tx * 16 + ty];  // Dx[i=tx][j=ty] = ρ·λx + tx
                    cy = (int64_t)sB[tx * 16 + ty];
                } else {
                    cx = ox * edge + tx;
                    cy = oy * edge + ty;
                }
            } else if (STRATEGY == NBB_STRATEGY_UNROLL) {
                const int64_t rank = ty * edge + tx;
                if (rank < a.local_members) {
                    int64_t lx, ly;
                    if (!GEN) {
                        uint32_t ux, uy;
                        lambda_arith((uint32_t)(rank % a.local_w), (uint32_t)(rank / a.local_w), ux, uy);
                        lx = ux;
                        ly = uy;
                    } else {
                        lambda_spec(a.spec, (uint64_t)(rank % a.local_w), (uint64_t)(rank / a.local_w),
                                    a.local_level, lx, ly);
                    }
                    cx = ox * edge + lx;
                    cy = oy * edge + ly;
                    active = true;
                }
            } else {  // LUT
                const int16_t lx = a.lut[2 * tid], ly = a.lut[2 * tid + 1];
                if (lx >= 0) {
                    cx = ox * edge + lx;
                    cy = oy * edge + ly;
                    active = true;
                }
            }
        }
    }

    // ---- payloads (dispatch.cpp:481-557) -----------------------------------------
    if (OP == OP_SW) {
        if (active) static_cast<Cell*>(a.dst)[cy * n + cx] = (Cell)1;
    } else if (OP == OP_RD) {
        unsigned long long v = 0;
        if (active) v = (unsigned long long)static_cast<const long long*>(a.src)[cy * n + cx];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        const int nw = (blockDim.x + 31) / 32;
        if (nw == 1) {
            if ((tid & 31) == 0 && v) atomicAdd(&a.partials[ordinal & 4095u], v);
        } else {
            if ((tid & 31) == 0) s_red[tid >> 5] = v;
            __syncthreads();
            if (tid < 32) {
                unsigned long long w = tid < nw ? s_red[tid] : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xFFFFFFFFu, w, o);
                if (tid == 0 && w) atomicAdd(&a.partials[ordinal & 4095u], w);
            }
        }
    } else {  // OP_CA: fractal-restricted Moore neighbourhood (dispatch.cpp:533-549)
        if (active) {
            const Cell* src = static_cast<const Cell*>(a.src);
            int live = 0;
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    if (dx == 0 && dy == 0) continue;
                    const int64_t nx = cx + dx, ny = cy + dy;
                    const bool m = !GEN ? gasket_member(nx, ny, n)
                                                 : member_spec(a.spec, nx, ny, a.r);
                    if (m && src[ny * n + nx] != (Cell)0) ++live;
                }
            const bool alive = src[cy * n + cx] != (Cell)0;
            const uint32_t bit = 1u << live;
            static_cast<Cell*>(a.dst)[cy * n + cx] =
                (((alive ? a.survive : a.birth) & bit) != 0u) ? (Cell)1 : (Cell)0;
        }
    }
}

__global__ void reduce_partials_kernel(const unsigned long long* partials, int count,
                                       unsigned long long* out) {
    unsigned long long v = 0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) v += partials[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    __shared__ unsigned long long s[32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x + 31) / 32 ? s[threadIdx.x] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (threadIdx.x == 0) *out = v;
    }
}

}  // namespace nbbgpu
