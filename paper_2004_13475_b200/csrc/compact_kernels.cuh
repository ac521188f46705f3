// compact_kernels.cuh — the compact (λ-ordered) codec and the shared stages of the CA on
// compact state (the pass kernel itself: compact_pass.cuh).
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
#include "util_kernels.cuh"

namespace nbbgpu {

// local λ at level 5 (ρ = 32 tile): packed x | y << 5 for local index li = ωy_l*27 + ωx_l
__constant__ uint16_t c_local_pos[243];
// inverse: local (x, y) -> li, or 0xFFFF for non-members
__constant__ uint16_t c_local_idx[1024];

template <bool GEN>
__device__ __forceinline__ void lambda_point(const DevSpec& sp, uint64_t ox, uint64_t oy, int level,
                                             int64_t& x, int64_t& y) {
    if (!GEN) {
        uint32_t lx, ly;
        lambda_arith((uint32_t)ox, (uint32_t)oy, lx, ly);
        x = lx;
        y = ly;
    } else {
        lambda_spec(sp, ox, oy, level, x, y);
    }
}

// compact[c] = embedded[λ(ω_c)], one thread per compact cell
template <bool GEN>
__global__ void compact_store_kernel(DevSpec sp, const long long* emb, long long* comp, int64_t n,
                                     uint64_t W, uint64_t total, int level) {
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < total;
         c += (uint64_t)gridDim.x * blockDim.x) {
        int64_t x, y;
        lambda_point<GEN>(sp, c % W, c / W, level, x, y);
        comp[c] = emb[y * n + x];
    }
}

// embedded[λ(ω_c)] = compact[c] (the non-member fill happens before)
template <bool GEN>
__global__ void compact_load_kernel(DevSpec sp, const long long* comp, long long* emb, int64_t n,
                                    uint64_t W, uint64_t total, int level) {
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < total;
         c += (uint64_t)gridDim.x * blockDim.x) {
        int64_t x, y;
        lambda_point<GEN>(sp, c % W, c / W, level, x, y);
        emb[y * n + x] = comp[c];
    }
}

// A shard of the compact state as memory segments: tiles u in [b, e) of the order
// u = ωx_b·H_b + ωy_b (a tile = 9 compact rows x 27 columns, a tile row = 9 full compact rows):
// a partial tile row at each end (9 segments of 27·k values each) and the full tile rows between
// (one contiguous segment) — at most 19 segments; the whole array is the single segment (0, 3^r).
constexpr int kMaxSegs = 20;
struct Segs {
    uint64_t off[kMaxSegs];
    uint64_t cnt[kMaxSegs];
    int n;
};

// Σ of the segments' values (int64, wrapping like the reference's accumulation): per segment
// an unaligned head, 32-byte sector loads, a tail; warp shuffle + block reduction, one atomic
// per block.
__global__ void __launch_bounds__(256) segment_sum_kernel(const long long* p, Segs sg, unsigned long long* out) {
    unsigned long long acc = 0;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (int k = 0; k < sg.n; ++k) {
        const uint64_t o = sg.off[k], c = sg.cnt[k];
        const uint64_t head = min(c, (4u - (o & 3u)) & 3u);
        const uint64_t vec = (c - head) / 4, body = o + head;
        for (uint64_t i = tid; i < head; i += stride) acc += (unsigned long long)p[o + i];
#pragma unroll 4
        for (uint64_t i = tid; i < vec; i += stride) acc += masked_sum4(ldg_sector(p + body + 4 * i), 0xFu);
        for (uint64_t i = body + 4 * vec + tid; i < o + c; i += stride) acc += (unsigned long long)p[i];
    }
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

// SW on the segments: every member value <- v (32-byte sector stores in the aligned body)
__global__ void __launch_bounds__(256) segment_fill_kernel(long long* p, Segs sg, long long v) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    Sector sv;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        sv.w[2 * i] = (uint32_t)(unsigned long long)v;
        sv.w[2 * i + 1] = (uint32_t)((unsigned long long)v >> 32);
    }
    for (int k = 0; k < sg.n; ++k) {
        const uint64_t o = sg.off[k], c = sg.cnt[k];
        const uint64_t head = min(c, (4u - (o & 3u)) & 3u);
        const uint64_t vec = (c - head) / 4, body = o + head;
        for (uint64_t i = tid; i < head; i += stride) p[o + i] = v;
        for (uint64_t i = tid; i < vec; i += stride) stg_sector(p + body + 4 * i, sv);
        for (uint64_t i = body + 4 * vec + tid; i < o + c; i += stride) p[i] = v;
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
    uint32_t tile_begin, tile_end;  // the CA step's shard of the tile order u (all: 0, tiles)
    uint32_t birth, survive;
};

// Base-3 value of a bit mask read as digits in {0,1}: the 8 values of 3 bits packed as nibbles.
__device__ __forceinline__ uint32_t bits_base3(uint32_t b) {
    constexpr uint32_t L = 0xDCA94310u;  // 0,1,3,4,9,10,12,13
    return ((L >> (4u * (b & 7u))) & 15u) + 27u * ((L >> (4u * ((b >> 3) & 7u))) & 15u) +
           729u * ((L >> (4u * ((b >> 6) & 7u))) & 15u);
}
// bits 0,2,4,... of v (< 2^18) packed together
__device__ __forceinline__ uint32_t even_bits(uint32_t v) {
    v &= 0x15555u;
    v = (v | (v >> 1)) & 0x13333u;
    v = (v | (v >> 2)) & 0x10F0Fu;
    v = (v | (v >> 4)) & 0x100FFu;
    return (v | (v >> 8)) & 0x1FFu;
}
// Compact offset (ωy·W + ωx) of a gasket member cell (x, y): λ⁻¹ at full level, where every
// digit is β = bit_x + bit_y (gasket offsets (0,0),(0,1),(1,1); block_map.cpp:113-148), odd
// levels μ (bit μ−1 even) feeding ωx and even levels feeding ωy. Valid for r ≤ 18.
__device__ __forceinline__ uint64_t gasket_compact_offset(uint32_t x, uint32_t y, uint32_t W) {
    const uint32_t ox = bits_base3(even_bits(x)) + bits_base3(even_bits(y));
    const uint32_t oy = bits_base3(even_bits(x >> 1)) + bits_base3(even_bits(y >> 1));
    return (uint64_t)oy * W + ox;
}

// ---- multi-GPU (P2P) step ordering -------------------------------------------------------
constexpr int kMaxP2P = 8;
struct P2PArgs {
    const long long* const* peer_src;  // [world] each rank's source buffer of this pass
    unsigned int* sync;                // this rank's {arrivals, done CTAs, error, unused}
    unsigned int* const* peer_flag;    // [world] every rank's sync word (arrival counter first)
    unsigned int wait_target;          // arrivals required before the pass may start (world x pass)
    unsigned int timeout_ms;
    int world, rank;
    FastDiv div_chunk;                 // tiles per rank: the owner of tile u is u / chunk
    unsigned int first_pass;           // first pass of a call: also wait for the previous grid
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// One thread per CTA: spin (bounded) until every rank finished the previous step. Every rank's
// last CTA of step i-1 adds one arrival here after its CTAs' stores, so world x i arrivals mean
// every peer's step i-1 output (this step's halo source) is complete AND no peer still reads the
// buffer this step overwrites (their step i-1 source). This rank's own arrival is included,
// which orders the step after this rank's previous kernel even when it was launched early (PDL).
__device__ __forceinline__ void p2p_wait(const P2PArgs& p) {
    if (p.wait_target == 0u) return;
    const unsigned long long t0 = global_ns();
    unsigned int v;
    for (;;) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p.sync) : "memory");
        if (v >= p.wait_target) break;
        if (global_ns() - t0 > 1000000ull * p.timeout_ms) {
            atomicExch(p.sync + 2, 1u);
            break;
        }
        __nanosleep(64);
    }
}

// After the CTA's last store: each CTA counts itself done with an acq_rel atomic at GPU scope
// (releasing its stores; peers read this GPU's memory through its L2); the last CTA — which has
// acquired every other CTA's release through that counter — fences once at system scope
// (cumulative over what it acquired) and announces the step to every rank with relaxed
// system-scope reductions: one GPU-scope atomic per CTA, one system fence per step.
__device__ __forceinline__ void p2p_arrive(const P2PArgs& p) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.sync + 1) : "memory");
        if (prev == gridDim.x - 1) {
            // the next step's CTAs count only after they pass their wait (which needs this
            // CTA's own arrival below, released after this store)
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(p.sync + 1) : "memory");
            asm volatile("fence.acq_rel.sys;" ::: "memory");
            for (int r = 0; r < p.world; ++r)
                asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(p.peer_flag[r]) : "memory");
        }
    }
}

// Programmatic dependent launch (the next step's CTAs are scheduled while this step drains
// and run their prologue; griddepcontrol.wait orders them after this grid's stores).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---- shared stage of the compact CA pass (compact_pass.cuh) --------------------------------
// One bit-sliced step of a tile held as row masks (lane = row y, bit x) with the 8 H1 halo
// bits h (order of compact_halo_table_kernel); members only.
__device__ __forceinline__ uint32_t compact_rows_step(uint32_t R, uint32_t h, int lane, uint32_t birth,
                                                      uint32_t survive) {
    uint64_t E = (uint64_t)R << 1;
    if (lane == 31) E |= ((h >> 3) & 1u) | ((uint64_t)((h >> 5) & 1u) << 33);
    if (lane == 30) E |= (uint64_t)((h >> 4) & 1u) << 33;
    const uint64_t top = (h & 1u) | (((h >> 1) & 1u) << 1) | (((h >> 2) & 1u) << 2);
    const uint64_t bottom = (((h >> 7) & 1u) << 1) | ((uint64_t)((h >> 6) & 1u) << 33);
    const uint64_t Eu = __shfl_up_sync(0xFFFFFFFFu, E, 1);
    const uint64_t Ed = __shfl_down_sync(0xFFFFFFFFu, E, 1);
    const uint64_t U = lane == 0 ? top : Eu;
    const uint64_t D = lane == 31 ? bottom : Ed;
    return life_rule((uint32_t)U, (uint32_t)(U >> 1), (uint32_t)(U >> 2), (uint32_t)E, (uint32_t)(E >> 2),
                     (uint32_t)D, (uint32_t)(D >> 1), (uint32_t)(D >> 2), (uint32_t)(E >> 1), birth, survive) &
           submask_bits((uint32_t)lane);
}

// ---- embedded member sectors <-> compact state, tile by tile ------------------------------
// Local compact index li = ωy_l·27 + ωx_l of member (x, y) of a ρ = 32 tile (x ⊆ y < 32).
__device__ __forceinline__ uint32_t tile_local_index(uint32_t x, uint32_t y) {
    const uint32_t wx = bits_base3(even_bits(x)) + bits_base3(even_bits(y));
    const uint32_t wy = bits_base3(even_bits(x >> 1)) + bits_base3(even_bits(y >> 1));
    return wy * 27u + wx;
}

// Slot e < 108 of a ρ = 32 int64 tile: the e-th member sector in row-major order,
// packed y | s << 5 (row y holds the 2^popc(y>>2) sectors s ⊆ y>>2).
__device__ __forceinline__ uint32_t tile_sector_slot(uint32_t e) {
    uint32_t y = 0;
    for (; y < 32u; ++y) {
        const uint32_t cnt = 1u << __popc(y >> 2);
        if (e < cnt) break;
        e -= cnt;
    }
    return y | (pdep32(e, y >> 2) << 5);
}

// Warp per λ tile: read the tile's 108 member sectors of an embedded int64 grid (device or
// mapped pinned host memory — every byte crossing PCIe is a member sector) and write its 243
// values as the tile's 9 x 27 compact sub-block. Replaces embedded -> compact_store for the
// host-buffer CA call (no 32 GiB embedded staging grid on the device).
__global__ void __launch_bounds__(256) compact_from_sectors_kernel(const long long* emb, long long* comp,
                                                                   CompactCaArgs a, FastDiv div_hb) {
    __shared__ long long s_v[8][256];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t slot[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t e = 32u * k + lane;
        slot[k] = e < 108u ? tile_sector_slot(e) : 0xFFFFFFFFu;
    }
    const uint32_t warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t warp_stride = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t u = warp_global; u < a.tiles; u += warp_stride) {
        const uint32_t wxb = fastdiv(u, div_hb), wyb = u - wxb * a.Hb;
        uint32_t bx, by;
        lambda_const(wxb, wyb, bx, by);
        const int64_t org = (int64_t)by * 32 * a.n + (int64_t)bx * 32;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (slot[k] == 0xFFFFFFFFu) continue;
            const uint32_t y = slot[k] & 31u, sx = slot[k] >> 5;
            const Sector v = ld_sector(emb + org + (int64_t)y * a.n + 4 * sx);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t x = 4u * sx + c;
                if ((x & ~y) == 0u)
                    s_v[wib][tile_local_index(x, y)] =
                        (long long)(((unsigned long long)v.w[2 * c + 1] << 32) | v.w[2 * c]);
            }
        }
        __syncwarp();
        const uint64_t base = (uint64_t)(9u * wxb) * a.W + 27u * wyb;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t li = 32u * k + lane;
            if (li < 243u) comp[base + (li / 27u) * a.W + li % 27u] = s_v[wib][li];
        }
        __syncwarp();
    }
}

// The inverse: compact sub-block of each tile -> its 108 member sectors of an embedded int64
// grid (non-member cells of those sectors written 0; other sectors untouched).
__global__ void __launch_bounds__(256) compact_to_sectors_kernel(const long long* comp, long long* emb,
                                                                 CompactCaArgs a, FastDiv div_hb) {
    __shared__ long long s_v[8][256];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t slot[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t e = 32u * k + lane;
        slot[k] = e < 108u ? tile_sector_slot(e) : 0xFFFFFFFFu;
    }
    const uint32_t warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t warp_stride = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t u = warp_global; u < a.tiles; u += warp_stride) {
        const uint32_t wxb = fastdiv(u, div_hb), wyb = u - wxb * a.Hb;
        const uint64_t base = (uint64_t)(9u * wxb) * a.W + 27u * wyb;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t li = 32u * k + lane;
            if (li < 243u) s_v[wib][li] = comp[base + (li / 27u) * a.W + li % 27u];
        }
        __syncwarp();
        uint32_t bx, by;
        lambda_const(wxb, wyb, bx, by);
        const int64_t org = (int64_t)by * 32 * a.n + (int64_t)bx * 32;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (slot[k] == 0xFFFFFFFFu) continue;
            const uint32_t y = slot[k] & 31u, sx = slot[k] >> 5;
            Sector v;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t x = 4u * sx + c;
                const unsigned long long q =
                    (x & ~y) == 0u ? (unsigned long long)s_v[wib][tile_local_index(x, y)] : 0ull;
                v.w[2 * c] = (uint32_t)q;
                v.w[2 * c + 1] = (uint32_t)(q >> 32);
            }
            stg_sector(emb + org + (int64_t)y * a.n + 4 * sx, v);
        }
        __syncwarp();
    }
}

// ---- embedded Grid <-> compact state in embedded ROW order (the host boundary) ----------------
// Warp per embedded row y: its member sectors s ⊆ (y >> 2) in increasing address order, member
// cells i ⊆ (y & 3) inside each. Used for the pinned host Grid of nbb_gpu_ca: walking the Grid
// row by row keeps consecutive zero-copy accesses on the same host pages, which the tile walk
// does not (a tile spans 32 rows 512 KB apart) — tools/probe_zero_copy.cu: member-sector reads
// 19.5 ms row-major vs 29 ms in tile order, writes 20.7 vs 27.4 ms, at n = 2^16. The compact
// side takes scattered 8-byte accesses in HBM (λ⁻¹ of each cell, gasket_compact_offset).
__global__ void __launch_bounds__(256) compact_from_rows_kernel(const long long* emb, long long* comp, int64_t n,
                                                                uint32_t W) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (uint32_t y = warp; y < (uint32_t)n; y += nwarps) {
        const uint32_t m = y >> 2, cnt = 1u << __popc(m);
        const uint32_t nib = submask_bits(y & 3u) & 0xFu;
#pragma unroll 4
        for (uint32_t j = (uint32_t)lane; j < cnt; j += 32u) {
            const uint32_t sx = pdep32(j, m);
            const Sector v = ld_sector(emb + (int64_t)y * n + 4 * (int64_t)sx);
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if ((nib >> c) & 1u)
                    comp[gasket_compact_offset(4u * sx + c, y, W)] =
                        (long long)(((unsigned long long)v.w[2 * c + 1] << 32) | v.w[2 * c]);
        }
    }
}

__global__ void __launch_bounds__(256) compact_to_rows_kernel(const long long* comp, long long* emb, int64_t n,
                                                              uint32_t W) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (uint32_t y = warp; y < (uint32_t)n; y += nwarps) {
        const uint32_t m = y >> 2, cnt = 1u << __popc(m);
        const uint32_t nib = submask_bits(y & 3u) & 0xFu;
#pragma unroll 4
        for (uint32_t j = (uint32_t)lane; j < cnt; j += 32u) {
            const uint32_t sx = pdep32(j, m);
            Sector v;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const unsigned long long q =
                    ((nib >> c) & 1u) ? (unsigned long long)__ldg(comp + gasket_compact_offset(4u * sx + c, y, W)) : 0ull;
                v.w[2 * c] = (uint32_t)q;
                v.w[2 * c + 1] = (uint32_t)(q >> 32);
            }
            stg_sector(emb + (int64_t)y * n + 4 * (int64_t)sx, v);
        }
    }
}

}  // namespace nbbgpu
