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
    const long long* const* peer_src;  // [world] each rank's source buffer of this step
    const uint8_t* halo_owner;         // [tiles * 8] rank owning each halo cell
    unsigned int* sync;                // this rank's {arrivals, done CTAs, error, unused}
    unsigned int* const* peer_flag;    // [world] every rank's sync word (arrival counter first)
    unsigned int wait_target;          // arrivals required before the step may start (world x step)
    unsigned int timeout_ms;
    int world, rank;
    unsigned int chunk;                // tiles per rank (ca_compact2_kernel: owner = tile / chunk)
    unsigned int own_lo, own_hi;       // compact offsets [lo, hi) inside this rank's whole tile rows
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

// The 8 halo cells of every ρ = 32 tile as compact offsets (-1: not a member / outside),
// [tile u][k] for the tile-local positions (-1,-1) (0,-1) (1,-1) (-1,31) (32,30) (32,31)
// (32,32) (0,32). Static per level; built once per device and level (5.7 MB at r = 16) so
// the CA step spends one 32-byte load per tile instead of λ + λ⁻¹ arithmetic.
__global__ void compact_halo_table_kernel(CompactCaArgs a, FastDiv div_hb, int32_t* tab) {
    const uint32_t nm1 = (uint32_t)(a.n - 1);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (uint64_t)a.tiles * 8u;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = (uint32_t)(i >> 3), hk = (uint32_t)i & 7u;
        const int hx = (hk == 0 || hk == 3) ? -1 : (hk == 1 || hk == 7) ? 0 : (hk == 2) ? 1 : 32;
        const int hy = (hk <= 2) ? -1 : (hk == 3 || hk == 5) ? 31 : (hk == 4) ? 30 : 32;
        const uint32_t wxb = fastdiv(u, div_hb), wyb = u - wxb * a.Hb;
        uint32_t bx, by;
        lambda_arith(wxb, wyb, bx, by);
        const uint32_t gx = bx * 32u + (uint32_t)hx, gy = by * 32u + (uint32_t)hy;  // wraps if < 0
        const bool ok = gx <= nm1 && gy <= nm1 && (gx & (nm1 - gy)) == 0u;
        tab[i] = ok ? (int32_t)gasket_compact_offset(gx, gy, a.W) : -1;
    }
}

// One warp per tile; tile u -> (ωx_b = u / Hb, ωy_b = u % Hb) so consecutive warps walk along a
// compact row block. 243 values per tile = slots k = 0..7 of lane l: li = 32k + l (k < 7 valid
// for every lane, k = 7 for lanes < 19).
//
// Per tile: 8 coalesced 8-byte loads per lane (compact rows of 27 values), the 8 halo cells
// (compact offsets from the per-level halo table), alive bits scattered as bytes into a per-warp
// 32 x 32 byte tile (non-member bytes stay 0, so no atomics and no clearing), rows packed back
// to bit masks (lane = row) for the bit-sliced rule, and 8 stores per lane. Software-pipelined
// (the next tile's loads fly during this tile's rule and stores) and launched with PDL; at
// n = 2^16 a step runs at 0.964 of the measured HBM copy peak, long-scoreboard the dominant
// stall (ncu: profiles/r1_ncu_ca_compact_v5.txt). Tried and slower on B200
// (profiles/r1_compact_ca_tuning.md): a cp.async ring (8-byte copies), L2 bulk prefetch one
// tile ahead, 64/48-register budgets, cp.async.bulk row copies into an mbarrier ring, all steps
// in one launch with tile-level dataflow, and exported boundary-cell bytes for the halo.
//
// P2P = true is the multi-GPU form (one kernel per step, no separate exchange): each rank
// owns a contiguous range of tiles in its own replica-sized buffers, the halo cells owned
// by other ranks are read straight from their buffers over NVLink (CUDA IPC mappings,
// ld.relaxed.sys), and a flag barrier in peer memory orders the steps: the kernel first
// waits until every rank has finished the previous step (world x i arrivals on this rank's
// counter before step i), and its last CTA to finish adds one arrival to every rank's flag.
template <bool P2P>
__global__ void __launch_bounds__(256, 3) ca_compact_kernel(CompactCaArgs a, FastDiv div_hb,
                                                             const int32_t* __restrict__ halo_tab,
                                                             P2PArgs p) {
    __shared__ __align__(16) uint8_t s_cell[8][32 * 32];
    __shared__ uint32_t s_new[8][32];
    __shared__ uint16_t s_pos[256];  // c_local_pos (per-lane constant-bank reads serialise)
    __shared__ const long long* s_peer[kMaxP2P];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint8_t* cell = s_cell[wib];
    pdl_trigger();
    s_pos[threadIdx.x] = threadIdx.x < 243 ? c_local_pos[threadIdx.x] : 0;
    if (P2P && p.wait_target != 0u) {
        // the arrival wait subsumes pdl_wait: this rank's own arrival for the previous step is
        // in it (its last CTA's stores released before it), so no grid-completion wait
        if (threadIdx.x < (unsigned)p.world) s_peer[threadIdx.x] = p.peer_src[threadIdx.x];
        if (threadIdx.x == 0) p2p_wait(p);
    } else {
        // plain steps, and the first P2P step of a sequence (its predecessor on the stream is
        // whatever produced the state, not a P2P step)
        if (P2P && threadIdx.x < (unsigned)p.world) s_peer[threadIdx.x] = p.peer_src[threadIdx.x];
        pdl_wait();
    }
    __syncthreads();
    uint32_t sl_off[8], sl_pos[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t li = 32u * k + lane;
        const bool ok = li < 243u;
        const uint32_t row = ok ? li / 27u : 0u, col = ok ? li % 27u : 0u;
        sl_off[k] = (row * a.W + col) * 8u;  // byte offset inside the tile's sub-block
        sl_pos[k] = s_pos[li];               // x | y << 5 = byte index in the 32 x 32 tile
    }
    const bool k7 = lane < 19;
#pragma unroll
    for (int i = 0; i < 8; ++i) reinterpret_cast<uint32_t*>(cell)[32 * i + lane] = 0u;
    const uint32_t warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t warp_stride = (gridDim.x * blockDim.x) >> 5;
    const char* src0 = reinterpret_cast<const char*>(a.src);
    char* dst0 = reinterpret_cast<char*>(a.dst);
    __syncwarp();

    // Software-pipelined over the warp's tiles: tile u+stride's loads (its 243 values and
    // halo cells) are issued as soon as tile u's values are in the byte tile — into the same
    // registers — so they fly while tile u's rule and stores run; the halo-table entries run
    // one more tile ahead (the halo load depends on them).
    auto tile_base = [&](uint32_t t) -> uint64_t {
        const uint32_t wxb = fastdiv(t, div_hb), wyb = t - wxb * a.Hb;
        return ((uint64_t)(9u * wxb) * a.W + 27u * wyb) * 8u;
    };
    long long v[8];
    auto load_tile = [&](uint64_t b) {
        const char* src = src0 + b;
#pragma unroll
        for (int k = 0; k < 7; ++k) v[k] = __ldg(reinterpret_cast<const long long*>(src + sl_off[k]));
        v[7] = k7 ? __ldg(reinterpret_cast<const long long*>(src + sl_off[7])) : 0ll;
    };
    auto load_halo = [&](int32_t off, uint32_t own) -> long long {
        long long hv = 0;
        if (off >= 0) {
            if (!P2P || own == (uint32_t)p.rank)
                hv = __ldg(a.src + off);
            else  // a cell of another rank's tile: read its buffer over NVLink
                asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(hv) : "l"(s_peer[own] + off));
        }
        return hv;
    };
    auto halo_entry = [&](uint32_t t, int32_t& off, uint32_t& own) {
        const bool ok = t < a.tile_end && lane < 8;
        off = ok ? __ldg(halo_tab + 8ull * t + lane) : -1;
        own = (P2P && ok) ? p.halo_owner[8ull * t + lane] : 0u;
    };

    uint32_t u = a.tile_begin + warp_global;
    uint64_t base = 0;
    long long hv = 0;
    int32_t hoff_n = -1;
    uint32_t hown_n = 0;
    if (u < a.tile_end) {
        base = tile_base(u);
        load_tile(base);
        int32_t off;
        uint32_t own;
        halo_entry(u, off, own);
        hv = load_halo(off, own);
        halo_entry(u + warp_stride, hoff_n, hown_n);
    }
    for (; u < a.tile_end; u += warp_stride) {
        const uint32_t un = u + warp_stride;
#pragma unroll
        for (int k = 0; k < 7; ++k) cell[sl_pos[k]] = v[k] != 0ll;
        if (k7) cell[sl_pos[7]] = v[7] != 0ll;
        const uint32_t h = __ballot_sync(0xFFFFFFFFu, hv != 0ll) & 0xFFu;
        uint64_t base_n = 0;
        if (un < a.tile_end) {  // warp-uniform
            base_n = tile_base(un);
            load_tile(base_n);
            hv = load_halo(hoff_n, hown_n);
            halo_entry(un + warp_stride, hoff_n, hown_n);
        }
        __syncwarp();
        uint32_t R;
        {   // 0/1 bytes -> bits (as in ca_compact2_kernel)
            const uint4 q0 = reinterpret_cast<const uint4*>(cell + 32 * lane)[0];
            const uint4 q1 = reinterpret_cast<const uint4*>(cell + 32 * lane)[1];
            const uint32_t p0 = (q0.x + (q0.y << 4)) * 0x01020408u, p1 = (q0.z + (q0.w << 4)) * 0x01020408u;
            const uint32_t p2 = (q1.x + (q1.y << 4)) * 0x01020408u, p3 = (q1.z + (q1.w << 4)) * 0x01020408u;
            R = __byte_perm(__byte_perm(p0, p1, 0x0073u), __byte_perm(p2, p3, 0x0073u), 0x5410u);
        }
        uint64_t E = (uint64_t)R << 1;
        if (lane == 31) E |= ((h >> 3) & 1u) | ((uint64_t)((h >> 5) & 1u) << 33);
        if (lane == 30) E |= (uint64_t)((h >> 4) & 1u) << 33;
        const uint64_t top = (h & 1u) | (((h >> 1) & 1u) << 1) | (((h >> 2) & 1u) << 2);
        const uint64_t bottom = (((h >> 7) & 1u) << 1) | ((uint64_t)((h >> 6) & 1u) << 33);
        const uint64_t Eu = __shfl_up_sync(0xFFFFFFFFu, E, 1);
        const uint64_t Ed = __shfl_down_sync(0xFFFFFFFFu, E, 1);
        const uint64_t U = lane == 0 ? top : Eu;
        const uint64_t D = lane == 31 ? bottom : Ed;
        s_new[wib][lane] = life_rule((uint32_t)U, (uint32_t)(U >> 1), (uint32_t)(U >> 2), (uint32_t)E,
                                     (uint32_t)(E >> 2), (uint32_t)D, (uint32_t)(D >> 1), (uint32_t)(D >> 2),
                                     (uint32_t)(E >> 1), a.birth, a.survive) &
                           submask_bits((uint32_t)lane);
        __syncwarp();
        char* dst = dst0 + base;
        base = base_n;
#pragma unroll
        for (int k = 0; k < 7; ++k)
            *reinterpret_cast<long long*>(dst + sl_off[k]) =
                (long long)((s_new[wib][sl_pos[k] >> 5] >> (sl_pos[k] & 31u)) & 1u);
        if (k7)
            *reinterpret_cast<long long*>(dst + sl_off[7]) =
                (long long)((s_new[wib][sl_pos[7] >> 5] >> (sl_pos[7] & 31u)) & 1u);
        __syncwarp();
    }
    if (P2P) p2p_arrive(p);
}


// ---- two CA steps per pass (temporal blocking of the compact step) ------------------------
// The radius-2 halo of a ρ = 32 tile: the 8 cells of compact_halo_table_kernel (H1, the
// member neighbours of the tile's members) followed by the 14 positions that can hold a member
// neighbour of an H1 cell outside the tile (H2; found by brute force over every tile of r = 6..11,
// the set is the same at every level by self-similarity). Tile-local (x, y).
constexpr int kHalo2 = 22, kHalo2Stride = 24;
__constant__ int8_t c_h2x[kHalo2] = {-1, 0, 1, -1, 32, 32, 32, 0, -2, -2, -2, -2, 0, 0, 1, 2, 2, 32, 32, 33, 33, 33};
__constant__ int8_t c_h2y[kHalo2] = {-1, -1, -1, 31, 30, 31, 32, 32, -2, -1, 30, 31, -2, 33, 33, -2, -1, 29, 33, 29, 31, 33};

// [tile u][k] compact offsets of the 22 halo positions (-1: not a member / outside), stride 24
__global__ void compact_halo2_table_kernel(CompactCaArgs a, FastDiv div_hb, int32_t* tab) {
    const uint32_t nm1 = (uint32_t)(a.n - 1);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (uint64_t)a.tiles * kHalo2Stride;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = (uint32_t)(i / kHalo2Stride), hk = (uint32_t)(i % kHalo2Stride);
        int32_t off = -1;
        if (hk < (uint32_t)kHalo2) {
            const uint32_t wxb = fastdiv(u, div_hb), wyb = u - wxb * a.Hb;
            uint32_t bx, by;
            lambda_arith(wxb, wyb, bx, by);
            const uint32_t gx = bx * 32u + (uint32_t)(int)c_h2x[hk], gy = by * 32u + (uint32_t)(int)c_h2y[hk];
            if (gx <= nm1 && gy <= nm1 && (gx & (nm1 - gy)) == 0u) off = (int32_t)gasket_compact_offset(gx, gy, a.W);
        }
        tab[i] = off;
    }
}

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

// Two CA steps per pass over the compact state: each warp loads its tile (243 values) and the
// 22 radius-2 halo cells once, computes step t+1 for the tile (bit-sliced) and for its 8 H1
// halo cells (lanes 0..7, scalar, from the step-t bytes), then step t+2 for the tile from those,
// and stores step t+2 — 8 B read + 8 B write per member per TWO steps. Same tile walk, software
// pipeline and PDL as ca_compact_kernel; the step-t+1 state never reaches HBM. The pass is
// ALU-bound, so the reference's default rule (CaRule{}: B3/S23) has its own instantiation with
// the rule masks known at compile time (the bit-sliced rule's leaves fold away); every other
// rule runs the generic one.
//
// P2P = true is the multi-GPU pass (as ca_compact_kernel<true>): the halo cells of other ranks'
// tiles are read from their buffers over NVLink, the owner computed from the compact offset
// (tile = (row / 9) H_b + col / 27, owner = tile / chunk), and the same flag barrier orders
// the passes (world x j arrivals before pass j).
template <bool CONWAY, bool P2P>
__global__ void __launch_bounds__(256, 3) ca_compact2_kernel(CompactCaArgs a, FastDiv div_hb,
                                                             const int32_t* __restrict__ halo_tab,
                                                             P2PArgs p) {
    const uint32_t birth = CONWAY ? (1u << 3) : a.birth;
    const uint32_t survive = CONWAY ? (1u << 2) | (1u << 3) : a.survive;
    __shared__ __align__(16) uint8_t s_cell[8][32 * 32];
    __shared__ uint32_t s_new[8][32];
    __shared__ uint16_t s_pos[256];
    // H1 cell k's neighbours: the halo slots among them (bit mask over the 22) and its <= 3
    // in-tile positions (byte index; padded with byte 1 = cell (1, 0), never a member, always 0)
    __shared__ uint32_t s_nb[8];
    __shared__ __align__(8) uint16_t s_nt[8][4];
    __shared__ const long long* s_peer[kMaxP2P];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint8_t* cell = s_cell[wib];
    pdl_trigger();
    if (P2P && threadIdx.x < (unsigned)p.world) s_peer[threadIdx.x] = p.peer_src[threadIdx.x];
    s_pos[threadIdx.x] = threadIdx.x < 243 ? c_local_pos[threadIdx.x] : 0;
    if (threadIdx.x < 8) {
        const int k = threadIdx.x;
        uint32_t nb = 0;
        int nt = 0;
        for (int i = 0; i < 4; ++i) s_nt[k][i] = 1;
        for (int dd = 0; dd < 9; ++dd) {  // the 8 neighbours of the 3 x 3 block, centre skipped
            if (dd == 4) continue;
            const int qx = c_h2x[k] + dd % 3 - 1, qy = c_h2y[k] + dd / 3 - 1;
            if (qx >= 0 && qx < 32 && qy >= 0 && qy < 32) {
                if (nt < 4) s_nt[k][nt++] = (uint16_t)(qy * 32 + qx);
            } else {
                for (int j = 0; j < kHalo2; ++j)
                    if (c_h2x[j] == qx && c_h2y[j] == qy) nb |= 1u << j;
            }
        }
        s_nb[k] = nb;
    }
    if (P2P && p.wait_target != 0u) {  // the arrival wait subsumes pdl_wait (ca_compact_kernel)
        if (threadIdx.x == 0) p2p_wait(p);
    } else {
        pdl_wait();
    }
    __syncthreads();
    uint32_t sl_off[8], sl_pos[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t li = 32u * k + lane;
        const bool ok = li < 243u;
        const uint32_t row = ok ? li / 27u : 0u, col = ok ? li % 27u : 0u;
        sl_off[k] = (row * a.W + col) * 8u;
        sl_pos[k] = s_pos[li];
    }
    const bool k7 = lane < 19;
#pragma unroll
    for (int i = 0; i < 8; ++i) reinterpret_cast<uint32_t*>(cell)[32 * i + lane] = 0u;
    const uint32_t warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t warp_stride = (gridDim.x * blockDim.x) >> 5;
    const char* src0 = reinterpret_cast<const char*>(a.src);
    char* dst0 = reinterpret_cast<char*>(a.dst);
    __syncwarp();

    auto tile_base = [&](uint32_t t) -> uint64_t {
        const uint32_t wxb = fastdiv(t, div_hb), wyb = t - wxb * a.Hb;
        return ((uint64_t)(9u * wxb) * a.W + 27u * wyb) * 8u;
    };
    long long v[8];
    auto load_tile = [&](uint64_t b) {
        const char* src = src0 + b;
#pragma unroll
        for (int k = 0; k < 7; ++k) v[k] = __ldg(reinterpret_cast<const long long*>(src + sl_off[k]));
        v[7] = k7 ? __ldg(reinterpret_cast<const long long*>(src + sl_off[7])) : 0ll;
    };
    auto halo_entry = [&](uint32_t t) -> int32_t {
        return (t < a.tile_end && lane < kHalo2) ? __ldg(halo_tab + (uint64_t)kHalo2Stride * t + lane) : -1;
    };
    auto load_halo = [&](int32_t off) -> long long {
        long long hv = 0;
        if (off >= 0) {
            uint32_t own = (uint32_t)p.rank;
            if (P2P && ((uint32_t)off < p.own_lo || (uint32_t)off >= p.own_hi)) {  // not surely ours
                const uint32_t row = (uint32_t)off / a.W, col = (uint32_t)off - row * a.W;
                own = ((row / 9u) * a.Hb + col / 27u) / p.chunk;
            }
            if (!P2P || own == (uint32_t)p.rank)
                hv = __ldg(a.src + off);
            else  // a cell of another rank's tile: read its buffer over NVLink
                asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(hv) : "l"(s_peer[own] + off));
        }
        return hv;
    };

    uint32_t u = a.tile_begin + warp_global;
    uint64_t base = 0;
    long long hv = 0;
    uint32_t hmem = 0;  // H1 slots that are members (bit k)
    int32_t hoff_n = -1;
    if (u < a.tile_end) {
        base = tile_base(u);
        load_tile(base);
        const int32_t off = halo_entry(u);
        hv = load_halo(off);
        hmem = __ballot_sync(0xFFFFFFFFu, off >= 0) & 0xFFu;
        hoff_n = halo_entry(u + warp_stride);
    }
    for (; u < a.tile_end; u += warp_stride) {
        const uint32_t un = u + warp_stride;
#pragma unroll
        for (int k = 0; k < 7; ++k) cell[sl_pos[k]] = v[k] != 0ll;
        if (k7) cell[sl_pos[7]] = v[7] != 0ll;
        const uint32_t hm = __ballot_sync(0xFFFFFFFFu, hv != 0ll);  // step-t halo alive bits
        const uint32_t hmem_cur = hmem;
        uint64_t base_n = 0;
        if (un < a.tile_end) {  // warp-uniform
            base_n = tile_base(un);
            load_tile(base_n);
            hv = load_halo(hoff_n);
            hmem = __ballot_sync(0xFFFFFFFFu, hoff_n >= 0) & 0xFFu;
            hoff_n = halo_entry(un + warp_stride);
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
        // step t+1: the tile (bit-sliced) and the H1 cells (lane k < 8, scalar)
        const uint32_t R1 = compact_rows_step(R, hm & 0xFFu, lane, birth, survive);
        uint32_t live;
        {
            const uint2 t = *reinterpret_cast<const uint2*>(s_nt[lane & 7]);
            live = __popc(hm & s_nb[lane & 7]) + cell[t.x & 0xFFFFu] + cell[t.x >> 16] + cell[t.y & 0xFFFFu];
        }
        const uint32_t rule = ((hm >> (lane & 7)) & 1u) ? survive : birth;
        const uint32_t h1 = __ballot_sync(0xFFFFFFFFu, lane < 8 && ((rule >> live) & 1u)) & hmem_cur;
        // step t+2: the tile only
        s_new[wib][lane] = compact_rows_step(R1, h1, lane, birth, survive);
        __syncwarp();
        char* dst = dst0 + base;
        base = base_n;
#pragma unroll
        for (int k = 0; k < 7; ++k)
            *reinterpret_cast<long long*>(dst + sl_off[k]) =
                (long long)((s_new[wib][sl_pos[k] >> 5] >> (sl_pos[k] & 31u)) & 1u);
        if (k7)
            *reinterpret_cast<long long*>(dst + sl_off[7]) =
                (long long)((s_new[wib][sl_pos[7] >> 5] >> (sl_pos[7] & 31u)) & 1u);
        __syncwarp();
    }
    if (P2P) p2p_arrive(p);
}

// The BOUNDING-BOX launch of the compact-state CA step (the comparison for ca_compact_kernel on
// the same storage): identical per-tile work, but the warps walk all (n/32)^2 box tiles, cull
// the non-member ones and address each member tile through λ⁻¹ — the inverse map the compact
// layout needs (block_map.cpp:113-148) — instead of enumerating the λ orthotope.
__global__ void __launch_bounds__(256, 3) ca_compact_bb_kernel(CompactCaArgs a, FastDiv div_hb,
                                                              const int32_t* __restrict__ halo_tab) {
    constexpr bool P2P = false;
    const P2PArgs p{};
    __shared__ __align__(16) uint8_t s_cell[8][32 * 32];
    __shared__ uint32_t s_new[8][32];
    __shared__ uint16_t s_pos[256];  // c_local_pos (per-lane constant-bank reads serialise)
    __shared__ const long long* s_peer[kMaxP2P];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint8_t* cell = s_cell[wib];
    pdl_trigger();
    s_pos[threadIdx.x] = threadIdx.x < 243 ? c_local_pos[threadIdx.x] : 0;
    if (P2P && p.wait_target != 0u) {
        // the arrival wait subsumes pdl_wait: this rank's own arrival for the previous step is
        // in it (its last CTA's stores released before it), so no grid-completion wait
        if (threadIdx.x < (unsigned)p.world) s_peer[threadIdx.x] = p.peer_src[threadIdx.x];
        if (threadIdx.x == 0) p2p_wait(p);
    } else {
        // plain steps, and the first P2P step of a sequence (its predecessor on the stream is
        // whatever produced the state, not a P2P step)
        if (P2P && threadIdx.x < (unsigned)p.world) s_peer[threadIdx.x] = p.peer_src[threadIdx.x];
        pdl_wait();
    }
    __syncthreads();
    uint32_t sl_off[8], sl_pos[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t li = 32u * k + lane;
        const bool ok = li < 243u;
        const uint32_t row = ok ? li / 27u : 0u, col = ok ? li % 27u : 0u;
        sl_off[k] = (row * a.W + col) * 8u;  // byte offset inside the tile's sub-block
        sl_pos[k] = s_pos[li];               // x | y << 5 = byte index in the 32 x 32 tile
    }
    const bool k7 = lane < 19;
#pragma unroll
    for (int i = 0; i < 8; ++i) reinterpret_cast<uint32_t*>(cell)[32 * i + lane] = 0u;
    const uint32_t warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t warp_stride = (gridDim.x * blockDim.x) >> 5;
    const char* src0 = reinterpret_cast<const char*>(a.src);
    char* dst0 = reinterpret_cast<char*>(a.dst);
    __syncwarp();

    // Software-pipelined over the warp's tiles: tile u+stride's loads (its 243 values and
    // halo cells) are issued as soon as tile u's values are in the byte tile — into the same
    // registers — so they fly while tile u's rule and stores run; the halo-table entries run
    // one more tile ahead (the halo load depends on them).
    auto tile_base = [&](uint32_t t) -> uint64_t {
        const uint32_t wxb = fastdiv(t, div_hb), wyb = t - wxb * a.Hb;
        return ((uint64_t)(9u * wxb) * a.W + 27u * wyb) * 8u;
    };
    long long v[8];
    auto load_tile = [&](uint64_t b) {
        const char* src = src0 + b;
#pragma unroll
        for (int k = 0; k < 7; ++k) v[k] = __ldg(reinterpret_cast<const long long*>(src + sl_off[k]));
        v[7] = k7 ? __ldg(reinterpret_cast<const long long*>(src + sl_off[7])) : 0ll;
    };
    auto load_halo = [&](int32_t off, uint32_t own) -> long long {
        long long hv = 0;
        if (off >= 0) {
            if (!P2P || own == (uint32_t)p.rank)
                hv = __ldg(a.src + off);
            else  // a cell of another rank's tile: read its buffer over NVLink
                asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(hv) : "l"(s_peer[own] + off));
        }
        return hv;
    };
    auto halo_entry = [&](uint32_t t, int32_t& off, uint32_t& own) {
        const bool ok = t < a.tile_end && lane < 8;
        off = ok ? __ldg(halo_tab + 8ull * t + lane) : -1;
        own = (P2P && ok) ? p.halo_owner[8ull * t + lane] : 0u;
    };

    // the bounding box of (n/32)^2 tiles, walked with an odd warp stride (tile_kernel); a box
    // tile holds members iff bx ⊆ (n/32 - 1 - by) — the others are culled, as the reference's
    // threads of such a block all fail their test — and a member tile finds its storage in the
    // compact state through λ⁻¹ of its block coordinates (u = ωx_b·H_b + ωy_b)
    const uint32_t nb = (uint32_t)(a.n >> 5), lg = 31u - __clz(nb), boxes = nb * nb;
    const uint32_t ustride = (warp_stride | 1u) - ((warp_stride & 1u) ? 0u : 2u);
    auto next_member = [&](uint32_t bi) -> uint32_t {
        while (bi < boxes && ((bi & (nb - 1u)) & (nb - 1u - (bi >> lg))) != 0u) bi += ustride;
        return bi;
    };
    auto tile_of_box = [&](uint32_t bi) -> uint32_t {
        const uint32_t bx = bi & (nb - 1u), by = bi >> lg;
        const uint32_t wx = bits_base3(even_bits(bx)) + bits_base3(even_bits(by));
        const uint32_t wy = bits_base3(even_bits(bx >> 1)) + bits_base3(even_bits(by >> 1));
        return wx * a.Hb + wy;
    };
    uint32_t bcur = next_member(warp_global < ustride ? warp_global : boxes);
    uint32_t bnext = bcur < boxes ? next_member(bcur + ustride) : boxes;
    uint32_t u = bcur < boxes ? tile_of_box(bcur) : 0u;
    uint32_t u_next = bnext < boxes ? tile_of_box(bnext) : 0u;
    uint64_t base = 0;
    long long hv = 0;
    int32_t hoff_n = -1;
    uint32_t hown_n = 0;
    if (bcur < boxes) {
        base = tile_base(u);
        load_tile(base);
        int32_t off;
        uint32_t own;
        halo_entry(u, off, own);
        hv = load_halo(off, own);
        halo_entry(bnext < boxes ? u_next : a.tile_end, hoff_n, hown_n);
    }
    while (bcur < boxes) {
        const uint32_t un = u_next, bn = bnext;
        const bool more = bn < boxes;
        const uint32_t bnn = more ? next_member(bn + ustride) : boxes;  // the tile after next
        u_next = bnn < boxes ? tile_of_box(bnn) : 0u;
#pragma unroll
        for (int k = 0; k < 7; ++k) cell[sl_pos[k]] = v[k] != 0ll;
        if (k7) cell[sl_pos[7]] = v[7] != 0ll;
        const uint32_t h = __ballot_sync(0xFFFFFFFFu, hv != 0ll) & 0xFFu;
        uint64_t base_n = 0;
        if (more) {  // warp-uniform
            base_n = tile_base(un);
            load_tile(base_n);
            hv = load_halo(hoff_n, hown_n);
            halo_entry(bnn < boxes ? u_next : a.tile_end, hoff_n, hown_n);
        }
        __syncwarp();
        uint32_t R;
        {   // 0/1 bytes -> bits (as in ca_compact2_kernel)
            const uint4 q0 = reinterpret_cast<const uint4*>(cell + 32 * lane)[0];
            const uint4 q1 = reinterpret_cast<const uint4*>(cell + 32 * lane)[1];
            const uint32_t p0 = (q0.x + (q0.y << 4)) * 0x01020408u, p1 = (q0.z + (q0.w << 4)) * 0x01020408u;
            const uint32_t p2 = (q1.x + (q1.y << 4)) * 0x01020408u, p3 = (q1.z + (q1.w << 4)) * 0x01020408u;
            R = __byte_perm(__byte_perm(p0, p1, 0x0073u), __byte_perm(p2, p3, 0x0073u), 0x5410u);
        }
        uint64_t E = (uint64_t)R << 1;
        if (lane == 31) E |= ((h >> 3) & 1u) | ((uint64_t)((h >> 5) & 1u) << 33);
        if (lane == 30) E |= (uint64_t)((h >> 4) & 1u) << 33;
        const uint64_t top = (h & 1u) | (((h >> 1) & 1u) << 1) | (((h >> 2) & 1u) << 2);
        const uint64_t bottom = (((h >> 7) & 1u) << 1) | ((uint64_t)((h >> 6) & 1u) << 33);
        const uint64_t Eu = __shfl_up_sync(0xFFFFFFFFu, E, 1);
        const uint64_t Ed = __shfl_down_sync(0xFFFFFFFFu, E, 1);
        const uint64_t U = lane == 0 ? top : Eu;
        const uint64_t D = lane == 31 ? bottom : Ed;
        s_new[wib][lane] = life_rule((uint32_t)U, (uint32_t)(U >> 1), (uint32_t)(U >> 2), (uint32_t)E,
                                     (uint32_t)(E >> 2), (uint32_t)D, (uint32_t)(D >> 1), (uint32_t)(D >> 2),
                                     (uint32_t)(E >> 1), a.birth, a.survive) &
                           submask_bits((uint32_t)lane);
        __syncwarp();
        char* dst = dst0 + base;
        base = base_n;
        u = un;
        bcur = bn;
        bnext = bnn;
#pragma unroll
        for (int k = 0; k < 7; ++k)
            *reinterpret_cast<long long*>(dst + sl_off[k]) =
                (long long)((s_new[wib][sl_pos[k] >> 5] >> (sl_pos[k] & 31u)) & 1u);
        if (k7)
            *reinterpret_cast<long long*>(dst + sl_off[7]) =
                (long long)((s_new[wib][sl_pos[7] >> 5] >> (sl_pos[7] & 31u)) & 1u);
        __syncwarp();
    }
    (void)p;
    (void)u;
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
