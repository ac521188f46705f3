/* nbb_launch.cuh — the reference's operator API, `launch(config, kernel)`, for DEVICE functors.
 *
 * Reference: `using Kernel = std::function<void(uint64_t block_ordinal, EmbeddedCoord cell)>;
 *             WorkReport launch(const DispatchConfig&, const Kernel&);`
 *            (include/nbb/dispatch.hpp:100-108; src/dispatch.cpp:209-467 launch_impl).
 *
 * A host std::function cannot run on the GPU, so the C ABI (nbb_gpu.h) draws the drop-in
 * boundary at the workload level. CUDA callers who need the operator itself get it here:
 * header-only, compiled by nvcc into the caller's own translation unit,
 *
 *     struct Write1 { int64_t* g; int64_t n;
 *         __device__ void operator()(uint64_t ordinal, nbb::gpu::EmbeddedCoord c) const {
 *             g[c.y * n + c.x] = 1; } };
 *     nbb_report rep;
 *     int rc = nbb::gpu::launch(cfg, Write1{d_grid, n}, &rep, stream);
 *
 * Semantics follow launch_impl for the gasket with the subbox strategy and the direct
 * backend (the path every workload of the reference defaults to):
 *   λ mode : one CTA of ρ x ρ threads per block ordinal o of the W x H orthotope
 *            (W = 3^ceil(r_b/2), o = ωy·W + ωx, dispatch.cpp:262-263); the block origin is
 *            ρ·λ(ω) (dispatch.cpp:309, 355, closed form SURVEY App. A.1); thread (tx, ty) is
 *            active iff the local subbox test passes (tx ⊆ ty, dispatch.cpp:361-374) and then
 *            receives (o, origin + (tx, ty)).
 *   BB mode: one CTA per block of the (n/ρ)^2 box; thread active iff its cell is a member
 *            (x & (n-1-y)) == 0 (dispatch.cpp:278-300).
 * The functor runs concurrently on all active threads (the reference runs it on `workers`
 * threads): it must be race-free, as the reference's kernels must be for workers > 1. The
 * counters come from the library's closed form (nbb_gpu_plan_report) — identical to the
 * reference's tallies. cfg.shard_begin/shard_count launch a contiguous range of ordinals.
 * Errors: the library's validation (nbb_gpu_validate) and NBB_ERR_INVALID_ARGUMENT for specs,
 * strategies or backends this operator does not cover; CUDA launch errors -> NBB_ERR_CUDA. */
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "nbb_gpu.h"

namespace nbb {
namespace gpu {

struct EmbeddedCoord {
    int64_t x, y;
};

namespace detail {

/* X(v), Y(v): bit 2j set iff base-3 digit j of v is 2 (X) / >= 1 (Y) — SURVEY App. A.1 */
__device__ __forceinline__ void xy_digits(uint64_t v, uint64_t& X, uint64_t& Y) {
    X = 0;
    Y = 0;
    for (int j = 0; v != 0; ++j) {
        const uint64_t q = v / 3u, d = v - 3u * q;
        X |= (uint64_t)(d == 2u) << (2 * j);
        Y |= (uint64_t)(d != 0u) << (2 * j);
        v = q;
    }
}

struct LaunchArgs {
    uint64_t begin, end;  /* block ordinals [begin, end) */
    uint64_t gw;          /* grid width: W (λ) or n/ρ (BB) */
    int64_t n;
    int edge;
    int bb;
};

template <class F>
__global__ void launch_kernel(LaunchArgs a, F f) {
    const int64_t tx = threadIdx.x, ty = threadIdx.y;
    for (uint64_t o = a.begin + blockIdx.x; o < a.end; o += gridDim.x) {
        const uint64_t gx = o % a.gw, gy = o / a.gw;
        int64_t x, y;
        bool active;
        if (a.bb) {
            x = (int64_t)gx * a.edge + tx;
            y = (int64_t)gy * a.edge + ty;
            active = (x & (a.n - 1 - y)) == 0;
        } else {
            uint64_t Xx, Yx, Xy, Yy;
            xy_digits(gx, Xx, Yx);
            xy_digits(gy, Xy, Yy);
            x = (int64_t)(Xx | Xy << 1) * a.edge + tx;
            y = (int64_t)(Yx | Yy << 1) * a.edge + ty;
            active = (tx & (a.edge - 1 - ty)) == 0;
        }
        if (active) f(o, EmbeddedCoord{x, y});
    }
}

}  // namespace detail

template <class F>
int launch(const nbb_config& cfg, F f, nbb_report* report = nullptr, cudaStream_t stream = 0) {
    int rc = nbb_gpu_validate(&cfg);
    if (rc != NBB_OK) return rc;
    nbb_spec g;  /* the gasket only (the device membership and λ below are its closed forms) */
    nbb_spec_sierpinski(&g);
    bool gasket = cfg.spec.k == g.k && cfg.spec.s == g.s;
    for (int i = 0; gasket && i < g.k; ++i)
        gasket = cfg.spec.offset_x[i] == g.offset_x[i] && cfg.spec.offset_y[i] == g.offset_y[i];
    if (!gasket) return NBB_ERR_INVALID_ARGUMENT;
    const bool bb = cfg.mode == NBB_MODE_BB;
    if (!bb && (cfg.strategy != NBB_STRATEGY_SUBBOX || cfg.backend != NBB_BACKEND_DIRECT))
        return NBB_ERR_INVALID_ARGUMENT;
    uint64_t blocks = 0;
    rc = nbb_gpu_launch_block_count(&cfg, &blocks);
    if (rc != NBB_OK) return rc;
    detail::LaunchArgs a;
    a.n = (int64_t)1 << cfg.r;
    a.edge = cfg.rho;
    a.bb = bb ? 1 : 0;
    int rb = 0;
    while ((1 << rb) < cfg.rho) ++rb;
    rb = cfg.r - rb;  /* map level r_b */
    uint64_t w = 1;
    for (int i = 0; i < (rb + 1) / 2; ++i) w *= 3u;
    a.gw = bb ? (uint64_t)(a.n / cfg.rho) : w;
    a.begin = 0;
    a.end = blocks;
    if (cfg.shard_count > 0) {
        a.begin = cfg.shard_begin < blocks ? cfg.shard_begin : blocks;
        a.end = a.begin + cfg.shard_count < blocks ? a.begin + cfg.shard_count : blocks;
    }
    if (report) {
        rc = nbb_gpu_plan_report(&cfg, report);
        if (rc != NBB_OK) return rc;
    }
    if (a.end > a.begin) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const uint64_t want = a.end - a.begin, cap = (uint64_t)sms * 32;
        const unsigned grid = (unsigned)(want < cap ? want : cap);
        detail::launch_kernel<F><<<grid, dim3(cfg.rho, cfg.rho), 0, stream>>>(a, f);
        if (cudaGetLastError() != cudaSuccess) return NBB_ERR_CUDA;
    }
    return NBB_OK;
}

}  // namespace gpu
}  // namespace nbb
