// nbb_capi.cu — the C ABI of include/nbb_gpu.h: validation, planning, device
// buffers, and dispatch to the sm_100a kernels.
//
// Kernel selection (NBB_KERNEL_AUTO):
//   tile kernel (tile_kernels.cuh) when the launch is BB, or λ with the subbox
//   strategy and direct backend, and the tile holds whole 32-byte sectors
//   (int64: ρ ∈ {8,16,32}; uint8: ρ = 32); otherwise the per-cell kernel
//   (percell_kernels.cuh), which covers every (strategy, backend) the reference
//   accepts. Both produce identical grids; WorkReports are the reference's
//   closed-form counters of the logical launch (nbb_host.cpp).
// There is no CPU fallback: without a CUDA device every compute call fails with
// NBB_ERR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "nbb_gpu.h"
#include "nbb_host.hpp"
#include "percell_kernels.cuh"
#include "tile_kernels.cuh"
#include "ca_pipe_kernel.cuh"
#include "bits_kernels.cuh"
#include "compact_kernels.cuh"
#include "compact_pass.cuh"
#include "compact_sliced.cuh"
#include "compact_cluster.cuh"
#include "util_kernels.cuh"

using namespace nbbgpu;
using nbbhost::Error;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
int fail(const Error& e) { return fail(e.code, e.msg); }

#define NBB_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t _e = (call);                                                                \
        if (_e != cudaSuccess) {                                                                \
            return fail(NBB_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorName(_e) + ": " + \
                                          cudaGetErrorString(_e) + " (" #call ")");             \
        }                                                                                       \
    } while (0)

#define NBB_TRY(...)                      \
    do {                                  \
        const Error _e = (__VA_ARGS__);   \
        if (!_e.ok()) return fail(_e);    \
    } while (0)

#define NBB_CHECK(...)                    \
    do {                                  \
        const int _rc = (__VA_ARGS__);    \
        if (_rc != NBB_OK) return _rc;    \
    } while (0)

// ---- per-device context ------------------------------------------------------
struct DeviceCtx {
    bool ready = false;
    int sms = 148;
    cudaStream_t stream = nullptr;
    unsigned long long* partials = nullptr;  // 4096 slots + 1 result
    void* bufs[3] = {nullptr, nullptr, nullptr};
    size_t buf_bytes[3] = {0, 0, 0};
    int16_t* lut[6] = {};                    // LocalCellTable per edge 2^i
    int32_t* nbr_tab[32] = {};               // compact CA neighbour-tile table per level r
};

std::mutex g_mutex;
std::vector<DeviceCtx> g_ctx;

int ensure_device(int device, DeviceCtx** out) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        return fail(NBB_ERR_CUDA, std::string("no CUDA device available (") +
                                      (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices") +
                                      "); the GPU path has no CPU fallback");
    }
    if (device < 0 || device >= count)
        return fail(NBB_ERR_INVALID_ARGUMENT, "device " + std::to_string(device) + " out of range");
    std::lock_guard<std::mutex> lock(g_mutex);
    if ((int)g_ctx.size() < count) g_ctx.resize(count);
    DeviceCtx& c = g_ctx[device];
    NBB_CUDA(cudaSetDevice(device));
    if (!c.ready) {
        cudaDeviceProp prop;
        NBB_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10) {
            return fail(NBB_ERR_CUDA, std::string("device ") + prop.name +
                                          " is not sm_100 (this library is built for sm_100a only)");
        }
        c.sms = prop.multiProcessorCount;
        uint32_t tab[729];
        for (uint32_t v = 0; v < 729; ++v) tab[v] = xy6_arith(v);
        NBB_CUDA(cudaMemcpyToSymbol(c_xy729, tab, sizeof(tab)));
        // local λ of a ρ = 32 tile (compact CA): li = ωy*27 + ωx <-> (x, y)
        uint16_t pos[243], idx[1024];
        for (int i = 0; i < 1024; ++i) idx[i] = 0xFFFF;
        for (uint32_t li = 0; li < 243; ++li) {
            const uint32_t ax = xy6_arith(li % 27), ay = xy6_arith(li / 27);
            const uint32_t x = (ax & 0xFFFF) | ((ay & 0xFFFF) << 1), y = (ax >> 16) | ((ay >> 16) << 1);
            pos[li] = (uint16_t)(x | (y << 5));
            idx[y * 32 + x] = (uint16_t)li;
        }
        NBB_CUDA(cudaMemcpyToSymbol(c_local_pos, pos, sizeof(pos)));
        NBB_CUDA(cudaMemcpyToSymbol(c_local_idx, idx, sizeof(idx)));
        // halo slots of the K-step compact pass (compact_pass.cuh)
        nbbhost::HaloSlots hs;
        NBB_TRY(nbbhost::halo_slots(&hs));
        for (int k = 1; k <= kPassMaxK; ++k)
            if (hs.upto[k] != pass_slots(k))
                return fail(NBB_ERR_RUNTIME, "halo slots: layer sizes differ from the compiled pass shapes");
        NBB_CUDA(cudaMemcpyToSymbol(c_slots, &hs, sizeof(hs)));
        nbbhost::SliceSlots ss;
        NBB_TRY(nbbhost::slice_slots(&ss));
        for (int d = 0; d < 8; ++d)
            if (ss.dir_upto[d][kSliceMaxK] > ((d == 2 || d == 5) ? 0 : kSliceDirMax))
                return fail(NBB_ERR_RUNTIME, "slice slots: a neighbouring tile holds more halo slots than compiled for");
        if (ss.upto[kSliceMaxK - 1] > 32 * kSliceMaxM)
            return fail(NBB_ERR_RUNTIME, "slice slots: more halo slots per step than compiled for");
        NBB_CUDA(cudaMemcpyToSymbol(c_sslots, &ss, sizeof(ss)));
        nbbhost::ClusterSlots cs;
        NBB_TRY(nbbhost::cluster_slots(&cs));
        if (cs.upto[kClMaxK - 1] > 32 * ClBox<kClMaxK>::kM || cs.upto[7] > 32 * ClBox<8>::kM ||
            cs.dir_upto[2][kClMaxK] != 0 || cs.dir_upto[5][kClMaxK] != 0)
            return fail(NBB_ERR_RUNTIME, "cluster slots: more halo slots per step than compiled for");
        NBB_CUDA(cudaMemcpyToSymbol(c_cslots, &cs, sizeof(cs)));
        NBB_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        NBB_CUDA(cudaMalloc(&c.partials, 4097 * sizeof(unsigned long long)));
        c.ready = true;
    }
    *out = &c;
    return NBB_OK;
}

int device_buffer(DeviceCtx& c, int slot, size_t bytes, void** out) {
    if (c.buf_bytes[slot] < bytes) {
        if (c.bufs[slot]) NBB_CUDA(cudaFree(c.bufs[slot]));
        c.bufs[slot] = nullptr;
        c.buf_bytes[slot] = 0;
        cudaError_t e = cudaMalloc(&c.bufs[slot], bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(NBB_ERR_RESOURCE, "device allocation of " + std::to_string(bytes) +
                                              " bytes failed: " + cudaGetErrorString(e));
        }
        c.buf_bytes[slot] = bytes;
    }
    *out = c.bufs[slot];
    return NBB_OK;
}

DevSpec dev_spec(const nbb_spec& s) {
    DevSpec d;
    std::memset(&d, 0, sizeof(d));
    d.k = s.k;
    d.s = s.s;
    for (int i = 0; i < 9; ++i) {
        d.ox[i] = i < s.k ? s.offset_x[i] : 0;
        d.oy[i] = i < s.k ? s.offset_y[i] : 0;
        d.replica_at[i] = -1;
    }
    for (int i = 0; i < s.k && i < 9; ++i) d.replica_at[s.offset_y[i] * s.s + s.offset_x[i]] = i;
    d.gasket = nbbhost::is_gasket(s) ? 1 : 0;
    return d;
}

int local_table(DeviceCtx& c, const nbb_spec& s, int edge, const int16_t** out) {
    int l = 0;
    while ((1 << l) < edge) ++l;
    if (!nbbhost::is_gasket(s)) {  // generic specs: refill a scratch table every call
        static thread_local int16_t* scratch = nullptr;
        if (!scratch) NBB_CUDA(cudaMalloc(&scratch, 32 * 32 * 2 * sizeof(int16_t)));
        std::vector<int16_t> h((size_t)edge * edge * 2);
        nbbhost::local_cell_table(s, edge, h.data());
        NBB_CUDA(cudaMemcpy(scratch, h.data(), h.size() * sizeof(int16_t), cudaMemcpyHostToDevice));
        *out = scratch;
        return NBB_OK;
    }
    if (!c.lut[l]) {
        std::vector<int16_t> h((size_t)edge * edge * 2);
        nbbhost::local_cell_table(s, edge, h.data());
        NBB_CUDA(cudaMalloc(&c.lut[l], h.size() * sizeof(int16_t)));
        NBB_CUDA(cudaMemcpy(c.lut[l], h.data(), h.size() * sizeof(int16_t), cudaMemcpyHostToDevice));
    }
    *out = c.lut[l];
    return NBB_OK;
}

// ---- timing ---------------------------------------------------------------------
struct Timer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t s = nullptr;
    bool on = false;
    Timer(bool enable, cudaStream_t st) : s(st), on(enable) {
        if (on) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, s);
        }
    }
    uint64_t stop_micros() {
        if (!on) return 0;
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        return (uint64_t)(ms * 1000.0f);
    }
    ~Timer() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

// ---- occupancy (resident CTAs per SM), cached per kernel and device -------------------
// Kern is the kernel itself (a non-type template parameter, so every kernel instantiation has
// its own cache even when two share a signature); dynamic_smem > 0 also raises the kernel's
// dynamic shared-memory limit on the device (an attribute that is per device).
template <auto Kern>
int occupancy(int threads, int dynamic_smem, int* out) {
    static std::atomic<int> cache[64];  // by device ordinal; 0 = not yet queried
    int dev = 0;
    NBB_CUDA(cudaGetDevice(&dev));
    int v = cache[dev & 63].load(std::memory_order_relaxed);
    if (v == 0) {
        if (dynamic_smem > 0)
            NBB_CUDA(cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dynamic_smem));
        NBB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, Kern, threads, dynamic_smem));
        if (v < 1) return fail(NBB_ERR_RESOURCE, "kernel does not fit on an SM");
        cache[dev & 63].store(v, std::memory_order_relaxed);
    }
    *out = v;
    return NBB_OK;
}

// ---- launch helpers -----------------------------------------------------------------
struct Launch {
    const nbb_config* cfg;
    nbbhost::Plan plan;
    int op;
    cudaStream_t stream;
    DeviceCtx* ctx;
};

bool tile_supported(const nbb_config& c, int op, int cell_width) {
    if (c.kernel == NBB_KERNEL_PERCELL) return false;
    if (!nbbhost::is_gasket(c.spec)) return false;  // tile kernels use the gasket bit structure
    if (c.mode == NBB_MODE_LAMBDA &&
        (c.strategy != NBB_STRATEGY_SUBBOX || c.backend != NBB_BACKEND_DIRECT))
        return false;
    if (c.r > 17) return false;
    if (cell_width == 8) return c.rho == 8 || c.rho == 16 || c.rho == 32;
    if (cell_width == 0) return c.rho == 32 && op == OP_CA;
    return c.rho == 32 && op != OP_RD;
}

// CA on the bit-packed state (bits_kernels.cuh)
template <bool BB, int ILP>
int run_ca_bits_ilp(const Launch& L, const TileArgs& a) {
    auto kern = ca_bits_kernel<BB, ILP>;
    int occ;
    NBB_CHECK(occupancy<ca_bits_kernel<BB, ILP>>(256, 0, &occ));
    const uint64_t units = (a.tiles + ILP - 1) / ILP;
    const uint64_t want = (units + 7) / 8;
    const uint64_t cap = (uint64_t)L.ctx->sms * (uint64_t)occ;
    const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min(want, cap));
    if (a.tiles == 0) return NBB_OK;
    kern<<<blocks, 256, 0, L.stream>>>(a);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

template <bool BB>
int run_ca_bits(const Launch& L, const TileArgs& a) {
    static int ilp = -1;
    if (ilp < 0) {
        const char* e = std::getenv("NBB_BITS_ILP");
        ilp = e ? std::atoi(e) : 0;
    }
    // Measured on B200 at n = 2^16 (profiles/r1_bits_ilp.json): λ tiles favour 8 words in
    // flight per thread (0.098 vs 0.108 ms at 4), the BB grid favours 2 (0.636 vs 0.718 ms).
    if (ilp == 0) return BB ? run_ca_bits_ilp<BB, 2>(L, a) : run_ca_bits_ilp<BB, 8>(L, a);
    if (ilp == 2) return run_ca_bits_ilp<BB, 2>(L, a);
    if (ilp == 8) return run_ca_bits_ilp<BB, 8>(L, a);
    return run_ca_bits_ilp<BB, 4>(L, a);
}


TileArgs make_tile_args(const Launch& L, const void* src, void* dst, unsigned long long* sum,
                        uint32_t birth, uint32_t survive, uint32_t tile_begin, uint32_t tiles) {
    TileArgs a;
    a.src = src;
    a.dst = dst;
    a.sum = sum;
    a.n = L.plan.n;
    a.tile_begin = tile_begin;
    a.tiles = tiles;
    a.gw = (uint32_t)L.plan.gw;
    nbbhost::fastdiv_magic(a.gw, &a.div_gw.m, &a.div_gw.s);
    a.div_gw.d = a.gw;
    a.birth = birth;
    a.survive = survive;
    return a;
}

// CA through the cp.async pipeline kernel (ca_pipe_kernel.cuh)
template <typename Cell, int RHO, bool BB, int STAGES, int WARPS>
int run_ca_pipe(const Launch& L, const TileArgs& a) {
    using P = CaPipeShape<Cell, RHO, BB, STAGES, WARPS>;
    auto kern = ca_pipe_kernel<Cell, RHO, BB, STAGES, WARPS>;
    int occ;
    NBB_CHECK((occupancy<ca_pipe_kernel<Cell, RHO, BB, STAGES, WARPS>>(WARPS * 32, P::SMEM, &occ)));
    constexpr int TPW = 32 / RHO;
    const uint64_t units = (a.tiles + TPW - 1) / TPW;
    const uint64_t want = (units + WARPS - 1) / WARPS;
    const uint64_t cap = (uint64_t)L.ctx->sms * (uint64_t)occ;
    const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min(want, cap));
    if (a.tiles == 0) return NBB_OK;
    kern<<<blocks, WARPS * 32, P::SMEM, L.stream>>>(a);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

// pipeline shape: NBB_CA_PIPE="stages,warps" (tuning), "0" = register-staged tile kernel
int ca_pipe_choice() {
    static int choice = -1;
    if (choice < 0) {
        choice = 1;
        if (const char* e = std::getenv("NBB_CA_PIPE")) {
            const std::string s(e);
            choice = s == "0" ? 0 : s == "2,8" ? 1 : s == "3,4" ? 2 : s == "4,4" ? 3 : s == "3,8" ? 4 : 1;
        }
    }
    return choice;
}

template <typename Cell, int RHO, bool BB>
int run_ca_tile(const Launch& L, const TileArgs& a) {
    switch (ca_pipe_choice()) {
        case 2: return run_ca_pipe<Cell, RHO, BB, 3, 4>(L, a);
        case 3: return run_ca_pipe<Cell, RHO, BB, 4, 4>(L, a);
        case 4: return run_ca_pipe<Cell, RHO, BB, 3, 8>(L, a);
        default: return run_ca_pipe<Cell, RHO, BB, 2, 8>(L, a);
    }
}

// rule masks travel in TileArgs; thin wrapper so CA can set them.
template <typename Cell, int RHO, int OP, bool BB>
int run_tile_rule(const Launch& L, const void* src, void* dst, unsigned long long* sum,
                  uint32_t birth, uint32_t survive, uint32_t tile_begin, uint32_t tiles) {
    if constexpr (OP == OP_CA && !BB) {  // BB keeps the register-staged kernel (faster for BB)
        if (ca_pipe_choice() != 0) {
            return run_ca_tile<Cell, RHO, BB>(
                L, make_tile_args(L, src, dst, sum, birth, survive, tile_begin, tiles));
        }
    }
    auto kern = tile_kernel<Cell, RHO, OP, BB>;
    int occ;
    NBB_CHECK((occupancy<tile_kernel<Cell, RHO, OP, BB>>(256, 0, &occ)));
    TileArgs a;
    a.src = src;
    a.dst = dst;
    a.sum = sum;
    a.n = L.plan.n;
    a.tile_begin = tile_begin;
    a.tiles = tiles;
    a.gw = (uint32_t)L.plan.gw;
    nbbhost::fastdiv_magic(a.gw, &a.div_gw.m, &a.div_gw.s);
    a.div_gw.d = a.gw;
    a.birth = birth;
    a.survive = survive;
    constexpr int TPW = 32 / RHO;
    const uint64_t units = (tiles + TPW - 1) / TPW;
    const uint64_t want = (units + 7) / 8;
    const uint64_t cap = (uint64_t)L.ctx->sms * (uint64_t)occ;
    const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min(want, cap));
    if (tiles == 0) return NBB_OK;
    kern<<<blocks, 256, 0, L.stream>>>(a);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

template <typename Cell, int OP, bool BB>
int dispatch_tile_rho(const Launch& L, const void* src, void* dst, unsigned long long* sum,
                      uint32_t birth, uint32_t survive, uint32_t tile_begin, uint32_t tiles) {
    if (sizeof(Cell) == 1) {
        if constexpr (OP != OP_RD) {
            return run_tile_rule<unsigned char, 32, OP, BB>(L, src, dst, sum, birth, survive,
                                                            tile_begin, tiles);
        }
        return fail(NBB_ERR_INVALID_ARGUMENT, "reduction needs int64 cells");
    }
    switch (L.cfg->rho) {
        case 8: return run_tile_rule<long long, 8, OP, BB>(L, src, dst, sum, birth, survive, tile_begin, tiles);
        case 16: return run_tile_rule<long long, 16, OP, BB>(L, src, dst, sum, birth, survive, tile_begin, tiles);
        case 32: return run_tile_rule<long long, 32, OP, BB>(L, src, dst, sum, birth, survive, tile_begin, tiles);
    }
    return fail(NBB_ERR_INVALID_ARGUMENT, "tile kernel needs rho in {8, 16, 32}");
}

// [lo, hi) block ordinals of this launch: the whole plan or the configured shard
void shard_range(const Launch& L, uint64_t* lo, uint64_t* hi) {
    const uint64_t total = L.plan.blocks();
    *lo = 0;
    *hi = total;
    if (L.cfg->shard_count > 0) {
        *lo = std::min<uint64_t>(L.cfg->shard_begin, total);
        *hi = std::min<uint64_t>(*lo + L.cfg->shard_count, total);
    }
}

template <typename Cell, int OP>
int launch_tile(const Launch& L, const void* src, void* dst, unsigned long long* sum,
                uint32_t birth, uint32_t survive) {
    uint64_t lo, hi;
    shard_range(L, &lo, &hi);
    const uint32_t tiles = (uint32_t)(hi - lo);
    // workers > 1: contiguous ordinal chunks (dispatch.cpp:419-427), run in order
    const uint32_t workers = (uint32_t)std::max(1, L.cfg->workers);
    const uint32_t chunk = (tiles + workers - 1) / workers;
    for (uint32_t w = 0; w < workers; ++w) {
        const uint32_t begin = (uint32_t)lo + w * chunk;
        if (w * chunk >= tiles) break;
        const uint32_t count = std::min(chunk, tiles - w * chunk);
        int rc = L.cfg->mode == NBB_MODE_BB
                     ? dispatch_tile_rho<Cell, OP, true>(L, src, dst, sum, birth, survive, begin, count)
                     : dispatch_tile_rho<Cell, OP, false>(L, src, dst, sum, birth, survive, begin, count);
        if (rc != NBB_OK) return rc;
    }
    return NBB_OK;
}

template <typename Cell, int OP, bool BB, int STRATEGY, int BACKEND>
int run_percell(const Launch& L, const PercellArgs& a) {
    const uint64_t B = a.launch_count;
    if (B == 0) return NBB_OK;
    const unsigned threads = (unsigned)std::max(32, a.edge * a.edge);
    const uint64_t X = std::min<uint64_t>(B, 65536);
    const uint64_t Y = std::min<uint64_t>((B + X - 1) / X, 65535);
    const uint64_t Z = (B + X * Y - 1) / (X * Y);
    dim3 grid((unsigned)X, (unsigned)Y, (unsigned)Z);
    // Generic (non-gasket) specs are a separate instantiation so the gasket kernels carry
    // no table-driven code; validate() restricts generic specs to int64 cells.
    if constexpr (sizeof(Cell) == 8) {
        if (!a.spec.gasket) {
            percell_kernel<Cell, OP, BB, STRATEGY, BACKEND, true><<<grid, threads, 0, L.stream>>>(a);
            NBB_CUDA(cudaGetLastError());
            return NBB_OK;
        }
    }
    percell_kernel<Cell, OP, BB, STRATEGY, BACKEND, false><<<grid, threads, 0, L.stream>>>(a);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

template <typename Cell, int OP>
int launch_percell(const Launch& L, const void* src, void* dst, uint32_t birth, uint32_t survive) {
    const nbb_config& c = *L.cfg;
    PercellArgs a;
    a.src = src;
    a.dst = dst;
    a.partials = L.ctx->partials;
    a.n = L.plan.n;
    a.total_blocks = L.plan.blocks();
    uint64_t lo, hi;
    shard_range(L, &lo, &hi);
    a.ordinal_base = lo;
    a.launch_count = hi - lo;
    a.gw = (uint64_t)L.plan.gw;
    a.edge = L.plan.edge;
    a.map_level = L.plan.map_level;
    a.local_level = L.plan.local_level;
    a.local_w = (int)L.plan.local_w;
    a.local_members = (int)L.plan.local_members;
    a.sub_w = L.plan.sub_w;
    a.sub_h = L.plan.sub_h;
    a.lut = nullptr;
    a.birth = birth;
    a.survive = survive;
    a.r = c.r;
    a.spec = dev_spec(c.spec);
    if (c.mode == NBB_MODE_LAMBDA && c.strategy == NBB_STRATEGY_LUT)
        NBB_CHECK(local_table(*L.ctx, c.spec, L.plan.edge, &a.lut));
    if (c.mode == NBB_MODE_BB)
        return run_percell<Cell, OP, true, NBB_STRATEGY_SUBBOX, NBB_BACKEND_DIRECT>(L, a);
#define NBB_PC_BACKENDS(ST)                                                                   \
    switch (c.backend) {                                                                      \
        case NBB_BACKEND_DIRECT: return run_percell<Cell, OP, false, ST, NBB_BACKEND_DIRECT>(L, a); \
        case NBB_BACKEND_MMA1: return run_percell<Cell, OP, false, ST, NBB_BACKEND_MMA1>(L, a); \
        case NBB_BACKEND_MMA2: return run_percell<Cell, OP, false, ST, NBB_BACKEND_MMA2>(L, a); \
    }
    switch (c.strategy) {
        case NBB_STRATEGY_SUBBOX:
            if (c.backend == NBB_BACKEND_MMA3)
                return run_percell<Cell, OP, false, NBB_STRATEGY_SUBBOX, NBB_BACKEND_MMA3>(L, a);
            NBB_PC_BACKENDS(NBB_STRATEGY_SUBBOX)
            break;
        case NBB_STRATEGY_UNROLL:
            NBB_PC_BACKENDS(NBB_STRATEGY_UNROLL)
            break;
        case NBB_STRATEGY_LUT:
            NBB_PC_BACKENDS(NBB_STRATEGY_LUT)
            break;
    }
#undef NBB_PC_BACKENDS
    return fail(NBB_ERR_INVALID_ARGUMENT, "unsupported strategy/backend combination");
}

// one workload launch (SW / RD / CA step) on device buffers
int launch_op(const Launch& L, int op, const void* src, void* dst, unsigned long long* d_sum,
              uint32_t birth, uint32_t survive) {
    const nbb_config& c = *L.cfg;
    const int cw = op == OP_RD ? 8 : c.cell_width;
    const bool tile = tile_supported(c, op, cw);
    if (c.kernel == NBB_KERNEL_TILE && !tile)
        return fail(NBB_ERR_INVALID_ARGUMENT,
                    "tile kernel needs bb or lambda/subbox/direct, rho in {8,16,32} (int64) or "
                    "rho = 32 (uint8), r <= 17");
    if (op == OP_RD) {
        if (tile) {
            NBB_CUDA(cudaMemsetAsync(d_sum, 0, sizeof(unsigned long long), L.stream));
            return launch_tile<long long, OP_RD>(L, src, nullptr, d_sum, 0, 0);
        }
        NBB_CUDA(cudaMemsetAsync(L.ctx->partials, 0, 4096 * sizeof(unsigned long long), L.stream));
        NBB_CHECK(launch_percell<long long, OP_RD>(L, src, nullptr, 0, 0));
        reduce_partials_kernel<<<1, 1024, 0, L.stream>>>(L.ctx->partials, 4096, d_sum);
        NBB_CUDA(cudaGetLastError());
        return NBB_OK;
    }
    if (cw == 0) {  // bit-packed alive state: CA through the ρ = 32 tile kernel only
        if (!tile)
            return fail(NBB_ERR_INVALID_ARGUMENT,
                        "the 1-bit packed state (cell_width 0) runs the CA step through the tile "
                        "kernel only: bb or lambda/subbox/direct with rho = 32");
        uint64_t lo, hi;
        shard_range(L, &lo, &hi);
        const uint32_t workers = (uint32_t)std::max(1, c.workers);
        const uint32_t tiles = (uint32_t)(hi - lo), chunk = (tiles + workers - 1) / workers;
        for (uint32_t w = 0; w < workers && w * chunk < tiles; ++w) {
            const TileArgs a = make_tile_args(L, src, dst, nullptr, birth, survive,
                                              (uint32_t)lo + w * chunk, std::min(chunk, tiles - w * chunk));
            NBB_CHECK(c.mode == NBB_MODE_BB ? run_ca_bits<true>(L, a) : run_ca_bits<false>(L, a));
        }
        return NBB_OK;
    }
    if (cw == 8) {
        if (tile) {
            return op == OP_SW ? launch_tile<long long, OP_SW>(L, src, dst, nullptr, 0, 0)
                               : launch_tile<long long, OP_CA>(L, src, dst, nullptr, birth, survive);
        }
        return op == OP_SW ? launch_percell<long long, OP_SW>(L, src, dst, 0, 0)
                           : launch_percell<long long, OP_CA>(L, src, dst, birth, survive);
    }
    if (tile) {
        return op == OP_SW ? launch_tile<unsigned char, OP_SW>(L, src, dst, nullptr, 0, 0)
                           : launch_tile<unsigned char, OP_CA>(L, src, dst, nullptr, birth, survive);
    }
    return op == OP_SW ? launch_percell<unsigned char, OP_SW>(L, src, dst, 0, 0)
                       : launch_percell<unsigned char, OP_CA>(L, src, dst, birth, survive);
}

// gasket_only: layout kernels (sanitize/pack/unpack/scatter) that use the gasket bit test
int prepare(const nbb_config* cfg, int op, Launch* L, bool need_budget, bool gasket_only = false) {
    if (cfg == nullptr) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    NBB_TRY(nbbhost::validate_spec(cfg->spec));
    NBB_TRY(nbbhost::validate(*cfg));
    if (gasket_only) NBB_TRY(nbbhost::require_gasket(cfg->spec));
    if (!nbbhost::is_gasket(cfg->spec) && cfg->cell_width != 8)
        return fail(NBB_ERR_INVALID_ARGUMENT,
                    "uint8 and 1-bit CA states run on the sierpinski gasket only; use cell_width 8 for '" +
                        std::string(cfg->spec.name) + "'");
    if (need_budget) NBB_TRY(nbbhost::member_mask_budget(cfg->spec, cfg->r, cfg->max_cells));
    L->cfg = cfg;
    L->op = op;
    NBB_TRY(nbbhost::make_plan(*cfg, &L->plan));
    if (L->plan.n > (int64_t(1) << 20))
        return fail(NBB_ERR_RESOURCE, "embedding side " + std::to_string(L->plan.n) +
                                          " exceeds the device path limit 2^20");
    NBB_CHECK(ensure_device(cfg->device, &L->ctx));
    return NBB_OK;
}

void fill_report(const nbb_config* cfg, nbb_report* r, uint64_t micros) {
    if (!r) return;
    nbbhost::plan_report(*cfg, r);
    r->micros = cfg->timing ? micros : 0;
}

int sanitize(const Launch& L, void* d_grid, int cell_width, cudaStream_t s) {
    const int blocks = L.ctx->sms * 8;
    if (!nbbhost::is_gasket(L.cfg->spec))
        sanitize_generic_kernel<<<blocks, 256, 0, s>>>(dev_spec(L.cfg->spec), (long long*)d_grid,
                                                       L.plan.n, L.cfg->r);
    else if (cell_width == 8)
        sanitize_kernel<long long><<<blocks, 256, 0, s>>>((long long*)d_grid, L.plan.n, 0);
    else if (cell_width == 1)
        sanitize_kernel<unsigned char><<<blocks, 256, 0, s>>>((unsigned char*)d_grid, L.plan.n, 0);
    else
        sanitize_bits_kernel<<<blocks, 256, 0, s>>>((uint32_t*)d_grid, L.plan.n);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

// bytes of an n x n grid of cw-byte cells (cw = 0: 1-bit packed, 32-bit words per row)
// Device-usable address of a pinned (page-locked, mapped) host buffer, or nullptr for
// pageable memory (then the whole grid is staged with cudaMemcpy).
void* mapped_host_ptr(const void* p) {
    cudaPointerAttributes a;
    if (p == nullptr || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (a.type != cudaMemoryTypeHost || a.devicePointer == nullptr) return nullptr;
    return a.devicePointer;
}

size_t grid_bytes(const Launch& L, int cw) {
    const size_t n = (size_t)L.plan.n;
    if (cw == 0) return n * std::max<size_t>(1, n / 32) * 4;
    return n * n * (size_t)cw;
}

}  // namespace

// ---- compact (λ-ordered) state ---------------------------------------------------------
namespace {
struct CompactShape {
    int64_t n = 1;
    uint64_t W = 1, H = 1, total = 1;
};
int compact_shape(const nbb_config* cfg, CompactShape* s) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    NBB_TRY(nbbhost::validate_spec(cfg->spec));
    if (cfg->r < 0) return fail(NBB_ERR_INVALID_ARGUMENT, "checked_pow: negative exponent");
    NBB_TRY(nbbhost::side_length(cfg->spec, cfg->r, &s->n));
    int64_t w, h;
    NBB_TRY(nbbhost::orthotope_dims(cfg->spec, cfg->r, &w, &h));
    s->W = (uint64_t)w;
    s->H = (uint64_t)h;
    s->total = s->W * s->H;
    if (s->n > (int64_t(1) << 20)) return fail(NBB_ERR_RESOURCE, "embedding too large for the device path");
    return NBB_OK;
}
// The compact-state memory of cfg's shard (all of it without a shard): Segs (compact_kernels.cuh)
int compact_segments(const nbb_config* cfg, Segs* sg) {
    CompactShape cs;
    NBB_CHECK(compact_shape(cfg, &cs));
    int64_t wb, hb;
    NBB_TRY(nbbhost::orthotope_dims(cfg->spec, cfg->r - 5, &wb, &hb));
    const uint64_t tiles = (uint64_t)wb * (uint64_t)hb, Hb = (uint64_t)hb, W = cs.W;
    uint64_t b = 0, e = tiles;
    if (cfg->shard_count > 0) {
        b = std::min<uint64_t>(cfg->shard_begin, tiles);
        e = std::min<uint64_t>(b + cfg->shard_count, tiles);
    }
    sg->n = 0;
    for (uint64_t u = b; u < e;) {
        const uint64_t wxb = u / Hb, c0 = u % Hb;
        if (c0 == 0 && e - u >= Hb) {  // whole tile rows: one contiguous run of compact rows
            const uint64_t k = (e - u) / Hb;
            sg->off[sg->n] = 9 * wxb * W;
            sg->cnt[sg->n] = 9 * W * k;
            ++sg->n;
            u += k * Hb;
        } else {  // part of one tile row: 9 row pieces of 27 values per tile
            const uint64_t c1 = std::min<uint64_t>(Hb, c0 + (e - u));
            for (uint64_t row = 0; row < 9; ++row) {
                sg->off[sg->n] = (9 * wxb + row) * W + 27 * c0;
                sg->cnt[sg->n] = 27 * (c1 - c0);
                ++sg->n;
            }
            u += c1 - c0;
        }
    }  // at most: a partial tile row (9) + whole tile rows (1) + a partial tile row (9) = 19
    return NBB_OK;
}
unsigned grid_for(const DeviceCtx* c, uint64_t work) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, (uint64_t)c->sms * 16));
}
// compact CA / RD / SW validity: the gasket, λ launch, ρ = 32 tiles inside (r >= 5)
// allow_bb: the CA step also runs as the bounding-box launch over the compact state
// (ca_compact_bb_kernel: box tiles culled, member tiles addressed through λ⁻¹), unsharded
int compact_workload_check(const nbb_config* cfg, bool allow_bb = false) {
    NBB_TRY(nbbhost::validate(*cfg));
    NBB_TRY(nbbhost::require_gasket(cfg->spec));
    if (cfg->r < 5)
        return fail(NBB_ERR_INVALID_ARGUMENT, "compact-state workloads need r >= 5 (32 x 32 tiles)");
    if (cfg->r > 18)  // 32-bit tile / halo indices (3^18 < 2^31)
        return fail(NBB_ERR_RESOURCE, "compact-state workloads support r <= 18");
    if (cfg->mode == NBB_MODE_BB && allow_bb) {
        if (cfg->shard_count > 0)
            return fail(NBB_ERR_INVALID_ARGUMENT, "the bounding-box launch over the compact state is unsharded");
        return NBB_OK;
    }
    if (cfg->mode != NBB_MODE_LAMBDA)
        return fail(NBB_ERR_INVALID_ARGUMENT, "the compact state is the lambda orthotope: lambda mode only");
    return NBB_OK;
}
CompactCaArgs compact_args(const nbb_config* cfg, const void* src, void* dst, uint16_t birth,
                           uint16_t survive, FastDiv* div_hb) {
    CompactCaArgs a;
    a.src = (const long long*)src;
    a.dst = (long long*)dst;
    int64_t w, h;
    nbbhost::orthotope_dims(cfg->spec, cfg->r, &w, &h);
    a.W = (uint32_t)w;
    a.rb = cfg->r - 5;
    int64_t wb, hb;
    nbbhost::orthotope_dims(cfg->spec, a.rb, &wb, &hb);
    a.Wb = (uint32_t)wb;
    a.Hb = (uint32_t)hb;
    a.n = (int64_t)1 << cfg->r;
    a.tiles = a.Wb * a.Hb;
    a.tile_begin = 0;
    a.tile_end = a.tiles;
    if (cfg->shard_count > 0) {
        a.tile_begin = (uint32_t)std::min<uint64_t>(cfg->shard_begin, a.tiles);
        a.tile_end = (uint32_t)std::min<uint64_t>(a.tile_begin + cfg->shard_count, a.tiles);
    }
    a.birth = birth;
    a.survive = survive;
    div_hb->d = a.Hb;
    nbbhost::fastdiv_magic(a.Hb, &div_hb->m, &div_hb->s);
    return a;
}

// The tile codec (compact_from/to_sectors_kernel) serves the gasket at r >= 5.
bool compact_tiles_ok(const nbb_config* cfg) { return nbbhost::is_gasket(cfg->spec) && cfg->r >= 5; }

int compact_from_sectors(DeviceCtx* ctx, const nbb_config* cfg, const void* emb, void* comp, cudaStream_t st) {
    FastDiv d;
    const CompactCaArgs a = compact_args(cfg, nullptr, nullptr, 0, 0, &d);
    const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((a.tiles + 7) / 8, (uint64_t)ctx->sms * 8));
    compact_from_sectors_kernel<<<blocks, 256, 0, st>>>((const long long*)emb, (long long*)comp, a, d);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

int compact_to_sectors(DeviceCtx* ctx, const nbb_config* cfg, const void* comp, void* emb, cudaStream_t st) {
    FastDiv d;
    const CompactCaArgs a = compact_args(cfg, nullptr, nullptr, 0, 0, &d);
    const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((a.tiles + 7) / 8, (uint64_t)ctx->sms * 8));
    compact_to_sectors_kernel<<<blocks, 256, 0, st>>>((const long long*)comp, (long long*)emb, a, d);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

// the per-level neighbour-tile table of ca_compact_pass_kernel (8 tile ordinals per tile),
// built once (then cached) per device and level
int compact_nbr_table(DeviceCtx* ctx, const nbb_config* cfg, const CompactCaArgs& a, const FastDiv& d,
                      const int32_t** out) {
    std::lock_guard<std::mutex> lock(g_mutex);
    int32_t*& t = ctx->nbr_tab[cfg->r];
    if (!t) {
        NBB_CUDA(cudaMalloc(&t, (size_t)a.tiles * 8 * sizeof(int32_t)));
        const uint64_t n = (uint64_t)a.tiles * 8;
        const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)ctx->sms * 16));
        compact_nbr_table_kernel<<<blocks, 256, 0, ctx->stream>>>(a, d, t);
        NBB_CUDA(cudaGetLastError());
        NBB_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    *out = t;
    return NBB_OK;
}

// Launch with programmatic stream serialization (PDL): the kernel may start while the previous
// kernel on the stream drains; kernels launched this way call griddepcontrol.wait before
// touching memory the previous kernel writes (ca_compact_pass_kernel: pdl_wait()).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_smem(void (*k)(KArgs...), unsigned grid, unsigned block, size_t dyn_smem, cudaStream_t st,
                            Args&&... args) {
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(grid);
    c.blockDim = dim3(block);
    c.dynamicSmemBytes = dyn_smem;
    c.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    c.attrs = at;
    c.numAttrs = 1;
    return cudaLaunchKernelEx(&c, k, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, cudaStream_t st, Args&&... args) {
    return launch_pdl_smem(k, grid, block, 0, st, std::forward<Args>(args)...);
}

bool is_conway(uint16_t birth, uint16_t survive) {  // CaRule{} (B3/S23): its own instantiation
    return birth == (1u << 3) && survive == ((1u << 2) | (1u << 3));
}

// the kernel of one pass: K steps, rule instantiation, walk (λ / BB / multi-GPU)
template <int K, bool P2P, bool BB>
using PassKernel = void (*)(CompactCaArgs, FastDiv, const int32_t*, P2PArgs);
template <int K, bool P2P, bool BB>
PassKernel<K, P2P, BB> pass_kernel(bool conway) {
    return conway ? ca_compact_pass_kernel<K, true, P2P, BB> : ca_compact_pass_kernel<K, false, P2P, BB>;
}
template <bool P2P, bool BB>
void (*pass_kernel_k(int k, bool conway))(CompactCaArgs, FastDiv, const int32_t*, P2PArgs) {
    switch (k) {
        case 1: return pass_kernel<1, P2P, BB>(conway);
        case 2: return pass_kernel<2, P2P, BB>(conway);
        case 3: return pass_kernel<3, P2P, BB>(conway);
        default: return pass_kernel<4, P2P, BB>(conway);
    }
}
// resident CTAs per SM of a pass kernel (cached per kernel pointer)
int pass_occupancy(const void* k, int* occ) {
    static std::mutex m;
    static std::vector<std::pair<const void*, int>> cache;
    std::lock_guard<std::mutex> lock(m);
    for (auto& e : cache)
        if (e.first == k) {
            *occ = e.second;
            return NBB_OK;
        }
    NBB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k, 256, 0));
    if (*occ < 1) *occ = 1;
    cache.push_back({k, *occ});
    return NBB_OK;
}

// The pass kernel: the tile-sliced kernel (compact_sliced.cuh, up to 8 steps per pass) unless
// NBB_PASS_IMPL=warp selects the warp-per-tile kernel (compact_pass.cuh, up to 4) for comparison.
bool sliced_impl() {
    static const bool v = [] {
        const char* e = std::getenv("NBB_PASS_IMPL");
        return !(e && std::strcmp(e, "warp") == 0);
    }();
    return v;
}
bool cluster_walk_ok(const CompactCaArgs& a);
// the most steps one pass of this config's kernel takes: the cluster walk 12 (λ over whole
// cluster columns, r >= 8), the tile-sliced walk 8, the warp-per-tile kernel 4
int impl_max_k(const nbb_config* cfg) {
    if (!sliced_impl()) return kPassMaxK;
    if (cfg && cfg->mode != NBB_MODE_BB && cfg->r >= 8 && cfg->r <= 20) {
        FastDiv d;
        if (cluster_walk_ok(compact_args(cfg, nullptr, nullptr, 0, 0, &d))) return kClMaxK;
    }
    return kSliceMaxK;
}
// steps per pass: cfg->pass_steps (0 = the default: the kernel's most), 1 with NBB_FLAG_SINGLE_STEP
int max_pass_steps(const nbb_config* cfg) {
    if (cfg->flags & NBB_FLAG_SINGLE_STEP) return 1;
    static const int env = [] {
        const char* e = std::getenv("NBB_PASS_STEPS");  // tuning
        return e ? std::atoi(e) : 0;
    }();
    // default 8: a pass of 8 steps still streams the state at >= 0.7 of the HBM peak; 12 steps
    // per pass (pass_steps = 12, cluster walk) are ~10% faster per step at ~0.6 of peak per pass
    const int kmax = impl_max_k(cfg);
    const int k = cfg->pass_steps ? (int)cfg->pass_steps : env > 0 ? env : kSliceMaxK;
    return std::max(1, std::min(k, kmax));
}
int check_pass_steps(const nbb_config* cfg) {
    if (cfg->pass_steps > (uint32_t)kClMaxK)
        return fail(NBB_ERR_INVALID_ARGUMENT, "pass_steps: at most 12 CA steps per pass over the compact state");
    return NBB_OK;
}

// the batches of the tile-sliced λ walk over this launch's shard [tile_begin, tile_end)
SliceBatches slice_batches(const CompactCaArgs& a, int k) {
    SliceBatches b{};
    b.K = k;
    b.rule = make_rule_tab(a.birth, a.survive);
    const uint32_t Hb = a.Hb;
    b.nb_row = (Hb + 31u) / 32u;
    b.div_nb_row.d = b.nb_row;
    nbbhost::fastdiv_magic(b.nb_row, &b.div_nb_row.m, &b.div_nb_row.s);
    if (a.tile_end <= a.tile_begin) return b;
    b.row0 = a.tile_begin / Hb;
    b.col0 = a.tile_begin % Hb;
    const uint32_t row_end = (b.row0 + 1u) * Hb;
    if (a.tile_end <= row_end) {
        b.cols0 = a.tile_end - a.tile_begin;
    } else {
        b.cols0 = Hb - b.col0;
        const uint32_t rem = a.tile_end - row_end;
        b.mid_rows = rem / Hb;
        b.last_cols = rem % Hb;
    }
    b.nb0 = (b.cols0 + 31u) / 32u;
    b.total = b.nb0 + b.mid_rows * b.nb_row + (b.last_cols + 31u) / 32u;
    return b;
}
template <bool P2P, bool BB>
void (*sliced_kernel(bool conway))(CompactCaArgs, SliceBatches, FastDiv, const int32_t*, P2PArgs) {
    return conway ? ca_compact_sliced_kernel<true, P2P, BB> : ca_compact_sliced_kernel<false, P2P, BB>;
}
// The cluster walk (compact_cluster.cuh): the single-device λ walk over the whole orthotope at
// r_b >= 3, unless NBB_PASS_IMPL=sliced keeps the 32-ordinal batches (comparison runs).
bool cluster_impl() {  // read per launch: comparison runs flip it inside one process
    const char* e = std::getenv("NBB_PASS_IMPL");
    return !(e && (std::strcmp(e, "sliced") == 0 || std::strcmp(e, "warp") == 0));
}
// ... over a shard of whole cluster columns (9 Hb tiles: the whole orthotope, or a multi-GPU
// chunk of nbbhost::compact_shard_chunk; an empty shard at the end also qualifies)
bool cluster_walk_ok(const CompactCaArgs& a) {
    if (!cluster_impl() || a.rb < 3 || a.Wb % 9u != 0 || a.Hb % 3u != 0) return false;
    const uint32_t col = 9u * a.Hb;
    return a.tile_begin % col == 0 && (a.tile_end % col == 0 || a.tile_end == a.tiles) && a.tile_begin <= a.tile_end;
}
ClusterWalk cluster_walk(const CompactCaArgs& a, int k) {
    ClusterWalk c{};
    c.K = k;
    c.ncy = a.Hb / 3u;
    c.div_ncy.d = c.ncy;
    nbbhost::fastdiv_magic(c.ncy, &c.div_ncy.m, &c.div_ncy.s);
    c.total = (a.Wb / 9u) * c.ncy;
    const uint32_t col = 9u * a.Hb;
    c.begin = a.tile_begin / col * c.ncy;
    c.end = std::min(c.total, (a.tile_end + col - 1) / col * c.ncy);
    return c;
}
int cluster_grid(DeviceCtx* ctx, const void* kern, size_t dyn, uint64_t batches, unsigned* grid) {
    static std::mutex m;
    static std::vector<std::pair<const void*, int>> cache;  // kernel -> resident CTAs per SM
    std::lock_guard<std::mutex> lock(m);
    int occ = 0;
    for (auto& e : cache)
        if (e.first == kern) occ = e.second;
    if (!occ) {
        NBB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        NBB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
        NBB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * kClWarps, dyn));
        if (occ < 1) occ = 1;
        cache.push_back({kern, occ});
    }
    const uint64_t wave = (uint64_t)ctx->sms * occ;
    *grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(wave, (batches + kClPipes - 1) / kClPipes));
    return NBB_OK;
}

// One pass of the cluster walk (P2P: a rank's pass of the multi-GPU step); `sharing` workers
// co-resident on the device get a share of one wave each and no PDL (they wait on each other).
// Passes of up to 8 steps run the 8-cell-frame kernel (two boxes per stepper), longer ones the
// 12-cell-frame kernel.
template <bool P2P, int F>
int launch_cluster_pass_f(DeviceCtx* ctx, const CompactCaArgs& a, int k, bool conway, const FastDiv& div_hb,
                          const int32_t* tab, const P2PArgs& p, cudaStream_t st, int sharing) {
    ClusterWalk cw = cluster_walk(a, k);
    cw.rule = make_rule_tab(a.birth, a.survive);
    auto kern = conway ? ca_compact_cluster_kernel<true, P2P, F> : ca_compact_cluster_kernel<false, P2P, F>;
    constexpr size_t dyn = cl_dyn_smem<F>();
    unsigned grid;
    NBB_CHECK(cluster_grid(ctx, (const void*)kern, dyn, std::max<uint64_t>(1, cw.end - cw.begin), &grid));
    if (sharing > 1) {
        grid = std::max(1u, grid / (unsigned)sharing);
        kern<<<grid, 32 * kClWarps, dyn, st>>>(a, cw, div_hb, tab, p);
        NBB_CUDA(cudaGetLastError());
        return NBB_OK;
    }
    NBB_CUDA(launch_pdl_smem(kern, grid, 32 * kClWarps, dyn, st, a, cw, div_hb, tab, p));
    return NBB_OK;
}
template <bool P2P>
int launch_cluster_pass(DeviceCtx* ctx, const CompactCaArgs& a, int k, bool conway, const FastDiv& div_hb,
                        const int32_t* tab, const P2PArgs& p, cudaStream_t st, int sharing = 1) {
    return k <= 8 ? launch_cluster_pass_f<P2P, 8>(ctx, a, k, conway, div_hb, tab, p, st, sharing)
                  : launch_cluster_pass_f<P2P, kClMaxK>(ctx, a, k, conway, div_hb, tab, p, st, sharing);
}

// grid of a tile-sliced launch: one wave of CTAs (kSlicePipes loader/stepper pipelines each),
// fewer when the batches are fewer
int sliced_grid(DeviceCtx* ctx, const void* kern, uint64_t batches, bool bb, unsigned* grid) {
    int occ;
    static std::mutex m;
    static std::vector<const void*> carved;  // carveout + dynamic smem limit raised once per kernel
    const size_t dyn = bb ? 0 : kSliceDynSmem;
    {
        std::lock_guard<std::mutex> lock(m);
        if (std::find(carved.begin(), carved.end(), kern) == carved.end()) {
            NBB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            NBB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
            carved.push_back(kern);
        }
    }
    {
        static std::mutex mo;
        static std::vector<std::pair<const void*, int>> cache;
        std::lock_guard<std::mutex> lock(mo);
        occ = 0;
        for (auto& e : cache)
            if (e.first == kern) occ = e.second;
        if (!occ) {
            NBB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * kSliceWarps, dyn));
            if (occ < 1) occ = 1;
            cache.push_back({kern, occ});
        }
    }
    const uint64_t wave = (uint64_t)ctx->sms * occ;
    *grid = (unsigned)std::max<uint64_t>(  // kSlicePipes batch pipelines per CTA
        1, bb ? wave : std::min<uint64_t>(wave, (batches + kSlicePipes - 1) / kSlicePipes));
    return NBB_OK;
}

// The passes of `steps` steps with at most kmax per pass: the fewest passes, steps spread evenly.
// With `parity`, the pass count has the parity of `steps` (the result then lands in the buffer a
// run of single steps leaves it in: the reference's double buffering), one pass more if needed.
std::vector<int> plan_passes(int32_t steps, int kmax, bool parity) {
    std::vector<int> out;
    if (steps <= 0) return out;
    int64_t p = (steps + kmax - 1) / kmax;
    if (parity && ((p ^ steps) & 1)) ++p;
    for (int64_t i = 0; i < p; ++i) out.push_back((int)(steps / p + (i < steps % p ? 1 : 0)));
    return out;
}

// One pass of k steps src -> dst on the compact state (λ or BB walk), this cfg's shard.
int launch_pass(DeviceCtx* ctx, const nbb_config* cfg, const void* src, void* dst, int k, uint16_t birth,
                uint16_t survive, cudaStream_t st) {
    FastDiv div_hb;
    const CompactCaArgs a = compact_args(cfg, src, dst, birth, survive, &div_hb);
    const int32_t* tab;
    NBB_CHECK(compact_nbr_table(ctx, cfg, a, div_hb, &tab));
    const uint64_t want = (a.tile_end - a.tile_begin + 7) / 8;
    if (want == 0) return NBB_OK;
    const bool bb = cfg->mode == NBB_MODE_BB;
    if (!bb && sliced_impl() && cluster_walk_ok(a))
        return launch_cluster_pass<false>(ctx, a, k, is_conway(birth, survive), div_hb, tab, P2PArgs{}, st);
    if (sliced_impl()) {
        const SliceBatches sb = slice_batches(a, k);
        auto kern = bb ? sliced_kernel<false, true>(is_conway(birth, survive))
                       : sliced_kernel<false, false>(is_conway(birth, survive));
        unsigned grid;
        NBB_CHECK(sliced_grid(ctx, (const void*)kern, sb.total, bb, &grid));
        NBB_CUDA(launch_pdl_smem(kern, grid, 32 * kSliceWarps, bb ? 0 : kSliceDynSmem, st, a, sb, div_hb, tab,
                                 P2PArgs{}));
        return NBB_OK;
    }
    auto kern = bb ? pass_kernel_k<false, true>(k, is_conway(birth, survive))
                   : pass_kernel_k<false, false>(k, is_conway(birth, survive));
    int occ;
    NBB_CHECK(pass_occupancy((const void*)kern, &occ));
    const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)ctx->sms * occ));
    NBB_CUDA(launch_pdl(kern, blocks, 256, st, a, div_hb, tab, P2PArgs{}));
    return NBB_OK;
}

// `steps` CA steps a <-> b on the compact state in passes (plan_passes); *result_in_b says where
// the result is; stats (optional) counts the launches.
int run_ca_compact(DeviceCtx* ctx, const nbb_config* cfg, void* d_a, void* d_b, int32_t steps, uint16_t birth,
                   uint16_t survive, cudaStream_t st, bool parity, nbb_pass_stats* stats) {
    NBB_CHECK(check_pass_steps(cfg));
    const std::vector<int> passes = plan_passes(steps, cfg->timing ? 1 : max_pass_steps(cfg), parity);
    nbb_pass_stats ps{};
    for (size_t i = 0; i < passes.size(); ++i) {
        NBB_CHECK(launch_pass(ctx, cfg, (i & 1) ? d_b : d_a, (i & 1) ? d_a : d_b, passes[i], birth, survive, st));
        ++ps.passes;
        ++ps.by_steps[passes[i]];
    }
    ps.result_in_b = (int32_t)(passes.size() & 1);
    if (stats) *stats = ps;
    return NBB_OK;
}

// The multi-GPU pass loop: `steps` steps in passes j = first_pass, first_pass + 1, ... of up to
// kmax steps (plan_passes, no parity constraint: pass j reads d_buf[j & 1] and writes
// d_buf[(j + 1) & 1] whatever its step count). Pass j waits for world x j arrivals.
int p2p_passes(const nbb_config* cfg, int64_t first_pass, int32_t steps, int kmax, uint16_t birth,
               uint16_t survive, const nbb_p2p* p2p, cudaStream_t stream, nbb_pass_stats* stats) {
    if (!cfg || !p2p) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    if (steps < 0) return fail(NBB_ERR_INVALID_ARGUMENT, "run_ca: steps must be non-negative");
    if (first_pass < 0) return fail(NBB_ERR_INVALID_ARGUMENT, "p2p: first_step must be non-negative");
    NBB_CHECK(compact_workload_check(cfg));
    NBB_CHECK(check_pass_steps(cfg));
    if (p2p->world < 1 || p2p->world > kMaxP2P || p2p->rank < 0 || p2p->rank >= p2p->world)
        return fail(NBB_ERR_INVALID_ARGUMENT, "p2p: need 1 <= world <= 8 and 0 <= rank < world");
    if (!p2p->d_buf[0] || !p2p->d_buf[1] || !p2p->d_peer_buf[0] || !p2p->d_peer_buf[1] || !p2p->d_sync ||
        !p2p->d_peer_flag)
        return fail(NBB_ERR_INVALID_ARGUMENT, "p2p: null device array");
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    FastDiv div_hb;
    CompactCaArgs a = compact_args(cfg, p2p->d_buf[0], p2p->d_buf[1], birth, survive, &div_hb);
    // the owner of a halo cell is its tile's ordinal / chunk: the shard must be the reference's
    // contiguous worker chunk (dispatch.cpp:419-427) of this rank, as every peer assumes
    const uint32_t chunk = (uint32_t)nbbhost::compact_shard_chunk(a.rb, a.tiles, a.Hb, p2p->world);
    const uint64_t want_b = std::min<uint64_t>((uint64_t)chunk * (uint64_t)p2p->rank, a.tiles);
    const uint64_t want_e = std::min<uint64_t>(want_b + chunk, a.tiles);
    if (cfg->shard_count == 0 || a.tile_begin != want_b || a.tile_end != want_e)
        return fail(NBB_ERR_INVALID_ARGUMENT,
                    "p2p: the shard must be the rank's contiguous chunk of tiles (nbb_gpu.h: ceil(tiles / world) "
                    "rounded up to whole 9 Hb-tile cluster columns when r >= 8): [" +
                        std::to_string(want_b) + ", " + std::to_string(want_e) + ")");
    const int32_t* tab;
    NBB_CHECK(compact_nbr_table(ctx, cfg, a, div_hb, &tab));
    P2PArgs p;
    p.sync = (unsigned int*)p2p->d_sync;
    p.peer_flag = (unsigned int* const*)p2p->d_peer_flag;
    p.timeout_ms = p2p->timeout_ms ? p2p->timeout_ms : 20000u;
    p.world = p2p->world;
    p.rank = p2p->rank;
    p.div_chunk.d = chunk;
    nbbhost::fastdiv_magic(chunk, &p.div_chunk.m, &p.div_chunk.s);
    const bool conway = is_conway(birth, survive);
    // every rank launches (and arrives) even with an empty shard: one CTA at least; at most one
    // resident wave, so CTAs spinning in the wait never keep a CTA of the same pass off an SM
    const uint64_t want = std::max<uint64_t>(1, (a.tile_end - a.tile_begin + 7) / 8);
    const std::vector<int> passes = plan_passes(steps, kmax, false);
    nbb_pass_stats ps{};
    int64_t j = first_pass;
    for (size_t i = 0; i < passes.size(); ++i, ++j) {
        const int par = (int)(j & 1);
        a.src = (const long long*)p2p->d_buf[par];
        a.dst = (long long*)p2p->d_buf[par ^ 1];
        p.peer_src = (const long long* const*)p2p->d_peer_buf[par];
        p.wait_target = (unsigned int)((uint64_t)p2p->world * (uint64_t)j);
        p.first_pass = i == 0 ? 1u : 0u;
        if (sliced_impl() && cluster_walk_ok(a)) {
            NBB_CHECK(launch_cluster_pass<true>(ctx, a, passes[i], conway, div_hb, tab, p, stream));
            ++ps.passes;
            ++ps.by_steps[passes[i]];
            continue;
        }
        if (sliced_impl()) {
            const SliceBatches sb = slice_batches(a, passes[i]);
            auto kern = sliced_kernel<true, false>(conway);
            unsigned grid;
            NBB_CHECK(sliced_grid(ctx, (const void*)kern, std::max<uint64_t>(1, sb.total), false, &grid));
            NBB_CUDA(launch_pdl_smem(kern, grid, 32 * kSliceWarps, kSliceDynSmem, stream, a, sb, div_hb, tab, p));
            ++ps.passes;
            ++ps.by_steps[passes[i]];
            continue;
        }
        auto kern = pass_kernel_k<true, false>(passes[i], conway);
        int occ;
        NBB_CHECK(pass_occupancy((const void*)kern, &occ));
        const unsigned blocks = (unsigned)std::min<uint64_t>(want, (uint64_t)ctx->sms * occ);
        NBB_CUDA(launch_pdl(kern, blocks, 256, stream, a, div_hb, tab, p));
        ++ps.passes;
        ++ps.by_steps[passes[i]];
    }
    ps.result_in_b = (int32_t)(j & 1);
    if (stats) *stats = ps;
    return NBB_OK;
}
}  // namespace

#include "nbb_multi.inc"

namespace {

// nbb_gpu_ca on the compact state: member sectors of the host Grid -> the λ-ordered compact array
// on devices[0] (2 x 8·3^r bytes, no embedded grid), passes over the orthotope (spread over the
// worker devices when ndev > 1), compact -> member sectors of out_grid.
int ca_compact_host(const nbb_config* cfg, Launch& L, const int64_t* initial, int64_t* out_grid, nbb_report* per_step,
                    int32_t steps, uint16_t birth, uint16_t survive, const long long* h_in, long long* h_out,
                    const int32_t* devices, int32_t ndev) {
    NBB_CHECK(compact_workload_check(cfg, ndev == 1));
    if (cfg->cell_width != 8) return fail(NBB_ERR_INVALID_ARGUMENT, "the compact state holds int64 values: cell_width 8");
    const size_t b64 = grid_bytes(L, 8);
    CompactShape cs;
    NBB_CHECK(compact_shape(cfg, &cs));
    void *ca, *cb, *stage = nullptr;
    NBB_CHECK(device_buffer(*L.ctx, 1, cs.total * 8, &ca));
    NBB_CHECK(device_buffer(*L.ctx, 2, cs.total * 8, &cb));
    const void* src = h_in;
    if (!src) {  // pageable input: stage the embedded grid in HBM
        NBB_CHECK(device_buffer(*L.ctx, 0, b64, &stage));
        NBB_CUDA(cudaMemcpyAsync(stage, initial, b64, cudaMemcpyHostToDevice, L.stream));
        src = stage;
    }
    // member sectors -> compact in embedded row order (host pages stay sequential)
    compact_from_rows_kernel<<<L.ctx->sms * 8, 256, 0, L.stream>>>((const long long*)src, (long long*)ca,
                                                                    (int64_t)cs.n, (uint32_t)cs.W);
    NBB_CUDA(cudaGetLastError());
    if (ndev > 1) {  // the worker split over devices
        nbb_pass_stats ps;
        NBB_CHECK(multi_device_passes(cfg, devices, ndev, ca, cb, steps, birth, survive, L.stream, &ps));
        if (per_step)
            for (int s = 0; s < steps; ++s) fill_report(cfg, &per_step[s], 0);
        if (ps.result_in_b) std::swap(ca, cb);
    } else if (cfg->timing) {  // per-step launch times: one launch per step
        NBB_CHECK(check_pass_steps(cfg));
        for (int s = 0; s < steps; ++s) {
            Timer t(true, L.stream);
            NBB_CHECK(launch_pass(L.ctx, cfg, ca, cb, 1, birth, survive, L.stream));
            const uint64_t us = t.stop_micros();
            if (per_step) fill_report(cfg, &per_step[s], us);
            std::swap(ca, cb);
        }
    } else {  // passes of up to pass_steps steps; the result in whichever buffer the last pass wrote
        nbb_pass_stats ps;
        NBB_CHECK(run_ca_compact(L.ctx, cfg, ca, cb, steps, birth, survive, L.stream, false, &ps));
        if (per_step)
            for (int s = 0; s < steps; ++s) fill_report(cfg, &per_step[s], 0);
        if (ps.result_in_b) std::swap(ca, cb);
    }
    if (h_out) {  // member sectors straight into the zeroed pinned output, row by row
        compact_to_rows_kernel<<<L.ctx->sms * 8, 256, 0, L.stream>>>((const long long*)ca, h_out, (int64_t)cs.n,
                                                                      (uint32_t)cs.W);
        NBB_CUDA(cudaGetLastError());
    } else {
        if (!stage) NBB_CHECK(device_buffer(*L.ctx, 0, b64, &stage));
        NBB_CUDA(cudaMemsetAsync(stage, 0, b64, L.stream));
        NBB_CHECK(compact_to_sectors(L.ctx, cfg, ca, stage, L.stream));
        NBB_CUDA(cudaMemcpyAsync(out_grid, stage, b64, cudaMemcpyDeviceToHost, L.stream));
    }
    NBB_CUDA(cudaStreamSynchronize(L.stream));
    return NBB_OK;
}
}  // namespace

// =====================================================================================
extern "C" {

int nbb_gpu_abi_version(void) { return NBB_GPU_ABI_VERSION; }
const char* nbb_gpu_last_error(void) { return g_last_error.c_str(); }

void nbb_spec_sierpinski(nbb_spec* s) {
    std::memset(s, 0, sizeof(*s));
    std::strcpy(s->name, "sierpinski");
    s->k = 3;
    s->s = 2;
    const int ox[] = {0, 0, 1}, oy[] = {0, 1, 1};
    for (int i = 0; i < 3; ++i) {
        s->offset_x[i] = ox[i];
        s->offset_y[i] = oy[i];
    }
}

void nbb_spec_vicsek(nbb_spec* s) {
    std::memset(s, 0, sizeof(*s));
    std::strcpy(s->name, "vicsek");
    s->k = 5;
    s->s = 3;
    const int ox[] = {1, 1, 1, 0, 2}, oy[] = {1, 0, 2, 1, 1};
    for (int i = 0; i < 5; ++i) {
        s->offset_x[i] = ox[i];
        s->offset_y[i] = oy[i];
    }
}

void nbb_spec_carpet(nbb_spec* s) {
    std::memset(s, 0, sizeof(*s));
    std::strcpy(s->name, "carpet");
    s->k = 8;
    s->s = 3;
    const int ox[] = {0, 1, 2, 0, 2, 0, 1, 2}, oy[] = {0, 0, 0, 1, 1, 2, 2, 2};
    for (int i = 0; i < 8; ++i) {
        s->offset_x[i] = ox[i];
        s->offset_y[i] = oy[i];
    }
}

void nbb_config_init(nbb_config* c) {
    std::memset(c, 0, sizeof(*c));
    nbb_spec_sierpinski(&c->spec);
    c->r = 0;
    c->rho = 1;
    c->mode = NBB_MODE_LAMBDA;
    c->strategy = NBB_STRATEGY_SUBBOX;
    c->backend = NBB_BACKEND_DIRECT;
    c->workers = 1;
    c->timing = 0;
    c->cell_width = 8;
    c->kernel = NBB_KERNEL_AUTO;
    c->device = 0;
    c->max_cells = (uint64_t)1 << 24;
}

int nbb_gpu_device_count(int32_t* count) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        c = 0;
    }
    *count = c;
    return NBB_OK;
}

int nbb_gpu_validate(const nbb_config* cfg) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    NBB_TRY(nbbhost::validate(*cfg));
    return NBB_OK;
}

int nbb_gpu_launch_block_count(const nbb_config* cfg, uint64_t* blocks) {
    NBB_TRY(nbbhost::validate(*cfg));
    nbbhost::Plan p;
    NBB_TRY(nbbhost::make_plan(*cfg, &p));
    *blocks = p.blocks();
    return NBB_OK;
}

int nbb_gpu_plan_report(const nbb_config* cfg, nbb_report* report) {
    NBB_TRY(nbbhost::plan_report(*cfg, report));
    return NBB_OK;
}

int nbb_gpu_work_quotient(const nbb_report* bb, const nbb_report* lam, int32_t weighted, double* q) {
    NBB_TRY(nbbhost::work_quotient(*bb, *lam, weighted != 0, q));
    return NBB_OK;
}

const char* nbb_gpu_csv_header(void) { return nbbhost::csv_header(); }

int nbb_gpu_report_csv_row(const nbb_report* report, char* buf, size_t len) {
    const std::string row = nbbhost::csv_row(*report);
    if (row.size() + 1 > len) return fail(NBB_ERR_INVALID_ARGUMENT, "csv buffer too small");
    std::memcpy(buf, row.c_str(), row.size() + 1);
    return NBB_OK;
}

int nbb_gpu_random_member_grid(const nbb_spec* spec, int32_t r, uint64_t seed, uint64_t modulus,
                               uint64_t max_cells, int64_t* out_grid) {
    NBB_TRY(nbbhost::random_member_grid(*spec, r, seed, modulus, max_cells, out_grid));
    return NBB_OK;
}

int nbb_gpu_random_member_values(const nbb_spec* spec, int32_t r, uint64_t seed, uint64_t modulus,
                                 int64_t* out_values) {
    NBB_TRY(nbbhost::random_member_values(*spec, r, seed, modulus, out_values));
    return NBB_OK;
}

// ---- device-resident workloads ---------------------------------------------------------
int nbb_gpu_single_write_dev(const nbb_config* cfg, void* d_grid, void* stream, nbb_report* report) {
    Launch L;
    NBB_CHECK(prepare(cfg, OP_SW, &L, cfg && cfg->mode == NBB_MODE_BB));
    L.stream = (cudaStream_t)stream;
    Timer t(cfg->timing != 0, L.stream);
    NBB_CHECK(launch_op(L, OP_SW, nullptr, d_grid, nullptr, 0, 0));
    fill_report(cfg, report, t.stop_micros());
    return NBB_OK;
}

int nbb_gpu_reduction_dev(const nbb_config* cfg, const void* d_grid, void* d_value, void* stream,
                          nbb_report* report) {
    Launch L;
    NBB_CHECK(prepare(cfg, OP_RD, &L, cfg && cfg->mode == NBB_MODE_BB));
    L.stream = (cudaStream_t)stream;
    Timer t(cfg->timing != 0, L.stream);
    NBB_CHECK(launch_op(L, OP_RD, d_grid, nullptr, (unsigned long long*)d_value, 0, 0));
    fill_report(cfg, report, t.stop_micros());
    return NBB_OK;
}

int nbb_gpu_ca_step_dev(const nbb_config* cfg, const void* d_src, void* d_dst, uint16_t birth,
                        uint16_t survive, void* stream, nbb_report* report) {
    Launch L;
    NBB_CHECK(prepare(cfg, OP_CA, &L, true));
    L.stream = (cudaStream_t)stream;
    Timer t(cfg->timing != 0, L.stream);
    NBB_CHECK(launch_op(L, OP_CA, d_src, d_dst, nullptr, birth, survive));
    fill_report(cfg, report, t.stop_micros());
    return NBB_OK;
}

int nbb_gpu_ca_run_dev(const nbb_config* cfg, void* d_a, void* d_b, int32_t steps, uint16_t birth, uint16_t survive,
                       void* stream, nbb_pass_stats* stats) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    if (steps < 0) return fail(NBB_ERR_INVALID_ARGUMENT, "run_ca: steps must be non-negative");
    Launch L;
    NBB_CHECK(prepare(cfg, OP_CA, &L, true));
    L.stream = (cudaStream_t)stream;
    void* res = (steps & 1) ? d_b : d_a;  // where a run of single steps leaves the result
    const bool blocked = nbbhost::is_gasket(cfg->spec) && cfg->cell_width == 8 && cfg->r >= 5 && cfg->r <= 18 &&
                         cfg->kernel == NBB_KERNEL_AUTO && !cfg->timing && cfg->shard_count == 0 && steps >= 2 &&
                         !(cfg->flags & NBB_FLAG_SINGLE_STEP);
    if (!blocked) {  // one launch per step on the embedded grid
        nbb_pass_stats ps{};
        void *src = d_a, *dst = d_b;
        for (int32_t s = 0; s < steps; ++s) {
            NBB_CHECK(launch_op(L, OP_CA, src, dst, nullptr, birth, survive));
            std::swap(src, dst);
            ++ps.passes;
            ++ps.by_steps[1];
        }
        ps.result_in_b = steps & 1;
        if (stats) *stats = ps;
        return NBB_OK;
    }
    // temporal blocking of the embedded state: its member sectors -> the λ-ordered compact state
    // (tile codec), passes of up to pass_steps steps there, compact -> the member sectors of the
    // result buffer (the same cells a run of single steps writes; non-member cells stay 0)
    NBB_CHECK(compact_workload_check(cfg, true));
    CompactShape cs;
    NBB_CHECK(compact_shape(cfg, &cs));
    void *ca, *cb;
    NBB_CHECK(device_buffer(*L.ctx, 1, cs.total * 8, &ca));
    NBB_CHECK(device_buffer(*L.ctx, 2, cs.total * 8, &cb));
    NBB_CHECK(compact_from_sectors(L.ctx, cfg, d_a, ca, L.stream));
    nbb_pass_stats ps;
    NBB_CHECK(run_ca_compact(L.ctx, cfg, ca, cb, steps, birth, survive, L.stream, false, &ps));
    NBB_CHECK(compact_to_sectors(L.ctx, cfg, ps.result_in_b ? cb : ca, res, L.stream));
    ps.result_in_b = steps & 1;
    if (stats) *stats = ps;
    return NBB_OK;
}

int nbb_gpu_sanitize_dev(const nbb_config* cfg, void* d_grid, void* stream) {
    Launch L;
    NBB_CHECK(prepare(cfg, OP_CA, &L, false, true));
    return sanitize(L, d_grid, cfg->cell_width, (cudaStream_t)stream);
}

int nbb_gpu_pack_alive_dev(const nbb_config* cfg, const void* d64, void* d8, void* stream) {
    Launch L;
    NBB_CHECK(prepare(cfg, OP_CA, &L, false, true));
    if (cfg->cell_width == 0)
        pack_bits_kernel<<<L.ctx->sms * 8, 256, 0, (cudaStream_t)stream>>>(
            (const long long*)d64, (uint32_t*)d8, L.plan.n);
    else
        pack_alive_kernel<<<L.ctx->sms * 8, 256, 0, (cudaStream_t)stream>>>(
            (const long long*)d64, (unsigned char*)d8, L.plan.n);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

int nbb_gpu_unpack_alive_dev(const nbb_config* cfg, const void* d8, void* d64, void* stream) {
    Launch L;
    NBB_CHECK(prepare(cfg, OP_CA, &L, false, true));
    if (cfg->cell_width == 0)  // writes member sectors only: d64's non-member cells must be 0
        unpack_bits_kernel<<<L.ctx->sms * 8, 256, 0, (cudaStream_t)stream>>>(
            (const uint32_t*)d8, (long long*)d64, L.plan.n);
    else
        unpack_alive_kernel<<<L.ctx->sms * 8, 256, 0, (cudaStream_t)stream>>>(
            (const unsigned char*)d8, (long long*)d64, L.plan.n);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

int nbb_gpu_scatter_members_dev(const nbb_config* cfg, const void* d_values, void* d_grid,
                                void* stream) {
    Launch L;
    NBB_CHECK(prepare(cfg, OP_CA, &L, false, true));
    scatter_members_kernel<<<L.ctx->sms * 8, 256, 0, (cudaStream_t)stream>>>(
        (const long long*)d_values, (long long*)d_grid, L.plan.n);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

int nbb_gpu_lambda_coords_dev(const nbb_config* cfg, int32_t level, void* d_xy, int32_t coord_bytes,
                              void* stream) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    NBB_TRY(nbbhost::validate_spec(cfg->spec));
    if (level < 0) return fail(NBB_ERR_INVALID_ARGUMENT, "lambda: negative level");
    if (!nbbhost::is_gasket(cfg->spec)) {  // table-driven digit loop for any NBB spec
        DeviceCtx* gctx;
        NBB_CHECK(ensure_device(cfg->device, &gctx));
        int64_t gw, gh;
        NBB_TRY(nbbhost::orthotope_dims(cfg->spec, level, &gw, &gh));
        const uint64_t gtotal = (uint64_t)gw * (uint64_t)gh;
        if (gtotal > (uint64_t(1) << 31)) return fail(NBB_ERR_RESOURCE, "orthotope too large for the map kernel");
        const unsigned gb = (unsigned)std::min<uint64_t>((gtotal + 255) / 256, (uint64_t)gctx->sms * 16);
        if (coord_bytes == 4)
            lambda_map_generic_kernel<int32_t><<<std::max(1u, gb), 256, 0, (cudaStream_t)stream>>>(
                dev_spec(cfg->spec), (int32_t*)d_xy, gtotal, (uint64_t)gw, level);
        else if (coord_bytes == 8)
            lambda_map_generic_kernel<long long><<<std::max(1u, gb), 256, 0, (cudaStream_t)stream>>>(
                dev_spec(cfg->spec), (long long*)d_xy, gtotal, (uint64_t)gw, level);
        else
            return fail(NBB_ERR_INVALID_ARGUMENT, "coord_bytes must be 4 or 8");
        NBB_CUDA(cudaGetLastError());
        return NBB_OK;
    }
    if (level > 17) return fail(NBB_ERR_RESOURCE, "lambda map kernel supports levels <= 17");
    if (coord_bytes != 4 && coord_bytes != 8)
        return fail(NBB_ERR_INVALID_ARGUMENT, "coord_bytes must be 4 or 8");
    const bool tc = cfg->backend == NBB_BACKEND_MMA1 || cfg->backend == NBB_BACKEND_MMA2;
    if (cfg->backend == NBB_BACKEND_MMA1 && level > 16)  // the paper's 16 x 16 fragment
        return fail(NBB_ERR_INVALID_ARGUMENT, "variant 1 encodes at most 16 levels, r_b = " +
                                                  std::to_string(level));
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    int64_t w, h;
    NBB_TRY(nbbhost::orthotope_dims(cfg->spec, level, &w, &h));
    const uint64_t total = (uint64_t)w * (uint64_t)h;
    FastDiv f;
    f.d = (uint32_t)w;
    nbbhost::fastdiv_magic(f.d, &f.m, &f.s);
    cudaStream_t s = (cudaStream_t)stream;
    // one wave at most, no more blocks than the work needs (small levels are launch-bound:
    // every block stages the 729-entry digit table)
    const uint64_t per_block = tc ? 16ull * 8 : 4ull * 256;  // ω per block and pass
    const int blocks = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ctx->sms * 8,
                                                                      (total + per_block - 1) / per_block));
    if (tc && cfg->backend == NBB_BACKEND_MMA2) {
        // K0-TC on tcgen05 (5th-gen tensor core, accumulator in TMEM): 128 ω per CTA tile,
        // 16 CTAs per SM (32 of the 512 TMEM columns and 13 KB smem each): the per-tile
        // build -> MMA -> tcgen05.ld chain is latency-bound, other CTAs fill the gaps
        const unsigned tc_blocks = (unsigned)std::max<uint64_t>(
            1, std::min<uint64_t>((uint64_t)ctx->sms * 16, (total + 127) / 128));
        if (coord_bytes == 4)
            lambda_map_tc5_kernel<int32_t><<<tc_blocks, 128, 0, s>>>((int32_t*)d_xy, total, (uint32_t)w, f);
        else
            lambda_map_tc5_kernel<long long><<<tc_blocks, 128, 0, s>>>((long long*)d_xy, total, (uint32_t)w, f);
    } else if (tc) {
        // K0-TC on the warp-level mma.sync path (the paper's 16 x 16 fragment product)
        if (coord_bytes == 4)
            lambda_map_tc_kernel<int32_t><<<blocks, 256, 0, s>>>((int32_t*)d_xy, total, (uint32_t)w, f, level);
        else
            lambda_map_tc_kernel<long long><<<blocks, 256, 0, s>>>((long long*)d_xy, total, (uint32_t)w, f, level);
    } else {
        if (coord_bytes == 4)
            lambda_map_kernel<int32_t><<<blocks, 256, 0, s>>>((int32_t*)d_xy, total, (uint32_t)w, f);
        else
            lambda_map_kernel<long long><<<blocks, 256, 0, s>>>((long long*)d_xy, total, (uint32_t)w, f);
    }
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

// ---- workloads on host buffers (drop-in for run_single_write / run_reduction / run_ca) ----
int nbb_gpu_single_write(const nbb_config* cfg, int64_t* out_grid, nbb_report* report) {
    if (cfg && cfg->r < 0) return fail(NBB_ERR_INVALID_ARGUMENT, "checked_pow: negative exponent");
    Launch L;
    NBB_CHECK(prepare(cfg, OP_SW, &L, cfg && cfg->mode == NBB_MODE_BB));
    L.stream = L.ctx->stream;
    nbb_config c8 = *cfg;
    c8.cell_width = 8;  // the result Grid is int64
    L.cfg = &c8;
    void* d;
    NBB_CHECK(device_buffer(*L.ctx, 0, grid_bytes(L, 8), &d));
    NBB_CUDA(cudaMemsetAsync(d, 0, grid_bytes(L, 8), L.stream));
    Timer t(cfg->timing != 0, L.stream);
    NBB_CHECK(launch_op(L, OP_SW, nullptr, d, nullptr, 0, 0));
    const uint64_t us = t.stop_micros();
    NBB_CUDA(cudaMemcpyAsync(out_grid, d, grid_bytes(L, 8), cudaMemcpyDeviceToHost, L.stream));
    NBB_CUDA(cudaStreamSynchronize(L.stream));
    fill_report(cfg, report, us);
    return NBB_OK;
}

int nbb_gpu_reduction(const nbb_config* cfg, const int64_t* grid, int32_t grid_level, int64_t* value,
                      nbb_report* report) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    NBB_TRY(nbbhost::validate(*cfg));
    if (grid_level != cfg->r)
        return fail(NBB_ERR_INVALID_ARGUMENT, "reduction: grid level " + std::to_string(grid_level) +
                                                  " does not match the configured r = " +
                                                  std::to_string(cfg->r));
    Launch L;
    NBB_CHECK(prepare(cfg, OP_RD, &L, cfg->mode == NBB_MODE_BB));
    L.stream = L.ctx->stream;
    void* d;
    NBB_CHECK(device_buffer(*L.ctx, 0, grid_bytes(L, 8), &d));
    NBB_CUDA(cudaMemcpyAsync(d, grid, grid_bytes(L, 8), cudaMemcpyHostToDevice, L.stream));
    unsigned long long* d_sum = L.ctx->partials + 4096;
    Timer t(cfg->timing != 0, L.stream);
    NBB_CHECK(launch_op(L, OP_RD, d, nullptr, d_sum, 0, 0));
    const uint64_t us = t.stop_micros();
    unsigned long long v = 0;
    NBB_CUDA(cudaMemcpyAsync(&v, d_sum, sizeof(v), cudaMemcpyDeviceToHost, L.stream));
    NBB_CUDA(cudaStreamSynchronize(L.stream));
    *value = (int64_t)v;
    fill_report(cfg, report, us);
    return NBB_OK;
}

int nbb_gpu_ca(const nbb_config* cfg, const int64_t* initial, int32_t initial_level, int32_t steps,
               uint16_t birth, uint16_t survive, int64_t* out_grid, nbb_report* per_step) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    NBB_TRY(nbbhost::validate(*cfg));
    if (initial_level != cfg->r)
        return fail(NBB_ERR_INVALID_ARGUMENT, "ca: grid level does not match the configured r");
    if (steps < 0) return fail(NBB_ERR_INVALID_ARGUMENT, "ca: negative step count");
    Launch L;
    NBB_CHECK(prepare(cfg, OP_CA, &L, true));
    L.stream = L.ctx->stream;
    const size_t b64 = grid_bytes(L, 8);
    if (steps == 0) {  // the input comes back unchanged (App. B.4)
        if (out_grid != initial) std::memmove(out_grid, initial, b64);
        return NBB_OK;
    }
    const int cw = cfg->cell_width;
    const int blocks = L.ctx->sms * 8;
    // zero-copy: pinned host buffers are read/written in place, member sectors only
    const bool gasket = nbbhost::is_gasket(cfg->spec);  // member-sector kernels need the gasket
    const long long* h_in = gasket ? (const long long*)mapped_host_ptr(initial) : nullptr;
    long long* h_out = (gasket && (cfg->flags & NBB_FLAG_OUT_ZEROED))
                           ? (long long*)mapped_host_ptr(out_grid) : nullptr;
    if ((cfg->flags & NBB_FLAG_COMPACT_STATE) && (cfg->flags & NBB_FLAG_EMBEDDED_STATE))
        return fail(NBB_ERR_INVALID_ARGUMENT, "ca: NBB_FLAG_COMPACT_STATE and NBB_FLAG_EMBEDDED_STATE exclude each other");
    // the compact state serves the call by default (nbb_gpu.h); the flags force either state
    const bool compact_ok = gasket && cw == 8 && cfg->r >= 5 && cfg->r <= 18 && cfg->kernel == NBB_KERNEL_AUTO &&
                            cfg->shard_count == 0;
    if ((cfg->flags & NBB_FLAG_COMPACT_STATE) || (compact_ok && !(cfg->flags & NBB_FLAG_EMBEDDED_STATE))) {
        return ca_compact_host(cfg, L, initial, out_grid, per_step, steps, birth, survive, h_in, h_out, nullptr, 1);
    }
    void *d64 = nullptr, *da, *db;
    if (cw == 8) {
        NBB_CHECK(device_buffer(*L.ctx, 0, b64, &da));
        NBB_CHECK(device_buffer(*L.ctx, 1, b64, &db));
        if (h_in) {
            NBB_CUDA(cudaMemsetAsync(da, 0, b64, L.stream));
            copy_member_sectors_kernel<<<blocks, 256, 0, L.stream>>>(h_in, (long long*)da, L.plan.n, 1);
            NBB_CUDA(cudaGetLastError());
        } else {
            NBB_CUDA(cudaMemcpyAsync(da, initial, b64, cudaMemcpyHostToDevice, L.stream));
            NBB_CHECK(sanitize(L, da, 8, L.stream));
        }
        NBB_CUDA(cudaMemsetAsync(db, 0, b64, L.stream));
    } else {
        const size_t bs = grid_bytes(L, cw);
        NBB_CHECK(device_buffer(*L.ctx, 1, bs, &da));
        NBB_CHECK(device_buffer(*L.ctx, 2, bs, &db));
        const long long* src64 = h_in;
        if (!src64) {  // stage the whole grid in HBM
            NBB_CHECK(device_buffer(*L.ctx, 0, b64, &d64));
            NBB_CUDA(cudaMemcpyAsync(d64, initial, b64, cudaMemcpyHostToDevice, L.stream));
            src64 = (const long long*)d64;
        }
        if (cw == 1)
            pack_alive_kernel<<<blocks, 256, 0, L.stream>>>(src64, (unsigned char*)da, L.plan.n);
        else
            pack_bits_kernel<<<blocks, 256, 0, L.stream>>>(src64, (uint32_t*)da, L.plan.n);
        NBB_CUDA(cudaGetLastError());
        NBB_CUDA(cudaMemsetAsync(db, 0, bs, L.stream));
    }
    for (int s = 0; s < steps; ++s) {
        Timer t(cfg->timing != 0, L.stream);
        NBB_CHECK(launch_op(L, OP_CA, da, db, nullptr, birth, survive));
        const uint64_t us = t.stop_micros();
        if (per_step) fill_report(cfg, &per_step[s], us);
        std::swap(da, db);
    }
    if (h_out) {  // member sectors straight into the (zeroed) pinned host grid
        if (cw == 8)
            copy_member_sectors_kernel<<<blocks, 256, 0, L.stream>>>((const long long*)da, h_out, L.plan.n, 0);
        else if (cw == 1)
            unpack_alive_kernel<<<blocks, 256, 0, L.stream>>>((const unsigned char*)da, h_out, L.plan.n, 1);
        else
            unpack_bits_kernel<<<blocks, 256, 0, L.stream>>>((const uint32_t*)da, h_out, L.plan.n);
        NBB_CUDA(cudaGetLastError());
        NBB_CUDA(cudaStreamSynchronize(L.stream));
        return NBB_OK;
    }
    if (cw != 8) {  // materialise the full int64 grid (non-members 0) in HBM
        NBB_CHECK(device_buffer(*L.ctx, 0, b64, &d64));
        NBB_CUDA(cudaMemsetAsync(d64, 0, b64, L.stream));
        if (cw == 1)
            unpack_alive_kernel<<<blocks, 256, 0, L.stream>>>((const unsigned char*)da, (long long*)d64,
                                                              L.plan.n, 1);
        else
            unpack_bits_kernel<<<blocks, 256, 0, L.stream>>>((const uint32_t*)da, (long long*)d64, L.plan.n);
        NBB_CUDA(cudaGetLastError());
        da = d64;
    }
    NBB_CUDA(cudaMemcpyAsync(out_grid, da, b64, cudaMemcpyDeviceToHost, L.stream));
    NBB_CUDA(cudaStreamSynchronize(L.stream));
    return NBB_OK;
}

int nbb_gpu_ca_multi(const nbb_config* cfg, const int32_t* devices, int32_t ndev, const int64_t* initial,
                     int32_t initial_level, int32_t steps, uint16_t birth, uint16_t survive, int64_t* out_grid,
                     nbb_report* per_step) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    NBB_CHECK(check_devices(devices, ndev));
    nbb_config c = *cfg;
    c.device = devices[0];
    if (ndev == 1) return nbb_gpu_ca(&c, initial, initial_level, steps, birth, survive, out_grid, per_step);
    NBB_TRY(nbbhost::validate(c));
    if (initial_level != c.r) return fail(NBB_ERR_INVALID_ARGUMENT, "ca: grid level does not match the configured r");
    if (steps < 0) return fail(NBB_ERR_INVALID_ARGUMENT, "ca: negative step count");
    if (c.shard_count > 0) return fail(NBB_ERR_INVALID_ARGUMENT, "multi: the devices split the whole tile range");
    if (c.flags & NBB_FLAG_EMBEDDED_STATE)
        return fail(NBB_ERR_INVALID_ARGUMENT, "multi: the worker split runs on the compact state");
    Launch L;
    NBB_CHECK(prepare(&c, OP_CA, &L, true));
    L.stream = L.ctx->stream;
    if (steps == 0) {
        if (out_grid != initial) std::memmove(out_grid, initial, grid_bytes(L, 8));
        return NBB_OK;
    }
    const long long* h_in = (const long long*)mapped_host_ptr(initial);
    long long* h_out = (c.flags & NBB_FLAG_OUT_ZEROED) ? (long long*)mapped_host_ptr(out_grid) : nullptr;
    return ca_compact_host(&c, L, initial, out_grid, per_step, steps, birth, survive, h_in, h_out, devices, ndev);
}

int nbb_gpu_reduction_multi(const nbb_config* cfg, const int32_t* devices, int32_t ndev, const int64_t* grid,
                            int32_t grid_level, int64_t* value, nbb_report* report) {
    if (!cfg || !value) return fail(NBB_ERR_INVALID_ARGUMENT, "null argument");
    NBB_CHECK(check_devices(devices, ndev));
    nbb_config c = *cfg;
    c.device = devices[0];
    if (ndev == 1) return nbb_gpu_reduction(&c, grid, grid_level, value, report);
    NBB_TRY(nbbhost::validate(c));
    if (grid_level != c.r)
        return fail(NBB_ERR_INVALID_ARGUMENT, "reduction: grid level " + std::to_string(grid_level) +
                                                  " does not match the configured r = " + std::to_string(c.r));
    NBB_CHECK(compact_workload_check(&c));
    Launch L;
    NBB_CHECK(prepare(&c, OP_RD, &L, false));
    L.stream = L.ctx->stream;
    CompactShape cs;
    NBB_CHECK(compact_shape(&c, &cs));
    const size_t b64 = grid_bytes(L, 8), bytes = (size_t)cs.total * 8;
    void *stage, *ca;
    NBB_CHECK(device_buffer(*L.ctx, 0, b64, &stage));
    NBB_CHECK(device_buffer(*L.ctx, 1, bytes, &ca));
    NBB_CUDA(cudaMemcpyAsync(stage, grid, b64, cudaMemcpyHostToDevice, L.stream));
    compact_from_rows_kernel<<<L.ctx->sms * 8, 256, 0, L.stream>>>((const long long*)stage, (long long*)ca,
                                                                    (int64_t)cs.n, (uint32_t)cs.W);
    NBB_CUDA(cudaGetLastError());
    NBB_CUDA(cudaStreamSynchronize(L.stream));
    // worker w sums its chunk of tiles on its device; the partial sums add up on the host (int64
    // addition wraps like the reference's accumulation, so any split gives the same value)
    FastDiv d;
    const CompactCaArgs a = compact_args(&c, nullptr, nullptr, 0, 0, &d);
    const uint32_t chunk = (uint32_t)nbbhost::compact_shard_chunk(a.rb, a.tiles, a.Hb, ndev);
    unsigned long long total = 0;
    for (int w = 0; w < ndev; ++w) {
        nbb_config wc = c;
        wc.device = devices[w];
        wc.shard_begin = std::min<uint64_t>((uint64_t)chunk * (uint64_t)w, a.tiles);
        wc.shard_count = std::min<uint64_t>((uint64_t)chunk, a.tiles - wc.shard_begin);
        if (wc.shard_count == 0) continue;
        DeviceCtx* ctx;
        NBB_CHECK(ensure_device(devices[w], &ctx));
        void* mine = ca;
        if (devices[w] != devices[0]) {
            NBB_CHECK(device_buffer(*ctx, 1, bytes, &mine));
            NBB_CUDA(cudaMemcpyPeerAsync(mine, devices[w], ca, devices[0], bytes, ctx->stream));
        }
        Segs sg;
        NBB_CHECK(compact_segments(&wc, &sg));
        unsigned long long* part = ctx->partials + 4096;
        NBB_CUDA(cudaMemsetAsync(part, 0, 8, ctx->stream));
        segment_sum_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>((const long long*)mine, sg, part);
        NBB_CUDA(cudaGetLastError());
        unsigned long long v = 0;
        NBB_CUDA(cudaMemcpyAsync(&v, part, 8, cudaMemcpyDeviceToHost, ctx->stream));
        NBB_CUDA(cudaStreamSynchronize(ctx->stream));
        total += v;
    }
    NBB_CUDA(cudaSetDevice(devices[0]));
    *value = (int64_t)total;
    fill_report(&c, report, 0);
    return NBB_OK;
}

int nbb_gpu_lambda_coords(const nbb_config* cfg, int32_t level, int64_t* xy) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    int64_t w, h;
    NBB_TRY(nbbhost::orthotope_dims(cfg->spec, level < 0 ? 0 : level, &w, &h));
    const size_t bytes = (size_t)w * (size_t)h * 16;
    void* d;
    NBB_CHECK(device_buffer(*ctx, 0, bytes, &d));
    NBB_CHECK(nbb_gpu_lambda_coords_dev(cfg, level, d, 8, ctx->stream));
    NBB_CUDA(cudaMemcpyAsync(xy, d, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    NBB_CUDA(cudaStreamSynchronize(ctx->stream));
    return NBB_OK;
}

int nbb_gpu_gather_cells_dev(const nbb_config* cfg, const void* d_grid, const int64_t* d_idx,
                             int64_t count, void* d_out, void* stream) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    if (count <= 0) return NBB_OK;
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    const unsigned blocks = (unsigned)std::min<int64_t>((count + 255) / 256, 65535);
    if (cfg->cell_width == 8)
        gather_cells_kernel<long long><<<blocks, 256, 0, (cudaStream_t)stream>>>(
            (const long long*)d_grid, (const long long*)d_idx, count, (long long*)d_out);
    else if (cfg->cell_width == 0)  // bit state: idx are 32-bit word indices
        gather_cells_kernel<uint32_t><<<blocks, 256, 0, (cudaStream_t)stream>>>(
            (const uint32_t*)d_grid, (const long long*)d_idx, count, (uint32_t*)d_out);
    else
        gather_cells_kernel<unsigned char><<<blocks, 256, 0, (cudaStream_t)stream>>>(
            (const unsigned char*)d_grid, (const long long*)d_idx, count, (unsigned char*)d_out);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

int nbb_gpu_scatter_cells_dev(const nbb_config* cfg, void* d_grid, const int64_t* d_idx,
                              int64_t count, const void* d_vals, void* stream) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    if (count <= 0) return NBB_OK;
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    const unsigned blocks = (unsigned)std::min<int64_t>((count + 255) / 256, 65535);
    if (cfg->cell_width == 8)
        scatter_cells_kernel<long long><<<blocks, 256, 0, (cudaStream_t)stream>>>(
            (long long*)d_grid, (const long long*)d_idx, count, (const long long*)d_vals);
    else if (cfg->cell_width == 0)
        scatter_cells_kernel<uint32_t><<<blocks, 256, 0, (cudaStream_t)stream>>>(
            (uint32_t*)d_grid, (const long long*)d_idx, count, (const uint32_t*)d_vals);
    else
        scatter_cells_kernel<unsigned char><<<blocks, 256, 0, (cudaStream_t)stream>>>(
            (unsigned char*)d_grid, (const long long*)d_idx, count, (const unsigned char*)d_vals);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}


int nbb_gpu_compact_store_dev(const nbb_config* cfg, const void* d_embedded, void* d_compact, void* stream) {
    CompactShape s;
    NBB_CHECK(compact_shape(cfg, &s));
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    if (compact_tiles_ok(cfg)) return compact_from_sectors(ctx, cfg, d_embedded, d_compact, (cudaStream_t)stream);
    if (nbbhost::is_gasket(cfg->spec))
        compact_store_kernel<false><<<grid_for(ctx, s.total), 256, 0, (cudaStream_t)stream>>>(
            dev_spec(cfg->spec), (const long long*)d_embedded, (long long*)d_compact, s.n, s.W, s.total, cfg->r);
    else
        compact_store_kernel<true><<<grid_for(ctx, s.total), 256, 0, (cudaStream_t)stream>>>(
            dev_spec(cfg->spec), (const long long*)d_embedded, (long long*)d_compact, s.n, s.W, s.total, cfg->r);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

int nbb_gpu_compact_load_dev(const nbb_config* cfg, const void* d_compact, int64_t empty_value,
                             void* d_embedded, void* stream) {
    CompactShape s;
    NBB_CHECK(compact_shape(cfg, &s));
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    const uint64_t cells = (uint64_t)s.n * (uint64_t)s.n;
    if (empty_value == 0) {
        NBB_CUDA(cudaMemsetAsync(d_embedded, 0, cells * 8, (cudaStream_t)stream));
        if (compact_tiles_ok(cfg)) return compact_to_sectors(ctx, cfg, d_compact, d_embedded, (cudaStream_t)stream);
    } else {
        fill_kernel<<<grid_for(ctx, cells), 256, 0, (cudaStream_t)stream>>>((long long*)d_embedded, cells, empty_value);
    }
    if (nbbhost::is_gasket(cfg->spec))
        compact_load_kernel<false><<<grid_for(ctx, s.total), 256, 0, (cudaStream_t)stream>>>(
            dev_spec(cfg->spec), (const long long*)d_compact, (long long*)d_embedded, s.n, s.W, s.total, cfg->r);
    else
        compact_load_kernel<true><<<grid_for(ctx, s.total), 256, 0, (cudaStream_t)stream>>>(
            dev_spec(cfg->spec), (const long long*)d_compact, (long long*)d_embedded, s.n, s.W, s.total, cfg->r);
    NBB_CUDA(cudaGetLastError());
    return NBB_OK;
}

int nbb_gpu_compact_store(const nbb_config* cfg, const int64_t* embedded, int64_t* compact) {
    CompactShape s;
    NBB_CHECK(compact_shape(cfg, &s));
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    const size_t be = (size_t)s.n * (size_t)s.n * 8, bc = (size_t)s.total * 8;
    void *de, *dc;
    NBB_CHECK(device_buffer(*ctx, 0, be, &de));
    NBB_CHECK(device_buffer(*ctx, 1, bc, &dc));
    NBB_CUDA(cudaMemcpyAsync(de, embedded, be, cudaMemcpyHostToDevice, ctx->stream));
    NBB_CHECK(nbb_gpu_compact_store_dev(cfg, de, dc, ctx->stream));
    NBB_CUDA(cudaMemcpyAsync(compact, dc, bc, cudaMemcpyDeviceToHost, ctx->stream));
    NBB_CUDA(cudaStreamSynchronize(ctx->stream));
    return NBB_OK;
}

int nbb_gpu_compact_load(const nbb_config* cfg, const int64_t* compact, int64_t empty_value,
                         int64_t* embedded) {
    CompactShape s;
    NBB_CHECK(compact_shape(cfg, &s));
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    const size_t be = (size_t)s.n * (size_t)s.n * 8, bc = (size_t)s.total * 8;
    void *de, *dc;
    NBB_CHECK(device_buffer(*ctx, 0, be, &de));
    NBB_CHECK(device_buffer(*ctx, 1, bc, &dc));
    NBB_CUDA(cudaMemcpyAsync(dc, compact, bc, cudaMemcpyHostToDevice, ctx->stream));
    NBB_CHECK(nbb_gpu_compact_load_dev(cfg, dc, empty_value, de, ctx->stream));
    NBB_CUDA(cudaMemcpyAsync(embedded, de, be, cudaMemcpyDeviceToHost, ctx->stream));
    NBB_CUDA(cudaStreamSynchronize(ctx->stream));
    return NBB_OK;
}

int nbb_gpu_lambda_inverse(const nbb_config* cfg, int32_t level, const int64_t* xy, uint64_t count,
                           int64_t* omega) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    NBB_TRY(nbbhost::validate_spec(cfg->spec));
    if (level < 0) return fail(NBB_ERR_INVALID_ARGUMENT, "lambda_inverse: negative level");
    int64_t n;
    NBB_TRY(nbbhost::side_length(cfg->spec, level, &n));
    if (count == 0) return NBB_OK;
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    void *dxy, *dom;
    NBB_CHECK(device_buffer(*ctx, 0, count * 16, &dxy));
    NBB_CHECK(device_buffer(*ctx, 1, count * 16 + count * 4, &dom));
    int* dst = (int*)((char*)dom + count * 16);
    NBB_CUDA(cudaMemcpyAsync(dxy, xy, count * 16, cudaMemcpyHostToDevice, ctx->stream));
    lambda_inverse_kernel<<<grid_for(ctx, count), 256, 0, ctx->stream>>>(
        dev_spec(cfg->spec), (const long long*)dxy, (long long*)dom, dst, count, level);
    NBB_CUDA(cudaGetLastError());
    std::vector<int> st(count);
    NBB_CUDA(cudaMemcpyAsync(omega, dom, count * 16, cudaMemcpyDeviceToHost, ctx->stream));
    NBB_CUDA(cudaMemcpyAsync(st.data(), dst, count * 4, cudaMemcpyDeviceToHost, ctx->stream));
    NBB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (uint64_t i = 0; i < count; ++i) {
        if (st[i] == NBB_ERR_OUT_OF_RANGE)
            return fail(NBB_ERR_OUT_OF_RANGE, "lambda_inverse: (" + std::to_string(xy[2 * i]) + "," +
                                                  std::to_string(xy[2 * i + 1]) + ") outside " +
                                                  std::to_string(n) + "^2");
        if (st[i] == NBB_ERR_DOMAIN)
            return fail(NBB_ERR_DOMAIN, "lambda_inverse: (" + std::to_string(xy[2 * i]) + "," +
                                            std::to_string(xy[2 * i + 1]) +
                                            ") is not a member cell at level " + std::to_string(level));
    }
    return NBB_OK;
}

int nbb_gpu_compact_write(const char* path, const nbb_spec* spec, int32_t level, const int64_t* values) {
    NBB_TRY(nbbhost::validate_spec(*spec));
    NBB_TRY(nbbhost::write_compact(path, *spec, level, values));
    return NBB_OK;
}

int nbb_gpu_compact_read(const char* path, const nbb_spec* spec, int32_t* level, int64_t* values,
                         uint64_t capacity) {
    NBB_TRY(nbbhost::validate_spec(*spec));
    int lv = 0;
    NBB_TRY(nbbhost::read_compact(path, *spec, &lv, values, capacity));
    *level = lv;
    return NBB_OK;
}

int nbb_gpu_ca_compact_step_dev(const nbb_config* cfg, const void* d_src, void* d_dst, uint16_t birth,
                                uint16_t survive, void* stream, nbb_report* report) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    NBB_CHECK(compact_workload_check(cfg, true));
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    Timer t(cfg->timing != 0, (cudaStream_t)stream);
    NBB_CHECK(launch_pass(ctx, cfg, d_src, d_dst, 1, birth, survive, (cudaStream_t)stream));
    fill_report(cfg, report, t.stop_micros());
    return NBB_OK;
}

int nbb_gpu_ca_compact_run_dev(const nbb_config* cfg, void* d_a, void* d_b, int32_t steps, uint16_t birth,
                               uint16_t survive, void* stream) {
    return nbb_gpu_ca_compact_passes_dev(cfg, d_a, d_b, steps, birth, survive, 1, stream, nullptr);
}

int nbb_gpu_ca_compact_passes_dev(const nbb_config* cfg, void* d_a, void* d_b, int32_t steps, uint16_t birth,
                                  uint16_t survive, int32_t parity, void* stream, nbb_pass_stats* stats) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    if (steps < 0) return fail(NBB_ERR_INVALID_ARGUMENT, "run_ca: steps must be non-negative");
    NBB_CHECK(compact_workload_check(cfg, true));
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    return run_ca_compact(ctx, cfg, d_a, d_b, steps, birth, survive, (cudaStream_t)stream, parity != 0, stats);
}

int nbb_gpu_pass_plan(const nbb_config* cfg, int32_t steps, int32_t parity, nbb_pass_stats* stats) {
    if (!cfg || !stats) return fail(NBB_ERR_INVALID_ARGUMENT, "null argument");
    if (steps < 0) return fail(NBB_ERR_INVALID_ARGUMENT, "run_ca: steps must be non-negative");
    NBB_CHECK(check_pass_steps(cfg));
    const std::vector<int> passes = plan_passes(steps, cfg->timing ? 1 : max_pass_steps(cfg), parity != 0);
    *stats = nbb_pass_stats{};
    for (int k : passes) {
        ++stats->passes;
        ++stats->by_steps[k];
    }
    stats->result_in_b = (int32_t)(passes.size() & 1);
    return NBB_OK;
}

int nbb_gpu_ca_compact_p2p_dev(const nbb_config* cfg, int64_t first_step, int32_t steps, uint16_t birth,
                               uint16_t survive, const nbb_p2p* p2p, void* stream) {
    return p2p_passes(cfg, first_step, steps, 1, birth, survive, p2p, (cudaStream_t)stream, nullptr);
}

int nbb_gpu_ca_compact_p2p_passes_dev(const nbb_config* cfg, int64_t first_pass, int32_t steps, uint16_t birth,
                                      uint16_t survive, const nbb_p2p* p2p, void* stream) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    return p2p_passes(cfg, first_pass, steps, max_pass_steps(cfg), birth, survive, p2p, (cudaStream_t)stream,
                      nullptr);
}

int nbb_gpu_p2p_check(const nbb_p2p* p2p, void* stream) {
    if (!p2p || !p2p->d_sync) return fail(NBB_ERR_INVALID_ARGUMENT, "p2p: null sync buffer");
    int err = 0;
    NBB_CUDA(cudaMemcpyAsync(&err, (const unsigned int*)p2p->d_sync + 2, sizeof(int), cudaMemcpyDeviceToHost,
                             (cudaStream_t)stream));
    NBB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    if (err) return fail(NBB_ERR_CUDA, "p2p: a step timed out waiting for the other ranks");
    return NBB_OK;
}

int nbb_gpu_malloc(int32_t device, uint64_t bytes, void** d_ptr) {
    if (!d_ptr) return fail(NBB_ERR_INVALID_ARGUMENT, "null output pointer");
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(device, &ctx));
    NBB_CUDA(cudaSetDevice(device));
    NBB_CUDA(cudaMalloc(d_ptr, bytes));
    NBB_CUDA(cudaMemset(*d_ptr, 0, bytes));
    return NBB_OK;
}

int nbb_gpu_free(int32_t device, void* d_ptr) {
    NBB_CUDA(cudaSetDevice(device));
    NBB_CUDA(cudaFree(d_ptr));
    return NBB_OK;
}

int nbb_gpu_ipc_handle(int32_t device, const void* d_ptr, uint8_t handle[64]) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    NBB_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    NBB_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
    std::memcpy(handle, &h, 64);
    return NBB_OK;
}

int nbb_gpu_ipc_open(int32_t device, const uint8_t handle[64], void** d_ptr) {
    NBB_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    NBB_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return NBB_OK;
}

int nbb_gpu_ipc_close(int32_t device, void* d_ptr) {
    NBB_CUDA(cudaSetDevice(device));
    NBB_CUDA(cudaIpcCloseMemHandle(d_ptr));
    return NBB_OK;
}

int nbb_gpu_reduction_compact_dev(const nbb_config* cfg, const void* d_compact, void* d_value, void* stream,
                                  nbb_report* report) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    NBB_CHECK(compact_workload_check(cfg));
    Segs sg;
    NBB_CHECK(compact_segments(cfg, &sg));
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    Timer t(cfg->timing != 0, (cudaStream_t)stream);
    NBB_CUDA(cudaMemsetAsync(d_value, 0, 8, (cudaStream_t)stream));
    segment_sum_kernel<<<ctx->sms * 4, 256, 0, (cudaStream_t)stream>>>((const long long*)d_compact, sg,
                                                                        (unsigned long long*)d_value);
    NBB_CUDA(cudaGetLastError());
    fill_report(cfg, report, t.stop_micros());
    return NBB_OK;
}

int nbb_gpu_single_write_compact_dev(const nbb_config* cfg, void* d_compact, void* stream, nbb_report* report) {
    if (!cfg) return fail(NBB_ERR_INVALID_ARGUMENT, "null config");
    NBB_CHECK(compact_workload_check(cfg));
    Segs sg;
    NBB_CHECK(compact_segments(cfg, &sg));
    DeviceCtx* ctx;
    NBB_CHECK(ensure_device(cfg->device, &ctx));
    Timer t(cfg->timing != 0, (cudaStream_t)stream);
    segment_fill_kernel<<<ctx->sms * 8, 256, 0, (cudaStream_t)stream>>>((long long*)d_compact, sg, 1);
    NBB_CUDA(cudaGetLastError());
    fill_report(cfg, report, t.stop_micros());
    return NBB_OK;
}

int nbb_gpu_release(void) {
    std::lock_guard<std::mutex> lock(g_mutex);
    for (size_t d = 0; d < g_ctx.size(); ++d) {
        DeviceCtx& c = g_ctx[d];
        if (!c.ready) continue;
        cudaSetDevice((int)d);
        for (int i = 0; i < 3; ++i) {
            if (c.bufs[i]) cudaFree(c.bufs[i]);
            c.bufs[i] = nullptr;
            c.buf_bytes[i] = 0;
        }
        for (auto& t : c.nbr_tab) {
            if (t) cudaFree(t);
            t = nullptr;
        }
    }
    return NBB_OK;
}

}  // extern "C"

#include "nbb_comm.inc"
