// probe_zero_copy.cu — microbenchmark (not product): zero-copy reads of the gasket's member
// data from a pinned, mapped host int64 Grid at n = 2^16 (the e2e boundary of nbb_gpu_ca), at
// three request granularities over the same λ tile walk (warp per ρ = 32 tile):
//   sector : the 108 member sectors of a tile (32 B each; what the product reads)  612 MB
//   chunk  : the 72 64-byte chunks holding a member                                 816 MB
//   line   : the 48 128-byte lines holding a member                                1088 MB
// the member sectors in embedded row-major order (sequential host pages), the same two walks for
// zero-copy WRITES (the D2H side), and the contiguous DMA (cudaMemcpy) of 612 MB as the link
// reference. One JSON line.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o probe_zero_copy probe_zero_copy.cu
#include <cuda_runtime.h>

#include <sys/mman.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__constant__ uint32_t c_slot[128];  // per granularity: (row y, unit index) packed y | u << 5
__constant__ int c_units;           // units per tile

__device__ __forceinline__ void xy(uint32_t v, uint32_t& X, uint32_t& Y) {
    X = Y = 0;
    for (int j = 0; v; ++j) {
        const uint32_t q = v / 3u, d = v - 3u * q;
        X |= (uint32_t)(d == 2u) << (2 * j);
        Y |= (uint32_t)(d != 0u) << (2 * j);
        v = q;
    }
}

// UNIT_BYTES: 32, 64 or 128; each unit read as 32-byte vectors by UNIT_BYTES/32 lanes
template <int UNIT_BYTES>
__global__ void read_units(const long long* grid, int64_t n, uint32_t tiles, unsigned long long* sink) {
    constexpr int L = UNIT_BYTES / 32;  // lanes per unit
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t stride = (gridDim.x * blockDim.x) >> 5;
    unsigned long long acc = 0;
    for (uint32_t t = warp; t < tiles; t += stride) {
        uint32_t Xx, Yx, Xy, Yy;
        xy(t % 729u, Xx, Yx);
        xy(t / 729u, Xy, Yy);
        const int64_t org = (int64_t)(Yx | Yy << 1) * 32 * n + (int64_t)(Xx | Xy << 1) * 32;
        for (int e = lane; e < c_units * L; e += 32) {
            const uint32_t s = c_slot[e / L];
            const int64_t y = s & 31u, u = s >> 5;
            const long long* p = grid + org + y * n + u * (UNIT_BYTES / 8) + 4 * (e % L);
            uint32_t w[8];
            asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                           "=r"(w[6]), "=r"(w[7])
                         : "l"(p));
            acc += w[0] ^ w[3] ^ w[7];
        }
    }
    if (acc == 0x1234567ull) *sink = acc;
}

// member sectors in embedded row-major order: warp per row y, lanes walk the row's member
// sectors s ⊆ ~M (M = (n-1-y) >> 2) in increasing address order — sequential host pages
__device__ __forceinline__ uint64_t pdep64(uint64_t k, uint64_t mask) {
    uint64_t r = 0;
    for (uint64_t bit = 1; mask; mask &= mask - 1, bit <<= 1)
        if (k & bit) r |= mask & (0 - mask);
    return r;
}
__global__ void read_rows(const long long* grid, int64_t n, unsigned long long* sink) {
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t stride = (gridDim.x * blockDim.x) >> 5;
    unsigned long long acc = 0;
    for (int64_t y = warp; y < n; y += stride) {
        const uint64_t free_bits = ~((uint64_t)(n - 1 - y) >> 2) & (uint64_t)(n / 4 - 1);
        const uint64_t count = 1ull << __popcll(free_bits);
        for (uint64_t k = lane; k < count; k += 32) {
            const long long* p = grid + y * n + 4 * pdep64(k, free_bits);
            uint32_t w[8];
            asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]),
                           "=r"(w[6]), "=r"(w[7])
                         : "l"(p));
            acc += w[0] ^ w[3] ^ w[7];
        }
    }
    if (acc == 0x1234567ull) *sink = acc;
}

// the D2H direction: member sectors written zero-copy in λ tile order vs row-major order
__global__ void write_tiles(long long* grid, int64_t n, uint32_t tiles) {
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t stride = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = warp; t < tiles; t += stride) {
        uint32_t Xx, Yx, Xy, Yy;
        xy(t % 729u, Xx, Yx);
        xy(t / 729u, Xy, Yy);
        const int64_t org = (int64_t)(Yx | Yy << 1) * 32 * n + (int64_t)(Xx | Xy << 1) * 32;
        for (int e = lane; e < c_units; e += 32) {
            const uint32_t s = c_slot[e];
            long long* p = grid + org + (int64_t)(s & 31u) * n + 4 * (int64_t)(s >> 5);
            asm volatile("st.global.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(t) : "memory");
        }
    }
}
__global__ void write_rows(long long* grid, int64_t n) {
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t stride = (gridDim.x * blockDim.x) >> 5;
    for (int64_t y = warp; y < n; y += stride) {
        const uint64_t free_bits = ~((uint64_t)(n - 1 - y) >> 2) & (uint64_t)(n / 4 - 1);
        const uint64_t count = 1ull << __popcll(free_bits);
        for (uint64_t k = lane; k < count; k += 32) {
            long long* p = grid + y * n + 4 * pdep64(k, free_bits);
            asm volatile("st.global.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"((uint32_t)y) : "memory");
        }
    }
}

int main() {
    const int64_t n = 1 << 16;
    const uint32_t tiles = 729u * 243u;
    const size_t bytes = (size_t)n * n * 8;
    long long *h, *d;
    const bool huge = getenv("PROBE_HUGE") != nullptr;  // THP-backed mmap + cudaHostRegister
    if (huge) {
        void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (p == MAP_FAILED) return 1;
        madvise(p, bytes, MADV_HUGEPAGE);
        std::memset(p, 0, bytes);
        if (cudaHostRegister(p, bytes, cudaHostRegisterMapped) != cudaSuccess) return 2;
        h = (long long*)p;
    } else if (cudaHostAlloc((void**)&h, bytes,
                             cudaHostAllocMapped | (getenv("PROBE_WC") ? cudaHostAllocWriteCombined : 0u)) !=
               cudaSuccess) {
        return 1;
    }
    for (size_t i = 0; i < bytes / 8; i += 512) h[i] = (long long)i;
    cudaHostGetDevicePointer((void**)&d, h, 0);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("{\"host_alloc\": \"%s\", ", huge ? "mmap+MADV_HUGEPAGE+cudaHostRegister" : getenv("PROBE_WC") ? "cudaHostAlloc(WriteCombined)" : "cudaHostAlloc");
    const char* names[3] = {"sector", "chunk", "line"};
    for (int g = 0; g < 3; ++g) {
        const int unit = 32 << g, per_row = 256 / unit;  // units per 256-byte tile row
        std::vector<uint32_t> slots;
        for (uint32_t y = 0; y < 32; ++y)
            for (int u = 0; u < per_row; ++u) {
                bool member = false;  // some sector s of the unit with s ⊆ y >> 2
                for (int s = u * (unit / 32); s < (u + 1) * (unit / 32); ++s) member |= (s & ~(y >> 2)) == 0;
                if (member) slots.push_back(y | (uint32_t)u << 5);
            }
        const int units = (int)slots.size();
        cudaMemcpyToSymbol(c_slot, slots.data(), units * 4);
        cudaMemcpyToSymbol(c_units, &units, 4);
        float best = 1e9f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (g == 0) read_units<32><<<148 * 8, 256>>>(d, n, tiles, sink);
            if (g == 1) read_units<64><<<148 * 8, 256>>>(d, n, tiles, sink);
            if (g == 2) read_units<128><<<148 * 8, 256>>>(d, n, tiles, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double mb = (double)tiles * units * unit / 1e6;
        printf("%s\"%s\": {\"units_per_tile\": %d, \"MB\": %.1f, \"ms\": %.2f, \"GBps\": %.1f}", g ? ", " : "",
               names[g], units, mb, best, mb / best);
    }
    {
        float best2 = 1e9f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            read_rows<<<148 * 8, 256>>>(d, n, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best2) best2 = ms;
        }
        printf(", \"sector_rowmajor\": {\"MB\": 612.2, \"ms\": %.2f, \"GBps\": %.1f}", best2, 612.22 / best2);
    }
    {
        std::vector<uint32_t> slots;
        for (uint32_t y = 0; y < 32; ++y)
            for (uint32_t u = 0; u < 8; ++u)
                if ((u & ~(y >> 2)) == 0) slots.push_back(y | u << 5);
        const int units = (int)slots.size();
        cudaMemcpyToSymbol(c_slot, slots.data(), units * 4);
        cudaMemcpyToSymbol(c_units, &units, 4);
        for (int v = 0; v < 2; ++v) {
            float b = 1e9f;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                if (v == 0) write_tiles<<<148 * 8, 256>>>(d, n, tiles);
                else write_rows<<<148 * 8, 256>>>(d, n);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < b) b = ms;
            }
            printf(", \"%s\": {\"MB\": 612.2, \"ms\": %.2f, \"GBps\": %.1f}",
                   v ? "write_sector_rowmajor" : "write_sector_tiles", b, 612.22 / b);
        }
    }
    void* dd;
    cudaMalloc(&dd, 612220032);
    float best = 1e9f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        cudaMemcpy(dd, h, 612220032, cudaMemcpyHostToDevice);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    printf(", \"dma_612MB\": {\"ms\": %.2f, \"GBps\": %.1f}}\n", best, 612.22 / best);
    return 0;
}
