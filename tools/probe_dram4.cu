// probe_dram4.cu — microbenchmark (not product): write forms for the gasket member pattern
// (int64, n = 2^16, λ tile order): sector vs full-line writes, cache hints, bulk (TMA) stores.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
struct S8 { uint32_t w[8]; };
__device__ __forceinline__ uint32_t pdep(uint32_t j, uint32_t m) {
    uint32_t r = 0;
    for (uint32_t bit = 1; m; m &= m - 1, bit <<= 1) if (j & bit) r |= m & (0u - m);
    return r;
}
__device__ void lam(uint32_t t, uint32_t W, uint32_t& lx, uint32_t& ly) {
    uint32_t ox = t % W, oy = t / W, X = 0, Y = 0;
    for (int j = 0; ox; ++j) { uint32_t d = ox % 3; ox /= 3; X |= (d == 2) << (2 * j); Y |= (d != 0) << (2 * j); }
    uint32_t X2 = 0, Y2 = 0;
    for (int j = 0; oy; ++j) { uint32_t d = oy % 3; oy /= 3; X2 |= (d == 2) << (2 * j); Y2 |= (d != 0) << (2 * j); }
    lx = X | (X2 << 1); ly = Y | (Y2 << 1);
}
template <int F> __device__ __forceinline__ void st(void* p, const S8& v) {
    if (F == 0) asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(v.w[0]),"r"(v.w[1]),"r"(v.w[2]),"r"(v.w[3]),"r"(v.w[4]),"r"(v.w[5]),"r"(v.w[6]),"r"(v.w[7]) : "memory");
    if (F == 1) asm volatile("st.global.cs.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(v.w[0]),"r"(v.w[1]),"r"(v.w[2]),"r"(v.w[3]),"r"(v.w[4]),"r"(v.w[5]),"r"(v.w[6]),"r"(v.w[7]) : "memory");
    if (F == 2) asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(v.w[0]),"r"(v.w[1]),"r"(v.w[2]),"r"(v.w[3]),"r"(v.w[4]),"r"(v.w[5]),"r"(v.w[6]),"r"(v.w[7]) : "memory");
    if (F == 3) asm volatile("st.global.L2::evict_last.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(v.w[0]),"r"(v.w[1]),"r"(v.w[2]),"r"(v.w[3]),"r"(v.w[4]),"r"(v.w[5]),"r"(v.w[6]),"r"(v.w[7]) : "memory");
    if (F == 4) asm volatile("st.global.wt.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.w[0]),"r"(v.w[1]),"r"(v.w[2]),"r"(v.w[3]) : "memory");
    if (F == 4) asm volatile("st.global.wt.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"((char*)p + 16), "r"(v.w[4]),"r"(v.w[5]),"r"(v.w[6]),"r"(v.w[7]) : "memory");
}

// G: 4 = member sectors, 16 = every sector of member 128 B lines, 32 = whole tile rows
template <int G, int F>
__global__ void __launch_bounds__(256) k_write(long long* dst, int64_t n, uint32_t tiles, uint32_t W) {
    constexpr int LOGG = G == 4 ? 2 : G == 16 ? 4 : 5;
    constexpr int SPG = G / 4;
    constexpr int NG = (G == 4) ? 108 : (G == 16) ? 48 : 32;
    constexpr int NS = NG * SPG, SLOTS = (NS + 31) / 32;
    const int lane = threadIdx.x & 31;
    uint32_t row[SLOTS], sec[SLOTS], ok = 0;
    for (int k = 0; k < SLOTS; ++k) {
        uint32_t e = k * 32 + lane, g = e / SPG, half = e % SPG, f = g, y = 0;
        for (y = 0; y < 32; ++y) { uint32_t c = 1u << __popc(y >> LOGG); if (f < c) break; f -= c; }
        if (e < NS) { ok |= 1u << k; row[k] = y; sec[k] = pdep(f, y >> LOGG) * SPG + half; } else { row[k] = 0; sec[k] = 0; }
    }
    S8 v; for (int i = 0; i < 8; ++i) v.w[i] = i;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = warp; t < tiles; t += nw) {
        uint32_t lx, ly; lam(t, W, lx, ly);
        const int64_t base = (int64_t)(ly * 32) * n + lx * 32;
#pragma unroll
        for (int k = 0; k < SLOTS; ++k) if (ok >> k & 1) st<F>(dst + base + row[k] * n + sec[k] * 4, v);
    }
}

// TMA bulk store: each lane stages its row's member run (contiguous sectors 0..span) in smem
// and issues cp.async.bulk.global.shared::cta for whole contiguous member-line runs of the row.
__global__ void __launch_bounds__(256) k_bulk(long long* dst, int64_t n, uint32_t tiles, uint32_t W) {
    __shared__ __align__(128) uint32_t buf[8][32][32];  // per warp: 32 rows x 128 B (reused)
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int i = 0; i < 32; ++i) buf[wib][lane][i] = i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t y = lane;
    const uint32_t lines = (y >> 4) ? 2 : 1;         // member 128 B lines in row y: l ⊆ (y >> 4)
    for (uint32_t t = warp; t < tiles; t += nw) {
        uint32_t lx, ly; lam(t, W, lx, ly);
        long long* rowp = dst + (int64_t)(ly * 32 + y) * n + lx * 32;
        const uint32_t s = (uint32_t)__cvta_generic_to_shared(&buf[wib][lane][0]);
        for (uint32_t l = 0; l < lines; ++l)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;" :: "l"(rowp + 16 * l), "r"(s) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class K> float timeit(K k, int reps) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k(); cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) k();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    const int64_t n = 1 << 16;
    const size_t words = (size_t)n * n;
    long long* b;
    CK(cudaMalloc(&b, words * 8));
    CK(cudaMemset(b, 0, words * 8));
    const uint32_t tiles = 177147, W = 729;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 8;
#define RUN(G, F, name, mb) { float ms = timeit([&] { k_write<G, F><<<grid, 256>>>(b, n, tiles, W); }, 5); printf("%-40s %8.3f ms  %7.1f GB/s (%d MB)\n", name, ms, mb / ms, (int)mb); }
    RUN(4, 0, "sector32 st.v8", 612.2); RUN(4, 1, "sector32 st.cs.v8", 612.2); RUN(4, 2, "sector32 st.noalloc.evict_first", 612.2);
    RUN(4, 3, "sector32 st.L2::evict_last", 612.2); RUN(4, 4, "sector32 st.wt 2xv4", 612.2);
    RUN(16, 0, "line128 st.v8 (zeros in non-member)", 1088.4); RUN(16, 1, "line128 st.cs.v8", 1088.4);
    RUN(32, 0, "row256 st.v8", 1451.2);
    { float ms = timeit([&] { k_bulk<<<grid, 256>>>(b, n, tiles, W); }, 5); printf("%-40s %8.3f ms  %7.1f GB/s (%d MB)\n", "line128 TMA bulk store", ms, 1088.4 / ms, 1088); }
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    return 0;
}
