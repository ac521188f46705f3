// probe_dram2.cu — microbenchmark (not product): 32 B sectors vs 64 B atoms for the
// gasket member pattern (int64, n = 2^16, λ tile order), and cudaLimitMaxL2FetchGranularity.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
struct S8 { uint32_t w[8]; };
__device__ __forceinline__ S8 ld(const void* p) {
    S8 r;
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r.w[0]),"=r"(r.w[1]),"=r"(r.w[2]),"=r"(r.w[3]),"=r"(r.w[4]),"=r"(r.w[5]),"=r"(r.w[6]),"=r"(r.w[7]) : "l"(p));
    return r;
}
__device__ __forceinline__ void st(void* p, const S8& v) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(v.w[0]),"r"(v.w[1]),"r"(v.w[2]),"r"(v.w[3]),"r"(v.w[4]),"r"(v.w[5]),"r"(v.w[6]),"r"(v.w[7]) : "memory");
}
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

// G = cells per access group (4: 32 B sectors, 8: 64 B atoms, 32: 256 B rows); sectors
// of every member group are moved (a group of 8 cells = 2 sectors = one 64 B atom).
// MODE 0 read, 1 write, 2 copy
template <int G, int MODE>
__global__ void __launch_bounds__(256) k_tile(const long long* src, long long* dst, int64_t n, uint32_t tiles, uint32_t W, unsigned long long* out) {
    constexpr int LOGG = G == 4 ? 2 : G == 8 ? 3 : 5;
    constexpr int SPG = G / 4;                      // sectors per group
    constexpr int NG = (G == 4) ? 108 : (G == 8) ? 72 : 32;  // member groups per tile
    constexpr int NS = NG * SPG;                    // sectors per tile
    constexpr int SLOTS = (NS + 31) / 32;
    const int lane = threadIdx.x & 31;
    uint32_t row[SLOTS], sec[SLOTS], ok = 0;
    for (int k = 0; k < SLOTS; ++k) {
        uint32_t e = k * 32 + lane, g = e / SPG, half = e % SPG, f = g, y = 0;
        for (y = 0; y < 32; ++y) { uint32_t c = 1u << __popc(y >> LOGG); if (f < c) break; f -= c; }
        if (e < NS) { ok |= 1u << k; row[k] = y; sec[k] = pdep(f, y >> LOGG) * SPG + half; } else { row[k] = 0; sec[k] = 0; }
    }
    unsigned long long acc = 0;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = warp; t < tiles; t += nw) {
        uint32_t lx, ly; lam(t, W, lx, ly);
        const int64_t base = (int64_t)(ly * 32) * n + lx * 32;
        S8 v[SLOTS];
        if (MODE != 1) {
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) if (ok >> k & 1) v[k] = ld(src + base + row[k] * n + sec[k] * 4);
        }
#pragma unroll
        for (int k = 0; k < SLOTS; ++k) if (ok >> k & 1) {
            if (MODE == 0) acc += v[k].w[0] + v[k].w[3] + v[k].w[7];
            else { if (MODE == 1) for (int i = 0; i < 8; ++i) v[k].w[i] = i; st(dst + base + row[k] * n + sec[k] * 4, v[k]); }
        }
    }
    if (MODE == 0 && acc == 12345) out[0] = acc;
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

int main(int argc, char** argv) {
    const int64_t n = 1 << 16;
    const size_t words = (size_t)n * n;
    long long *a, *b; unsigned long long* out;
    CK(cudaMalloc(&a, words * 8)); CK(cudaMalloc(&b, words * 8)); CK(cudaMalloc(&out, 8));
    CK(cudaMemset(a, 1, words * 8)); CK(cudaMemset(b, 0, words * 8));
    const uint32_t tiles = 177147, W = 729;
    const double B32 = 32.0 * 4 * 4782969;   // 32 B-sector layout bytes per pass
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 8;
    for (int gran : {0, 32, 64, 128}) {
        if (gran) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran));
        size_t cur = 0; cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity);
        printf("--- L2 fetch granularity limit = %zu\n", cur);
#define RUN(name, launch, passes) { float ms = timeit([&] { launch; }, 10); printf("%-28s %8.3f ms  %7.1f GB/s vs 32B-layout bytes\n", name, ms, passes * B32 / (ms * 1e6)); }
        RUN("sector32 read", (k_tile<4, 0><<<grid, 256>>>(a, b, n, tiles, W, out)), 1);
        RUN("sector32 write", (k_tile<4, 1><<<grid, 256>>>(a, b, n, tiles, W, out)), 1);
        RUN("sector32 copy", (k_tile<4, 2><<<grid, 256>>>(a, b, n, tiles, W, out)), 2);
        RUN("atom64 read", (k_tile<8, 0><<<grid, 256>>>(a, b, n, tiles, W, out)), 1);
        RUN("atom64 write", (k_tile<8, 1><<<grid, 256>>>(a, b, n, tiles, W, out)), 1);
        RUN("atom64 copy", (k_tile<8, 2><<<grid, 256>>>(a, b, n, tiles, W, out)), 2);
        RUN("row256 copy", (k_tile<32, 2><<<grid, 256>>>(a, b, n, tiles, W, out)), 2);
    }
    CK(cudaGetLastError());
    return 0;
}
