// probe_dram3.cu — microbenchmark (not product): which global-load forms fetch only the
// requested 32 B sectors (vs whole 128 B lines) for the gasket member-sector pattern.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

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

// sum of one 32 B sector via load form F
template <int F> __device__ __forceinline__ uint32_t ldsum(const void* p) {
    uint32_t a, b, c, d, e, f, g, h;
    const char* q = (const char*)p;
    if (F == 0) asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d),"=r"(e),"=r"(f),"=r"(g),"=r"(h) : "l"(q));
    if (F == 1) { asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d) : "l"(q)); asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(e),"=r"(f),"=r"(g),"=r"(h) : "l"(q + 16)); }
    if (F == 2) { asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d) : "l"(q)); asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(e),"=r"(f),"=r"(g),"=r"(h) : "l"(q + 16)); }
    if (F == 3) { asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d) : "l"(q)); asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(e),"=r"(f),"=r"(g),"=r"(h) : "l"(q + 16)); }
    if (F == 4) { asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d) : "l"(q)); asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(e),"=r"(f),"=r"(g),"=r"(h) : "l"(q + 16)); }
    if (F == 5) { asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d) : "l"(q)); asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(e),"=r"(f),"=r"(g),"=r"(h) : "l"(q + 16)); }
    if (F == 6) { asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(a),"=r"(b) : "l"(q)); asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(c),"=r"(d) : "l"(q+8)); asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(e),"=r"(f) : "l"(q+16)); asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(g),"=r"(h) : "l"(q+24)); }
    if (F == 7) asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d),"=r"(e),"=r"(f),"=r"(g),"=r"(h) : "l"(q));
    if (F == 8) asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d) : "l"(q)); if (F == 8 || F == 9) { e = f = g = h = 0; }
    if (F == 9) asm volatile("ld.global.lu.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a),"=r"(b),"=r"(c),"=r"(d) : "l"(q)); if (F == 8 || F == 9) { e = f = g = h = 0; }
    return a + b + c + d + e + f + g + h;
}

template <int F>
__global__ void __launch_bounds__(256) k_read(const long long* src, int64_t n, uint32_t tiles, uint32_t W, unsigned long long* out) {
    const int lane = threadIdx.x & 31;
    uint32_t row[4], sec[4], ok = 0;
    for (int k = 0; k < 4; ++k) {
        uint32_t e = k * 32 + lane, f = e, y = 0;
        for (y = 0; y < 32; ++y) { uint32_t c = 1u << __popc(y >> 2); if (f < c) break; f -= c; }
        if (e < 108) { ok |= 1u << k; row[k] = y; sec[k] = pdep(f, y >> 2); } else { row[k] = 0; sec[k] = 0; }
    }
    uint32_t acc = 0;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = warp; t < tiles; t += nw) {
        uint32_t lx, ly; lam(t, W, lx, ly);
        const int64_t base = (int64_t)(ly * 32) * n + lx * 32;
#pragma unroll
        for (int k = 0; k < 4; ++k) if (ok >> k & 1) acc += ldsum<F>(src + base + row[k] * n + sec[k] * 4);
    }
    if (acc == 12345) out[0] = acc;
}

// cp.async.cg 16 B x2 into a per-warp smem ring, then sum from smem
__global__ void __launch_bounds__(256) k_cpasync(const long long* src, int64_t n, uint32_t tiles, uint32_t W, unsigned long long* out) {
    __shared__ __align__(16) uint32_t buf[8][4][32][8];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t row[4], sec[4], ok = 0;
    for (int k = 0; k < 4; ++k) {
        uint32_t e = k * 32 + lane, f = e, y = 0;
        for (y = 0; y < 32; ++y) { uint32_t c = 1u << __popc(y >> 2); if (f < c) break; f -= c; }
        if (e < 108) { ok |= 1u << k; row[k] = y; sec[k] = pdep(f, y >> 2); } else { row[k] = 0; sec[k] = 0; }
    }
    uint32_t acc = 0;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = warp; t < tiles; t += nw) {
        uint32_t lx, ly; lam(t, W, lx, ly);
        const int64_t base = (int64_t)(ly * 32) * n + lx * 32;
#pragma unroll
        for (int k = 0; k < 4; ++k) if (ok >> k & 1) {
            const char* g = (const char*)(src + base + row[k] * n + sec[k] * 4);
            uint32_t s = (uint32_t)__cvta_generic_to_shared(&buf[wib][k][lane][0]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s), "l"(g));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s + 16), "l"(g + 16));
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
        for (int k = 0; k < 4; ++k) if (ok >> k & 1) acc += buf[wib][k][lane][0] + buf[wib][k][lane][7];
    }
    if (acc == 12345) out[0] = acc;
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
    long long* a; unsigned long long* out;
    CK(cudaMalloc(&a, words * 8)); CK(cudaMalloc(&out, 8));
    CK(cudaMemset(a, 1, words * 8));
    const uint32_t tiles = 177147, W = 729;
    const double B32 = 32.0 * 4 * 4782969;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 8;
#define RUN(F, name) { float ms = timeit([&] { k_read<F><<<grid, 256>>>(a, n, tiles, W, out); }, 5); printf("%-36s %8.3f ms %7.1f GB/s\n", name, ms, B32 / (ms * 1e6)); }
    RUN(0, "v8 default"); RUN(1, "2 x v4 default"); RUN(2, "2 x v4 .cg"); RUN(3, "2 x v4 .cs");
    RUN(4, "2 x v4 .cv"); RUN(5, "2 x v4 relaxed.gpu"); RUN(6, "4 x v2 default");
    RUN(7, "v8 L1::no_allocate.L2::evict_first"); RUN(8, "v4 volatile (half sector)"); RUN(9, "v4 .lu (half sector)");
    { float ms = timeit([&] { k_cpasync<<<grid, 256>>>(a, n, tiles, W, out); }, 5); printf("%-36s %8.3f ms %7.1f GB/s\n", "cp.async.cg 2 x 16B", ms, B32 / (ms * 1e6)); }
    CK(cudaGetLastError());
    return 0;
}
