// probe_dram.cu — microbenchmark (not product): DRAM efficiency of the gasket's
// member-sector access pattern on the embedded int64 grid at n = 2^16.
//   traversal: (a) λ tile order, warp per 32x32 tile (the product's order)
//              (b) row-major over member sectors (max DRAM page locality)
//   load flavour: .nc.L1::no_allocate v8 / plain v8 / .nc v8 / 2 x v4
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_dram probe_dram.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct S8 { uint32_t w[8]; };

template <int F> __device__ __forceinline__ S8 ld(const void* p) {
    S8 r;
    if (F == 0) asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r.w[0]),"=r"(r.w[1]),"=r"(r.w[2]),"=r"(r.w[3]),"=r"(r.w[4]),"=r"(r.w[5]),"=r"(r.w[6]),"=r"(r.w[7]) : "l"(p));
    if (F == 1) asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r.w[0]),"=r"(r.w[1]),"=r"(r.w[2]),"=r"(r.w[3]),"=r"(r.w[4]),"=r"(r.w[5]),"=r"(r.w[6]),"=r"(r.w[7]) : "l"(p));
    if (F == 2) asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r.w[0]),"=r"(r.w[1]),"=r"(r.w[2]),"=r"(r.w[3]),"=r"(r.w[4]),"=r"(r.w[5]),"=r"(r.w[6]),"=r"(r.w[7]) : "l"(p));
    if (F == 3) {
        asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.w[0]),"=r"(r.w[1]),"=r"(r.w[2]),"=r"(r.w[3]) : "l"(p));
        asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.w[4]),"=r"(r.w[5]),"=r"(r.w[6]),"=r"(r.w[7]) : "l"((const char*)p + 16));
    }
    if (F == 4) asm volatile("ld.global.L1::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r.w[0]),"=r"(r.w[1]),"=r"(r.w[2]),"=r"(r.w[3]),"=r"(r.w[4]),"=r"(r.w[5]),"=r"(r.w[6]),"=r"(r.w[7]) : "l"(p));
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

// (a) λ tile order; MODE 0 read, 1 write, 2 read+write (copy src->dst)
template <int F, int MODE>
__global__ void __launch_bounds__(256) k_lambda(const long long* src, long long* dst, int64_t n, uint32_t tiles, uint32_t W, unsigned long long* out) {
    const int lane = threadIdx.x & 31;
    uint32_t row[4], sec[4], ok = 0;
    for (int k = 0; k < 4; ++k) {
        uint32_t e = k * 32 + lane, f = e, y = 0;
        for (y = 0; y < 32; ++y) { uint32_t c = 1u << __popc(y >> 2); if (f < c) break; f -= c; }
        if (e < 108) { ok |= 1u << k; row[k] = y; sec[k] = pdep(f, y >> 2); } else { row[k] = 0; sec[k] = 0; }
    }
    unsigned long long acc = 0;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = warp; t < tiles; t += nw) {
        uint32_t lx, ly; lam(t, W, lx, ly);
        const int64_t base = (int64_t)(ly * 32) * n + lx * 32;
        S8 v[4];
        if (MODE != 1) {
#pragma unroll
            for (int k = 0; k < 4; ++k) if (ok >> k & 1) v[k] = ld<F>(src + base + row[k] * n + sec[k] * 4);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) if (ok >> k & 1) {
            if (MODE == 0) acc += v[k].w[0] + v[k].w[3] + v[k].w[7];
            else { if (MODE == 1) for (int i = 0; i < 8; ++i) v[k].w[i] = i; st(dst + base + row[k] * n + sec[k] * 4, v[k]); }
        }
    }
    if (MODE == 0 && acc == 12345) out[0] = acc;
}

// (b) row-major member sectors: warp per row
template <int F, int MODE>
__global__ void __launch_bounds__(256) k_rows(const long long* src, long long* dst, int64_t n, unsigned long long* out) {
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    unsigned long long acc = 0;
    for (uint32_t y = warp; y < (uint32_t)n; y += nw) {
        const uint32_t m = y >> 2, cnt = 1u << __popc(m);
        for (uint32_t j = lane; j < cnt; j += 32) {
            const int64_t off = (int64_t)y * n + pdep(j, m) * 4;
            if (MODE == 0) { S8 v = ld<F>(src + off); acc += v.w[0] + v.w[3] + v.w[7]; }
            else if (MODE == 1) { S8 v; for (int i = 0; i < 8; ++i) v.w[i] = i; st(dst + off, v); }
            else { S8 v = ld<F>(src + off); st(dst + off, v); }
        }
    }
    if (acc == 12345) out[0] = acc;
}

__global__ void k_dense_read(const long long* src, size_t words, unsigned long long* out) {
    unsigned long long acc = 0;
    for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < words; i += (size_t)gridDim.x * blockDim.x * 4) {
        S8 v = ld<1>(src + i); acc += v.w[0];
    }
    if (acc == 12345) out[0] = acc;
}

template <class K>
float timeit(K k, int reps) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k(); cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) k();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    const int r = 16; const int64_t n = 1 << r;
    const size_t words = (size_t)n * n;
    long long *a, *b; unsigned long long* out;
    CK(cudaMalloc(&a, words * 8)); CK(cudaMalloc(&b, words * 8)); CK(cudaMalloc(&out, 8));
    CK(cudaMemset(a, 1, words * 8)); CK(cudaMemset(b, 0, words * 8));
    const uint32_t tiles = 177147, W = 729;
    const double B = 32.0 * 4 * 4782969;  // layout bytes per pass (19,131,876 sectors)
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 8;
    printf("dense read 32GiB: %.1f GB/s\n", words * 8 / (timeit([&] { k_dense_read<<<grid, 256>>>(a, words, out); }, 3) * 1e6));
#define RUN(name, launch, passes) { float ms = timeit([&] { launch; }, 10); printf("%-34s %8.3f ms  %7.1f GB/s (alg)\n", name, ms, passes * B / (ms * 1e6)); }
    RUN("lambda read nc.noalloc v8", (k_lambda<0, 0><<<grid, 256>>>(a, b, n, tiles, W, out)), 1);
    RUN("lambda read plain v8", (k_lambda<1, 0><<<grid, 256>>>(a, b, n, tiles, W, out)), 1);
    RUN("lambda read nc v8", (k_lambda<2, 0><<<grid, 256>>>(a, b, n, tiles, W, out)), 1);
    RUN("lambda read 2 x v4", (k_lambda<3, 0><<<grid, 256>>>(a, b, n, tiles, W, out)), 1);
    RUN("lambda read L1::evict_first v8", (k_lambda<4, 0><<<grid, 256>>>(a, b, n, tiles, W, out)), 1);
    RUN("lambda write v8", (k_lambda<1, 1><<<grid, 256>>>(a, b, n, tiles, W, out)), 1);
    RUN("lambda copy plain v8", (k_lambda<1, 2><<<grid, 256>>>(a, b, n, tiles, W, out)), 2);
    RUN("lambda copy nc.noalloc v8", (k_lambda<0, 2><<<grid, 256>>>(a, b, n, tiles, W, out)), 2);
    RUN("rows read nc.noalloc v8", (k_rows<0, 0><<<grid, 256>>>(a, b, n, out)), 1);
    RUN("rows read plain v8", (k_rows<1, 0><<<grid, 256>>>(a, b, n, out)), 1);
    RUN("rows write v8", (k_rows<1, 1><<<grid, 256>>>(a, b, n, out)), 1);
    RUN("rows copy plain v8", (k_rows<1, 2><<<grid, 256>>>(a, b, n, out)), 2);
    for (int g : {1, 2, 4, 16, 32}) {
        char nm[64]; snprintf(nm, 64, "lambda copy plain grid=%dxSM", g * 8 / 8);
        float ms = timeit([&] { k_lambda<1, 2><<<sms * g, 256>>>(a, b, n, tiles, W, out); }, 10);
        printf("%-34s %8.3f ms  %7.1f GB/s (alg)\n", nm, ms, 2 * B / (ms * 1e6));
    }
    CK(cudaGetLastError());
    return 0;
}
