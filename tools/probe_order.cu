// probe_order.cu — microbenchmark (not product): member-sector copy of the int64 gasket
// (n = 2^16, ρ = 32 tiles) with the member tiles visited in different orders:
//   lambda : ordinal order of the λ orthotope (the product's order)
//   band   : embedded row-major order of member tiles (by-major, bx-minor)
//   random : a fixed random permutation
// The tile list is precomputed on the host; each warp copies one tile's 108 sectors.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
struct S8 { uint32_t w[8]; };
__device__ __forceinline__ S8 ld(const void* p) {
    S8 r;
    asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r.w[0]),"=r"(r.w[1]),"=r"(r.w[2]),"=r"(r.w[3]),"=r"(r.w[4]),"=r"(r.w[5]),"=r"(r.w[6]),"=r"(r.w[7]) : "l"(p));
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
__global__ void __launch_bounds__(256) k_copy(const long long* src, long long* dst, int64_t n, const uint2* tiles, uint32_t ntiles) {
    const int lane = threadIdx.x & 31;
    uint32_t row[4], sec[4], ok = 0;
    for (int k = 0; k < 4; ++k) {
        uint32_t e = k * 32 + lane, f = e, y = 0;
        for (y = 0; y < 32; ++y) { uint32_t c = 1u << __popc(y >> 2); if (f < c) break; f -= c; }
        if (e < 108) { ok |= 1u << k; row[k] = y; sec[k] = pdep(f, y >> 2); } else { row[k] = 0; sec[k] = 0; }
    }
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = warp; t < ntiles; t += nw) {
        const uint2 b = tiles[t];
        const int64_t base = (int64_t)(b.y * 32) * n + b.x * 32;
        S8 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) if (ok >> k & 1) v[k] = ld(src + base + row[k] * n + sec[k] * 4);
#pragma unroll
        for (int k = 0; k < 4; ++k) if (ok >> k & 1) st(dst + base + row[k] * n + sec[k] * 4, v[k]);
    }
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

static void lam(uint32_t t, uint32_t W, uint32_t& lx, uint32_t& ly) {
    uint32_t ox = t % W, oy = t / W, X = 0, Y = 0, X2 = 0, Y2 = 0;
    for (int j = 0; ox; ++j) { uint32_t d = ox % 3; ox /= 3; X |= (d == 2) << (2 * j); Y |= (d != 0) << (2 * j); }
    for (int j = 0; oy; ++j) { uint32_t d = oy % 3; oy /= 3; X2 |= (d == 2) << (2 * j); Y2 |= (d != 0) << (2 * j); }
    lx = X | (X2 << 1); ly = Y | (Y2 << 1);
}

int main() {
    const int64_t n = 1 << 16;
    const size_t words = (size_t)n * n;
    long long *a, *b;
    CK(cudaMalloc(&a, words * 8)); CK(cudaMalloc(&b, words * 8));
    CK(cudaMemset(a, 1, words * 8)); CK(cudaMemset(b, 0, words * 8));
    const uint32_t T = 177147, W = 729;
    std::vector<uint2> lam_order(T), band(T), rnd;
    for (uint32_t t = 0; t < T; ++t) { uint32_t x, y; lam(t, W, x, y); lam_order[t] = make_uint2(x, y); }
    band = lam_order;
    std::sort(band.begin(), band.end(), [](uint2 p, uint2 q) { return p.y != q.y ? p.y < q.y : p.x < q.x; });
    rnd = lam_order;
    std::shuffle(rnd.begin(), rnd.end(), std::mt19937(7));
    // "column" order: bx-major
    std::vector<uint2> col = lam_order;
    std::sort(col.begin(), col.end(), [](uint2 p, uint2 q) { return p.x != q.x ? p.x < q.x : p.y < q.y; });
    uint2* d_t;
    CK(cudaMalloc(&d_t, T * sizeof(uint2)));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double B = 2.0 * 32 * 4 * 4782969;
    struct { const char* name; std::vector<uint2>* v; } cases[] = {{"lambda", &lam_order}, {"band (row-major)", &band}, {"column-major", &col}, {"random", &rnd}};
    for (auto& c : cases) {
        CK(cudaMemcpy(d_t, c.v->data(), T * sizeof(uint2), cudaMemcpyHostToDevice));
        for (int g : {4, 8, 16}) {
            float ms = timeit([&] { k_copy<<<sms * g, 256>>>(a, b, n, d_t, T); }, 10);
            printf("%-18s grid=%2dxSM  %7.3f ms  %7.1f GB/s alg\n", c.name, g, ms, B / (ms * 1e6));
        }
    }
    CK(cudaGetLastError());
    return 0;
}
