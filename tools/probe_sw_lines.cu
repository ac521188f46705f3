// probe_sw_lines.cu — microbenchmark (not product): the single-write payload on the embedded int64
// grid at n = 2^16 in λ tile order, warp per 32x32 tile: (a) the member sectors only (108 per
// tile, 612 MB: what tile_kernel<int64,32,SW> writes) vs (b) every 128-byte line holding a member
// (48 per tile, 1,088 MB, zeros in the non-member cells) — does DRAM take whole lines faster?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_sw_lines tools/probe_sw_lines.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void st8(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e, uint32_t f,
                                    uint32_t g, uint32_t h) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d), "r"(e),
                 "r"(f), "r"(g), "r"(h) : "memory");
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
// sector (y, s) of a tile: 4 cells x = 4s..4s+3, member iff x ⊆ y; value 1 / 0
__device__ __forceinline__ void put(char* tile, int64_t n, uint32_t y, uint32_t s) {
    uint32_t w[8];
    for (int c = 0; c < 4; ++c) {
        const uint32_t x = 4 * s + c;
        w[2 * c] = (x & ~y) == 0u ? 1u : 0u;
        w[2 * c + 1] = 0u;
    }
    st8(tile + ((int64_t)y * n + 4 * s) * 8, w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7]);
}
template <int LINES>
__global__ void __launch_bounds__(256) k_sw(long long* dst, int64_t n, uint32_t tiles, uint32_t W) {
    const int lane = threadIdx.x & 31;
    constexpr int SL = LINES ? 6 : 4;  // slots per lane: 192 or 108 sectors per tile
    uint32_t row[SL], sec[SL], ok = 0;
    for (int k = 0; k < SL; ++k) {
        const uint32_t e = k * 32 + lane;
        uint32_t y = 0, s = 0;
        bool v;
        if (LINES) {  // line l: rows 0..15 one line (sectors 0-3), rows 16..31 two (0-3, 4-7)
            const uint32_t l = e / 4, q = e % 4;
            v = e < 192;
            if (l < 16) { y = l; s = q; } else { y = 16 + (l - 16) / 2; s = ((l - 16) % 2) * 4 + q; }
        } else {
            uint32_t f = e;
            for (y = 0; y < 32; ++y) { const uint32_t c = 1u << __popc(y >> 2); if (f < c) break; f -= c; }
            v = e < 108;
            if (v) s = pdep(f, y >> 2);
        }
        row[k] = v ? y : 0; sec[k] = v ? s : 0; ok |= (v ? 1u : 0u) << k;
    }
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = warp; t < tiles; t += nw) {
        uint32_t lx, ly; lam(t, W, lx, ly);
        char* base = reinterpret_cast<char*>(dst) + ((int64_t)(ly * 32) * n + lx * 32) * 8;
        for (int k = 0; k < SL; ++k) if ((ok >> k) & 1u) put(base, n, row[k], sec[k]);
    }
}
int main() {
    const int r = 16; const int64_t n = 1 << r;
    uint32_t W = 1, H = 1; for (int i = 0; i < (r - 5 + 1) / 2; ++i) W *= 3; for (int i = 0; i < (r - 5) / 2; ++i) H *= 3;
    const uint32_t tiles = W * H;
    long long* d; CK(cudaMalloc(&d, (size_t)n * n * 8)); CK(cudaMemset(d, 0, (size_t)n * n * 8));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep)
        for (int lines = 0; lines < 2; ++lines)
            for (int g : {4, 8, 16}) {
                auto go = [&] { if (lines) k_sw<1><<<sms * g, 256>>>(d, n, tiles, W); else k_sw<0><<<sms * g, 256>>>(d, n, tiles, W); };
                go(); CK(cudaDeviceSynchronize());
                cudaEventRecord(e0); for (int i = 0; i < 10; ++i) go(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
                float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
                const double mb = lines ? 1088.4 : 612.2;
                printf("%s grid=%2dxSM  %.4f ms  %7.1f GB/s moved  (member sectors 612.2 MB: %7.1f GB/s)\n",
                       lines ? "lines  " : "sectors", g, ms, mb / ms, 612.2 / ms);
            }
    CK(cudaGetLastError());
    return 0;
}
