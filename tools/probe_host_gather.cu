// Host-side probe for the e2e path at n = 2^16 (int64 embedded Grid, 32 GiB pinned):
//  (1) contiguous pinned cudaMemcpy H2D / D2H bandwidth (612 MB),
//  (2) multi-threaded CPU gather of the 19.1 M member sectors (32 B) into a contiguous pinned
//      staging buffer in tile order, and the matching scatter, for 1..T threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o probe_host_gather probe_host_gather.cu
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// X(v), Y(v) of SURVEY App. A.1 (bit 2j set iff base-3 digit j is 2 / >= 1)
static void xy(uint32_t v, uint32_t& X, uint32_t& Y) {
    X = Y = 0;
    for (int j = 0; v; ++j, v /= 3) {
        const uint32_t d = v % 3;
        X |= (d == 2u) << (2 * j);
        Y |= (d != 0u) << (2 * j);
    }
}

int main() {
    const int r = 16, rb = 11;
    const int64_t n = 1 << r;
    const uint32_t Wb = 729, Hb = 243, tiles = Wb * Hb;  // ρ = 32 tiles, block orthotope
    // 108 member sectors of a tile: (row y, sector s ⊆ y >> 2)
    std::vector<uint32_t> slot;
    for (uint32_t y = 0; y < 32; ++y)
        for (uint32_t s = 0; s < 8; ++s)
            if ((s & ~(y >> 2)) == 0) slot.push_back(y | s << 5);
    std::vector<int64_t> org(tiles);
    for (uint32_t u = 0; u < tiles; ++u) {
        const uint32_t wx = u % Wb, wy = u / Wb;
        uint32_t Xx, Yx, Xy, Yy;
        xy(wx, Xx, Yx);
        xy(wy, Xy, Yy);
        const int64_t bx = Xx | Xy << 1, by = Yx | Yy << 1;
        org[u] = by * 32 * n + bx * 32;
    }
    const size_t grid_bytes = (size_t)n * n * 8, stage_bytes = (size_t)tiles * slot.size() * 32;
    int64_t *grid, *stage, *dev;
    if (cudaHostAlloc((void**)&grid, grid_bytes, cudaHostAllocMapped) != cudaSuccess) return 1;
    cudaHostAlloc((void**)&stage, stage_bytes, 0);
    cudaMalloc((void**)&dev, stage_bytes);
    std::memset(grid, 1, grid_bytes);
    std::memset(stage, 0, stage_bytes);
    printf("{\"stage_MB\": %.1f", stage_bytes / 1e6);
    for (int rep = 0; rep < 2; ++rep) {
        double t0 = now();
        cudaMemcpy(dev, stage, stage_bytes, cudaMemcpyHostToDevice);
        double t1 = now();
        cudaMemcpy(stage, dev, stage_bytes, cudaMemcpyDeviceToHost);
        double t2 = now();
        if (rep) printf(", \"h2d_GBps\": %.1f, \"d2h_GBps\": %.1f", stage_bytes / (t1 - t0) / 1e9,
                        stage_bytes / (t2 - t1) / 1e9);
    }
    const int hw = (int)std::thread::hardware_concurrency();
    printf(", \"hw_threads\": %d", hw);
    for (int T : {1, 4, 8, hw, 2 * hw}) {
        for (int dir = 0; dir < 2; ++dir) {
            double best = 1e9;
            for (int rep = 0; rep < 2; ++rep) {
                std::atomic<uint32_t> next{0};
                const double t0 = now();
                std::vector<std::thread> th;
                for (int w = 0; w < T; ++w)
                    th.emplace_back([&] {
                        for (;;) {
                            const uint32_t u0 = next.fetch_add(256);
                            if (u0 >= tiles) break;
                            for (uint32_t u = u0; u < u0 + 256 && u < tiles; ++u) {
                                int64_t* st = stage + (size_t)u * slot.size() * 4;
                                for (size_t e = 0; e < slot.size(); ++e) {
                                    const uint32_t y = slot[e] & 31, s = slot[e] >> 5;
                                    int64_t* g = grid + org[u] + (int64_t)y * n + 4 * s;
                                    if (dir == 0) std::memcpy(st + 4 * e, g, 32);
                                    else std::memcpy(g, st + 4 * e, 32);
                                }
                            }
                        }
                    });
                for (auto& t : th) t.join();
                best = std::min(best, now() - t0);
            }
            printf(", \"%s_T%d_ms\": %.2f", dir ? "scatter" : "gather", T, best * 1e3);
        }
    }
    printf("}\n");
    return 0;
}
