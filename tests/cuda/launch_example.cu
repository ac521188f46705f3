// The reference's launch(config, kernel) with device functors (include/nbb_launch.cuh):
// single write and reduction written as functors, run over the λ and BB launches.
//   launch_example <r> <rho> <lambda|bb> <seed>   -> "sw <fnv> rd <sum> blocks <b> active <a>"
//   launch_example --host-only                    -> exit 0 iff the launch fails loudly (no GPU)
#include <cstdio>
#include <cstring>
#include <vector>

#include "nbb_launch.cuh"

struct Write1 {  // run_single_write's kernel (dispatch.cpp:481-488)
    int64_t* g;
    int64_t n;
    __device__ void operator()(uint64_t, nbb::gpu::EmbeddedCoord c) const { g[c.y * n + c.x] = 1; }
};

struct Sum {  // run_reduction's per-cell accumulation (dispatch.cpp:490-515), int64 wrap-around
    const int64_t* g;
    int64_t n;
    unsigned long long* acc;
    __device__ void operator()(uint64_t, nbb::gpu::EmbeddedCoord c) const {
        atomicAdd(acc, (unsigned long long)g[c.y * n + c.x]);
    }
};

static uint64_t fnv1a64(const void* p, size_t bytes) {
    uint64_t h = 0xcbf29ce484222325ull;
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < bytes; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
    return h;
}

int main(int argc, char** argv) {
    nbb_config cfg;
    nbb_config_init(&cfg);
    if (argc > 1 && std::strcmp(argv[1], "--host-only") == 0) {
        cfg.r = 6;
        cfg.rho = 4;
        const int rc = nbb::gpu::launch(cfg, Write1{nullptr, 64});
        std::printf("launch without a device: rc=%d\n", rc);
        return rc == NBB_ERR_CUDA ? 0 : 1;
    }
    if (argc < 5) return 2;
    cfg.r = std::atoi(argv[1]);
    cfg.rho = std::atoi(argv[2]);
    cfg.mode = std::strcmp(argv[3], "bb") == 0 ? NBB_MODE_BB : NBB_MODE_LAMBDA;
    const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    const int64_t n = (int64_t)1 << cfg.r;
    cfg.max_cells = (uint64_t)(n * n);
    const size_t bytes = (size_t)(n * n) * 8;
    std::vector<int64_t> host((size_t)(n * n));
    if (nbb_gpu_random_member_grid(&cfg.spec, cfg.r, seed, 1000, (uint64_t)(n * n), host.data())) return 3;
    int64_t *d_sw, *d_in;
    unsigned long long* d_acc;
    cudaMalloc(&d_sw, bytes);
    cudaMalloc(&d_in, bytes);
    cudaMalloc(&d_acc, 8);
    cudaMemset(d_sw, 0, bytes);
    cudaMemset(d_acc, 0, 8);
    cudaMemcpy(d_in, host.data(), bytes, cudaMemcpyHostToDevice);
    nbb_report rep;
    if (nbb::gpu::launch(cfg, Write1{d_sw, n}, &rep)) return 4;
    if (nbb::gpu::launch(cfg, Sum{d_in, n, d_acc})) return 5;
    unsigned long long acc = 0;
    cudaMemcpy(host.data(), d_sw, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(&acc, d_acc, 8, cudaMemcpyDeviceToHost);
    if (cudaDeviceSynchronize() != cudaSuccess) return 6;
    std::printf("sw %016llx rd %lld blocks %llu active %llu\n",
                (unsigned long long)fnv1a64(host.data(), bytes), (long long)acc,
                (unsigned long long)rep.blocks_launched, (unsigned long long)rep.threads_active);
    return 0;
}
