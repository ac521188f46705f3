// Example reference-style program against the C++ shim (include/nbb_gpu.hpp).
// Compiled by tests/test_capi.py (CPU: --host-only) and run on the GPU by
// tests/test_gpu_parity.py::test_cpp_shim_on_gpu.
#include <cstdio>
#include <cstring>
#include <cstdint>
#include <numeric>
#include <vector>

#include "nbb_gpu.hpp"

int main(int argc, char** argv) {
    namespace g = nbb::gpu;
    const bool host_only = argc > 1 && std::strcmp(argv[1], "--host-only") == 0;
    g::DispatchConfig cfg;
    cfg.r = 8;
    std::printf("%s\n", g::WorkReport::csv_header().c_str());
    std::printf("%s\n", g::plan_report(cfg).csv_row().c_str());
    try {
        g::DispatchConfig bad = cfg;
        bad.rho = 3;
        bad.validate();
        return 1;
    } catch (const std::invalid_argument& e) {
        std::printf("invalid_argument: %s\n", e.what());
    }
    if (host_only) return 0;

    cfg.r = 10;
    cfg.rho = 32;
    const auto sw = g::run_single_write(cfg);
    const long long sum = std::accumulate(sw.grid.values().begin(), sw.grid.values().end(), 0LL);
    std::printf("sw sum %lld\n", sum);
    const auto rd_grid = g::random_member_grid(cfg.spec, 10, 11, 100);
    std::printf("rd %lld\n", (long long)g::run_reduction(cfg, rd_grid).value);
    const auto ca_grid = g::random_member_grid(cfg.spec, 10, 11, 2);
    const auto ca = g::run_ca(cfg, ca_grid, 10);
    const long long pop = std::accumulate(ca.grid.values().begin(), ca.grid.values().end(), 0LL);
    std::printf("ca pop %lld gen %llu reports %zu\n", pop, (unsigned long long)ca.grid.generation(),
                ca.reports.size());
    // n = 2^13: the default device state (compact, passes of up to 8 steps), the explicit compact
    // state with 3 steps per pass, and the embedded int64 grid; FNV-1a of each result, which the
    // test compares with the C oracle's trajectory
    g::DispatchConfig c13 = cfg;
    c13.r = 13;
    c13.max_cells = 1ull << 26;
    const auto init13 = g::random_member_grid(c13.spec, 13, 14, 2, c13.max_cells);
    auto fnv = [](const std::vector<std::int64_t>& v) {
        std::uint64_t h = 0xcbf29ce484222325ull;
        for (std::int64_t x : v)
            for (int b = 0; b < 8; ++b) {
                h ^= (std::uint64_t)((unsigned long long)x >> (8 * b)) & 0xFFu;
                h *= 0x100000001b3ull;
            }
        return h;
    };
    std::printf("ca13 default %016llx\n", (unsigned long long)fnv(g::run_ca(c13, init13, 20).grid.values()));
    c13.state = g::DispatchConfig::State::Compact;
    c13.pass_steps = 3;
    std::printf("ca13 compact3 %016llx\n", (unsigned long long)fnv(g::run_ca(c13, init13, 20).grid.values()));
    c13.state = g::DispatchConfig::State::Embedded;
    std::printf("ca13 embedded %016llx\n", (unsigned long long)fnv(g::run_ca(c13, init13, 20).grid.values()));
    // the reference's workers as devices: 3 workers (on device 0 when it is the only GPU)
    c13.state = g::DispatchConfig::State::Auto;
    c13.pass_steps = 0;
    int ndev = 0;
    g::check(nbb_gpu_device_count(&ndev));
    const std::vector<int> devs = {0, 1 % ndev, 2 % ndev};
    std::printf("ca13 workers %016llx\n",
                (unsigned long long)fnv(g::run_ca(c13, init13, 20, g::CaRule{}, devs).grid.values()));
    return (sum == 59049 && pop == 10398) ? 0 : 2;
}
