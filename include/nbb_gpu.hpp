// nbb_gpu.hpp — header-only C++ shim over the C ABI (nbb_gpu.h) that re-exposes
// the reference's public API (/root/reference/proj/include/nbb/dispatch.hpp,
// fractal.hpp) in namespace nbb::gpu with the same signatures and exception
// types, so a reference user switches by changing the namespace:
//
//   nbb::DispatchConfig / run_single_write / run_reduction / run_ca / ...
//   -> nbb::gpu::DispatchConfig / run_single_write / run_reduction / run_ca / ...
//
// Status codes are rethrown as the reference's exception types
// (std::invalid_argument, std::out_of_range, nbb::gpu::ResourceError,
// std::domain_error, std::overflow_error, std::runtime_error).
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "nbb_gpu.h"

namespace nbb::gpu {

class ResourceError : public std::runtime_error {  // fractal.hpp:16-19
public:
    using std::runtime_error::runtime_error;
};

class CudaError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == NBB_OK) return;
    const std::string msg = nbb_gpu_last_error();
    switch (rc) {
        case NBB_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case NBB_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        case NBB_ERR_RESOURCE: throw ResourceError(msg);
        case NBB_ERR_DOMAIN: throw std::domain_error(msg);
        case NBB_ERR_OVERFLOW: throw std::overflow_error(msg);
        case NBB_ERR_CUDA:
        case NBB_ERR_NCCL: throw CudaError(msg);
        default: throw std::runtime_error(msg);
    }
}

enum class MapMode { BoundingBox = NBB_MODE_BB, Lambda = NBB_MODE_LAMBDA };
enum class LambdaBackend {
    Direct = NBB_BACKEND_DIRECT,
    MmaV1 = NBB_BACKEND_MMA1,
    MmaV2 = NBB_BACKEND_MMA2,
    MmaV3 = NBB_BACKEND_MMA3
};
enum class IntraBlockStrategy {
    FurtherUnrolling = NBB_STRATEGY_UNROLL,
    SharedLookupTable = NBB_STRATEGY_LUT,
    BoundingSubBoxes = NBB_STRATEGY_SUBBOX
};

inline constexpr std::uint64_t kEnumerateBudget = std::uint64_t{1} << 24;

class FractalSpec {  // fractal.hpp:53-102 (the shipped built-ins)
public:
    static FractalSpec sierpinski() { FractalSpec f; nbb_spec_sierpinski(&f.c_); return f; }
    static FractalSpec vicsek() { FractalSpec f; nbb_spec_vicsek(&f.c_); return f; }
    static FractalSpec carpet() { FractalSpec f; nbb_spec_carpet(&f.c_); return f; }
    std::string name() const { return c_.name; }
    int replica_count() const { return c_.k; }
    int scale_factor() const { return c_.s; }
    std::int64_t side_length(int level) const {
        if (level < 0) throw std::invalid_argument("checked_pow: negative exponent");
        std::int64_t v = 1;
        for (int i = 0; i < level; ++i) v *= c_.s;
        return v;
    }
    std::uint64_t volume(int level) const {
        std::uint64_t v = 1;
        for (int i = 0; i < level; ++i) v *= (std::uint64_t)c_.k;
        return v;
    }
    const nbb_spec& c() const { return c_; }

private:
    nbb_spec c_{};
};

struct DispatchConfig {  // dispatch.hpp:25-38
    FractalSpec spec = FractalSpec::sierpinski();
    int r = 0;
    int rho = 1;
    MapMode mode = MapMode::Lambda;
    IntraBlockStrategy strategy = IntraBlockStrategy::BoundingSubBoxes;
    LambdaBackend backend = LambdaBackend::Direct;
    int workers = 1;
    bool timing = false;
    std::uint64_t max_cells = kEnumerateBudget;
    int cell_width = 8;  // device-side extensions
    int kernel = NBB_KERNEL_AUTO;
    int device = 0;
    // Device state of run_ca (nbb_gpu.h): Auto = the compact (λ-ordered) state whenever it
    // serves the call, Compact = require it, Embedded = the reference's n x n layout.
    enum class State { Auto, Compact, Embedded } state = State::Auto;
    std::uint32_t flags = 0;       // further NBB_FLAG_* (e.g. NBB_FLAG_OUT_ZEROED)
    std::uint32_t pass_steps = 0;  // compact state: steps per pass, 1..12 (0 = 8; > 8: cluster walk only)

    nbb_config c() const {
        nbb_config out;
        nbb_config_init(&out);
        out.spec = spec.c();
        out.r = r;
        out.rho = rho;
        out.mode = (int)mode;
        out.strategy = (int)strategy;
        out.backend = (int)backend;
        out.workers = workers;
        out.timing = timing ? 1 : 0;
        out.max_cells = max_cells;
        out.cell_width = cell_width;
        out.kernel = kernel;
        out.device = device;
        out.flags = flags | (state == State::Compact ? NBB_FLAG_COMPACT_STATE : 0u) |
                    (state == State::Embedded ? NBB_FLAG_EMBEDDED_STATE : 0u);
        out.pass_steps = pass_steps;
        return out;
    }
    void validate() const {
        const nbb_config cc = c();
        check(nbb_gpu_validate(&cc));
    }
};

struct WorkReport {  // dispatch.hpp:44-61
    nbb_report c{};
    static std::string csv_header() { return nbb_gpu_csv_header(); }
    std::string csv_row() const {
        char buf[512];
        check(nbb_gpu_report_csv_row(&c, buf, sizeof buf));
        return buf;
    }
};

class Grid {  // dispatch.hpp:65-93
public:
    Grid(const FractalSpec& spec, int r) : r_(r), n_(spec.side_length(r)) {
        values_.assign((std::size_t)n_ * (std::size_t)n_, 0);
    }
    int level() const { return r_; }
    std::int64_t side() const { return n_; }
    std::uint64_t generation() const { return generation_; }
    void bump_generation() { ++generation_; }
    std::int64_t& at(std::int64_t x, std::int64_t y) { return values_[(std::size_t)(y * n_ + x)]; }
    std::int64_t at(std::int64_t x, std::int64_t y) const { return values_[(std::size_t)(y * n_ + x)]; }
    const std::vector<std::int64_t>& values() const { return values_; }
    std::vector<std::int64_t>& values() { return values_; }
    bool operator==(const Grid& o) const { return r_ == o.r_ && n_ == o.n_ && values_ == o.values_; }
    void set_generation(std::uint64_t g) { generation_ = g; }

private:
    int r_ = 0;
    std::int64_t n_ = 1;
    std::uint64_t generation_ = 0;
    std::vector<std::int64_t> values_;
};

inline Grid random_member_grid(const FractalSpec& spec, int r, std::uint64_t seed,
                               std::uint64_t modulus, std::uint64_t max_cells = kEnumerateBudget) {
    Grid g(spec, r);
    check(nbb_gpu_random_member_grid(&spec.c(), r, seed, modulus, max_cells, g.values().data()));
    return g;
}

inline std::uint64_t launch_block_count(const DispatchConfig& config) {
    const nbb_config c = config.c();
    std::uint64_t b = 0;
    check(nbb_gpu_launch_block_count(&c, &b));
    return b;
}

struct SingleWriteResult {
    Grid grid;
    WorkReport report;
};
inline SingleWriteResult run_single_write(const DispatchConfig& config) {
    SingleWriteResult res{Grid(config.spec, config.r), {}};
    const nbb_config c = config.c();
    check(nbb_gpu_single_write(&c, res.grid.values().data(), &res.report.c));
    return res;
}

struct ReductionResult {
    std::int64_t value = 0;
    WorkReport report;
};
inline ReductionResult run_reduction(const DispatchConfig& config, const Grid& grid) {
    ReductionResult res;
    const nbb_config c = config.c();
    check(nbb_gpu_reduction(&c, grid.values().data(), grid.level(), &res.value, &res.report.c));
    return res;
}

struct CaRule {  // dispatch.hpp:131-134
    std::uint16_t birth = 1u << 3;
    std::uint16_t survive = (1u << 2) | (1u << 3);
};
struct CaResult {
    Grid grid;
    std::vector<WorkReport> reports;
};
inline CaResult run_ca(const DispatchConfig& config, const Grid& initial, int steps,
                       CaRule rule = CaRule{}) {
    CaResult res{initial, {}};
    const nbb_config c = config.c();
    std::vector<nbb_report> reps((std::size_t)(steps > 0 ? steps : 0));
    check(nbb_gpu_ca(&c, initial.values().data(), initial.level(), steps, rule.birth, rule.survive,
                     res.grid.values().data(), reps.empty() ? nullptr : reps.data()));
    for (const auto& r : reps) res.reports.push_back(WorkReport{r});
    res.grid.set_generation(initial.generation() + (std::uint64_t)(steps > 0 ? steps : 0));
    return res;
}

// The reference's `workers` as devices of this process (nbb_gpu_ca_multi): contiguous chunks of
// the compact tile range, halos over peer memory; byte-identical for any device list.
inline CaResult run_ca(const DispatchConfig& config, const Grid& initial, int steps, CaRule rule,
                       const std::vector<int>& devices) {
    CaResult res{initial, {}};
    const nbb_config c = config.c();
    std::vector<std::int32_t> devs(devices.begin(), devices.end());
    std::vector<nbb_report> reps((std::size_t)(steps > 0 ? steps : 0));
    check(nbb_gpu_ca_multi(&c, devs.data(), (std::int32_t)devs.size(), initial.values().data(), initial.level(),
                           steps, rule.birth, rule.survive, res.grid.values().data(),
                           reps.empty() ? nullptr : reps.data()));
    for (const auto& r : reps) res.reports.push_back(WorkReport{r});
    res.grid.set_generation(initial.generation() + (std::uint64_t)(steps > 0 ? steps : 0));
    return res;
}
inline ReductionResult run_reduction(const DispatchConfig& config, const Grid& grid, const std::vector<int>& devices) {
    ReductionResult res;
    const nbb_config c = config.c();
    std::vector<std::int32_t> devs(devices.begin(), devices.end());
    check(nbb_gpu_reduction_multi(&c, devs.data(), (std::int32_t)devs.size(), grid.values().data(), grid.level(),
                                  &res.value, &res.report.c));
    return res;
}

inline double work_quotient(const WorkReport& bounding_box, const WorkReport& lambda,
                            bool weighted = false) {
    double q = 0;
    check(nbb_gpu_work_quotient(&bounding_box.c, &lambda.c, weighted ? 1 : 0, &q));
    return q;
}

inline WorkReport plan_report(const DispatchConfig& config) {
    WorkReport w;
    const nbb_config c = config.c();
    check(nbb_gpu_plan_report(&c, &w.c));
    return w;
}

}  // namespace nbb::gpu
