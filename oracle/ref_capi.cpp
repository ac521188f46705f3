// ref_capi.cpp — TEST INFRASTRUCTURE ONLY (checker / CPU baseline, never product).
//
// A thin extern "C" wrapper over the UNMODIFIED reference library built from
// /root/reference/proj/src/{fractal,block_map,mma,dispatch}.cpp by
// oracle/Makefile into oracle/_ref/libnbbref.so. It exists so that pytest (via
// ctypes) and bench.py's reference arm can call the reference's own entry points
// with the same nbb_config / nbb_report PODs the product C ABI uses
// (include/nbb_gpu.h). Nothing here re-implements reference logic: every call
// forwards to nbb::run_single_write / run_reduction / run_ca / lambda_map /
// map_thread / encode_variant* / compact_store ... (dispatch.hpp:111-148,
// block_map.hpp:25-132, mma.hpp:16-76).
#include <chrono>
#include <cstring>
#include <fstream>
#include <new>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "nbb/block_map.hpp"
#include "nbb/dispatch.hpp"
#include "nbb/fractal.hpp"
#include "nbb/mma.hpp"
#include "nbb_gpu.h"

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return NBB_OK;
    } catch (const nbb::ResourceError& e) {
        g_error = e.what();
        return NBB_ERR_RESOURCE;
    } catch (const std::bad_alloc& e) {
        g_error = e.what();
        return NBB_ERR_RESOURCE;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return NBB_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_error = e.what();
        return NBB_ERR_OUT_OF_RANGE;
    } catch (const std::domain_error& e) {
        g_error = e.what();
        return NBB_ERR_DOMAIN;
    } catch (const std::overflow_error& e) {
        g_error = e.what();
        return NBB_ERR_OVERFLOW;
    } catch (const std::exception& e) {
        g_error = e.what();
        return NBB_ERR_RUNTIME;
    }
}

nbb::FractalSpec to_spec(const nbb_spec& s) {
    std::vector<nbb::ReplicaOffset> offs;
    for (int i = 0; i < s.k && i < NBB_MAX_REPLICAS; ++i) {
        offs.push_back({s.offset_x[i], s.offset_y[i]});
    }
    return nbb::FractalSpec(std::string(s.name), s.k, s.s, offs);
}

nbb::DispatchConfig to_config(const nbb_config& c) {
    nbb::DispatchConfig d;
    d.spec = to_spec(c.spec);
    d.r = c.r;
    d.rho = c.rho;
    d.mode = c.mode == NBB_MODE_BB ? nbb::MapMode::BoundingBox : nbb::MapMode::Lambda;
    switch (c.strategy) {
        case NBB_STRATEGY_UNROLL: d.strategy = nbb::IntraBlockStrategy::FurtherUnrolling; break;
        case NBB_STRATEGY_LUT: d.strategy = nbb::IntraBlockStrategy::SharedLookupTable; break;
        default: d.strategy = nbb::IntraBlockStrategy::BoundingSubBoxes; break;
    }
    switch (c.backend) {
        case NBB_BACKEND_MMA1: d.backend = nbb::LambdaBackend::MmaV1; break;
        case NBB_BACKEND_MMA2: d.backend = nbb::LambdaBackend::MmaV2; break;
        case NBB_BACKEND_MMA3: d.backend = nbb::LambdaBackend::MmaV3; break;
        default: d.backend = nbb::LambdaBackend::Direct; break;
    }
    d.workers = c.workers;
    d.timing = c.timing != 0;
    d.max_cells = c.max_cells;
    return d;
}

void from_report(const nbb::WorkReport& w, nbb_report* out) {
    if (out == nullptr) return;
    std::memset(out, 0, sizeof(*out));
    std::strncpy(out->spec_name, w.spec_name.c_str(), sizeof(out->spec_name) - 1);
    out->r = w.r;
    out->rho = w.rho;
    out->mode = w.mode == nbb::MapMode::BoundingBox ? NBB_MODE_BB : NBB_MODE_LAMBDA;
    switch (w.strategy) {
        case nbb::IntraBlockStrategy::FurtherUnrolling: out->strategy = NBB_STRATEGY_UNROLL; break;
        case nbb::IntraBlockStrategy::SharedLookupTable: out->strategy = NBB_STRATEGY_LUT; break;
        case nbb::IntraBlockStrategy::BoundingSubBoxes: out->strategy = NBB_STRATEGY_SUBBOX; break;
    }
    switch (w.backend) {
        case nbb::LambdaBackend::Direct: out->backend = NBB_BACKEND_DIRECT; break;
        case nbb::LambdaBackend::MmaV1: out->backend = NBB_BACKEND_MMA1; break;
        case nbb::LambdaBackend::MmaV2: out->backend = NBB_BACKEND_MMA2; break;
        case nbb::LambdaBackend::MmaV3: out->backend = NBB_BACKEND_MMA3; break;
    }
    out->map_levels = w.map_levels;
    out->blocks_launched = w.blocks_launched;
    out->threads_launched = w.threads_launched;
    out->threads_active = w.threads_active;
    out->threads_wasted = w.threads_wasted;
    out->map_ops = w.map_ops;
    out->micros = w.micros;
}

nbb::WorkReport to_report(const nbb_report& r) {
    nbb::WorkReport w;
    w.spec_name = r.spec_name;
    w.r = r.r;
    w.rho = r.rho;
    w.mode = r.mode == NBB_MODE_BB ? nbb::MapMode::BoundingBox : nbb::MapMode::Lambda;
    w.strategy = r.strategy == NBB_STRATEGY_UNROLL ? nbb::IntraBlockStrategy::FurtherUnrolling
                 : r.strategy == NBB_STRATEGY_LUT  ? nbb::IntraBlockStrategy::SharedLookupTable
                                                   : nbb::IntraBlockStrategy::BoundingSubBoxes;
    w.backend = r.backend == NBB_BACKEND_MMA1   ? nbb::LambdaBackend::MmaV1
                : r.backend == NBB_BACKEND_MMA2 ? nbb::LambdaBackend::MmaV2
                : r.backend == NBB_BACKEND_MMA3 ? nbb::LambdaBackend::MmaV3
                                                : nbb::LambdaBackend::Direct;
    w.map_levels = r.map_levels;
    w.blocks_launched = r.blocks_launched;
    w.threads_launched = r.threads_launched;
    w.threads_active = r.threads_active;
    w.threads_wasted = r.threads_wasted;
    w.map_ops = r.map_ops;
    w.micros = r.micros;
    return w;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_error.c_str(); }

// ---- grids held by the reference's own nbb::Grid (no copies for big runs) ----
void* ref_grid_create(const nbb_spec* spec, int32_t r) {
    void* out = nullptr;
    guarded([&] { out = new nbb::Grid(to_spec(*spec), r); });
    return out;
}
void ref_grid_destroy(void* g) { delete static_cast<nbb::Grid*>(g); }
int64_t* ref_grid_data(void* g) { return static_cast<nbb::Grid*>(g)->values().data(); }
uint64_t ref_grid_generation(void* g) { return static_cast<nbb::Grid*>(g)->generation(); }

int ref_validate(const nbb_config* cfg) {
    return guarded([&] { to_config(*cfg).validate(); });
}

int ref_launch_block_count(const nbb_config* cfg, uint64_t* out) {
    return guarded([&] { *out = nbb::launch_block_count(to_config(*cfg)); });
}

int ref_single_write(const nbb_config* cfg, int64_t* out_grid, nbb_report* report,
                     double* call_seconds) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        auto res = nbb::run_single_write(to_config(*cfg));
        if (call_seconds) *call_seconds = seconds_since(t0);
        if (out_grid) {
            std::memcpy(out_grid, res.grid.values().data(), res.grid.values().size() * 8);
        }
        from_report(res.report, report);
    });
}

// grid_handle: an nbb::Grid from ref_grid_create (avoids a copy at large r).
int ref_reduction_h(const nbb_config* cfg, void* grid_handle, int64_t* value, nbb_report* report,
                    double* call_seconds) {
    return guarded([&] {
        const auto& grid = *static_cast<nbb::Grid*>(grid_handle);
        const auto t0 = std::chrono::steady_clock::now();
        auto res = nbb::run_reduction(to_config(*cfg), grid);
        if (call_seconds) *call_seconds = seconds_since(t0);
        *value = res.value;
        from_report(res.report, report);
    });
}

int ref_reduction(const nbb_config* cfg, const int64_t* grid_values, int32_t level, int64_t* value,
                  nbb_report* report) {
    return guarded([&] {
        const auto spec = to_spec(cfg->spec);
        nbb::Grid grid(spec, level);
        std::memcpy(grid.values().data(), grid_values, grid.values().size() * 8);
        auto res = nbb::run_reduction(to_config(*cfg), grid);
        *value = res.value;
        from_report(res.report, report);
    });
}

int ref_ca_h(const nbb_config* cfg, void* initial_handle, int32_t steps, uint16_t birth,
             uint16_t survive, void* out_handle, nbb_report* per_step, double* call_seconds) {
    return guarded([&] {
        const auto& initial = *static_cast<nbb::Grid*>(initial_handle);
        nbb::CaRule rule;
        rule.birth = birth;
        rule.survive = survive;
        const auto t0 = std::chrono::steady_clock::now();
        auto res = nbb::run_ca(to_config(*cfg), initial, steps, rule);
        if (call_seconds) *call_seconds = seconds_since(t0);
        if (out_handle) {
            auto& out = *static_cast<nbb::Grid*>(out_handle);
            out.values().swap(res.grid.values());
        }
        if (per_step) {
            for (std::size_t i = 0; i < res.reports.size(); ++i) from_report(res.reports[i], &per_step[i]);
        }
    });
}

int ref_ca(const nbb_config* cfg, const int64_t* initial_values, int32_t level, int32_t steps,
           uint16_t birth, uint16_t survive, int64_t* out_grid, nbb_report* per_step,
           uint64_t* generation) {
    return guarded([&] {
        const auto spec = to_spec(cfg->spec);
        nbb::Grid initial(spec, level);
        std::memcpy(initial.values().data(), initial_values, initial.values().size() * 8);
        nbb::CaRule rule;
        rule.birth = birth;
        rule.survive = survive;
        auto res = nbb::run_ca(to_config(*cfg), initial, steps, rule);
        std::memcpy(out_grid, res.grid.values().data(), res.grid.values().size() * 8);
        if (generation) *generation = res.grid.generation();
        if (per_step) {
            for (std::size_t i = 0; i < res.reports.size(); ++i) from_report(res.reports[i], &per_step[i]);
        }
    });
}

int ref_random_member_grid(const nbb_spec* spec, int32_t r, uint64_t seed, uint64_t modulus,
                           uint64_t max_cells, int64_t* out_grid) {
    return guarded([&] {
        auto g = nbb::random_member_grid(to_spec(*spec), r, seed, modulus, max_cells);
        std::memcpy(out_grid, g.values().data(), g.values().size() * 8);
    });
}

int ref_lambda_map(const nbb_spec* spec, int32_t level, int64_t ox, int64_t oy, int64_t* x,
                   int64_t* y) {
    return guarded([&] {
        const auto p = nbb::lambda_map(to_spec(*spec), level, {ox, oy});
        *x = p.x;
        *y = p.y;
    });
}

// Every ω of the level orthotope, ordinal-major (o = ωy*W + ωx).
int ref_lambda_coords(const nbb_spec* spec, int32_t level, int64_t* xy) {
    return guarded([&] {
        const auto s = to_spec(*spec);
        const auto [w, h] = s.orthotope_dims(level);
        std::size_t o = 0;
        for (std::int64_t oy = 0; oy < h; ++oy) {
            for (std::int64_t ox = 0; ox < w; ++ox, ++o) {
                const auto p = nbb::lambda_map(s, level, {ox, oy});
                xy[2 * o] = p.x;
                xy[2 * o + 1] = p.y;
            }
        }
    });
}

int ref_lambda_inverse(const nbb_spec* spec, int32_t level, int64_t x, int64_t y, int64_t* ox,
                       int64_t* oy) {
    return guarded([&] {
        const auto w = nbb::lambda_inverse(to_spec(*spec), level, {x, y});
        *ox = w.x;
        *oy = w.y;
    });
}

int ref_is_member(const nbb_spec* spec, int32_t level, int64_t x, int64_t y, int32_t* member) {
    return guarded([&] { *member = to_spec(*spec).is_member({x, y}, level) ? 1 : 0; });
}

int ref_map_thread(const nbb_spec* spec, int32_t r, int32_t rho, int64_t ox, int64_t oy,
                   int64_t tx, int64_t ty, int32_t strategy, int64_t* x, int64_t* y,
                   int32_t* active) {
    return guarded([&] {
        const auto s = to_spec(*spec);
        const auto geom = nbb::BlockGeometry::create(s, r, rho);
        const auto st = strategy == NBB_STRATEGY_UNROLL ? nbb::IntraBlockStrategy::FurtherUnrolling
                        : strategy == NBB_STRATEGY_LUT ? nbb::IntraBlockStrategy::SharedLookupTable
                                                       : nbb::IntraBlockStrategy::BoundingSubBoxes;
        const auto cell = nbb::map_thread(s, geom, {ox, oy}, {tx, ty}, st);
        *active = cell.has_value() ? 1 : 0;
        if (cell) {
            *x = cell->x;
            *y = cell->y;
        }
    });
}

// D = A*B (+C) of the reference encodings; fragments are 16x16 row-major doubles.
int ref_mma_variant1(const nbb_spec* spec, int32_t level, int64_t ox, int64_t oy, double* d) {
    return guarded([&] {
        const auto enc = nbb::encode_variant1(to_spec(*spec), level, {ox, oy});
        const auto out = nbb::mma_eval(enc.a, enc.b, nbb::Fragment{});
        std::memcpy(d, out.cells.data(), sizeof(double) * 256);
    });
}

int ref_mma_variant2(const nbb_spec* spec, int32_t level, const int64_t* omegas, int32_t count,
                     double* d, int32_t* active) {
    return guarded([&] {
        std::vector<nbb::OrthotopeCoord> coords;
        for (int i = 0; i < count; ++i) coords.push_back({omegas[2 * i], omegas[2 * i + 1]});
        const auto enc = nbb::encode_variant2(to_spec(*spec), level, coords);
        const auto out = nbb::mma_eval(enc.a, enc.b, nbb::Fragment{});
        std::memcpy(d, out.cells.data(), sizeof(double) * 256);
        for (int i = 0; i < 8; ++i) active[i] = enc.active[static_cast<std::size_t>(i)] ? 1 : 0;
    });
}

int ref_mma_variant3(const nbb_spec* spec, int32_t r, int32_t rho, int64_t ox, int64_t oy,
                     double* dx, double* dy) {
    return guarded([&] {
        const auto s = to_spec(*spec);
        const auto geom = nbb::BlockGeometry::create(s, r, rho);
        const auto enc = nbb::encode_variant3(s, geom, {ox, oy});
        const auto fx = nbb::mma_eval(enc.a, enc.bx, enc.cx);
        const auto fy = nbb::mma_eval(enc.a, enc.by, enc.cy);
        std::memcpy(dx, fx.cells.data(), sizeof(double) * 256);
        std::memcpy(dy, fy.cells.data(), sizeof(double) * 256);
    });
}

int ref_work_quotient(const nbb_report* bb, const nbb_report* lam, int32_t weighted,
                      double* out) {
    return guarded([&] { *out = nbb::work_quotient(to_report(*bb), to_report(*lam), weighted != 0); });
}

int ref_csv_row(const nbb_report* report, char* buf, size_t len) {
    return guarded([&] {
        const auto row = to_report(*report).csv_row();
        if (row.size() + 1 > len) throw std::length_error("csv buffer too small");
        std::memcpy(buf, row.c_str(), row.size() + 1);
    });
}

// std::ostream << double, as nbbmap bench formats the quotient column (nbbmap.cpp:611-613)
int ref_format_double(double v, char* buf, size_t len) {
    return guarded([&] {
        std::ostringstream s;
        s << v;
        const auto str = s.str();
        if (str.size() + 1 > len) throw std::length_error("buffer too small");
        std::memcpy(buf, str.c_str(), str.size() + 1);
    });
}

const char* ref_csv_header(void) {
    static const std::string h = nbb::WorkReport::csv_header();
    return h.c_str();
}

// compact codec (block_map.cpp:238-282): embedded <-> orthotope-ordered values
int ref_compact_store(const nbb_spec* spec, int32_t level, const int64_t* embedded, int64_t* compact) {
    return guarded([&] {
        const auto s = to_spec(*spec);
        const std::int64_t n = s.side_length(level);
        std::vector<std::int64_t> e(embedded, embedded + n * n);
        const auto c = nbb::compact_store(s, level, e);
        std::memcpy(compact, c.values().data(), c.values().size() * 8);
    });
}

// NBBC file through the reference's own writer (block_map.cpp:327-338)
int ref_write_compact(const nbb_spec* spec, int32_t level, const int64_t* values, const char* path) {
    return guarded([&] {
        const auto s = to_spec(*spec);
        nbb::CompactGrid g(s, level);
        std::memcpy(g.values().data(), values, g.values().size() * 8);
        std::ofstream out(path, std::ios::binary);
        nbb::write_compact(out, s, g);
    });
}

// NBBC reader (block_map.cpp:340-362); values must hold k^level entries
int ref_read_compact(const nbb_spec* spec, const char* path, int32_t* level, int64_t* values,
                     uint64_t capacity) {
    return guarded([&] {
        std::ifstream in(path, std::ios::binary);
        const auto g = nbb::read_compact(in, to_spec(*spec));
        if (g.values().size() > capacity) throw std::length_error("capacity");
        std::memcpy(values, g.values().data(), g.values().size() * 8);
        *level = g.level();
    });
}

}  // extern "C"
