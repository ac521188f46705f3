// nbb_host.cpp — host-side logic of the engine; see nbb_host.hpp.
#include "nbb_host.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <random>
#include <sstream>
#include <vector>

namespace nbbhost {

bool is_gasket(const nbb_spec& s) {
    return s.k == 3 && s.s == 2 && s.offset_x[0] == 0 && s.offset_y[0] == 0 &&
           s.offset_x[1] == 0 && s.offset_y[1] == 1 && s.offset_x[2] == 1 && s.offset_y[2] == 1;
}

Error require_gasket(const nbb_spec& s) {
    if (!is_gasket(s)) {
        return err(NBB_ERR_INVALID_ARGUMENT,
                   std::string("fractal '") + s.name +
                       "': the GPU path runs the sierpinski gasket only (k=3, s=2, offsets "
                       "(0,0),(0,1),(1,1)); there is no CPU fallback");
    }
    return {};
}

Error validate_spec(const nbb_spec& s) {
    if (s.k < 2) return err(NBB_ERR_INVALID_ARGUMENT, "FractalSpec: replica count must be >= 2");
    if (s.s < 2) return err(NBB_ERR_INVALID_ARGUMENT, "FractalSpec: scale factor must be >= 2");
    if ((int64_t)s.k > (int64_t)s.s * s.s)
        return err(NBB_ERR_INVALID_ARGUMENT, "FractalSpec: more replicas than step-box cells (k > s^2)");
    if (s.k > NBB_MAX_REPLICAS)
        return err(NBB_ERR_INVALID_ARGUMENT, "FractalSpec: at most 9 replicas on the GPU path");
    bool seen[NBB_MAX_REPLICAS] = {};
    for (int i = 0; i < s.k; ++i) {
        const int x = s.offset_x[i], y = s.offset_y[i];
        if (x < 0 || y < 0 || x >= s.s || y >= s.s)
            return err(NBB_ERR_INVALID_ARGUMENT, "FractalSpec: replica offset (" + std::to_string(x) +
                                                     "," + std::to_string(y) + ") outside [0," +
                                                     std::to_string(s.s - 1) + "]");
        if (seen[y * s.s + x])
            return err(NBB_ERR_INVALID_ARGUMENT, "FractalSpec: replica offsets overlap at (" +
                                                     std::to_string(x) + "," + std::to_string(y) + ")");
        seen[y * s.s + x] = true;
    }
    return {};
}

Error checked_pow(uint64_t base, int exp, uint64_t* out) {
    if (exp < 0) return err(NBB_ERR_INVALID_ARGUMENT, "checked_pow: negative exponent");
    uint64_t r = 1;
    for (int i = 0; i < exp; ++i) {
        if (base != 0 && r > std::numeric_limits<uint64_t>::max() / base) {
            return err(NBB_ERR_OVERFLOW, "checked_pow: " + std::to_string(base) + "^" +
                                             std::to_string(exp) + " overflows 64 bits");
        }
        r *= base;
    }
    *out = r;
    return {};
}

Error level_for_size(int64_t n, int s, int* level) {
    if (s < 2) return err(NBB_ERR_INVALID_ARGUMENT, "level_for_size: scale factor must be >= 2");
    if (n < 1) return err(NBB_ERR_INVALID_ARGUMENT, "level_for_size: side length must be >= 1");
    int l = 0;
    int64_t v = n;
    while (v > 1) {
        if (v % s != 0) {
            return err(NBB_ERR_INVALID_ARGUMENT, "level_for_size: " + std::to_string(n) +
                                                     " is not a power of " + std::to_string(s));
        }
        v /= s;
        ++l;
    }
    *level = l;
    return {};
}

Error side_length(const nbb_spec& s, int level, int64_t* n) {
    uint64_t v;
    Error e = checked_pow((uint64_t)s.s, level, &v);
    if (!e.ok()) return e;
    if (v > (uint64_t)std::numeric_limits<int64_t>::max())
        return err(NBB_ERR_OVERFLOW, "side_length overflows int64");
    *n = (int64_t)v;
    return {};
}

Error orthotope_dims(const nbb_spec& s, int level, int64_t* w, int64_t* h) {
    if (level < 0) return err(NBB_ERR_INVALID_ARGUMENT, "orthotope_dims: negative level");
    uint64_t a, b;
    Error e = checked_pow((uint64_t)s.k, (level + 1) / 2, &a);
    if (!e.ok()) return e;
    e = checked_pow((uint64_t)s.k, level / 2, &b);
    if (!e.ok()) return e;
    *w = (int64_t)a;
    *h = (int64_t)b;
    return {};
}

Error validate(const nbb_config& c) {
    const int rho = c.rho;
    if (!(rho == 1 || rho == 2 || rho == 4 || rho == 8 || rho == 16 || rho == 32))
        return err(NBB_ERR_INVALID_ARGUMENT,
                   "rho " + std::to_string(rho) + " is not one of 1, 2, 4, 8, 16, 32");
    if (c.r < 0) return err(NBB_ERR_INVALID_ARGUMENT, "negative scale level");
    if (c.workers < 1) return err(NBB_ERR_INVALID_ARGUMENT, "workers must be >= 1");
    int64_t n;
    Error e = side_length(c.spec, c.r, &n);
    if (!e.ok()) return e;
    if (n % rho != 0)
        return err(NBB_ERR_INVALID_ARGUMENT,
                   "rho " + std::to_string(rho) + " does not divide n = " + std::to_string(n));
    if (c.cell_width != 8 && c.cell_width != 1 && c.cell_width != 0)
        return err(NBB_ERR_INVALID_ARGUMENT, "cell_width " + std::to_string(c.cell_width) +
                                                 " is not 8 (int64), 1 (uint8) or 0 (1-bit packed)");
    if (c.mode == NBB_MODE_BB) {
        if (c.backend != NBB_BACKEND_DIRECT)
            return err(NBB_ERR_INVALID_ARGUMENT, "lambda backends apply to lambda mode only");
        return {};
    }
    int r_t;
    e = level_for_size(rho, c.spec.s, &r_t);
    if (!e.ok()) return e;
    if (r_t > c.r)
        return err(NBB_ERR_INVALID_ARGUMENT, "block geometry: rho " + std::to_string(rho) +
                                                 " exceeds the embedding side " + std::to_string(n));
    const int r_b = c.r - r_t;
    switch (c.backend) {
        case NBB_BACKEND_DIRECT:
            break;
        case NBB_BACKEND_MMA1:
            if (r_b > 16)
                return err(NBB_ERR_INVALID_ARGUMENT,
                           "variant 1 encodes at most 16 levels, r_b = " + std::to_string(r_b));
            break;
        case NBB_BACKEND_MMA2: {
            if (rho < 2)
                return err(NBB_ERR_INVALID_ARGUMENT, "variant 2 needs sub-blocks of edge rho/2 >= 1");
            int sub_rt;
            if (!level_for_size(rho / 2, c.spec.s, &sub_rt).ok())
                return err(NBB_ERR_INVALID_ARGUMENT,
                           "variant 2 sub-block edge " + std::to_string(rho / 2) +
                               " is not a power of s = " + std::to_string(c.spec.s));
            if (c.r - sub_rt > 16)
                return err(NBB_ERR_INVALID_ARGUMENT, "variant 2 encodes at most 16 levels");
            break;
        }
        case NBB_BACKEND_MMA3:
            if (rho != 16)
                return err(NBB_ERR_INVALID_ARGUMENT,
                           "variant 3 runs at rho = 16 only, got " + std::to_string(rho));
            if (c.strategy != NBB_STRATEGY_SUBBOX)
                return err(NBB_ERR_INVALID_ARGUMENT,
                           "variant 3 emits sub-box thread coordinates; use the subbox strategy");
            if (r_b > 16) return err(NBB_ERR_INVALID_ARGUMENT, "variant 3 encodes at most 16 levels");
            break;
        default:
            return err(NBB_ERR_INVALID_ARGUMENT, "unknown backend " + std::to_string(c.backend));
    }
    if (c.strategy < NBB_STRATEGY_UNROLL || c.strategy > NBB_STRATEGY_SUBBOX)
        return err(NBB_ERR_INVALID_ARGUMENT, "unknown strategy " + std::to_string(c.strategy));
    return {};
}

Error make_plan(const nbb_config& c, Plan* p) {
    Plan plan;
    Error e = side_length(c.spec, c.r, &plan.n);
    if (!e.ok()) return e;
    if (c.mode == NBB_MODE_BB) {
        plan.gw = plan.gh = plan.n / c.rho;
        plan.edge = c.rho;
        *p = plan;
        return {};
    }
    int r_t;
    e = level_for_size(c.rho, c.spec.s, &r_t);
    if (!e.ok()) return e;
    if (c.backend == NBB_BACKEND_MMA2) {
        int sub_rt;
        e = level_for_size(c.rho / 2, c.spec.s, &sub_rt);
        if (!e.ok()) return e;
        const int r_sb = c.r - sub_rt;
        int64_t w, h;
        e = orthotope_dims(c.spec, r_sb, &w, &h);
        if (!e.ok()) return e;
        plan.gw = (w + 1) / 2 * 2;
        plan.gh = (h + 1) / 2 * 2;
        plan.sub_w = w;
        plan.sub_h = h;
        plan.edge = c.rho / 2;
        plan.map_level = r_sb;
        plan.local_level = sub_rt;
    } else {
        int64_t w, h;
        e = orthotope_dims(c.spec, c.r - r_t, &w, &h);
        if (!e.ok()) return e;
        plan.gw = w;
        plan.gh = h;
        plan.edge = c.rho;
        plan.map_level = c.r - r_t;
        plan.local_level = r_t;
    }
    int64_t lw, lh;
    e = orthotope_dims(c.spec, plan.local_level, &lw, &lh);
    if (!e.ok()) return e;
    plan.local_w = lw;
    e = checked_pow((uint64_t)c.spec.k, plan.local_level, &plan.local_members);
    if (!e.ok()) return e;
    *p = plan;
    return {};
}

Error plan_report(const nbb_config& c, nbb_report* r) {
    Error e = validate(c);
    if (!e.ok()) return e;
    Plan p;
    e = make_plan(c, &p);
    if (!e.ok()) return e;
    std::memset(r, 0, sizeof(*r));
    std::strncpy(r->spec_name, c.spec.name, sizeof(r->spec_name) - 1);
    r->r = c.r;
    r->rho = c.rho;
    r->mode = c.mode;
    r->strategy = c.strategy;
    r->backend = c.backend;
    uint64_t members;
    e = checked_pow((uint64_t)c.spec.k, c.r, &members);
    if (!e.ok()) return e;
    const uint64_t blocks = p.blocks();
    const uint64_t edge2 = (uint64_t)p.edge * (uint64_t)p.edge;
    r->blocks_launched = blocks;
    r->threads_launched = blocks * edge2;
    r->threads_active = members;
    r->threads_wasted = r->threads_launched - members;
    if (c.mode == NBB_MODE_BB) {
        r->map_ops = r->threads_launched;  // one membership predicate per thread
        r->map_levels = 0;
        return {};
    }
    const uint64_t inrange =
        c.backend == NBB_BACKEND_MMA2 ? (uint64_t)p.sub_w * (uint64_t)p.sub_h : blocks;
    uint64_t ops = inrange * (uint64_t)p.map_level;
    switch (c.strategy) {
        case NBB_STRATEGY_SUBBOX: ops += inrange * edge2; break;
        case NBB_STRATEGY_UNROLL: ops += members * (uint64_t)p.local_level; break;
        case NBB_STRATEGY_LUT: ops += p.local_members * (uint64_t)p.local_level; break;
    }
    r->map_ops = ops;
    r->map_levels = p.map_level;
    return {};
}

Error member_mask_budget(const nbb_spec& s, int level, uint64_t max_cells) {
    int64_t n;
    Error e = side_length(s, level, &n);
    if (!e.ok()) return e;
    const uint64_t area = (uint64_t)n * (uint64_t)n;
    if (area > max_cells)
        return err(NBB_ERR_RESOURCE, "MemberMask: embedding of " + std::to_string(area) +
                                         " cells exceeds the budget of " + std::to_string(max_cells));
    return {};
}

static const char* mode_name(int m) { return m == NBB_MODE_BB ? "bb" : "lambda"; }
static const char* strategy_name(int s) {
    return s == NBB_STRATEGY_UNROLL ? "unroll" : s == NBB_STRATEGY_LUT ? "lut" : "subbox";
}
static const char* backend_name(int b) {
    return b == NBB_BACKEND_MMA1 ? "mma1" : b == NBB_BACKEND_MMA2 ? "mma2" : b == NBB_BACKEND_MMA3 ? "mma3" : "direct";
}

std::string csv_row(const nbb_report& r) {
    std::ostringstream out;
    out << r.spec_name << ',' << r.r << ',' << r.rho << ',' << mode_name(r.mode) << ','
        << strategy_name(r.strategy) << ',' << backend_name(r.backend) << ',' << r.blocks_launched
        << ',' << r.threads_launched << ',' << r.threads_active << ',' << r.threads_wasted << ','
        << r.map_ops << ',' << r.micros;
    return out.str();
}

const char* csv_header() {
    return "# spec,r,rho,mode,strategy,backend,blocks,threads,active,wasted,map_ops,micros";
}

Error work_quotient(const nbb_report& bb, const nbb_report& lam, bool weighted, double* q) {
    if (bb.mode != NBB_MODE_BB || lam.mode != NBB_MODE_LAMBDA)
        return err(NBB_ERR_INVALID_ARGUMENT, "work_quotient takes one bb report and one lambda report");
    if (std::strncmp(bb.spec_name, lam.spec_name, sizeof(bb.spec_name)) != 0 || bb.r != lam.r ||
        bb.rho != lam.rho)
        return err(NBB_ERR_INVALID_ARGUMENT, "work_quotient: the reports describe different launches");
    double denom = (double)lam.threads_launched;
    if (weighted) denom *= (double)(lam.map_levels > 1 ? lam.map_levels : 1);
    *q = (double)bb.threads_launched / denom;
    return {};
}

static bool member_generic(const nbb_spec& s, int level, int64_t x, int64_t y, int64_t n) {
    int64_t scale = n / s.s;
    for (int mu = level; mu >= 1; --mu) {
        const int cx = (int)(x / scale), cy = (int)(y / scale);
        bool hit = false;
        for (int i = 0; i < s.k; ++i) hit |= (s.offset_x[i] == cx && s.offset_y[i] == cy);
        if (!hit) return false;
        x -= cx * scale;
        y -= cy * scale;
        scale /= s.s;
    }
    return true;
}

Error random_member_values(const nbb_spec& s, int r, uint64_t seed, uint64_t modulus, int64_t* out) {
    if (modulus == 0) return err(NBB_ERR_INVALID_ARGUMENT, "random_member_grid: modulus must be positive");
    Error e = require_gasket(s);
    if (!e.ok()) return e;
    int64_t n;
    e = side_length(s, r, &n);
    if (!e.ok()) return e;
    std::mt19937_64 rng(seed);
    uint64_t k = 0;
    for (int64_t y = 0; y < n; ++y) {
        int64_t x = 0;
        do {
            out[k++] = (int64_t)(rng() % modulus);
            x = (x - y) & y;
        } while (x != 0);
    }
    return {};
}

Error random_member_grid(const nbb_spec& s, int r, uint64_t seed, uint64_t modulus,
                         uint64_t max_cells, int64_t* grid) {
    if (modulus == 0) return err(NBB_ERR_INVALID_ARGUMENT, "random_member_grid: modulus must be positive");
    int64_t n;
    Error e = side_length(s, r, &n);
    if (!e.ok()) return e;
    e = member_mask_budget(s, r, max_cells);
    if (!e.ok()) return e;
    std::memset(grid, 0, (size_t)n * (size_t)n * sizeof(int64_t));
    std::mt19937_64 rng(seed);
    if (is_gasket(s)) {
        for (int64_t y = 0; y < n; ++y) {
            int64_t x = 0;
            do {
                grid[y * n + x] = (int64_t)(rng() % modulus);
                x = (x - y) & y;
            } while (x != 0);
        }
        return {};
    }
    for (int64_t y = 0; y < n; ++y)
        for (int64_t x = 0; x < n; ++x)
            if (member_generic(s, r, x, y, n)) grid[y * n + x] = (int64_t)(rng() % modulus);
    return {};
}

void local_cell_table(const nbb_spec& s, int edge, int16_t* out) {
    int r_t = 0;
    level_for_size(edge, s.s, &r_t);
    uint64_t members = 1;
    checked_pow((uint64_t)s.k, r_t, &members);
    int64_t w, h;
    orthotope_dims(s, r_t, &w, &h);
    for (int64_t ty = 0; ty < edge; ++ty) {
        for (int64_t tx = 0; tx < edge; ++tx) {
            const uint64_t rank = (uint64_t)ty * (uint64_t)edge + (uint64_t)tx;
            int16_t* e = out + 2 * (ty * edge + tx);
            if (rank >= members) {
                e[0] = e[1] = -1;
                continue;
            }
            // λ at the local level (block_map.cpp:25-37, 77-111)
            int64_t dx = (int64_t)(rank % (uint64_t)w), dy = (int64_t)(rank / (uint64_t)w);
            int64_t px = 0, py = 0, scale = 1;
            for (int mu = 1; mu <= r_t; ++mu) {
                int beta;
                if (mu % 2 == 1) {
                    beta = (int)(dx % s.k);
                    dx /= s.k;
                } else {
                    beta = (int)(dy % s.k);
                    dy /= s.k;
                }
                px += s.offset_x[beta] * scale;
                py += s.offset_y[beta] * scale;
                scale *= s.s;
            }
            e[0] = (int16_t)px;
            e[1] = (int16_t)py;
        }
    }
}

static void put_u32(std::vector<unsigned char>& b, uint32_t v) {
    for (int i = 0; i < 4; ++i) b.push_back((unsigned char)(v >> (8 * i)));
}

Error write_compact(const char* path, const nbb_spec& s, int level, const int64_t* values) {
    uint64_t count;
    Error e = checked_pow((uint64_t)s.k, level, &count);
    if (!e.ok()) return e;
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return err(NBB_ERR_RUNTIME, std::string("cannot open '") + path + "' for writing");
    std::vector<unsigned char> head = {'N', 'B', 'B', 'C'};
    put_u32(head, (uint32_t)s.k);
    put_u32(head, (uint32_t)s.s);
    put_u32(head, (uint32_t)level);
    bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
    std::vector<unsigned char> buf;
    buf.reserve(1 << 20);
    for (uint64_t i = 0; i < count && ok; ++i) {
        const uint64_t v = (uint64_t)values[i];
        for (int b = 0; b < 8; ++b) buf.push_back((unsigned char)(v >> (8 * b)));
        if (buf.size() >= (1 << 20) || i + 1 == count) {
            ok = std::fwrite(buf.data(), 1, buf.size(), f) == buf.size();
            buf.clear();
        }
    }
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) return err(NBB_ERR_RUNTIME, "compact file: write failed");
    return {};
}

Error read_compact(const char* path, const nbb_spec& s, int* level, int64_t* values, uint64_t capacity) {
    std::FILE* f = std::fopen(path, "rb");
    if (!f) return err(NBB_ERR_INVALID_ARGUMENT, std::string("cannot open '") + path + "'");
    unsigned char head[16];
    const size_t got = std::fread(head, 1, 16, f);
    auto u32 = [&](int o) {
        return (uint32_t)head[o] | ((uint32_t)head[o + 1] << 8) | ((uint32_t)head[o + 2] << 16) |
               ((uint32_t)head[o + 3] << 24);
    };
    if (got < 4 || std::memcmp(head, "NBBC", 4) != 0) {
        std::fclose(f);
        return err(NBB_ERR_INVALID_ARGUMENT, "compact file: bad magic");
    }
    if (got < 16) {
        std::fclose(f);
        return err(NBB_ERR_INVALID_ARGUMENT, "compact file: truncated header");
    }
    const uint32_t k = u32(4), ss = u32(8), lv = u32(12);
    if (k != (uint32_t)s.k || ss != (uint32_t)s.s) {
        std::fclose(f);
        return err(NBB_ERR_INVALID_ARGUMENT, "compact file: header (k=" + std::to_string(k) + ", s=" +
                                                 std::to_string(ss) + ") does not match spec '" +
                                                 s.name + "'");
    }
    if (lv > 64) {
        std::fclose(f);
        return err(NBB_ERR_INVALID_ARGUMENT, "compact file: implausible level " + std::to_string(lv));
    }
    uint64_t count;
    Error e = checked_pow((uint64_t)s.k, (int)lv, &count);
    if (!e.ok()) {
        std::fclose(f);
        return e;
    }
    if (count > capacity) {
        std::fclose(f);
        return err(NBB_ERR_RESOURCE, "compact file: " + std::to_string(count) +
                                         " values exceed the buffer of " + std::to_string(capacity));
    }
    std::vector<unsigned char> buf(8);
    for (uint64_t i = 0; i < count; ++i) {
        if (std::fread(buf.data(), 1, 8, f) != 8) {
            std::fclose(f);
            return err(NBB_ERR_INVALID_ARGUMENT, "compact file: truncated payload");
        }
        uint64_t v = 0;
        for (int b = 0; b < 8; ++b) v |= (uint64_t)buf[b] << (8 * b);
        values[i] = (int64_t)v;
    }
    std::fclose(f);
    *level = (int)lv;
    return {};
}

void fastdiv_magic(uint32_t d, uint32_t* m, uint32_t* s) {
    if (d == 0) d = 1;
    if ((d & (d - 1)) == 0) {
        uint32_t l = 0;
        while ((1u << l) < d) ++l;
        *m = 0;
        *s = l;
        return;
    }
    uint32_t l = 0;
    while ((2u << l) <= d) ++l;  // 2^l < d < 2^(l+1)
    const unsigned __int128 num = (unsigned __int128)1 << (32 + l);
    *m = (uint32_t)((num + d - 1) / d);
    *s = l;
}

}  // namespace nbbhost

// ---- halo slots (see nbb_host.hpp) ---------------------------------------------------------
namespace nbbhost {
namespace {
uint32_t tile_local_index_host(uint32_t x, uint32_t y) {  // λ⁻¹ inside a ρ = 32 gasket tile
    auto b3 = [](uint32_t bits) {  // even bits of `bits` read as base-3 digits in {0, 1}
        uint32_t v = 0, p = 1;
        for (int j = 0; j < 16; j += 2, p *= 3) v += ((bits >> j) & 1u) * p;
        return v;
    };
    const uint32_t wx = b3(x) + b3(y), wy = b3(x >> 1) + b3(y >> 1);
    return wy * 27u + wx;
}
}  // namespace

Error halo_slots(HaloSlots* out) {
    constexpr int L = 13, T = 32, K = kPassMaxK;
    const int64_t n = int64_t(1) << L, nb = n / T;
    auto member = [&](int64_t x, int64_t y) { return x >= 0 && y >= 0 && x < n && y < n && (x & y) == x; };
    // the first 8 slots keep the order of the one-step halo (compact_rows_step's h bits)
    const int h1x[8] = {-1, 0, 1, -1, 32, 32, 32, 0}, h1y[8] = {-1, -1, -1, 31, 30, 31, 32, 32};
    constexpr int E = T + 2 * K;  // the tile and a K-cell frame, (x, y) -> (x + K, y + K)
    std::vector<int> best(E * E, 99);
    std::vector<int> layer(E * E);
    for (int64_t by = 0; by < nb; ++by)
        for (int64_t bx = 0; bx < nb; ++bx) {
            if ((bx & by) != bx) continue;
            std::fill(layer.begin(), layer.end(), -1);
            for (int y = 0; y < T; ++y)
                for (int x = 0; x < T; ++x)
                    if ((x & y) == x) layer[(y + K) * E + x + K] = 0;
            for (int d = 1; d <= K; ++d)
                for (int y = -K; y < T + K; ++y)
                    for (int x = -K; x < T + K; ++x) {
                        const int i = (y + K) * E + x + K;
                        if (layer[i] >= 0 || !member(bx * T + x, by * T + y)) continue;
                        bool adj = false;
                        for (int dy = -1; dy <= 1 && !adj; ++dy)
                            for (int dx = -1; dx <= 1 && !adj; ++dx) {
                                const int qx = x + dx, qy = y + dy;
                                if ((dx || dy) && qx >= -K && qy >= -K && qx < T + K && qy < T + K)
                                    adj = layer[(qy + K) * E + qx + K] == d - 1;
                            }
                        if (adj) layer[i] = d;
                    }
            for (int i = 0; i < E * E; ++i)
                if (layer[i] > 0) best[i] = std::min(best[i], layer[i]);
        }
    std::vector<std::pair<int, int>> pos;  // (layer, index)
    for (int i = 0; i < E * E; ++i)
        if (best[i] <= K) pos.push_back({best[i], i});
    std::vector<int> order;
    for (int k = 0; k < 8; ++k) order.push_back((h1y[k] + K) * E + h1x[k] + K);
    std::stable_sort(pos.begin(), pos.end(), [](auto a, auto b) { return a.first < b.first; });
    for (auto& pi : pos)
        if (std::find(order.begin(), order.end(), pi.second) == order.end()) order.push_back(pi.second);
    if ((int)order.size() > kPassSlots || (int)pos.size() != (int)order.size())
        return err(NBB_ERR_RUNTIME, "halo slots: unexpected layer structure");
    HaloSlots h{};
    h.count = (int32_t)order.size();
    for (int d = 0; d <= K; ++d)
        for (auto& pi : pos) h.upto[d] += pi.first <= d;
    for (int s = 0; s < h.count; ++s) {
        const int x = order[s] % E - K, y = order[s] / E - K;
        if (s < 8 ? best[order[s]] != 1 : best[order[s]] < 2)
            return err(NBB_ERR_RUNTIME, "halo slots: H_1 is not the one-step halo");
        h.x[s] = (int8_t)x;
        h.y[s] = (int8_t)y;
        const int dx = x < 0 ? -1 : x >= T ? 1 : 0, dy = y < 0 ? -1 : y >= T ? 1 : 0;
        const int d9 = (dy + 1) * 3 + dx + 1;
        h.dir[s] = (uint8_t)(d9 > 4 ? d9 - 1 : d9);
        h.li[s] = (uint8_t)tile_local_index_host((uint32_t)(x - dx * T), (uint32_t)(y - dy * T));
        for (int t = 0; t < h.count; ++t) {
            const int tx = order[t] % E - K, ty = order[t] / E - K;
            if (t != s && std::abs(tx - x) <= 1 && std::abs(ty - y) <= 1) {
                if (t < 32) h.nb_lo[s] |= 1u << t; else h.nb_hi[s] |= 1u << (t - 32);
            }
        }
        for (int qy = y - 1; qy <= y + 1; ++qy)
            for (int qx = x - 1; qx <= x + 1; ++qx) {
                if (qx < 0 || qy < 0 || qx >= T || qy >= T || (qx & qy) != qx) continue;
                if (s >= 8) return err(NBB_ERR_RUNTIME, "halo slots: in-tile neighbour beyond H_1");
                if (qy == 0) h.m0[s] |= 1u << qx;
                else if (qy == 30) h.m30[s] |= 1u << qx;
                else if (qy == 31) h.m31[s] |= 1u << qx;
                else return err(NBB_ERR_RUNTIME, "halo slots: in-tile neighbour outside rows 0/30/31");
            }
    }
    *out = h;
    return {};
}
}  // namespace nbbhost

// ---- halo slots of the tile-sliced pass (see nbb_host.hpp) ----------------------------------
namespace nbbhost {
template <class S>
Error build_slot_table(S* out) {
    constexpr int L = 12, T = 32, K = S::kMaxK, E = T + 2 * K;
    const int64_t n = int64_t(1) << L, nb = n / T;
    auto member = [&](int64_t x, int64_t y) { return x >= 0 && y >= 0 && x < n && y < n && (x & y) == x; };
    std::vector<int> best(E * E, 99), layer(E * E);
    std::vector<int> front, next;
    for (int64_t by = 0; by < nb; ++by)
        for (int64_t bx = 0; bx < nb; ++bx) {
            if ((bx & by) != bx) continue;
            std::fill(layer.begin(), layer.end(), -1);
            front.clear();
            for (int y = 0; y < T; ++y)
                for (int x = 0; x < T; ++x)
                    if ((x & y) == x) {
                        layer[(y + K) * E + x + K] = 0;
                        front.push_back((y + K) * E + x + K);
                    }
            for (int d = 1; d <= K; ++d) {
                next.clear();
                for (int i : front) {
                    const int x = i % E - K, y = i / E - K;
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            const int qx = x + dx, qy = y + dy;
                            if ((!dx && !dy) || qx < -K || qy < -K || qx >= T + K || qy >= T + K) continue;
                            const int q = (qy + K) * E + qx + K;
                            if (layer[q] >= 0 || !member(bx * T + qx, by * T + qy)) continue;
                            layer[q] = d;
                            next.push_back(q);
                        }
                }
                front.swap(next);
                for (int q : front) best[q] = std::min(best[q], d);
            }
        }
    std::vector<std::pair<int, int>> pos;  // (layer, index), index in row-major frame order
    for (int i = 0; i < E * E; ++i)
        if (best[i] <= K) pos.push_back({best[i], i});
    std::stable_sort(pos.begin(), pos.end(), [](auto a, auto b) { return a.first < b.first; });
    if ((int)pos.size() > S::kSlots) return err(NBB_ERR_RUNTIME, "slice slots: too many halo positions");
    S h{};
    h.count = (int32_t)pos.size();
    for (int s = 0; s < h.count; ++s) {
        const int x = pos[s].second % E - K, y = pos[s].second / E - K, d = pos[s].first;
        h.x[s] = (int8_t)x;
        h.y[s] = (int8_t)y;
        h.layer[s] = (uint8_t)d;
        const int dx = x < 0 ? -1 : x >= T ? 1 : 0, dy = y < 0 ? -1 : y >= T ? 1 : 0;
        const int d9 = (dy + 1) * 3 + dx + 1;
        const int dir = d9 > 4 ? d9 - 1 : d9;
        h.dir_of[s] = (uint8_t)dir;
        h.li[s] = (uint8_t)tile_local_index_host((uint32_t)(x - dx * T), (uint32_t)(y - dy * T));
        if (h.dir_upto[dir][K] >= S::kDirMax) return err(NBB_ERR_RUNTIME, "slice slots: too many in one tile");
        h.by_dir[dir][h.dir_upto[dir][K]++] = (uint16_t)s;
        for (int k = d; k <= K; ++k) ++h.upto[k];
    }
    for (int dir = 0; dir < 8; ++dir)  // the per-tile lists are in slot (= layer) order
        for (int k = 0; k <= K; ++k) {
            int c = 0;
            for (int i = 0; i < h.dir_upto[dir][K]; ++i) c += h.layer[h.by_dir[dir][i]] <= k;
            h.dir_upto[dir][k] = c;
        }
    *out = h;
    return {};
}
Error slice_slots(SliceSlots* out) { return build_slot_table(out); }
Error cluster_slots(ClusterSlots* out) { return build_slot_table(out); }
}  // namespace nbbhost

// ---- halo exchange lists of the multi-process compact CA (see nbb_host.hpp) ----------------
namespace nbbhost {
namespace {
uint64_t digits_to_bits(uint64_t v, bool two_only) {  // X(v) (digit 2) / Y(v) (digit >= 1) at even bits
    uint64_t out = 0;
    for (int j = 0; v; ++j, v /= 3) {
        const uint64_t d = v % 3;
        if (two_only ? d == 2 : d >= 1) out |= 1ull << (2 * j);
    }
    return out;
}
uint64_t even_bits_base3(uint64_t b) {  // bits 0, 2, 4, ... of b read as base-3 digits in {0, 1}
    uint64_t v = 0, p = 1;
    for (int j = 0; j < 64; j += 2, p *= 3) v += ((b >> j) & 1u) * p;
    return v;
}
}  // namespace

Error halo_exchange_lists(int r, int world, int rank, int kmax, std::vector<std::vector<uint32_t>>* send,
                          std::vector<std::vector<uint32_t>>* recv) {
    if (r < 5 || r > 18) return err(NBB_ERR_INVALID_ARGUMENT, "halo exchange: 5 <= r <= 18");
    if (world < 1 || rank < 0 || rank >= world) return err(NBB_ERR_INVALID_ARGUMENT, "halo exchange: 0 <= rank < world");
    if (kmax < 1 || kmax > kSliceMaxK) return err(NBB_ERR_INVALID_ARGUMENT, "halo exchange: 1 <= kmax <= 8");
    SliceSlots ss;
    Error e = slice_slots(&ss);
    if (!e.ok()) return e;
    const int rb = r - 5;
    uint64_t W = 1, Wb = 1, Hb = 1;
    for (int i = 0; i < (r + 1) / 2; ++i) W *= 3;
    for (int i = 0; i < (rb + 1) / 2; ++i) Wb *= 3;
    for (int i = 0; i < rb / 2; ++i) Hb *= 3;
    const uint64_t tiles = Wb * Hb, nb = uint64_t(1) << rb;
    const uint64_t chunk = compact_shard_chunk(rb, tiles, Hb, world);
    auto owner = [&](uint64_t u) { return (int)(u / chunk); };
    auto base = [&](uint64_t u) { return 9 * (u / Hb) * W + 27 * (u % Hb); };
    // slot offsets inside a neighbouring tile, per direction, layers <= kmax
    std::vector<uint32_t> loc[8];
    for (int d = 0; d < 8; ++d)
        for (int j = 0; j < ss.dir_upto[d][kmax]; ++j) {
            const uint32_t li = ss.li[ss.by_dir[d][j]];
            loc[d].push_back((uint32_t)((li / 27) * W + li % 27));
        }
    auto neighbour = [&](uint64_t u, int d, uint64_t* out) {  // tile ordinal in direction d, if any
        const int d9 = d < 4 ? d : d + 1;
        const uint64_t wx = u / Hb, wy = u % Hb;
        const uint64_t bx = digits_to_bits(wx, true) | digits_to_bits(wy, true) << 1;
        const uint64_t by = digits_to_bits(wx, false) | digits_to_bits(wy, false) << 1;
        const int64_t qx = (int64_t)bx + d9 % 3 - 1, qy = (int64_t)by + d9 / 3 - 1;
        if (qx < 0 || qy < 0 || (uint64_t)qx >= nb || (uint64_t)qy >= nb || ((uint64_t)qx & (uint64_t)qy) != (uint64_t)qx)
            return false;
        *out = (even_bits_base3((uint64_t)qx) + even_bits_base3((uint64_t)qy)) * Hb +
               even_bits_base3((uint64_t)qx >> 1) + even_bits_base3((uint64_t)qy >> 1);
        return true;
    };
    send->assign((size_t)world, {});
    recv->assign((size_t)world, {});
    for (uint64_t u = 0; u < tiles; ++u) {  // the halo cells every tile reads from another rank
        const int need = owner(u);
        for (int d = 0; d < 8; ++d) {
            uint64_t v;
            if (loc[d].empty() || !neighbour(u, d, &v)) continue;
            const int has = owner(v);
            if (has == need || (need != rank && has != rank)) continue;
            auto& lst = need == rank ? (*recv)[(size_t)has] : (*send)[(size_t)need];
            for (uint32_t o : loc[d]) lst.push_back((uint32_t)(base(v) + o));
        }
    }
    for (auto* side : {send, recv})
        for (auto& l : *side) {
            std::sort(l.begin(), l.end());
            l.erase(std::unique(l.begin(), l.end()), l.end());
        }
    return {};
}
}  // namespace nbbhost
