/*
 * nbb_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU checker for the GPU path.
 *
 * A plain-C restatement of the reference's hot-path algorithm
 * (/root/reference/proj/src/{fractal,block_map,dispatch,mma}.cpp). Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it, and
 * only as the checker; the product library never links or calls it.
 * Pinned against the reference itself (oracle/_ref/libnbbref.so) and the
 * golden digests of SURVEY.md App. B by tests/test_oracle.py.
 */
#include "nbb_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---- std::mt19937_64 ([rand.eng.mers]; used by dispatch.cpp:140) ---------- */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i) {
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    }
    g->idx = MT_N;
}

uint64_t orc_mt64_next(orc_mt64* g) {
    if (g->idx >= MT_N) {
        for (int i = 0; i < MT_N; ++i) {
            const uint64_t x = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

uint64_t orc_fnv1a64(const void* data, size_t bytes) {
    const unsigned char* p = (const unsigned char*)data;
    uint64_t h = 0xcbf29ce484222325ULL;
    for (size_t i = 0; i < bytes; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* ---- fractal-core (fractal.cpp) ------------------------------------------- */
static uint64_t ipow_u(uint64_t b, int e) {
    uint64_t v = 1;
    for (int i = 0; i < e; ++i) v *= b;
    return v;
}

int64_t orc_side_length(const nbb_spec* spec, int level) {           /* fractal.cpp:165-171 */
    return (int64_t)ipow_u((uint64_t)spec->s, level);
}

void orc_orthotope_dims(const nbb_spec* spec, int level, int64_t* w, int64_t* h) { /* :181-192 */
    *w = (int64_t)ipow_u((uint64_t)spec->k, (level + 1) / 2);
    *h = (int64_t)ipow_u((uint64_t)spec->k, level / 2);
}

static int replica_at(const nbb_spec* spec, int cx, int cy) {
    for (int i = 0; i < spec->k; ++i) {
        if (spec->offset_x[i] == cx && spec->offset_y[i] == cy) return i;
    }
    return -1;
}

int orc_is_member(const nbb_spec* spec, int level, int64_t x, int64_t y) { /* fractal.cpp:194-214 */
    const int64_t n = orc_side_length(spec, level);
    if (x < 0 || y < 0 || x >= n || y >= n) return 0;
    int64_t scale = n / spec->s;
    for (int mu = level; mu >= 1; --mu) {
        const int cx = (int)(x / scale);
        const int cy = (int)(y / scale);
        if (replica_at(spec, cx, cy) < 0) return 0;
        x -= cx * scale;
        y -= cy * scale;
        scale /= spec->s;
    }
    return 1;
}

/* The gasket bit test: x is a bitwise submask of y (acceptance.cpp:88-102). */
int orc_gasket_bit_test(int level, int64_t x, int64_t y) {
    const int64_t n = (int64_t)1 << level;
    if (x < 0 || y < 0 || x >= n || y >= n) return 0;
    return (x & (n - 1 - y)) == 0;
}

static int is_gasket(const nbb_spec* s) {
    return s->k == 3 && s->s == 2 && s->offset_x[0] == 0 && s->offset_y[0] == 0 &&
           s->offset_x[1] == 0 && s->offset_y[1] == 1 && s->offset_x[2] == 1 && s->offset_y[2] == 1;
}

static int member(const nbb_spec* spec, int level, int64_t x, int64_t y) {
    return is_gasket(spec) ? orc_gasket_bit_test(level, x, y) : orc_is_member(spec, level, x, y);
}

/* ---- block-map (block_map.cpp) -------------------------------------------- */
int orc_beta_index(const nbb_spec* spec, int64_t ox, int64_t oy, int mu) { /* :57-65 */
    if (mu < 1) return -1;
    const int64_t value = (mu % 2 == 1) ? ox : oy;
    const int64_t divisor = (int64_t)ipow_u((uint64_t)spec->k, (mu + 1) / 2 - 1);
    return (int)((value / divisor) % spec->k);
}

int orc_lambda_map(const nbb_spec* spec, int level, int64_t ox, int64_t oy, int64_t* x,
                   int64_t* y) {                                            /* :77-111 */
    if (level < 0) return NBB_ERR_INVALID_ARGUMENT;
    int64_t w, h;
    orc_orthotope_dims(spec, level, &w, &h);
    if (ox < 0 || oy < 0 || ox >= w || oy >= h) return NBB_ERR_OUT_OF_RANGE;
    int64_t dx = ox, dy = oy, scale = 1, px = 0, py = 0;
    for (int mu = 1; mu <= level; ++mu) {
        int beta;
        if (mu % 2 == 1) {
            beta = (int)(dx % spec->k);
            dx /= spec->k;
        } else {
            beta = (int)(dy % spec->k);
            dy /= spec->k;
        }
        px += spec->offset_x[beta] * scale;
        py += spec->offset_y[beta] * scale;
        scale *= spec->s;
    }
    *x = px;
    *y = py;
    return NBB_OK;
}

int orc_lambda_inverse(const nbb_spec* spec, int level, int64_t x, int64_t y, int64_t* ox,
                       int64_t* oy) {                                       /* :113-148 */
    if (level < 0) return NBB_ERR_INVALID_ARGUMENT;
    const int64_t n = orc_side_length(spec, level);
    if (x < 0 || y < 0 || x >= n || y >= n) return NBB_ERR_OUT_OF_RANGE;
    int64_t scale = n / spec->s, wx = 0, wy = 0;
    for (int mu = level; mu >= 1; --mu) {
        const int cx = (int)(x / scale), cy = (int)(y / scale);
        const int beta = replica_at(spec, cx, cy);
        if (beta < 0) return NBB_ERR_DOMAIN;
        const int64_t digit_scale = (int64_t)ipow_u((uint64_t)spec->k, (mu + 1) / 2 - 1);
        if (mu % 2 == 1) wx += beta * digit_scale; else wy += beta * digit_scale;
        x -= cx * scale;
        y -= cy * scale;
        scale /= spec->s;
    }
    *ox = wx;
    *oy = wy;
    return NBB_OK;
}

void orc_lambda_coords(const nbb_spec* spec, int level, int64_t* xy) {
    int64_t w, h;
    orc_orthotope_dims(spec, level, &w, &h);
    size_t o = 0;
    for (int64_t oy = 0; oy < h; ++oy) {
        for (int64_t ox = 0; ox < w; ++ox, ++o) {
            orc_lambda_map(spec, level, ox, oy, &xy[2 * o], &xy[2 * o + 1]);
        }
    }
}

static int level_for_size(int64_t n, int s) {                 /* fractal.cpp:27-45 */
    if (n < 1) return -1;
    int level = 0;
    while (n > 1) {
        if (n % s != 0) return -1;
        n /= s;
        ++level;
    }
    return level;
}

/* Linearised further unrolling (block_map.cpp:25-37). */
static int unrolled_local_cell(const nbb_spec* spec, int r_t, int rho, int64_t tx, int64_t ty,
                               int64_t* x, int64_t* y) {
    const uint64_t members = ipow_u((uint64_t)spec->k, r_t);
    const uint64_t rank = (uint64_t)ty * (uint64_t)rho + (uint64_t)tx;
    if (rank >= members) return 0;
    int64_t w, h;
    orc_orthotope_dims(spec, r_t, &w, &h);
    orc_lambda_map(spec, r_t, (int64_t)(rank % (uint64_t)w), (int64_t)(rank / (uint64_t)w), x, y);
    return 1;
}

int orc_map_thread(const nbb_spec* spec, int r, int rho, int64_t ox, int64_t oy, int64_t tx,
                   int64_t ty, int strategy, int64_t* x, int64_t* y) { /* :208-236 */
    const int r_t = level_for_size(rho, spec->s);
    const int r_b = r - r_t;
    int64_t px, py, lx = 0, ly = 0;
    orc_lambda_map(spec, r_b, ox, oy, &px, &py);
    int active;
    if (strategy == NBB_STRATEGY_SUBBOX) {
        active = orc_is_member(spec, r_t, tx, ty);
        lx = tx;
        ly = ty;
    } else {
        active = unrolled_local_cell(spec, r_t, rho, tx, ty, &lx, &ly); /* lut == memoised unroll */
    }
    if (!active) return 0;
    *x = px * rho + lx;
    *y = py * rho + ly;
    return 1;
}

/* ---- sim-harness workloads (dispatch.cpp) ---------------------------------- */
/* random_member_grid (dispatch.cpp:133-149): members in row-major order draw
 * rng() % modulus. For the gasket, the members of row y are the submasks x of y
 * (App. A.3), enumerated in increasing order. */
void orc_random_member_grid(const nbb_spec* spec, int r, uint64_t seed, uint64_t modulus,
                            int64_t* out) {
    const int64_t n = orc_side_length(spec, r);
    memset(out, 0, (size_t)(n * n) * sizeof(int64_t));
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    if (is_gasket(spec)) {
        for (int64_t y = 0; y < n; ++y) {
            int64_t x = 0;
            do {
                out[y * n + x] = (int64_t)(orc_mt64_next(&g) % modulus);
                x = (x - y) & y;
            } while (x != 0);
        }
        return;
    }
    for (int64_t y = 0; y < n; ++y)
        for (int64_t x = 0; x < n; ++x)
            if (orc_is_member(spec, r, x, y)) out[y * n + x] = (int64_t)(orc_mt64_next(&g) % modulus);
}

void orc_single_write(const nbb_spec* spec, int r, int64_t* out) {  /* dispatch.cpp:481-488 */
    const int64_t n = orc_side_length(spec, r);
    for (int64_t y = 0; y < n; ++y)
        for (int64_t x = 0; x < n; ++x) out[y * n + x] = member(spec, r, x, y) ? 1 : 0;
}

/* Σ over member cells (dispatch.cpp:490-515; non-members ignored, App. B.4).
 * Integer + is associative mod 2^64, so the fixed pairwise tree of
 * dispatch.cpp:501-513 and this sequential sum give the same bits. */
int64_t orc_reduction(const nbb_spec* spec, int r, const int64_t* grid) {
    const int64_t n = orc_side_length(spec, r);
    uint64_t sum = 0;
    for (int64_t y = 0; y < n; ++y)
        for (int64_t x = 0; x < n; ++x)
            if (member(spec, r, x, y)) sum += (uint64_t)grid[y * n + x];
    return (int64_t)sum;
}

/* Dense masked automaton (tests/test_dispatch.cpp:42-64, dispatch.cpp:533-549). */
void orc_ca_step(const nbb_spec* spec, int r, const int64_t* src, int64_t* dst, uint16_t birth,
                 uint16_t survive) {
    const int64_t n = orc_side_length(spec, r);
    for (int64_t y = 0; y < n; ++y) {
        for (int64_t x = 0; x < n; ++x) {
            if (!member(spec, r, x, y)) {
                dst[y * n + x] = 0;
                continue;
            }
            int live = 0;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    if (dx == 0 && dy == 0) continue;
                    const int64_t nx = x + dx, ny = y + dy;
                    if (member(spec, r, nx, ny) && src[ny * n + nx] != 0) ++live;
                }
            const uint16_t bit = (uint16_t)(1u << live);
            dst[y * n + x] = (((src[y * n + x] != 0) ? survive : birth) & bit) ? 1 : 0;
        }
    }
}

int64_t orc_ca_compact_check(const nbb_spec* spec, int r, const int64_t* src, const int64_t* dst,
                             const int64_t* offsets, int64_t count, uint16_t birth, uint16_t survive) {
    int64_t W, H, bad = 0;
    orc_orthotope_dims(spec, r, &W, &H);
    for (int64_t i = 0; i < count; ++i) {
        const int64_t c = offsets[i];
        int64_t x, y;
        if (c < 0 || c >= W * H || orc_lambda_map(spec, r, c % W, c / W, &x, &y) != 0) {
            ++bad;
            continue;
        }
        int live = 0;
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                if (dx == 0 && dy == 0) continue;
                int64_t ox, oy;
                if (member(spec, r, x + dx, y + dy) &&
                    orc_lambda_inverse(spec, r, x + dx, y + dy, &ox, &oy) == 0 && src[oy * W + ox] != 0)
                    ++live;
            }
        const uint16_t bit = (uint16_t)(1u << live);
        const int64_t want = (((src[c] != 0) ? survive : birth) & bit) ? 1 : 0;
        if (dst[c] != want) ++bad;
    }
    return bad;
}

/* λ and λ⁻¹ of the gasket (k = 3, s = 2, offsets (0,0) (0,1) (1,1)): the digit loops of
 * block_map.cpp:77-111 / :113-148 with the spec's constants folded in (same arithmetic as
 * orc_lambda_map / orc_lambda_inverse, which test_oracle.py pins to the reference). */
static void gasket_lambda(int level, int64_t ox64, int64_t oy64, int64_t* x, int64_t* y) {
    static const int tx[3] = {0, 0, 1}, ty[3] = {0, 1, 1};
    uint32_t ox = (uint32_t)ox64, oy = (uint32_t)oy64;  /* < 3^10 for level <= 20 */
    int64_t px = 0, py = 0;
    for (int mu = 1; mu <= level; ++mu) {
        int beta;
        if (mu & 1) {
            beta = (int)(ox % 3);
            ox /= 3;
        } else {
            beta = (int)(oy % 3);
            oy /= 3;
        }
        px += (int64_t)tx[beta] << (mu - 1);
        py += (int64_t)ty[beta] << (mu - 1);
    }
    *x = px;
    *y = py;
}

static void gasket_lambda_inverse(int level, int64_t x, int64_t y, int64_t* ox, int64_t* oy) {
    int64_t wx = 0, wy = 0, dx = 1, dy = 1;
    for (int mu = 1; mu <= level; ++mu) {  /* digit of level mu: replica (bit_x, bit_y) */
        const int bx = (int)((x >> (mu - 1)) & 1), by = (int)((y >> (mu - 1)) & 1);
        const int beta = bx + by;           /* (0,0) -> 0, (0,1) -> 1, (1,1) -> 2 */
        if (mu & 1) {
            wx += beta * dx;
            dx *= 3;
        } else {
            wy += beta * dy;
            dy *= 3;
        }
    }
    *ox = wx;
    *oy = wy;
}

/* ---- whole-trajectory checker on the compact state (full-size C3 / C5 parity) ---------------
 * random_member_grid (dispatch.cpp:133-149) written straight into compact order: the reference
 * walks the n x n grid row-major and draws rng() % modulus for each member cell; for the gasket
 * the members of row y are the submasks x of y, visited in increasing order by x = (x - y) & y
 * (SURVEY App. A.3). Each value lands at the cell's compact offset ωy·W + ωx, ω = λ⁻¹(x, y)
 * (block_map.cpp:113-148), i.e. CompactGrid of the reference's Grid (block_map.cpp:245-263). */
int orc_random_member_compact(const nbb_spec* spec, int r, uint64_t seed, uint64_t modulus,
                              int64_t* out) {
    if (!is_gasket(spec) || r < 0 || r > 20 || modulus == 0) return NBB_ERR_INVALID_ARGUMENT;
    const int64_t n = (int64_t)1 << r;
    int64_t W, H;
    orc_orthotope_dims(spec, r, &W, &H);
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    for (int64_t y = 0; y < n; ++y) {
        int64_t x = 0;
        do {
            int64_t ox, oy;
            gasket_lambda_inverse(r, x, y, &ox, &oy);
            out[oy * W + ox] = (int64_t)(orc_mt64_next(&g) % modulus);
            x = (x - y) & y;
        } while (x != 0);
    }
    return NBB_OK;
}

/* run_ca (dispatch.cpp:517-557) on a CompactGrid: `steps` double-buffered steps of the
 * reference rule (dispatch.cpp:530-550: live = #member Moore neighbours with value != 0,
 * next = ((alive ? survive : birth) >> live) & 1, non-members stay 0), returned as the compact
 * values of the final grid. The state between steps is the alive bit of every embedded cell
 * (one bit per cell, n²/8 bytes: 512 MiB at r = 16, 2 GiB at r = 17) — exact because the rule
 * reads only `value != 0` and writes 0/1; the compact <-> embedded mapping is the reference's
 * λ (block_map.cpp:77-111), evaluated once per cell at entry and exit. steps == 0 copies. */
static int bit_at(const uint64_t* b, int64_t n, int64_t x, int64_t y) {
    const uint64_t i = (uint64_t)(y * n + x);
    return (int)((b[i >> 6] >> (i & 63u)) & 1u);
}

int orc_ca_compact(const nbb_spec* spec, int r, const int64_t* src, int steps, uint16_t birth,
                   uint16_t survive, int64_t* out) {
    if (!is_gasket(spec) || r < 0 || r > 18 || steps < 0) return NBB_ERR_INVALID_ARGUMENT;
    const int64_t n = (int64_t)1 << r;
    int64_t W, H;
    orc_orthotope_dims(spec, r, &W, &H);
    const int64_t total = W * H;
    if (steps == 0) {
        memcpy(out, src, (size_t)total * sizeof(int64_t));
        return NBB_OK;
    }
    const size_t words = (size_t)((n * n + 63) / 64);
    uint64_t* a = (uint64_t*)calloc(words, sizeof(uint64_t));
    uint64_t* b = (uint64_t*)calloc(words, sizeof(uint64_t));
    if (!a || !b) {
        free(a);
        free(b);
        return NBB_ERR_RESOURCE;
    }
    for (int64_t c = 0; c < total; ++c) {
        int64_t x, y;
        gasket_lambda(r, c % W, c / W, &x, &y);
        if (src[c] != 0) {
            const uint64_t i = (uint64_t)(y * n + x);
            a[i >> 6] |= 1ull << (i & 63u);
        }
    }
    for (int s = 0; s < steps; ++s) {
        memset(b, 0, words * sizeof(uint64_t));
        for (int64_t y = 0; y < n; ++y) {
            int64_t x = 0;
            do {  /* the member cells of row y */
                int live = 0;
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        if (dx == 0 && dy == 0) continue;
                        const int64_t nx = x + dx, ny = y + dy;
                        if (orc_gasket_bit_test(r, nx, ny) && bit_at(a, n, nx, ny)) ++live;
                    }
                const uint16_t rule = bit_at(a, n, x, y) ? survive : birth;
                if ((rule >> live) & 1u) {
                    const uint64_t i = (uint64_t)(y * n + x);
                    b[i >> 6] |= 1ull << (i & 63u);
                }
                x = (x - y) & y;
            } while (x != 0);
        }
        uint64_t* t = a;
        a = b;
        b = t;
    }
    for (int64_t c = 0; c < total; ++c) {
        int64_t x, y;
        gasket_lambda(r, c % W, c / W, &x, &y);
        out[c] = bit_at(a, n, x, y);
    }
    free(a);
    free(b);
    return NBB_OK;
}

void orc_ca(const nbb_spec* spec, int r, const int64_t* initial, int steps, uint16_t birth,
            uint16_t survive, int64_t* out) {
    const int64_t n = orc_side_length(spec, r);
    const size_t bytes = (size_t)(n * n) * sizeof(int64_t);
    memcpy(out, initial, bytes);
    if (steps <= 0) return;
    int64_t* tmp = (int64_t*)malloc(bytes);
    for (int s = 0; s < steps; ++s) {
        orc_ca_step(spec, r, out, tmp, birth, survive);
        memcpy(out, tmp, bytes);
    }
    free(tmp);
}

/* ---- config validation and counters ----------------------------------------- */
static int fail(char* msg, size_t len, int code, const char* text) {
    if (msg && len) snprintf(msg, len, "%s", text);
    return code;
}

int orc_validate(const nbb_config* cfg, char* msg, size_t len) {   /* dispatch.cpp:50-114 */
    char buf[256];
    const int rho = cfg->rho;
    if (!(rho == 1 || rho == 2 || rho == 4 || rho == 8 || rho == 16 || rho == 32)) {
        snprintf(buf, sizeof buf, "rho %d is not one of 1, 2, 4, 8, 16, 32", rho);
        return fail(msg, len, NBB_ERR_INVALID_ARGUMENT, buf);
    }
    if (cfg->r < 0) return fail(msg, len, NBB_ERR_INVALID_ARGUMENT, "negative scale level");
    if (cfg->workers < 1) return fail(msg, len, NBB_ERR_INVALID_ARGUMENT, "workers must be >= 1");
    const int64_t n = orc_side_length(&cfg->spec, cfg->r);
    if (n % rho != 0) {
        snprintf(buf, sizeof buf, "rho %d does not divide n = %lld", rho, (long long)n);
        return fail(msg, len, NBB_ERR_INVALID_ARGUMENT, buf);
    }
    if (cfg->mode == NBB_MODE_BB) {
        if (cfg->backend != NBB_BACKEND_DIRECT)
            return fail(msg, len, NBB_ERR_INVALID_ARGUMENT, "lambda backends apply to lambda mode only");
        return NBB_OK;
    }
    const int r_t = level_for_size(rho, cfg->spec.s);
    if (r_t < 0) {
        snprintf(buf, sizeof buf, "level_for_size: %d is not a power of %d", rho, cfg->spec.s);
        return fail(msg, len, NBB_ERR_INVALID_ARGUMENT, buf);
    }
    if (r_t > cfg->r) {
        snprintf(buf, sizeof buf, "block geometry: rho %d exceeds the embedding side %lld", rho,
                 (long long)n);
        return fail(msg, len, NBB_ERR_INVALID_ARGUMENT, buf);
    }
    const int r_b = cfg->r - r_t;
    switch (cfg->backend) {
        case NBB_BACKEND_MMA1:
            if (r_b > 16) {
                snprintf(buf, sizeof buf, "variant 1 encodes at most 16 levels, r_b = %d", r_b);
                return fail(msg, len, NBB_ERR_INVALID_ARGUMENT, buf);
            }
            break;
        case NBB_BACKEND_MMA2: {
            if (rho < 2)
                return fail(msg, len, NBB_ERR_INVALID_ARGUMENT,
                            "variant 2 needs sub-blocks of edge rho/2 >= 1");
            const int sub_rt = level_for_size(rho / 2, cfg->spec.s);
            if (sub_rt < 0) {
                snprintf(buf, sizeof buf, "variant 2 sub-block edge %d is not a power of s = %d",
                         rho / 2, cfg->spec.s);
                return fail(msg, len, NBB_ERR_INVALID_ARGUMENT, buf);
            }
            if (cfg->r - sub_rt > 16)
                return fail(msg, len, NBB_ERR_INVALID_ARGUMENT, "variant 2 encodes at most 16 levels");
            break;
        }
        case NBB_BACKEND_MMA3:
            if (rho != 16) {
                snprintf(buf, sizeof buf, "variant 3 runs at rho = 16 only, got %d", rho);
                return fail(msg, len, NBB_ERR_INVALID_ARGUMENT, buf);
            }
            if (cfg->strategy != NBB_STRATEGY_SUBBOX)
                return fail(msg, len, NBB_ERR_INVALID_ARGUMENT,
                            "variant 3 emits sub-box thread coordinates; use the subbox strategy");
            if (r_b > 16)
                return fail(msg, len, NBB_ERR_INVALID_ARGUMENT, "variant 3 encodes at most 16 levels");
            break;
        default:
            break;
    }
    return NBB_OK;
}

/* make_plan (dispatch.cpp:165-197) + the tallies of launch_impl (:240-466),
 * summed in closed form. */
int orc_plan_report(const nbb_config* cfg, nbb_report* out) {
    const int rc = orc_validate(cfg, NULL, 0);
    if (rc != NBB_OK) return rc;
    memset(out, 0, sizeof *out);
    snprintf(out->spec_name, sizeof out->spec_name, "%s", cfg->spec.name);
    out->r = cfg->r;
    out->rho = cfg->rho;
    out->mode = cfg->mode;
    out->strategy = cfg->strategy;
    out->backend = cfg->backend;
    const uint64_t k = (uint64_t)cfg->spec.k;
    const uint64_t members = ipow_u(k, cfg->r);
    if (cfg->mode == NBB_MODE_BB) {
        const uint64_t n = (uint64_t)orc_side_length(&cfg->spec, cfg->r);
        const uint64_t nb = n / (uint64_t)cfg->rho;
        out->blocks_launched = nb * nb;
        out->threads_launched = n * n;
        out->threads_active = members;
        out->threads_wasted = n * n - members;
        out->map_ops = n * n;
        out->map_levels = 0;
        return NBB_OK;
    }
    const int r_t = level_for_size(cfg->rho, cfg->spec.s);
    int map_level, local_level;
    uint64_t edge, gw, gh, inrange;
    if (cfg->backend == NBB_BACKEND_MMA2) {
        local_level = level_for_size(cfg->rho / 2, cfg->spec.s);
        map_level = cfg->r - local_level;
        int64_t sw, sh;
        orc_orthotope_dims(&cfg->spec, map_level, &sw, &sh);
        gw = (uint64_t)((sw + 1) / 2 * 2);
        gh = (uint64_t)((sh + 1) / 2 * 2);
        inrange = (uint64_t)(sw * sh);
        edge = (uint64_t)cfg->rho / 2;
    } else {
        local_level = r_t;
        map_level = cfg->r - r_t;
        int64_t w, h;
        orc_orthotope_dims(&cfg->spec, map_level, &w, &h);
        gw = (uint64_t)w;
        gh = (uint64_t)h;
        inrange = gw * gh;
        edge = (uint64_t)cfg->rho;
    }
    const uint64_t local_members = ipow_u(k, local_level);
    out->blocks_launched = gw * gh;
    out->threads_launched = gw * gh * edge * edge;
    out->threads_active = inrange * local_members;
    out->threads_wasted = out->threads_launched - out->threads_active;
    uint64_t ops = inrange * (uint64_t)map_level;
    switch (cfg->strategy) {
        case NBB_STRATEGY_SUBBOX: ops += inrange * edge * edge; break;
        case NBB_STRATEGY_UNROLL: ops += inrange * local_members * (uint64_t)local_level; break;
        case NBB_STRATEGY_LUT: ops += local_members * (uint64_t)local_level; break;
        default: break;
    }
    out->map_ops = ops;
    out->map_levels = map_level;
    return NBB_OK;
}

uint64_t orc_launch_block_count(const nbb_config* cfg) {
    nbb_report r;
    if (orc_plan_report(cfg, &r) != NBB_OK) return 0;
    return r.blocks_launched;
}

double orc_work_quotient(const nbb_report* bb, const nbb_report* lam, int weighted) { /* :559-572 */
    double denom = (double)lam->threads_launched;
    if (weighted) denom *= (double)(lam->map_levels > 1 ? lam->map_levels : 1);
    return (double)bb->threads_launched / denom;
}

void orc_csv_row(const nbb_report* r, char* buf, size_t len) {  /* dispatch.cpp:120-127 */
    static const char* modes[] = {"bb", "lambda"};
    static const char* strategies[] = {"unroll", "lut", "subbox"};
    static const char* backends[] = {"direct", "mma1", "mma2", "mma3"};
    snprintf(buf, len, "%s,%d,%d,%s,%s,%s,%llu,%llu,%llu,%llu,%llu,%llu", r->spec_name, r->r, r->rho,
             modes[r->mode], strategies[r->strategy], backends[r->backend],
             (unsigned long long)r->blocks_launched, (unsigned long long)r->threads_launched,
             (unsigned long long)r->threads_active, (unsigned long long)r->threads_wasted,
             (unsigned long long)r->map_ops, (unsigned long long)r->micros);
}

/* ---- mma-encode (mma.cpp) ------------------------------------------------------ */
#define F 16
void orc_mma_eval(const double* a, const double* b, const double* c, double* d) { /* :18-32 */
    memcpy(d, c, sizeof(double) * F * F);
    for (int i = 0; i < F; ++i)
        for (int m = 0; m < F; ++m) {
            const double av = a[i * F + m];
            if (av == 0.0) continue;
            for (int j = 0; j < F; ++j) d[i * F + j] += av * b[m * F + j];
        }
}

int orc_encode_variant1(const nbb_spec* spec, int level, int64_t ox, int64_t oy, double* a,
                        double* b) {                                      /* mma.cpp:34-47 */
    if (level > F) return NBB_ERR_RESOURCE;
    int64_t x, y;
    const int rc = orc_lambda_map(spec, level, ox, oy, &x, &y);
    if (rc != NBB_OK) return rc;
    memset(a, 0, sizeof(double) * F * F);
    memset(b, 0, sizeof(double) * F * F);
    double power = 1.0;
    for (int mu = 1; mu <= level; ++mu) {
        a[mu - 1] = power;
        power *= spec->s;
        const int beta = orc_beta_index(spec, ox, oy, mu);
        b[(mu - 1) * F + 0] = spec->offset_x[beta];
        b[(mu - 1) * F + 1] = spec->offset_y[beta];
    }
    return NBB_OK;
}

int orc_encode_variant2(const nbb_spec* spec, int level, const int64_t* omegas, int count,
                        double* a, double* b, int32_t* active) {         /* mma.cpp:49-77 */
    if (level > F || count > 8) return NBB_ERR_RESOURCE;
    memset(a, 0, sizeof(double) * F * F);
    memset(b, 0, sizeof(double) * F * F);
    for (int i = 0; i < 8; ++i) active[i] = 0;
    int64_t w, h;
    orc_orthotope_dims(spec, level, &w, &h);
    double power = 1.0;
    for (int mu = 1; mu <= level; ++mu) {
        a[mu - 1] = power;
        power *= spec->s;
    }
    for (int i = 0; i < count; ++i) {
        const int64_t ox = omegas[2 * i], oy = omegas[2 * i + 1];
        if (ox < 0 || oy < 0 || ox >= w || oy >= h) continue;
        active[i] = 1;
        for (int mu = 1; mu <= level; ++mu) {
            const int beta = orc_beta_index(spec, ox, oy, mu);
            b[(mu - 1) * F + 2 * i] = spec->offset_x[beta];
            b[(mu - 1) * F + 2 * i + 1] = spec->offset_y[beta];
        }
    }
    return NBB_OK;
}

int orc_encode_variant3(const nbb_spec* spec, int r, int rho, int64_t ox, int64_t oy, double* a,
                        double* bx, double* cx, double* by, double* cy) { /* mma.cpp:91-118 */
    if (rho != F) return NBB_ERR_INVALID_ARGUMENT;
    const int r_t = level_for_size(rho, spec->s);
    const int r_b = r - r_t;
    if (r_b > F) return NBB_ERR_RESOURCE;
    int64_t x, y;
    const int rc = orc_lambda_map(spec, r_b, ox, oy, &x, &y);
    if (rc != NBB_OK) return rc;
    memset(a, 0, sizeof(double) * F * F);
    memset(bx, 0, sizeof(double) * F * F);
    memset(by, 0, sizeof(double) * F * F);
    double power = rho;
    for (int mu = 1; mu <= r_b; ++mu) {
        for (int i = 0; i < F; ++i) a[i * F + mu - 1] = power;
        power *= spec->s;
        const int beta = orc_beta_index(spec, ox, oy, mu);
        for (int j = 0; j < F; ++j) {
            bx[(mu - 1) * F + j] = spec->offset_x[beta];
            by[(mu - 1) * F + j] = spec->offset_y[beta];
        }
    }
    for (int i = 0; i < F; ++i)
        for (int j = 0; j < F; ++j) {
            cx[i * F + j] = i;
            cy[i * F + j] = j;
        }
    return NBB_OK;
}
