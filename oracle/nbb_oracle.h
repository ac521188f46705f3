/*
 * nbb_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's hot-path algorithm, used only by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * CHECKER. It is never linked into, loaded by, or called from the product
 * library (paper_2004_13475_b200/libnbbgpu.so). Each function cites the
 * reference file:line (under /root/reference/proj) it restates.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against
 *  - the reference itself, compiled unmodified into oracle/_ref/libnbbref.so, and
 *  - the golden digests of SURVEY.md App. B (committed in tests/golden/).
 */
#ifndef NBB_ORACLE_H
#define NBB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "nbb_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* std::mt19937_64 ([rand.eng.mers], the engine behind dispatch.cpp:140). */
typedef struct orc_mt64 {
    uint64_t mt[312];
    int idx;
} orc_mt64;
void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);

uint64_t orc_fnv1a64(const void* data, size_t bytes);

int64_t orc_side_length(const nbb_spec* spec, int level);          /* fractal.cpp:165-171 */
void orc_orthotope_dims(const nbb_spec* spec, int level, int64_t* w, int64_t* h); /* :181-192 */
int orc_is_member(const nbb_spec* spec, int level, int64_t x, int64_t y);          /* :194-214 */
int orc_gasket_bit_test(int level, int64_t x, int64_t y);       /* tests/acceptance.cpp:88-102 */

/* block_map.cpp:57-65 / :77-111 / :113-148 / :150-155 */
int orc_beta_index(const nbb_spec* spec, int64_t ox, int64_t oy, int mu);
int orc_lambda_map(const nbb_spec* spec, int level, int64_t ox, int64_t oy, int64_t* x, int64_t* y);
int orc_lambda_inverse(const nbb_spec* spec, int level, int64_t x, int64_t y, int64_t* ox,
                       int64_t* oy);
void orc_lambda_coords(const nbb_spec* spec, int level, int64_t* xy);
/* map_thread (block_map.cpp:208-236); returns 1 if active */
int orc_map_thread(const nbb_spec* spec, int r, int rho, int64_t ox, int64_t oy, int64_t tx,
                   int64_t ty, int strategy, int64_t* x, int64_t* y);

/* dispatch.cpp:133-149 (member cells in row-major order get rng() % modulus) */
void orc_random_member_grid(const nbb_spec* spec, int r, uint64_t seed, uint64_t modulus,
                            int64_t* out);

/* Workload semantics (dispatch.cpp:481-557, tests/test_dispatch.cpp:28-64). */
void orc_single_write(const nbb_spec* spec, int r, int64_t* out);
int64_t orc_reduction(const nbb_spec* spec, int r, const int64_t* grid);
void orc_ca_step(const nbb_spec* spec, int r, const int64_t* src, int64_t* dst, uint16_t birth,
                 uint16_t survive);
/* One CA step checked on the compact state (CompactGrid, block_map.hpp:82-110: value(ω) =
 * embedded(λ(ω)) at offset ωy·W + ωx): for each sampled offset, the reference rule
 * (dispatch.cpp:530-550) over the cell's member Moore neighbours located by λ⁻¹. Returns the
 * number of sampled offsets whose dst value differs (size-independent full-size check). */
int64_t orc_ca_compact_check(const nbb_spec* spec, int r, const int64_t* src, const int64_t* dst,
                             const int64_t* offsets, int64_t count, uint16_t birth, uint16_t survive);
/* Full-size trajectory checker on the compact state (gasket only): random_member_grid
 * (dispatch.cpp:133-149) emitted in compact order (λ⁻¹ per member, block_map.cpp:113-148), and
 * run_ca (dispatch.cpp:517-557) from a compact state to a compact state through a one-bit-per-cell
 * embedded raster. Return nbb_status. */
int orc_random_member_compact(const nbb_spec* spec, int r, uint64_t seed, uint64_t modulus,
                              int64_t* out);
int orc_ca_compact(const nbb_spec* spec, int r, const int64_t* src, int steps, uint16_t birth,
                   uint16_t survive, int64_t* out);
/* steps == 0 copies the input unchanged (B.4) */
void orc_ca(const nbb_spec* spec, int r, const int64_t* initial, int steps, uint16_t birth,
            uint16_t survive, int64_t* out);

/* Config validation (dispatch.cpp:50-114); message into msg. Returns nbb_status. */
int orc_validate(const nbb_config* cfg, char* msg, size_t len);
/* make_plan + launch counters in closed form (dispatch.cpp:165-197, 240-466) */
int orc_plan_report(const nbb_config* cfg, nbb_report* out);
uint64_t orc_launch_block_count(const nbb_config* cfg);
double orc_work_quotient(const nbb_report* bb, const nbb_report* lam, int weighted);
void orc_csv_row(const nbb_report* r, char* buf, size_t len);

/* mma.cpp:18-118 (16x16 row-major double fragments) */
void orc_mma_eval(const double* a, const double* b, const double* c, double* d);
int orc_encode_variant1(const nbb_spec* spec, int level, int64_t ox, int64_t oy, double* a,
                        double* b);
int orc_encode_variant2(const nbb_spec* spec, int level, const int64_t* omegas, int count,
                        double* a, double* b, int32_t* active);
int orc_encode_variant3(const nbb_spec* spec, int r, int rho, int64_t ox, int64_t oy, double* a,
                        double* bx, double* cx, double* by, double* cy);

#ifdef __cplusplus
}
#endif

#endif
