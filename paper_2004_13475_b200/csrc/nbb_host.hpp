// nbb_host.hpp — host-side logic of the engine (no CUDA): config validation,
// launch planning, closed-form work counters, CSV rows, seeded grids.
// Mirrors the reference's dispatch/fractal/block_map host code paths
// (dispatch.cpp:50-197, 116-149, 559-572; fractal.cpp:12-45, 165-192) with the
// same names, argument meaning and error text; errors are reported as
// (nbb_status, message) instead of C++ exceptions so they cross the C ABI.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "nbb_gpu.h"

namespace nbbhost {

struct Error {
    int code = NBB_OK;
    std::string msg;
    bool ok() const { return code == NBB_OK; }
};

inline Error err(int code, std::string msg) { return Error{code, std::move(msg)}; }

bool is_gasket(const nbb_spec& s);
Error require_gasket(const nbb_spec& s);
// FractalSpec constructor checks (fractal.cpp:47-78)
Error validate_spec(const nbb_spec& s);
Error checked_pow(uint64_t base, int exp, uint64_t* out);    // fractal.cpp:12-25
Error level_for_size(int64_t n, int s, int* level);          // fractal.cpp:27-45
Error side_length(const nbb_spec& s, int level, int64_t* n); // fractal.cpp:165-171
Error orthotope_dims(const nbb_spec& s, int level, int64_t* w, int64_t* h); // :181-192

// DispatchConfig::validate (dispatch.cpp:50-114)
Error validate(const nbb_config& c);

// make_plan (dispatch.cpp:153-197)
struct Plan {
    int64_t n = 1;
    int64_t gw = 1, gh = 1;  // launch grid (blocks or mma2 sub-block slots)
    int edge = 1;
    int map_level = 0;
    int local_level = 0;
    int64_t local_w = 1;
    uint64_t local_members = 1;
    int64_t sub_w = -1, sub_h = -1;  // mma2 in-range bounds
    uint64_t blocks() const { return (uint64_t)gw * (uint64_t)gh; }
};
Error make_plan(const nbb_config& c, Plan* p);

// WorkReport of one launch in closed form
Error plan_report(const nbb_config& c, nbb_report* r);

// MemberMask budget (fractal.cpp:249-256): n^2 cells must fit max_cells
Error member_mask_budget(const nbb_spec& s, int level, uint64_t max_cells);

std::string csv_row(const nbb_report& r);                 // dispatch.cpp:120-127
const char* csv_header();                                 // dispatch.cpp:116-118
Error work_quotient(const nbb_report& bb, const nbb_report& lam, bool weighted, double* q);

// random_member_grid (dispatch.cpp:133-149) — gasket rows enumerated as submasks.
Error random_member_values(const nbb_spec& s, int r, uint64_t seed, uint64_t modulus, int64_t* out);
Error random_member_grid(const nbb_spec& s, int r, uint64_t seed, uint64_t modulus,
                         uint64_t max_cells, int64_t* grid);

// LocalCellTable (block_map.cpp:197-206): edge*edge (x, y) int16 pairs, -1 = spare
void local_cell_table(const nbb_spec& s, int edge, int16_t* out);

// NBBC compact file (block_map.cpp:284-362)
Error write_compact(const char* path, const nbb_spec& s, int level, const int64_t* values);
Error read_compact(const char* path, const nbb_spec& s, int* level, int64_t* values, uint64_t capacity);

// ---- halo slots of the multi-step compact CA pass (compact_pass.cuh) ----------------------
// The member cells outside a ρ = 32 gasket tile that can reach one of its members within K <= 4
// steps: the chain layers H_1 (member neighbours of the tile's members), H_2 (member neighbours
// of H_1 outside the tile), ... found by brute force over every tile of level 13 (the 3 x 3
// tile neighbourhoods repeat by self-similarity), each position labelled with its smallest
// layer d over all tiles and sorted by d, so the slots of a K-step pass are a prefix
// (8 / 22 / 36 / 58 for K = 1..4). Per slot: tile-local position, the neighbouring tile it lies
// in (0..7, (dy+1)*3 + dx+1 with the centre skipped), its local compact index there, the
// other slots adjacent to it (bit mask), and — for H_1 — its in-tile member neighbours as bit
// masks over tile rows 0, 30 and 31 (the only rows they touch).
constexpr int kPassMaxK = 4;
constexpr int kPassSlots = 64;
struct HaloSlots {
    int32_t count;                 // slots with layer <= kPassMaxK
    int32_t upto[kPassMaxK + 1];   // upto[d] = slots with layer <= d
    int8_t x[kPassSlots], y[kPassSlots];
    uint8_t dir[kPassSlots];       // neighbouring tile, 0..7
    uint8_t li[kPassSlots];        // local compact index (ωy_l * 27 + ωx_l) in that tile
    uint32_t nb_lo[kPassSlots], nb_hi[kPassSlots];  // adjacent slots
    uint32_t m0[8], m30[8], m31[8];                 // H_1: in-tile neighbours in rows 0, 30, 31
};
Error halo_slots(HaloSlots* out);

// The same layers for the multi-step passes over the compact state: positions sorted by layer,
// and per neighbouring tile the slots lying in it, sorted by layer (the halo loads walk one
// neighbour at a time). 8 / 22 / 36 / 58 / 76 / 104 / 128 / 166 / 184 / 212 / 240 / 288 slots for
// K = 1..12, at most 54 of them in one neighbouring tile.
template <int MAXK, int SLOTS, int DIRMAX>
struct SlotTable {
    static constexpr int kMaxK = MAXK, kSlots = SLOTS, kDirMax = DIRMAX;
    int32_t count;                      // slots with layer <= MAXK
    int32_t upto[MAXK + 1];             // upto[d] = slots with layer <= d
    int8_t x[SLOTS], y[SLOTS];
    uint8_t layer[SLOTS];
    uint8_t li[SLOTS];                  // local compact index in the neighbouring tile
    uint8_t dir_of[SLOTS];              // neighbouring tile, 0..7 ((dy+1)*3 + dx+1, centre skipped)
    uint16_t by_dir[8][DIRMAX];         // per neighbouring tile: its slots, by layer
    int32_t dir_upto[8][MAXK + 1];      // per neighbouring tile: slots with layer <= d
};
// the tile-sliced pass (compact_sliced.cuh): up to 8 steps
constexpr int kSliceMaxK = 8;
constexpr int kSliceSlots = 192;
using SliceSlots = SlotTable<kSliceMaxK, kSliceSlots, kSliceSlots>;
Error slice_slots(SliceSlots* out);
// the cluster pass (compact_cluster.cuh): up to 12 steps
constexpr int kClMaxK = 12;
constexpr int kClSlots = 320;
constexpr int kClDirSlots = 64;
using ClusterSlots = SlotTable<kClMaxK, kClSlots, kClDirSlots>;
Error cluster_slots(ClusterSlots* out);

// Tiles per rank of the multi-GPU compact CA (the reference's contiguous worker chunks,
// dispatch.cpp:419-427, in the tile order u = ωx_b·Hb + ωy_b): ceil(tiles / world), rounded up to
// whole cluster columns (9·Hb tiles: every rank then owns whole level-3 clusters, the batches of
// compact_cluster.cuh) when r_b >= 3. Results are identical for any split; this one is shared by
// every multi-GPU entry point (peer passes, workers as devices, the NCCL communicator's lists).
inline uint64_t compact_shard_chunk(int rb, uint64_t tiles, uint64_t Hb, int world) {
    if (world < 1) world = 1;
    if (rb >= 3 && Hb % 3 == 0 && tiles % (9 * Hb) == 0) {
        const uint64_t col = 9 * Hb, ncol = tiles / col;
        return ((ncol + (uint64_t)world - 1) / (uint64_t)world) * col;
    }
    return (tiles + (uint64_t)world - 1) / (uint64_t)world;
}
// Halo exchange of the multi-process compact CA (NCCL transport): with `world` ranks owning
// contiguous chunks of compact_shard_chunk ρ = 32 tiles (dispatch.cpp:419-427), recv[j] = the
// compact offsets of rank j's cells that lie in a halo slot of layer <= kmax of one of `rank`'s
// tiles, send[j] = the offsets of `rank`'s cells that rank j needs; sorted, unique. send[j] on
// rank i equals recv[i] on rank j by construction.
Error halo_exchange_lists(int r, int world, int rank, int kmax, std::vector<std::vector<uint32_t>>* send,
                          std::vector<std::vector<uint32_t>>* recv);

// precomputed fast division magic (see common.cuh FastDiv), exact for x < 2^31
void fastdiv_magic(uint32_t d, uint32_t* m, uint32_t* s);

}  // namespace nbbhost
