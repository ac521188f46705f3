/*
 * nbb_gpu.h — C ABI of the B200-native λ(ω) / bounding-box launch engine.
 *
 * Drop-in boundary for the reference's workload entry points
 * (/root/reference/proj/include/nbb/dispatch.hpp). The reference's operator API
 * is `launch(const DispatchConfig&, const Kernel&)` with a host std::function
 * kernel (dispatch.hpp:100-108); a host closure cannot run on the device, so the
 * boundary sits one level up, at the three workloads the reference ships
 * (SURVEY.md §8(b)):
 *
 *   reference (C++, dispatch.hpp)                         replaced by (this header)
 *   -----------------------------------------------------------------------------
 *   DispatchConfig::validate()          dispatch.cpp:50-114  nbb_gpu_validate
 *   launch_block_count(config)          dispatch.cpp:475-479 nbb_gpu_launch_block_count
 *   run_single_write(config)            dispatch.cpp:481-488 nbb_gpu_single_write
 *   run_reduction(config, grid)         dispatch.cpp:490-515 nbb_gpu_reduction
 *   run_ca(config, initial, steps, rule) dispatch.cpp:517-557 nbb_gpu_ca
 *   work_quotient(bb, lambda, weighted) dispatch.cpp:559-572 nbb_gpu_work_quotient
 *   WorkReport::csv_header/csv_row      dispatch.cpp:116-127 nbb_gpu_csv_header / nbb_gpu_report_csv_row
 *   random_member_grid(spec,r,seed,mod) dispatch.cpp:133-149 nbb_gpu_random_member_grid
 *   lambda_map over a whole orthotope   block_map.cpp:77-111 nbb_gpu_lambda_coords
 *
 * plus device-resident variants (`*_dev`) that take device pointers and a
 * cudaStream_t (as void*) so that no PCIe traffic sits inside a timed region.
 *
 * All buffers are plain pointers + sizes; no torch types. Grids are the
 * reference's dense row-major embedding (index = y*n + x, n = 2^r) of int64
 * cells (dispatch.hpp:74-79). Every entry point returns an nbb_status; on
 * failure nbb_gpu_last_error() holds a thread-local message that mirrors the
 * reference's exception text. There is no CPU fallback: without a CUDA device
 * every compute entry point returns NBB_ERR_CUDA.
 */
#ifndef NBB_GPU_H
#define NBB_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NBB_GPU_ABI_VERSION 4  /* 4: nbb_pass_stats.by_steps[13], passes of up to 12 steps */
#define NBB_MAX_REPLICAS 9

/* Status codes; the C++ shim (nbb_gpu.hpp) rethrows the matching std:: type. */
typedef enum nbb_status {
    NBB_OK = 0,
    NBB_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument            */
    NBB_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range                */
    NBB_ERR_RESOURCE = 3,         /* nbb::ResourceError / bad_alloc   */
    NBB_ERR_CUDA = 4,             /* CUDA runtime failure / no device */
    NBB_ERR_NCCL = 5,             /* collective failure               */
    NBB_ERR_DOMAIN = 6,           /* std::domain_error                */
    NBB_ERR_OVERFLOW = 7,         /* std::overflow_error              */
    NBB_ERR_RUNTIME = 8           /* std::runtime_error               */
} nbb_status;

/* MapMode (dispatch.hpp:16) */
enum { NBB_MODE_BB = 0, NBB_MODE_LAMBDA = 1 };
/* IntraBlockStrategy (block_map.hpp:46-50), same enumerator order */
enum { NBB_STRATEGY_UNROLL = 0, NBB_STRATEGY_LUT = 1, NBB_STRATEGY_SUBBOX = 2 };
/* LambdaBackend (dispatch.hpp:17) */
enum { NBB_BACKEND_DIRECT = 0, NBB_BACKEND_MMA1 = 1, NBB_BACKEND_MMA2 = 2, NBB_BACKEND_MMA3 = 3 };
/* Device kernel family (new; not in the reference):
 *  AUTO    — fastest implementation of the requested (mode, strategy, backend)
 *  PERCELL — the paper's one-thread-per-cell blocks of rho x rho threads
 *  TILE    — warp-per-tile, 32-byte-sector vectorised payload (subbox/direct only) */
enum { NBB_KERNEL_AUTO = 0, NBB_KERNEL_PERCELL = 1, NBB_KERNEL_TILE = 2 };

/* FractalSpec (fractal.hpp:53-102). Only the gasket runs on the GPU path. */
typedef struct nbb_spec {
    char name[32];
    int32_t k;                       /* replica count  */
    int32_t s;                       /* scale factor   */
    int32_t offset_x[NBB_MAX_REPLICAS];
    int32_t offset_y[NBB_MAX_REPLICAS];
} nbb_spec;

/* DispatchConfig (dispatch.hpp:25-38) extended with device-side knobs. */
typedef struct nbb_config {
    nbb_spec spec;
    int32_t r;          /* scale level, n = s^r                                */
    int32_t rho;        /* block edge, one of 1,2,4,8,16,32                     */
    int32_t mode;       /* NBB_MODE_*                                          */
    int32_t strategy;   /* NBB_STRATEGY_*                                      */
    int32_t backend;    /* NBB_BACKEND_*                                       */
    int32_t workers;    /* reference: host threads (>= 1); here the ordinal range is
                         * split into that many contiguous chunks (dispatch.cpp:419-427),
                         * launched in order on `device` — results identical for any
                         * count; across GPUs: one process per GPU with shard_* below */
    int32_t timing;     /* nonzero: fill report.micros from CUDA events         */
    int32_t cell_width; /* device cell bytes: 8 (int64, drop-in) or 1 (uint8)   */
    int32_t kernel;     /* NBB_KERNEL_*                                        */
    int32_t device;     /* CUDA device ordinal of the first worker              */
    uint64_t max_cells; /* membership-raster budget (reference kEnumerateBudget) */
    /* Shard: launch only block ordinals [shard_begin, shard_begin + shard_count)
     * of the plan (0/0 = all). The multi-GPU path gives each rank one contiguous
     * chunk, as the reference splits ordinals over workers (dispatch.cpp:419-427). */
    uint64_t shard_begin;
    uint64_t shard_count;
    uint32_t flags;     /* NBB_FLAG_* */
    uint32_t pass_steps; /* compact-state CA: at most this many steps per pass over the
                          * state (1..12; 0 = 8; above 8 only the cluster walk — gasket,
                          * lambda, r >= 8 — the others cap at 8). See
                          * nbb_gpu_ca_compact_passes_dev. */
} nbb_config;

/* nbb_config.flags
 * NBB_FLAG_OUT_ZEROED: the caller guarantees that the non-member cells of the host
 *   out_grid are already 0 (e.g. a reused output buffer, or one allocated zeroed); host
 *   calls may then write member cells only. With pinned (cudaHostAlloc/-Register)
 *   buffers the kernels then move only member sectors over PCIe (zero-copy) instead of
 *   the whole n*n grid. Without the flag out_grid is always written in full. */
#define NBB_FLAG_OUT_ZEROED 1u
/* Device state of nbb_gpu_ca. By default (neither flag) the CA state lives on the device in the
 *   compact (λ-ordered CompactGrid) layout between the two conversions — int64 values, every
 *   byte a member — whenever that layout serves the call: the gasket, cell_width 8,
 *   5 <= r <= 18, kernel AUTO, no shard. Lambda mode walks the orthotope (the compact array's
 *   own order); BB mode walks the bounding box, culls empty tiles and addresses member tiles
 *   through λ⁻¹ (the comparison launch). Other calls use the embedded grid of cell_width.
 * NBB_FLAG_COMPACT_STATE: require the compact state (NBB_ERR_INVALID_ARGUMENT if the call
 *   cannot use it).
 * NBB_FLAG_EMBEDDED_STATE: opt out — step the reference's embedded n x n layout of cell_width
 *   (int64, uint8 or 1-bit) with the tile / per-cell kernels (kernel, strategy, backend). */
#define NBB_FLAG_COMPACT_STATE 2u
#define NBB_FLAG_EMBEDDED_STATE 8u
/* NBB_FLAG_SINGLE_STEP: compact-state CA runs (nbb_gpu_ca with NBB_FLAG_COMPACT_STATE,
 *   nbb_gpu_ca_compact_*_dev) launch one kernel per step (= pass_steps 1). Without it,
 *   untimed runs advance up to pass_steps (default 8) steps per pass over the state
 *   (ca_compact_cluster_kernel / ca_compact_sliced_kernel: the tile and its radius-K halo are
 *   read once, the intermediate
 *   steps stay on chip) — the same result. */
#define NBB_FLAG_SINGLE_STEP 4u

/* WorkReport (dispatch.hpp:44-61) */
typedef struct nbb_report {
    char spec_name[32];
    int32_t r;
    int32_t rho;
    int32_t mode;
    int32_t strategy;
    int32_t backend;
    int32_t map_levels;
    uint64_t blocks_launched;
    uint64_t threads_launched;
    uint64_t threads_active;
    uint64_t threads_wasted;
    uint64_t map_ops;
    uint64_t micros;
} nbb_report;

/* What a pass sequence did: launches, launches per step count, where the result is. */
typedef struct nbb_pass_stats {
    int32_t passes;       /* kernel launches (passes over the state)                  */
    int32_t by_steps[13]; /* by_steps[k]: passes that advanced k steps (k = 1..12)     */
    int32_t result_in_b;  /* 1: the state after `steps` steps is in d_b; 0: in d_a     */
} nbb_pass_stats;

/* ---- library / config helpers ------------------------------------------ */
int nbb_gpu_abi_version(void);
const char* nbb_gpu_last_error(void);
/* gasket, r=0, rho=1, lambda, subbox, direct, workers=1, cell_width=8, 2^24 budget */
void nbb_config_init(nbb_config* cfg);
/* FractalSpec::sierpinski/vicsek/carpet (fractal.cpp:80-91) */
void nbb_spec_sierpinski(nbb_spec* spec);
void nbb_spec_vicsek(nbb_spec* spec);
void nbb_spec_carpet(nbb_spec* spec);
/* Number of CUDA devices visible (0 when none). */
int nbb_gpu_device_count(int32_t* count);

/* ---- host logic (no device needed) --------------------------------------- */
int nbb_gpu_validate(const nbb_config* cfg);
int nbb_gpu_launch_block_count(const nbb_config* cfg, uint64_t* blocks);
/* Closed-form WorkReport of one launch; micros = 0. */
int nbb_gpu_plan_report(const nbb_config* cfg, nbb_report* report);
int nbb_gpu_work_quotient(const nbb_report* bb, const nbb_report* lambda, int32_t weighted,
                          double* quotient);
const char* nbb_gpu_csv_header(void);
/* Writes WorkReport::csv_row() into buf (NUL-terminated); len >= 256 suffices. */
int nbb_gpu_report_csv_row(const nbb_report* report, char* buf, size_t len);
/* random_member_grid (dispatch.cpp:133-149), bit-identical, O(3^r) host loop.
 * out_grid: n*n int64, fully written (non-members 0). */
int nbb_gpu_random_member_grid(const nbb_spec* spec, int32_t r, uint64_t seed, uint64_t modulus,
                               uint64_t max_cells, int64_t* out_grid);
/* Member values only, in row-major member order (length 3^r): the same stream
 * random_member_grid assigns, without the n*n embedding. */
int nbb_gpu_random_member_values(const nbb_spec* spec, int32_t r, uint64_t seed,
                                 uint64_t modulus, int64_t* out_values);

/* ---- workloads on host buffers (drop-in) -------------------------------- */
/* run_single_write: out_grid (n*n int64) receives the whole result grid. */
int nbb_gpu_single_write(const nbb_config* cfg, int64_t* out_grid, nbb_report* report);
/* run_reduction: grid (n*n int64) at level grid_level (must equal cfg->r). */
int nbb_gpu_reduction(const nbb_config* cfg, const int64_t* grid, int32_t grid_level,
                      int64_t* value, nbb_report* report);
/* run_ca: `steps` double-buffered steps; per_step receives `steps` reports
 * (may be NULL). out_grid may alias initial. */
int nbb_gpu_ca(const nbb_config* cfg, const int64_t* initial, int32_t initial_level,
               int32_t steps, uint16_t birth, uint16_t survive, int64_t* out_grid,
               nbb_report* per_step);
/* run_ca / run_reduction with the reference's `workers` mapped to DEVICES of this process
 * (dispatch.cpp:416-432: contiguous ordinal chunks — ceil(total / workers), rounded up to whole
 * cluster columns as for nbb_gpu_ca_compact_p2p_passes_dev — result independent
 * of the count — byte-identical for any ndev). The compact tiles are split into ndev contiguous
 * chunks; worker w advances chunk w on devices[w] in passes of up to pass_steps steps and reads
 * the halo cells other workers own from their buffers over NVLink (peer access) inside the pass
 * kernel; a flag barrier in device memory orders the passes. devices may repeat (several
 * chunks on one GPU). Gasket, lambda mode, cell_width 8, 5 <= r <= 18; ndev <= 8; the host
 * buffers as for nbb_gpu_ca / nbb_gpu_reduction (devices[0] converts them). */
int nbb_gpu_ca_multi(const nbb_config* cfg, const int32_t* devices, int32_t ndev,
                     const int64_t* initial, int32_t initial_level, int32_t steps, uint16_t birth,
                     uint16_t survive, int64_t* out_grid, nbb_report* per_step);
int nbb_gpu_reduction_multi(const nbb_config* cfg, const int32_t* devices, int32_t ndev,
                            const int64_t* grid, int32_t grid_level, int64_t* value,
                            nbb_report* report);
/* λ(ω) for every ω of the level-`level` orthotope, ordinal-major
 * (xy[2*o], xy[2*o+1], o = ωy*W + ωx). Uses cfg->backend (direct or mma1/mma2). */
int nbb_gpu_lambda_coords(const nbb_config* cfg, int32_t level, int64_t* xy);

/* ---- device-resident variants (pointers are device pointers) -------------- */
/* stream: cudaStream_t or NULL for the legacy default stream. */
int nbb_gpu_single_write_dev(const nbb_config* cfg, void* d_grid, void* stream,
                             nbb_report* report);
/* *d_value (device int64) receives the sum; no host synchronisation. */
int nbb_gpu_reduction_dev(const nbb_config* cfg, const void* d_grid, void* d_value,
                          void* stream, nbb_report* report);
/* One CA step d_src -> d_dst. Non-member cells of d_dst must already be 0
 * (true after nbb_gpu_sanitize_dev / a zeroed allocation); they stay 0. */
int nbb_gpu_ca_step_dev(const nbb_config* cfg, const void* d_src, void* d_dst, uint16_t birth,
                        uint16_t survive, void* stream, nbb_report* report);
/* `steps` CA steps on an embedded device grid (the reference's layout, d_a initial): the result
 * is where a run of single steps leaves it (d_a when steps is even, else d_b); the other buffer is
 * scratch. For the gasket's int64 grid (5 <= r <= 18, kernel AUTO, unsharded, untimed, steps >= 2)
 * the run is temporally blocked: the member sectors go once into the λ-ordered compact state,
 * the steps run there in passes of up to pass_steps, and the result comes back into the member
 * sectors — bit-identical to stepping the embedded grid; otherwise one launch per step. Non-member
 * cells of both buffers must be 0 (they stay 0). stats (optional): the passes issued. */
int nbb_gpu_ca_run_dev(const nbb_config* cfg, void* d_a, void* d_b, int32_t steps, uint16_t birth,
                       uint16_t survive, void* stream, nbb_pass_stats* stats);
/* Zero every non-member cell of a device grid of cfg->cell_width cells. */
int nbb_gpu_sanitize_dev(const nbb_config* cfg, void* d_grid, void* stream);
/* int64 grid -> uint8 alive grid (cell != 0) and back (0/1 -> int64). */
int nbb_gpu_pack_alive_dev(const nbb_config* cfg, const void* d_grid64, void* d_grid8,
                           void* stream);
int nbb_gpu_unpack_alive_dev(const nbb_config* cfg, const void* d_grid8, void* d_grid64,
                             void* stream);
/* Scatter member values given in row-major member order into a zeroed
 * embedded device grid (inverse of the host generator's order). */
int nbb_gpu_scatter_members_dev(const nbb_config* cfg, const void* d_values, void* d_grid,
                                void* stream);
/* λ map of the whole level-`level` orthotope into device memory.
 * coord_bytes = 4 (int32 pairs) or 8 (int64 pairs). */
int nbb_gpu_lambda_coords_dev(const nbb_config* cfg, int32_t level, void* d_xy,
                              int32_t coord_bytes, void* stream);
/* ---- compact (λ-ordered) state: CompactGrid, block_map.hpp:82-132 ----------------
 * The k^r member values row-major over the packing orthotope (W = k^ceil(r/2) wide),
 * value(ω) = embedded(λ(ω)). Level = cfg->r, any valid spec. */
/* compact_store (block_map.cpp:245-262): embedded n*n -> compact k^r */
int nbb_gpu_compact_store(const nbb_config* cfg, const int64_t* embedded, int64_t* compact);
/* compact_load (block_map.cpp:264-282): compact -> embedded, non-members = empty_value */
int nbb_gpu_compact_load(const nbb_config* cfg, const int64_t* compact, int64_t empty_value,
                         int64_t* embedded);
int nbb_gpu_compact_store_dev(const nbb_config* cfg, const void* d_embedded, void* d_compact,
                              void* stream);
int nbb_gpu_compact_load_dev(const nbb_config* cfg, const void* d_compact, int64_t empty_value,
                             void* d_embedded, void* stream);
/* lambda_inverse (block_map.cpp:113-148) of `count` points xy[2i], xy[2i+1] at `level`;
 * omega receives (ωx, ωy) pairs. Returns NBB_ERR_OUT_OF_RANGE / NBB_ERR_DOMAIN for the
 * first offending point (message names it), NBB_OK otherwise. */
int nbb_gpu_lambda_inverse(const nbb_config* cfg, int32_t level, const int64_t* xy, uint64_t count,
                           int64_t* omega);
/* NBBC file (block_map.cpp:284-362): "NBBC", k, s, level (LE u32), values (LE i64) */
int nbb_gpu_compact_write(const char* path, const nbb_spec* spec, int32_t level,
                          const int64_t* values);
/* reads into values (capacity entries); *level receives the file's level */
int nbb_gpu_compact_read(const char* path, const nbb_spec* spec, int32_t* level, int64_t* values,
                         uint64_t capacity);
/* Workloads on device-resident compact state (gasket; CA needs r >= 5): one CA step
 * d_src -> d_dst, the member sum, the single write (every member value = 1).
 * The CA step honours shard_begin/shard_count over the compact tile order
 * u = ωx_b·H_b + ωy_b of the ρ = 32 tiles (a contiguous u range = contiguous compact
 * rows), so each rank of the multi-GPU path updates one slab of the compact array. */
int nbb_gpu_ca_compact_step_dev(const nbb_config* cfg, const void* d_src, void* d_dst,
                                uint16_t birth, uint16_t survive, void* stream, nbb_report* report);
/* `steps` compact CA steps ping-ponging between d_a and d_b, issued back to back from C++
 * (the reference's run_ca step loop, dispatch.cpp:517-557) as passes of up to pass_steps
 * steps each; the result is in d_a when steps is even, else in d_b (as stepping one by one:
 * the pass count then has the parity of `steps`, which may cost one pass more). */
int nbb_gpu_ca_compact_run_dev(const nbb_config* cfg, void* d_a, void* d_b, int32_t steps,
                               uint16_t birth, uint16_t survive, void* stream);
/* The same run with parity = 0: the fewest passes (ceil(steps / pass_steps)), the result in
 * whichever buffer stats->result_in_b names; parity != 0 behaves as nbb_gpu_ca_compact_run_dev.
 * stats may be NULL. */
int nbb_gpu_ca_compact_passes_dev(const nbb_config* cfg, void* d_a, void* d_b, int32_t steps,
                                  uint16_t birth, uint16_t survive, int32_t parity, void* stream,
                                  nbb_pass_stats* stats);
/* Host only: the passes the two calls above (parity as given) issue for `steps` steps. */
int nbb_gpu_pass_plan(const nbb_config* cfg, int32_t steps, int32_t parity, nbb_pass_stats* stats);
int nbb_gpu_reduction_compact_dev(const nbb_config* cfg, const void* d_compact, void* d_value,
                                  void* stream, nbb_report* report);
int nbb_gpu_single_write_compact_dev(const nbb_config* cfg, void* d_compact, void* stream,
                                     nbb_report* report);

/* Halo exchange helpers for sharded CA (multi-GPU): gather d_grid[idx[i]] into
 * d_out[i] and scatter d_vals[i] into d_grid[idx[i]], count cells of
 * cfg->cell_width bytes; idx are flat cell indices (y*n + x) in device memory. */
int nbb_gpu_gather_cells_dev(const nbb_config* cfg, const void* d_grid, const int64_t* d_idx,
                             int64_t count, void* d_out, void* stream);
int nbb_gpu_scatter_cells_dev(const nbb_config* cfg, void* d_grid, const int64_t* d_idx,
                              int64_t count, const void* d_vals, void* stream);
/* Free the device buffers cached by the host-buffer entry points. */
int nbb_gpu_release(void);

/* ---- multi-GPU compact CA over peer memory (one process per GPU) ----------------------
 * The reference splits block ordinals over worker threads sharing one Grid
 * (dispatch.cpp:416-432); across GPUs the shared grid becomes CUDA IPC mappings of every
 * rank's compact buffers. nbb_gpu_ca_compact_p2p_dev runs `steps` steps of
 * nbb_gpu_ca_compact_step_dev for this rank's shard (cfg.shard_begin/shard_count over the
 * compact tile order), ONE kernel per step issued back to back from C++: each kernel waits
 * until every rank finished the previous step (flag barrier in peer memory: world x i arrivals
 * before step i, bounded by timeout_ms -> error flag), reads the
 * halo cells other ranks own straight from their buffers over NVLink, and announces its own
 * completion to every rank. Step i (first_step <= i < first_step + steps) reads d_buf[i & 1]
 * and writes d_buf[(i + 1) & 1]; first_step must equal the number of steps this d_sync has
 * already run. All d_* arrays are device-resident; world <= 8. */
typedef struct nbb_p2p {
    int32_t world, rank;
    void* d_buf[2];              /* this rank's two compact buffers (3^r int64 each)            */
    const void* d_peer_buf[2];   /* [world] const int64_t*: every rank's buffer 0 / buffer 1   */
    const void* reserved;        /* unused (ABI 2: a halo owner table; the owner of a halo cell
                                  * is now its tile ordinal / the shard chunk below)          */
    void* d_sync;                /* this rank's uint32[4] {arrivals, done, error, 0}, zeroed    */
    const void* d_peer_flag;     /* [world] uint32*: every rank's d_sync (arrival counter)      */
    uint32_t timeout_ms;         /* bound on each wait; 0 = 20000                               */
} nbb_p2p;
int nbb_gpu_ca_compact_p2p_dev(const nbb_config* cfg, int64_t first_step, int32_t steps,
                               uint16_t birth, uint16_t survive, const nbb_p2p* p2p, void* stream);
/* The same step sequence in PASSES of up to cfg->pass_steps steps (default 8; the
 * ca_compact_cluster_kernel — ca_compact_sliced_kernel for r < 8 — over peer memory: the
 * radius-K halo read once, the intermediate
 * steps kept on chip): ceil(steps / K) passes, steps spread evenly. Pass j (first_pass <= j)
 * reads d_buf[j & 1], writes d_buf[(j + 1) & 1] and waits for world x j arrivals; first_pass
 * must equal the number of passes (either entry point: a step of nbb_gpu_ca_compact_p2p_dev
 * is one pass) this d_sync has already run. The shard must be the rank's contiguous chunk:
 * shard_begin = rank * chunk, shard_count = chunk (clipped), chunk = ceil(tiles / world)
 * rounded up to a multiple of 9 * Hb tiles (whole level-3 cluster columns, Hb = 3^floor((r-5)/2))
 * when r >= 8, plain ceil(tiles / world) below — the owner of every halo cell is derived from it
 * (NBB_ERR_INVALID_ARGUMENT otherwise). Results are identical for any split.
 * nbb_gpu_pass_plan(cfg, steps, 0, &stats) names the passes. */
int nbb_gpu_ca_compact_p2p_passes_dev(const nbb_config* cfg, int64_t first_pass, int32_t steps,
                                      uint16_t birth, uint16_t survive, const nbb_p2p* p2p, void* stream);
/* error flag of d_sync after a step sequence (synchronises the stream): 0 ok, 1 timed out */
int nbb_gpu_p2p_check(const nbb_p2p* p2p, void* stream);
/* device memory that can be exported (cudaMalloc: the IPC handle names the allocation) */
int nbb_gpu_malloc(int32_t device, uint64_t bytes, void** d_ptr);
int nbb_gpu_free(int32_t device, void* d_ptr);
/* CUDA IPC: 64-byte handle of an nbb_gpu_malloc allocation; open a peer's handle */
int nbb_gpu_ipc_handle(int32_t device, const void* d_ptr, uint8_t handle[64]);
int nbb_gpu_ipc_open(int32_t device, const uint8_t handle[64], void** d_ptr);
int nbb_gpu_ipc_close(int32_t device, void* d_ptr);

/* ---- multi-GPU compact CA over NCCL (one process per GPU) ---------------------------------
 * The north_star's transport: NCCL over NVLink only for the CA boundary halos and the final
 * reduction. A communicator spans `world` processes (ncclCommInitRank; the 128-byte id comes from
 * nbb_gpu_comm_unique_id on one rank and reaches the others through the caller's launcher).
 * Rank i owns the contiguous compact tile chunk [i * chunk, min((i + 1) * chunk, tiles)),
 * chunk as for nbb_gpu_ca_compact_p2p_passes_dev (dispatch.cpp:419-427 rounded up to whole cluster
 * columns; cfg->shard_* are set from it). Before every
 * pass of up to pass_steps (<= 8) steps the halo cells the rank's tiles read from other ranks
 * within 8 steps are gathered, exchanged with ncclSend / ncclRecv in one group on `stream` and
 * scattered into the pass's source buffer; d_a / d_b are replica-sized (3^r int64) buffers in
 * which this rank's tiles are current; the result buffer is named by stats->result_in_b. NCCL
 * is bound at run time (libnccl.so.2); without it these calls return NBB_ERR_NCCL. */
typedef struct nbb_comm nbb_comm;
int nbb_gpu_comm_unique_id(uint8_t id[128]);
int nbb_gpu_comm_init(const uint8_t id[128], int32_t world, int32_t rank, int32_t device,
                      nbb_comm** comm);
int nbb_gpu_comm_destroy(nbb_comm* comm);
int nbb_gpu_ca_compact_comm_dev(const nbb_config* cfg, nbb_comm* comm, void* d_a, void* d_b,
                                int32_t steps, uint16_t birth, uint16_t survive, void* stream,
                                nbb_pass_stats* stats);
/* Σ of the rank's tiles + one ncclAllReduce (int64 sum): *d_value on every rank. */
int nbb_gpu_reduction_compact_comm_dev(const nbb_config* cfg, nbb_comm* comm, const void* d_compact,
                                       void* d_value, void* stream);
/* Host only: the halo exchange of rank `rank` for passes of up to kmax steps — cells sent to /
 * received from every peer (counts[world]) and the sorted compact offsets for one peer. */
int nbb_gpu_halo_exchange_counts(const nbb_config* cfg, int32_t world, int32_t rank, int32_t kmax,
                                 uint64_t* send_counts, uint64_t* recv_counts);
int nbb_gpu_halo_exchange_lists(const nbb_config* cfg, int32_t world, int32_t rank, int32_t kmax,
                                int32_t peer, uint32_t* send, uint32_t* recv);

#ifdef __cplusplus
}
#endif

#endif /* NBB_GPU_H */
