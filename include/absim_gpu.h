/* absim_gpu.h — C ABI of the B200 (sm_100a) mechanical-step engine.
 *
 * Drop-in boundary for the reference's neighbour-search / mechanical-forces
 * path. The reference has no C ABI (static C++ lib, proj/src/CMakeLists.txt:1-21)
 * and its per-agent virtual visitor (environment.hpp:12-16) cannot cross to a
 * GPU, so the boundary is batched at step granularity. Each entry point names
 * the reference interface it replaces:
 *
 *   abs_gpu_create          Simulation::Simulation(SimulationParams)      simulation.hpp:91, params.hpp:17-52
 *                           + make_environment(kUniformGrid)                simulation.cpp:40-53
 *   abs_gpu_upload          Simulation::add_agent (+ Behavior attach)       simulation.hpp:107, simulation.cpp:131-141
 *   abs_gpu_simulate        Simulation::simulate(iterations)                simulation.hpp:121, simulation.cpp:222-322
 *                           = Environment::update → [staticness] → behaviours
 *                             → run_forces → run_integration → run_commit
 *   abs_gpu_stats           Simulation::report() counters                   report.hpp:32-40
 *   abs_gpu_download        ResourceManager::for_each_agent + Agent getters resource_manager.hpp:70, agent.hpp:31-110
 *   abs_gpu_run_frames      add_agent -> simulate -> read agents, repeated over
 *                           independent host frames with copy/compute overlap simulation.hpp:107-121
 *   abs_gpu_env_update      Environment::update (UniformGrid::update)       environment.hpp:40, uniform_grid.cpp:59-170
 *   abs_gpu_grid_info       UniformGrid::{origin, box_length, dims, largest_agent_diameter}  uniform_grid.hpp:40-49
 *   abs_gpu_cell_ids        UniformGrid::box_index_of (per agent)           uniform_grid.cpp:28-37
 *   abs_gpu_neighbors       Environment::for_each_neighbor (batched; force
 *                           query radius 0.5 (d + dmax), simulation.cpp:469) uniform_grid.cpp:172-230
 *   abs_gpu_sort            sort_and_balance (one domain)                   sort_balance.cpp:22-148
 *   abs_gpu_remove          CommitBuffer removals / remove_agents_parallel  commit.cpp:14-106
 *   abs_gpu_set_defer_commit / abs_gpu_division_marks / abs_gpu_commit
 *                           CommitBuffer::commit additions, split so ranks
 *                           agree on daughter uids                          commit.cpp:186-222, simulation.cpp:64-91
 *   abs_gpu_download_storage_keys
 *                           each agent's slot in ResourceManager's agent
 *                           vector (the order for_each_agent walks and that
 *                           decides daughter uids and survivor slots)        resource_manager.hpp:19-101
 *   abs_gpu_create with environment = ABS_ENV_BRUTE_FORCE / ABS_ENV_KD_TREE
 *                           make_environment(kBruteForce / kKdTree)          simulation.cpp:40-53, environment.hpp:53-80,
 *                                                                            kdtree_env.cpp:8-86
 *   abs_gpu_comm_init / abs_gpu_comm_set_transport / abs_gpu_simulate_decomposed / abs_gpu_decomp_info
 *                           the reference's per-domain partition of one
 *                           address space (ResourceManager domains, box-aligned
 *                           shares) as one z slab per GPU                    resource_manager.hpp:95, sort_balance.cpp:61-77
 *   abs_gpu_export_layers / abs_gpu_import / abs_gpu_drop_ghosts / abs_gpu_set_grid_override
 *                           the same slab exchange step by step, for hosts
 *                           that bring their own transport
 *
 * Conventions: int status (ABS_OK == 0), no exceptions across the ABI, one
 * host thread per context, device memory owned by the context, host buffers
 * borrowed for the duration of the call only. All work is ordered on the
 * context's CUDA stream; calls that return host data synchronise it.
 * Agent order in download/cell_ids/neighbors is the device storage order
 * (cell order); identity is the uid.
 */
#ifndef ABSIM_GPU_H
#define ABSIM_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define ABS_OK 0
#define ABS_ERR_INVALID_ARGUMENT 1  /* std::invalid_argument in the reference */
#define ABS_ERR_CUDA 2
#define ABS_ERR_NONFINITE 3          /* "agent positions are not finite"  uniform_grid.cpp:112-116 */
#define ABS_ERR_FIXED_BOX 4          /* fixed box < largest diameter     uniform_grid.cpp:118-125 */
#define ABS_ERR_BOX_BUDGET 5         /* > 2^31 boxes                      uniform_grid.cpp:139-141 */
#define ABS_ERR_CAPACITY 6           /* device agent capacity exhausted */
#define ABS_ERR_NO_DEVICE 7
#define ABS_ERR_STATE 8              /* std::logic_error in the reference */

/* agent flags (download), same bits as the oracles' dumps */
#define ABS_FLAG_STATIC 1u
#define ABS_FLAG_MOVED 2u
#define ABS_FLAG_GREW 4u
#define ABS_FLAG_NEWLY_ADDED 8u
#define ABS_FLAG_NEIGHBOR_VIOLATION 16u
#define ABS_FLAG_NEW_NEIGHBOR 32u
#define ABS_FLAG_GHOST 128u /* multi-domain halo copy: a candidate, never stepped */
#define ABS_FLAG_REMOVED 64u /* internal: removal staged this iteration (never seen after the commit) */

/* device behaviour models (BASELINE configs; models.hpp:69-83 for GROW) */
#define ABS_MODEL_NONE 0
#define ABS_MODEL_PROLIFERATION 1 /* mp[0] volume rate, mp[1] division volume */
#define ABS_MODEL_DRIVE 2         /* mp[0..2] centre, mp[3] max speed */
#define ABS_MODEL_GROW 3          /* mp[0] growth rate, mp[1] diameter cap */
#define ABS_MODEL_SIR 4           /* mp[0] L (periodic cube), mp[1] radius, mp[2] step, mp[3] recovery, mp[4] p */
#define ABS_MODEL_GROW_DIVIDE 5   /* the reference's models::GrowDivide (models.hpp:15-37): mp[0] growth rate,
                                     mp[1] division threshold, mp[2] initial diameter; daughters from the
                                     agent's own RandomStream (tag copied, counter advanced by 2) */
#define ABS_MODEL_GROW_DIVIDE_DIE 7 /* models::GrowDivide (mp[0..2] as above) whose agents also remove themselves
                                     (AgentContext::remove_self, simulation.cpp:64-66) with probability mp[3]
                                     per iteration: u01(rng_word(seed, uid, ABS_RNG_DEATH(it))) < mp[3]; the
                                     commit applies removals (remove_agents_parallel) before additions */
#define ABS_MODEL_COHERE 6        /* the reference's models::Cohere (models.hpp:42-64): mp[0] attraction
                                     radius (<= box length, e.g. fixed_box_length), mp[1] speed; same-tag
                                     neighbours only */

/* environment kinds (params.hpp:9 EnvironmentKind; simulation.cpp:40-53 make_environment) */
#define ABS_ENV_UNIFORM_GRID 0  /* UniformGrid: the B200 cell table */
#define ABS_ENV_BRUTE_FORCE 1   /* BruteForceEnvironment (environment.hpp:53-80): every agent is a
                                   candidate, no maximum query radius; O(N^2) comparison baseline.
                                   Sorting (params.cpp:52-55) and cell ids need the grid. */
#define ABS_ENV_KD_TREE 2       /* KdTreeEnvironment (kdtree_env.cpp:8-86): a balanced kd-tree over the
                                   agent array, rebuilt every environment update (median splits along the
                                   widest axis, leaves of 32); the force query descends it with the exact
                                   d2 <= r^2 at the leaves. Same query contract as brute force (no maximum
                                   radius); the paper's grid-vs-tree comparison baseline. */

typedef struct abs_gpu_ctx abs_gpu_ctx;

/* SimulationParams (params.hpp:17-52), hot-path subset + device knobs */
typedef struct {
  uint64_t seed;                 /* 42 */
  double simulation_time_step;   /* 0.1 */
  double repulsion_coefficient;  /* 2.0 */
  double max_displacement;       /* 3.0 */
  double force_threshold;        /* 0.0 */
  double fixed_box_length;       /* 0.0 = follow the largest diameter */
  uint64_t sorting_frequency;    /* 0 = never; f > 0: the reference's Morton sort_and_balance order is
                                    applied before every iteration with iteration % f == 0
                                    (simulation.cpp:246-247); storage is re-binned every step anyway */
  int32_t detect_static_agents;  /* 0 */
  int32_t model;                 /* ABS_MODEL_* */
  double model_params[8];
  uint64_t capacity;             /* agent capacity hint; grows on demand */
  int32_t record_forces;         /* keep Agent::last_force (parity); 0 skips the 24 B/agent write */
  int32_t bins_per_box;          /* internal sub-bins per box edge along y and z: 0 auto, 1..4 */
  int32_t bins_per_box_x;        /* internal sub-bins per box edge along x: 0 auto, 1..4 */
  int32_t environment;           /* ABS_ENV_* (SimulationParams::environment_kind), default grid */
  int32_t neighbor_list;         /* 0 auto: per-agent candidate lists between environment rebuilds when
                                    the diameters are constant (no behaviours, no static detection, one
                                    domain) and the observed displacement rate lets a build serve >= 3 steps;
                                    1 always (build whenever the lists do not cover the step); -1 off
                                    (re-bin + cell-table walk every iteration). The visited neighbour
                                    sets are identical either way */
  double neighbor_skin;          /* list skin (absolute length); 0 = 0.2 x the largest diameter */
} abs_gpu_config;

/* SimulationReport counters (report.hpp:32-40) */
typedef struct {
  uint64_t agents;
  uint64_t uid_count;
  uint64_t iterations;
  uint64_t force_evaluations;
  uint64_t force_skips;
  uint64_t agents_added;
  uint64_t agents_removed;
  uint64_t kernel_launches; /* kernels this context launched so far */
  uint64_t agent_iterations; /* sum over iterations since the last upload of the agents at iteration start
                                (the metric's numerator, exact for growing populations) */
} abs_step_stats;

void abs_gpu_default_config(abs_gpu_config* cfg);
int abs_gpu_create(const abs_gpu_config* cfg, int device, abs_gpu_ctx** out);
int abs_gpu_destroy(abs_gpu_ctx* ctx);
/* message of the last failure on ctx (or of the last failed create if ctx == NULL) */
const char* abs_gpu_last_error(const abs_gpu_ctx* ctx);

/* Replace the population with n agents copied from host arrays. uid == NULL
 * assigns uids 0..n-1 in array order (Simulation::add_agent order);
 * behaviour_mask == NULL attaches the model behaviour to every agent;
 * volume/flags/partners may be NULL (volume defaults to the sphere volume).
 * uid_count: uids ever assigned (every uid < uid_count, checked on the
 * device -> ABS_ERR_INVALID_ARGUMENT); 0 with explicit uids = derive it from
 * the uids on the host. Page-locked host arrays are copied by plain DMA. */
int abs_gpu_upload(abs_gpu_ctx* ctx, uint64_t n, const uint64_t* uid, const double* x,
                   const double* y, const double* z, const double* d,
                   const uint8_t* behaviour_mask, const double* volume,
                   const uint8_t* flags, const uint32_t* partners, uint64_t uid_count);

/* Same, from device pointers already resident in HBM (no host copies);
 * explicit uids need uid_count > 0. */
int abs_gpu_upload_device(abs_gpu_ctx* ctx, uint64_t n, const uint64_t* uid, const double* x,
                          const double* y, const double* z, const double* d,
                          const uint8_t* behaviour_mask, uint64_t uid_count);

/* Agent::tag and the per-agent RandomStream counter (agent.hpp:35-36, 145;
 * used by ABS_MODEL_GROW_DIVIDE / ABS_MODEL_COHERE), host arrays in the
 * current storage order (after abs_gpu_upload: upload order); either
 * pointer may be NULL. Uploads reset both to 0. */
int abs_gpu_set_agent_ext(abs_gpu_ctx* ctx, const uint32_t* tags, const uint64_t* rng_counters);
int abs_gpu_download_ext(abs_gpu_ctx* ctx, uint32_t* tags, uint64_t* rng_counters);

/* Multi-domain additions (commit.cpp:186-222). With defer != 0
 * a proliferation context's abs_gpu_simulate(ctx, 1) stops with the
 * iteration's daughters staged. The caller copies this rank's uid-indexed
 * division marks (uid_count entries, 1 = that uid divided here) with
 * abs_gpu_division_marks into a device buffer, sums the buffers of all ranks
 * (e.g. an NCCL all-reduce) and passes the sum to abs_gpu_commit: daughter
 * uids are then uid_count + the parent's rank among ALL dividing parents,
 * exactly the single-domain numbering. global_marks == NULL commits with
 * this rank's marks alone. Static detection with deferred additions is
 * rejected (new-neighbour marks would stay local). */
int abs_gpu_set_defer_commit(abs_gpu_ctx* ctx, int defer);
int abs_gpu_division_marks(abs_gpu_ctx* ctx, uint32_t* out_device, uint64_t cap, uint64_t* len);
int abs_gpu_commit(abs_gpu_ctx* ctx, const uint32_t* global_marks_device, uint64_t len);

/* Multi-domain: force the grid computed over all ranks
 * (grid[0..2] origin, grid[3] box length, grid[4] largest diameter; dims)
 * instead of the local bounds; grid == NULL restores the local grid. */
int abs_gpu_set_grid_override(abs_gpu_ctx* ctx, const double* grid, const uint32_t* dims);
/* Local bounds of the current population: out[0..2] min xyz, out[3..5]
 * max xyz, out[6] largest diameter (uniform_grid.cpp:74-110 pass 1). */
int abs_gpu_local_bounds(abs_gpu_ctx* ctx, double* out7);

/* Device-resident multi-domain exchange. Agents travel as
 * packed 96-byte records (ABS_RECORD_BYTES) in caller-owned DEVICE buffers.
 * abs_gpu_export_layers classifies agents by reference-box z-layer under the
 * given global grid (grid[0..2] origin, grid[3] box; dims):
 *   mode 0 (migrate): owned agents with layer < lo -> out_lo, >= hi -> out_hi,
 *                     removed from this context;
 *   mode 1 (halo):    owned agents with layer == lo -> out_lo, == hi-1 -> out_hi.
 *   mode | 2:         periodic z (a ring of layers, config 5): a migrant
 *                     leaves through the nearer side modulo dims[2].
 * Returns ABS_ERR_CAPACITY when a count exceeds cap (counts are still set). */
#define ABS_RECORD_BYTES 96
int abs_gpu_export_layers(abs_gpu_ctx* ctx, const double* grid, const uint32_t* dims, int64_t lo, int64_t hi,
                          int mode, void* out_lo, void* out_hi, uint64_t cap, uint64_t* n_lo, uint64_t* n_hi);
/* Append count records (device pointer) as owned agents or as ghosts. */
int abs_gpu_import(abs_gpu_ctx* ctx, const void* records, uint64_t count, int as_ghost);
/* Remove every ghost agent (order-preserving compaction). */
int abs_gpu_drop_ghosts(abs_gpu_ctx* ctx);

/* Multi-GPU slab decomposition driven by the library: one
 * context per GPU / rank; per iteration a device all-reduce of the bounds
 * gives the single-domain grid, an all-reduced z-layer histogram gives
 * equal-count slab edges (sort_balance.cpp:61-77 analogue), one export pass
 * and one exchange move emigrants (owned) and boundary layers (ghosts) to the
 * neighbouring slabs, then the iteration runs and the ghosts are dropped.
 * Transport: the built-in NCCL one (abs_gpu_comm_init, unique id from
 * abs_gpu_nccl_unique_id on one rank, shared by the caller), or callbacks.
 * All device pointers; counts are host values; `stream` is the context's
 * CUDA stream (cudaStream_t). Callbacks return 0 on success. */
#define ABS_DT_F64_MAX 0 /* element-wise MAX of doubles */
#define ABS_DT_U64_SUM 1
#define ABS_DT_U32_SUM 2
typedef struct {
  void* user;
  int (*allreduce)(void* user, void* dev, uint64_t count, int dtype, void* stream);
  /* send n_lo / n_hi to the lo / hi neighbour slab, return what they send here */
  int (*counts)(void* user, uint64_t n_lo, uint64_t n_hi, uint64_t* got_lo, uint64_t* got_hi, void* stream);
  /* ABS_RECORD_BYTES-byte records: send_lo[n_lo] -> lo peer, send_hi[n_hi] -> hi peer;
     receive got_lo records from the lo peer into recv_lo, got_hi from the hi peer into recv_hi */
  int (*records)(void* user, const void* send_lo, uint64_t n_lo, const void* send_hi, uint64_t n_hi, void* recv_lo,
                 uint64_t got_lo, void* recv_hi, uint64_t got_hi, void* stream);
} abs_gpu_transport;
int abs_gpu_nccl_unique_id(void* id_128_bytes);
int abs_gpu_comm_init(abs_gpu_ctx* ctx, const void* nccl_unique_id, int rank, int nranks);
int abs_gpu_comm_set_transport(abs_gpu_ctx* ctx, const abs_gpu_transport* transport, int rank, int nranks);
/* Reserve exchange records per direction (grown automatically otherwise). */
int abs_gpu_comm_reserve(abs_gpu_ctx* ctx, uint64_t records);
/* `iterations` decomposed iterations (the population is this rank's slab;
 * uids global, uid_count the global count). */
int abs_gpu_simulate_decomposed(abs_gpu_ctx* ctx, uint64_t iterations);
/* Slab edges of the last iteration (nranks + 1 z-layers) and the owned agents. */
int abs_gpu_decomp_info(abs_gpu_ctx* ctx, int64_t* layer_bounds, uint64_t* owned);
/* Stream-ordered copy between any two pointers (host or device), then a
 * synchronisation of `stream` (for transport callbacks staging through host memory). */
int abs_gpu_memcpy(void* dst, const void* src, uint64_t bytes, void* stream);

/* Config 5 (SIR): S/I/R counts after the last iteration, and the per-agent
 * state (0 S, 1 I, 2 R) + infection iteration in download order. */
int abs_gpu_sir_counts(abs_gpu_ctx* ctx, uint64_t* out3);
int abs_gpu_sir_state(abs_gpu_ctx* ctx, uint8_t* state, uint32_t* t_infected);

/* Set the global iteration counter (checkpoint resume / teacher forcing;
 * the counter drives frequency gating and the RNG counters, simulation.hpp:117-121). */
int abs_gpu_set_iteration(abs_gpu_ctx* ctx, uint64_t iteration);

/* Run `iterations` full iterations (stream-ordered). */
int abs_gpu_simulate(abs_gpu_ctx* ctx, uint64_t iterations);
int abs_gpu_stats(abs_gpu_ctx* ctx, abs_step_stats* out);
int abs_gpu_synchronize(abs_gpu_ctx* ctx);

/* Copy the population to host arrays (any pointer may be NULL); *n_out = agents. */
int abs_gpu_download(abs_gpu_ctx* ctx, uint64_t* n_out, uint64_t* uid, double* x, double* y,
                     double* z, double* d, double* fx, double* fy, double* fz,
                     uint32_t* partners, uint8_t* flags, double* volume);

/* Host-boundary pipeline (end-to-end use with host buffers). Each frame is
 * exactly abs_gpu_upload (uids 0..n-1, no mask) + abs_gpu_set_iteration(
 * first_iteration + f * iterations) + abs_gpu_simulate(iterations) +
 * abs_gpu_download(x, y, z); frames run in order on this context. The H2D of
 * frame f+1 and the D2H of frame f-1 run on two copy streams while frame f
 * computes (double-buffered device staging), so PCIe and HBM work overlap.
 * Host arrays should be page-locked (plain DMA). Output order is the device
 * storage order (cell order), as abs_gpu_download. */
typedef struct {
  uint64_t n;                    /* agents in this frame */
  const double *x, *y, *z, *d;   /* host inputs */
  double *out_x, *out_y, *out_z; /* host outputs: positions after the iterations */
  uint64_t out_cap;              /* entries each output array holds (>= n unless a model adds agents) */
  uint64_t* n_out;               /* agents after the iterations (may be NULL) */
  uint64_t* out_uid;             /* uids in output order (may be NULL; out_cap entries) */
} abs_frame;
int abs_gpu_run_frames(abs_gpu_ctx* ctx, const abs_frame* frames, uint64_t count, uint64_t iterations,
                       uint64_t first_iteration);

/* Teacher-forced environment: build the grid for the current state. */
int abs_gpu_env_update(abs_gpu_ctx* ctx);
/* grid[0..2] origin, grid[3] box length, grid[4] largest diameter */
int abs_gpu_grid_info(abs_gpu_ctx* ctx, double* grid, uint32_t* dims);
/* reference box index per agent (download order); requires abs_gpu_env_update;
 * ABS_ERR_STATE under ABS_ENV_BRUTE_FORCE (no grid) */
int abs_gpu_cell_ids(abs_gpu_ctx* ctx, uint64_t* out);
/* CSR of sorted neighbour uids per agent (download order) within the force
 * query radius; offsets has n+1 entries. *total receives the number of uids;
 * uids == NULL only sizes the result; returns ABS_ERR_CAPACITY (and the
 * needed total) when cap is too small. */
int abs_gpu_neighbors(abs_gpu_ctx* ctx, uint64_t* offsets, uint64_t* uids, uint64_t cap,
                      uint64_t* total);
/* Reorder storage into sort_and_balance order: boxes by Morton rank, agents in
 * a box by descending current storage index (sort_balance.cpp:88-128). */
int abs_gpu_sort(abs_gpu_ctx* ctx);
/* Remove agents by uid with the reference's five-step slot semantics. */
int abs_gpu_remove(abs_gpu_ctx* ctx, const uint64_t* uids, uint64_t count);

/* CUDA stream used by the context (cudaStream_t); may be replaced. */
void* abs_gpu_stream(abs_gpu_ctx* ctx);
int abs_gpu_set_stream(abs_gpu_ctx* ctx, void* stream);

/* Timing of the dominant kernel (mechanical force) recorded with CUDA events
 * on the context stream: cumulative ms and launch count since the last reset. */
int abs_gpu_force_kernel_time(abs_gpu_ctx* ctx, double* total_ms, uint64_t* launches);
/* SimulationReport wall-time categories (report.hpp:12-23) as device time
 * of the iterations run while timing is enabled (abs_gpu_reset_timers(ctx, 1)):
 * out4 = {environment update, sorting, agent operations (staticness marking,
 * behaviours, forces, integration), setup/teardown (commit of additions)} ms;
 * per_iteration_ms[0 .. min(cap, *n)) with *n = iterations recorded (a
 * rolled-back attempt counts as one). */
int abs_gpu_phase_times(abs_gpu_ctx* ctx, double* out4, double* per_iteration_ms, uint64_t cap, uint64_t* n);
int abs_gpu_reset_timers(abs_gpu_ctx* ctx, int enable);
/* Parity hook: with enable != 0 every iteration records each agent's force
 * evaluations (run_forces' ++evals, simulation.cpp:473) — the size of its
 * neighbour set at the force radius; static agents record 0.
 * abs_gpu_download_evaluations copies the last iteration's counts in
 * download (storage) order. */
int abs_gpu_record_evaluations(abs_gpu_ctx* ctx, int enable);
int abs_gpu_download_evaluations(abs_gpu_ctx* ctx, uint32_t* out, uint64_t cap);
/* Each agent's slot in the REFERENCE's storage order (ResourceManager's agent
 * vector, resource_manager.hpp:19-101), download order. The device keeps its
 * own storage in cell order; the reference's order — which decides daughter
 * uids (commit.cpp:186-222) and survivor slots (remove_agents_parallel,
 * commit.cpp:14-106) — is carried as this key through uploads (slot = upload
 * order), appends, removals and exact Morton sorts (abs_gpu_sort, and in-loop
 * sorts of models that add or remove agents). Sorting a download by it gives
 * the reference's for_each_agent order. Single-domain contexts only
 * (decomposed contexts carry global keys). */
int abs_gpu_download_storage_keys(abs_gpu_ctx* ctx, uint32_t* out, uint64_t cap);
/* Neighbour-list statistics: out4 = {list builds, list
 * steps (iterations served from the lists), build launches timed, largest
 * candidate count of the last build}; *build_ms = CUDA-event time of the
 * timed builds (abs_gpu_reset_timers(ctx, 1)). Counts since creation. */
int abs_gpu_list_stats(abs_gpu_ctx* ctx, uint64_t* out4, double* build_ms);

#ifdef __cplusplus
}
#endif

#endif /* ABSIM_GPU_H */
