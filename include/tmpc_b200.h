/* tmpc_b200 — C ABI of the B200 batched candidate-rollout planner.
 *
 * This is the drop-in boundary under the reference planner entry points
 * `solve_ocp` / `plan_step`.  Everything
 * from "parallel over candidates k" down to the per-GPU arg-min runs on the
 * device behind these calls; the host side keeps the reference's structs
 * (VehicleParams/TireParams dynamics.hpp:20-58, ConstraintConfig
 * constraints.hpp:42-58, GridSpec/Heightmap/SignedDistanceMap
 * terrain.hpp:20-75,230-239) and the SPEC types (CostWeights, Goal,
 * PlannerConfig, RolloutResult: SPEC.md:348-367) and marshals them into the
 * plain-old-data mirrors below.  No torch types cross this boundary.
 *
 * Conventions
 *  - Return codes (errors.hpp:8-27):
 *      TMPC_OK 0, TMPC_ERR_NUMERIC 1 (all candidates diverged),
 *      TMPC_ERR_CONFIG 2 (same rules as the reference validate() methods),
 *      TMPC_ERR_RUNTIME 3 (CUDA / NCCL failure).  Message: tmpc_last_error().
 *  - The caller owns every host buffer; the library copies and never keeps a
 *    host pointer.  Terrain and params are immutable between set_* calls
 *    (terrain.hpp:54-55).
 *  - One context = one planning problem on one or several GPUs; not
 *    reentrant.  Results are identical for any GPU count
 *    because every candidate draws its controls from its GLOBAL index and
 *    every reduction is order-independent.
 */
#ifndef TMPC_B200_H_
#define TMPC_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TMPC_OK 0
#define TMPC_ERR_NUMERIC 1
#define TMPC_ERR_CONFIG 2
#define TMPC_ERR_RUNTIME 3

#define TMPC_STATE_DIM 13 /* SrbState::kDim, dynamics.hpp:174 */

/* Per-candidate flag bits (tmpc_get_costs). */
#define TMPC_FLAG_FEASIBLE 1u /* never diverged, ESM > 0 and every wheel sd > 0 */
#define TMPC_FLAG_DIVERGED 2u /* non-finite state or gimbal guard -> cost +inf */
#define TMPC_FLAG_GOAL 4u     /* rollout truncated at the goal circle */

/* Sampler kinds (SPEC.md:377-383 plus BASELINE-defined extensions). */
#define TMPC_SAMPLE_UNIFORM 0     /* i.i.d. U(-rate_max, rate_max) per step   */
#define TMPC_SAMPLE_RANDOM_WALK 1 /* clip(prev + U(-walk_step, walk_step))     */
#define TMPC_SAMPLE_WARM_GAUSS 2  /* clip(base + N(0, sigma^2)), k=0 unperturbed */

/* Arithmetic of the rollout kernel.  FP32: fp32 math over
 * fp32 terrain fields with fp64 state/cost storage (the fast path).  FP64:
 * fp64 math over fp64 fields, matching the fp64 reference to ~1e-12 even on
 * chaotic (rollover) candidates — the certification mode. */
#define TMPC_PRECISION_FP32 0
#define TMPC_PRECISION_FP64 1

/* Vehicle model of the rollouts.  SRB: the 13-state
 * single rigid body (dynamics.hpp:308-398) with the ESM rollover constraint
 * (constraints.hpp:16-23).  EST: the paper's baseline 7-state extended
 * single-track model on the local tangent plane (dynamics.hpp:213-275) with
 * the lateral-acceleration rollover constraint (constraints.hpp:62-65,78-80);
 * its state is read from / written to the SrbState slots x, y, psi, v_by,
 * omega_bz, delta, v_bx of the 13-vector. */
#define TMPC_MODEL_SRB 0
#define TMPC_MODEL_EST 1

/* Integration scheme of each dt_int substep, integrate_step's Scheme
 * (dynamics.hpp:419,446-468): forward Euler (the paper's planner,
 * PAPER.md:1065) or classical RK4.  The running cost is
 * the rectangle rule at the substep's start state in both. */
#define TMPC_SCHEME_EULER 0
#define TMPC_SCHEME_RK4 1

/* Selection order of the arg-min. */
#define TMPC_SELECT_FEASIBLE_FIRST 0 /* key (infeasible, J, k)            */
#define TMPC_SELECT_PLAIN 1          /* key (J, k): the reference's order */

/* Everything one rollout needs besides the state, terrain and sampler.
 * Field-for-field mirror of VehicleParams (dynamics.hpp:20-36), TireParams
 * (dynamics.hpp:50-52), ConstraintConfig (constraints.hpp:42-49), SPEC
 * CostWeights, Goal and the integration grid
 * (ControlSequence::dt_zoh dynamics.hpp:137, PlannerConfig dt_int
 * SPEC.md:361). */
typedef struct tmpc_params {
  /* VehicleParams */
  double M, J_xx, J_yy, J_zz, L_f, L_r, e, h, R, k_f, k_r, b_f, b_r;
  double delta_max, delta_rate_max, g;
  /* TireParams */
  double C, mu;
  /* ConstraintConfig (esm_nominal must be > 0: SURVEY App. A D10) */
  double a_by_bar, esm_nominal, eps_dist, sigma, safety_factor;
  int32_t enable_dist, enable_rollover;
  /* CostWeights */
  double w_t, w_c, w_g;
  /* Goal */
  double goal_x, goal_y, goal_r;
  /* Horizon: n_steps ZOH segments of dt_zoh, each integrated with
   * dt_zoh/dt_int forward-Euler substeps (dynamics.hpp:472-481). */
  double dt_zoh, dt_int;
  int32_t n_steps;
  int32_t selection; /* TMPC_SELECT_* */
  int32_t model;     /* TMPC_MODEL_SRB (default) or TMPC_MODEL_EST       */
  int32_t scheme;    /* TMPC_SCHEME_EULER (default) or TMPC_SCHEME_RK4   */
} tmpc_params;

/* Control sampler of one planning cycle.  Candidate k (GLOBAL index) uses the
 * counter stream RngStream(substream(seed, k)) (rng.hpp:10-48); per ZOH step
 * it consumes 1 draw (uniform / walk) or 2 draws (Gaussian, Box-Muller) per
 * control channel; the v_bx_rate channel is sampled only when
 * vdot_max > 0 (the reference fixes v_bx_rate = 0). */
typedef struct tmpc_sampling {
  int32_t kind; /* TMPC_SAMPLE_* */
  int32_t _pad0;
  uint64_t seed;
  double vdot_max;        /* bound of v_bx_rate samples; 0 => v_bx_rate = 0 */
  double walk_step;       /* random walk increment bound a                  */
  double warm_sigma_frac; /* Gaussian sigma as a fraction of the range      */
  const double* warm_seq; /* n_steps x 2 (delta_rate, v_bx_rate) or NULL   */
  int64_t k_begin;        /* first global candidate index of this shard     */
  int64_t k_count;        /* candidates in this shard                       */
  int64_t k_total;        /* candidates of the whole problem (all shards);
                           * 0 => k_count.  The fp32 lane layout is picked
                           * from it, so per-candidate results are bitwise
                           * independent of the shard count  */
} tmpc_sampling;

/* Row-major heightmap / signed-distance grid (terrain.hpp:20-29,56-75,
 * 230-239).  sdist may be NULL: SignedDistanceMap::has_features == false. */
typedef struct tmpc_terrain {
  const double* heights; /* ny*nx, index j*nx+i */
  const double* sdist;   /* ny*nx or NULL       */
  int32_t nx, ny;
  double origin_x, origin_y, resolution;
} tmpc_terrain;

/* Outcome of one planning cycle (SPEC RolloutResult + solver stats,
 * SPEC.md:365-367,386,414). */
typedef struct tmpc_result {
  int64_t best_index; /* global candidate index                */
  double best_cost;   /* J of the winner (+inf never returned) */
  int32_t best_feasible;
  float best_margin;
  int64_t n_candidates; /* over all ranks                         */
  int64_t n_feasible;
  int64_t n_diverged;
  int64_t n_goal;
  double min_cost;  /* over non-diverged candidates            */
  double mean_cost; /* over non-diverged candidates            */
  int64_t substeps_executed;
  double kernel_ms; /* device time of the cycle's kernels (CUDA events;
                     * max over the context's GPUs)                     */
  double cycle_ms;  /* host wall time of tmpc_solve                 */
} tmpc_result;

/* Context options.
 *
 * Two multi-GPU modes, both with contiguous candidate shards
 * and results bit-identical for any GPU count:
 *  - one process drives n_devices GPUs (devices[]): tmpc_solve splits its
 *    candidates over them, launches every GPU from the calling thread and
 *    folds the per-GPU reduction records on the host in device order
 *    (one blocking solve_ocp call);
 *  - one process per GPU (rank / world_size + nccl_id): every rank's record
 *    is exchanged with one ncclAllGather and folded in rank order.  A
 *    collective that does not complete within timeout_ms (a peer failed
 *    before reaching it) aborts the communicator and returns
 *    TMPC_ERR_RUNTIME instead of hanging. */
typedef struct tmpc_opts {
  int32_t device;      /* CUDA ordinal (when devices == NULL)             */
  int32_t rank;        /* this process's rank among world_size           */
  int32_t world_size;  /* >1 => cross-GPU arg-min through NCCL            */
  int32_t lanes;       /* 0 = auto, 1 = thread per candidate, 4 = quad   */
  int64_t k_max;       /* largest shard (candidates) this ctx will solve */
  int32_t n_steps_max; /* largest horizon                                */
  int32_t precision;   /* TMPC_PRECISION_FP32 (default) or _FP64          */
  const void* nccl_id; /* 128-byte ncclUniqueId, required if world_size>1
                        * (given with world_size == 1: a 1-rank communicator) */
  int32_t ordering;    /* TMPC_ORDER_AUTO (default), _OFF or _ON: assign
                        * candidates to threads by predicted path (terrain
                        * locality of the fp32 kernel; outputs unchanged) */
  int32_t n_devices;   /* GPUs this context drives (0 or 1: one GPU)      */
  const int32_t* devices; /* n_devices CUDA ordinals (may repeat an ordinal:
                           * several shards on one GPU), or NULL => {device} */
  int32_t timeout_ms;  /* NCCL collective watchdog; 0 => 60000             */
  int32_t graphs;      /* TMPC_GRAPHS_AUTO (default: replay the cycle as a
                        * CUDA graph) or TMPC_GRAPHS_OFF (direct launches) */
  int32_t exchange;    /* one process per GPU: TMPC_EXCHANGE_NCCL (default
                        * with nccl_id) or TMPC_EXCHANGE_PEER -- the rollout
                        * kernel itself stores its record into every rank's
                        * mailbox over peer memory (NVLink) and waits for
                        * theirs (tmpc_peer_export / tmpc_peer_connect)    */
  int32_t _pad1;
} tmpc_opts;

#define TMPC_EXCHANGE_NCCL 0
#define TMPC_EXCHANGE_PEER 1

#define TMPC_GRAPHS_AUTO 0
#define TMPC_GRAPHS_OFF 1

#define TMPC_ORDER_AUTO 0
#define TMPC_ORDER_OFF 1
#define TMPC_ORDER_ON 2

typedef struct tmpc_ctx tmpc_ctx;

/* ---- context lifecycle ---------------------------------------------- */
int tmpc_ctx_create(const tmpc_opts* opts, tmpc_ctx** out);
void tmpc_ctx_destroy(tmpc_ctx* ctx);
const char* tmpc_last_error(const tmpc_ctx* ctx); /* ctx may be NULL */

/* ---- configuration (host validation mirrors the reference validate()) -- */
/* Validates like VehicleParams::validate (dynamics.hpp:38-47),
 * TireParams::validate (54-57), ConstraintConfig::validate
 * (constraints.hpp:51-57) plus esm_nominal > 0, dt_int | dt_zoh
 * (dynamics.hpp:477-481), n_steps >= 1, goal_r > 0.  No device needed. */
int tmpc_validate_params(const tmpc_params* p, char* msg, size_t msg_len);
int tmpc_validate_terrain(const tmpc_terrain* t, char* msg, size_t msg_len);
int tmpc_set_params(tmpc_ctx* ctx, const tmpc_params* p);
/* Copies, pads by 2 replicated cells, precomputes the node gradient field
 * and uploads the terrain store. */
int tmpc_set_terrain(tmpc_ctx* ctx, const tmpc_terrain* t);

/* ---- the hot path ---------------------------------------------------- */
/* One planning cycle: samples, rolls out and scores candidates
 * [k_begin, k_begin+k_count), arg-min on this GPU, then across ranks.
 * Blocking.  s0: 13 doubles in SrbState::as_array order
 * (dynamics.hpp:175-178).  best_controls (nullable): n_steps x 2 floats
 * (delta_rate, v_bx_rate) of the winner, regenerated on the host from
 * (seed, best_index). */
int tmpc_solve(tmpc_ctx* ctx, const double* s0, const tmpc_sampling* smp,
               tmpc_result* out, double* best_controls);

/* Asynchronous variant for device-resident timing: s0 and the sampler are
 * staged first with tmpc_stage_cycle; tmpc_launch_cycle then only enqueues
 * the rollout kernel + arg-min on the context stream (no host sync, no
 * copies).  tmpc_finish_cycle synchronises and fills `out`. */
int tmpc_stage_cycle(tmpc_ctx* ctx, const double* s0, const tmpc_sampling* smp);
int tmpc_launch_cycle(tmpc_ctx* ctx);
int tmpc_finish_cycle(tmpc_ctx* ctx, tmpc_result* out);

/* Per-candidate results of the last cycle (parity / debugging); each array
 * has k_count entries of this shard.  Any pointer may be NULL. */
int tmpc_get_costs(tmpc_ctx* ctx, double* cost, uint8_t* flags, float* margin);

/* Device stream of the context's first GPU (cudaStream_t), for event timing. */
void* tmpc_get_stream(tmpc_ctx* ctx);
/* Number of GPUs the context drives, and the stream / ordinal of GPU i. */
int tmpc_num_devices(const tmpc_ctx* ctx);
void* tmpc_get_device_stream(tmpc_ctx* ctx, int32_t i);
int tmpc_get_device_ordinal(const tmpc_ctx* ctx, int32_t i);
/* Number of kernels tmpc_launch_cycle enqueues per cycle. */
int tmpc_kernels_per_cycle(const tmpc_ctx* ctx);

/* ---- host helpers (no device) ---------------------------------------- */
/* Control sequence of global candidate k exactly as the device draws it
 * (SPEC.md:377-383 + tmpc_sampling).  out: n_steps x 2 doubles. */
int tmpc_sample_controls(const tmpc_params* p, const tmpc_sampling* smp, int64_t k,
                         double* out);
/* Arg-min key of one candidate: hi = infeasible << 63 | IEEE bits of the
 * fp64 cost (>= 0 or +inf, so bits order like values), paired with the
 * global index as lo; the lexicographic MIN of (hi, lo) is the
 * (infeasible, J, k) arg-min with lowest-index ties on the exact cost. */
uint64_t tmpc_key_hi(double cost, int feasible, int selection);

/* Per-GPU reduction record of one cycle (what one GPU's rollout kernel
 * reduces its shard to; exchanged between GPUs / ranks and folded).
 * Every field is an order-independent reduction (integer sums, MINs). */
typedef struct tmpc_rank_record {
  uint64_t key_lo, key_hi; /* arg-min pair; (~0, ~0) = no candidate      */
  uint64_t min_cost_bits;  /* bits of the least finite cost (+inf bits)  */
  uint64_t done_blocks;    /* kernel-internal ticket                      */
  uint64_t n_feasible, n_diverged, n_goal, n_finite, substeps;
  uint64_t cost_limb[3];   /* finite costs on the 2^-24 grid, 32-bit limbs */
  double best_cost;        /* the shard winner's exact cost, flags, margin */
  float best_margin;
  int32_t best_flags;
  int64_t k_begin, k_count; /* the shard                                  */
} tmpc_rank_record;

/* Host mirror of one GPU's reduction: the record of the per-candidate
 * outputs of shard [k_begin, k_begin + k_count) (substeps may be NULL). */
int tmpc_make_record(const double* cost, const uint8_t* flags, const float* margin,
                     const int64_t* substeps, int64_t k_begin, int64_t k_count, int selection,
                     tmpc_rank_record* out);
/* Fold n records (in order) into the cycle's result: global arg-min, counts,
 * min / mean cost, the winner's fields.  TMPC_ERR_NUMERIC when every
 * candidate diverged. */
int tmpc_fold_records(const tmpc_rank_record* recs, int32_t n, tmpc_result* out);

/* Peer-memory exchange (opts.exchange == TMPC_EXCHANGE_PEER): export this
 * rank's mailbox as a 64-byte CUDA IPC handle; the caller all-gathers the
 * world_size handles (any channel) and connects every rank to all of them in
 * rank order.  Every cycle the rollout kernel's last block then stores this
 * GPU's reduction record into all mailboxes (NVLink stores), publishes the
 * cycle's sequence number and waits for every rank's record -- the
 * compute step and its collective in one kernel; a rank that never delivers
 * fails the call after timeout_ms. */
int tmpc_peer_export(tmpc_ctx* ctx, void* handle64);
int tmpc_peer_connect(tmpc_ctx* ctx, const void* handles, int32_t n);
/* Inspect this rank's own mailbox: the record rank src_rank stored for
 * sequence number seq (buffer seq & 1) and the sequence number src_rank last
 * published (diagnostics of the exchange; the kernel never waits on it). */
int tmpc_peer_inspect(tmpc_ctx* ctx, int32_t src_rank, uint64_t seq, tmpc_rank_record* out,
                      uint64_t* published_seq);

/* NCCL unique id for world_size > 1 (rank 0 creates, caller broadcasts). */
int tmpc_nccl_unique_id(void* out128);

/* ---- workload setup (host, runs once per terrain) --- */
/* Additive synthetic heightmap (all components optional, zero amplitude =>
 * absent), row-major j*nx+i, fp64, deterministic in `seed` (streams derived
 * with substream(seed, tag) like synth_terrain, terrain.hpp:309):
 *   sine    h += sine_amp * sin(2 pi (x-ox)/L + p1) * sin(2 pi (y-oy)/L + p2)
 *   noise   h += U(-noise_amp, noise_amp) per cell
 *   fractal h += value noise, `fractal_octaves` octaves, lattice spacing
 *           fractal_lattice / 2^o, amplitude fractal_persistence^o,
 *           smoothstep interpolation, rescaled to fractal_pp peak-to-peak
 *   slopes  h += sinusoidal side slopes alternating between +-tan(slope_deg),
 *           period slope_period along direction slope_dir
 *   berms   h += n_berms capsule berms (height berm_height, length
 *           berm_length, raised-cosine cross-section of half-width
 *           berm_halfwidth) at seeded positions/orientations */
typedef struct tmpc_synth_spec {
  int32_t nx, ny;
  double origin_x, origin_y, resolution;
  uint64_t seed;
  double sine_amp, sine_wavelength;
  double noise_amp;
  int32_t fractal_octaves;
  int32_t _pad0;
  double fractal_persistence, fractal_lattice, fractal_pp;
  double slope_deg, slope_period, slope_dir;
  int32_t n_berms;
  int32_t _pad1;
  double berm_height, berm_length, berm_halfwidth;
} tmpc_synth_spec;
int tmpc_synth_heightmap(const tmpc_synth_spec* spec, double* out);

/* Seeded cylinder obstacles as regular n-gon perimeters:
 * centres uniform in [x_min,x_max]x[y_min,y_max] outside the keep-out circle
 * (clear_x, clear_y, clear_r), radius U(r_min, r_max).
 * circles: n x 3 (cx, cy, r); verts: n x n_gon x 2 (counter-clockwise). */
typedef struct tmpc_obstacle_spec {
  uint64_t seed;
  int32_t n, n_gon;
  double r_min, r_max;
  double x_min, x_max, y_min, y_max;
  double clear_x, clear_y, clear_r;
} tmpc_obstacle_spec;
int tmpc_synth_obstacles(const tmpc_obstacle_spec* spec, double* circles, double* verts);
/* Adds `height` to every cell whose centre lies inside an obstacle polygon. */
int tmpc_stamp_obstacles(const tmpc_terrain* grid, double* heights, int32_t n_poly,
                         const int32_t* poly_off, const double* verts, double height);
/* build_sdist_map (terrain.hpp:241-260): per-cell MIN of signed_distance
 * (terrain.hpp:186-224) over perimeters (kinds: 0 obstacle, 1 path
 * boundary), bit-identical to the reference; bounding-circle culling keeps it
 * exact.  n_poly == 0 => every cell +inf. */
int tmpc_build_sdist_map(int32_t nx, int32_t ny, double origin_x, double origin_y,
                         double resolution, int32_t n_poly, const int32_t* poly_off,
                         const double* verts, const int32_t* kinds, double* out,
                         int32_t n_threads);

/* ---- device terrain preprocessing --------------------- */
/* gaussian_smooth (terrain.hpp:102-138) on GPU `device`: separable Gaussian,
 * taps truncated at 3 sigma and renormalised, replicate padding; host fp64
 * heights in, host fp64 heights out, bit-identical to the reference.
 * sigma_m == 0 copies; sigma_m < 0 => TMPC_ERR_CONFIG (terrain.hpp:105). */
int tmpc_gaussian_smooth(int32_t device, const double* heights, int32_t nx, int32_t ny,
                         double resolution, double sigma_m, double* out);
/* build_sdist_map (terrain.hpp:241-260) on GPU `device`: same arguments and
 * bit-identical result as tmpc_build_sdist_map (one thread per cell,
 * bounding-circle culling that never changes the minimum). */
int tmpc_build_sdist_map_gpu(int32_t device, int32_t nx, int32_t ny, double origin_x,
                             double origin_y, double resolution, int32_t n_poly,
                             const int32_t* poly_off, const double* verts, const int32_t* kinds,
                             double* out);

/* ---- closed loop (BASELINE c5) ------------------------ */
/* Plant between planning cycles: advances `state` (13 doubles, in place) by
 * n_steps RK4 steps of dt under the held control (delta_rate, v_bx_rate),
 * the reference integrate_step<SrbModel> kRk4 + clamp_steering
 * (dynamics.hpp:446-468) over height_at/gradient_at (terrain.hpp:79-93), fp64
 * on the host (SPEC.md:447-453 plant_step).  Returns TMPC_ERR_NUMERIC on the
 * gimbal guard or a non-finite state. */
int tmpc_plant_step(const tmpc_params* p, const tmpc_terrain* t, const double* control, double dt,
                    int32_t n_steps, double* state);

/* ---- open-loop model error analysis ------------------ */
/* open_loop_errors for n_traj
 * trajectories on the context's (first) GPU: each starts from s0[13 t..] and
 * applies controls[2 n_steps t..] (n_steps ZOH pairs of the context's
 * params); the plant is the SRB model with RK4 at plant_dt (must divide
 * dt_int; the harness plant), the model is `model`
 * (TMPC_MODEL_SRB / _EST) with the params' scheme at dt_int.  Per trajectory
 * the time averages over the horizon of the location error |p^ - p| and of
 * |U^_ESM - U_ESM| (EST: ESM of its local-plane attitude), sampled at every
 * model substep start.  flags: 1 model diverged, 2 plant diverged (errors
 * NaN).  Needs a TMPC_PRECISION_FP64 context (fp64 math and terrain). */
int tmpc_open_loop_errors(tmpc_ctx* ctx, int32_t model, const double* s0, const double* controls,
                          int64_t n_traj, double plant_dt, double* loc_err, double* esm_err,
                          uint8_t* flags);
/* The plant's own terrain LOD for tmpc_open_loop_errors (the paper's
 * unsmoothed plant LOD vs the smoothed model LODs); same
 * grid as the context's terrain; NULL => the plant uses the context's
 * terrain.  FP64 contexts only. */
int tmpc_set_plant_terrain(tmpc_ctx* ctx, const tmpc_terrain* t);

/* FP32 FFMA throughput of `device` in TFLOP/s (roofline denominator of the
 * FP32-SIMT-bound rollout kernel; bench.py measures it on the same box). */
int tmpc_fp32_peak(int32_t device, double* tflops);

/* Library identification (build flags, arch) for logs. */
const char* tmpc_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* TMPC_B200_H_ */
