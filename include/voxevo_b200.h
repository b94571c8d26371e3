/* voxevo_b200.h — C ABI of the B200-native (sm_100a) voxevo hot path.
 *
 * Drop-in boundary for the data-parallel path of arXiv 2405.00698's reference
 * (`voxevo`, /root/reference/proj/include/voxevo).  The reference exposes no
 * plugin/FFI; its API is the header-only `voxevo::` C++ surface.  Every entry
 * point below names the reference function(s) it replaces (file:line, paths
 * relative to proj/include/voxevo).  Batch-granular because per-robot calls are
 * too fine for a GPU.
 *
 * Conventions
 *  - Status codes only; no exceptions cross the ABI.  vx_last_error() returns
 *    the calling thread's last message.  The C++ shim (voxevo_b200/voxevo_shim.hpp)
 *    maps codes back to the reference exception types.
 *  - `_dev` entry points take DEVICE pointers (caller-owned, e.g. torch
 *    tensors) and are stream-ordered on the context stream (vx_set_stream);
 *    they never synchronize.  Other entry points take HOST pointers, copy
 *    in/out and synchronize before returning.
 *  - Opaque handles own their device memory.  Not thread-safe per context.
 *  - All arithmetic is FP64 in the reference's operation order (parity mode,
 *    no FMA contraction) unless a function says otherwise.
 */
#ifndef VOXEVO_B200_H
#define VOXEVO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VX_ABI_VERSION 3
#define VX_MAX_HIDDEN 8
#define VX_NMAT 5

typedef enum {
    VX_OK = 0,
    VX_EINVAL = 1,   /* std::invalid_argument in the reference (validate()) */
    VX_ECUDA = 2,    /* CUDA runtime error */
    VX_EOOM = 3,     /* device allocation failed */
    VX_EEMPTY = 4,   /* empty_robot (morphology.hpp:17-19, :230) */
    VX_ESHAPE = 5,   /* shape_mismatch (genome.hpp:19-21) */
    VX_ESTATE = 6,   /* call made in the wrong state (e.g. finish before begin) */
    VX_ENODEV = 7,   /* no CUDA device / extension unusable */
    VX_ENCCL = 8     /* NCCL missing or failed (vx_comm_*) */
} vx_status;

typedef struct vx_ctx vx_ctx;     /* one per device: stream, scratch, counters */
typedef struct vx_batch vx_batch; /* device-resident batch of MassSpringSystems */
typedef struct vx_evo vx_evo;     /* device-resident EvolutionState */
typedef struct vx_comm vx_comm;   /* NCCL communicator of one rank (one GPU) */

/* EncodingSpec + hidden widths (genome.hpp:25-35, sample_genome :146) */
typedef struct {
    int32_t m;        /* frequency rows; features = 2m */
    int32_t n_hidden; /* <= VX_MAX_HIDDEN */
    int32_t hidden[VX_MAX_HIDDEN];
    double sigma;
} vx_arch;

/* MaterialTable (morphology.hpp:45-65) */
typedef struct {
    double k_muscle, k_soft, k_bone, damping_ratio, amp_max, phase_max, voxel_edge, mass_per_vertex;
} vx_materials;

/* GroundPlane (morphology.hpp:124-129) */
typedef struct {
    double k, damping_ratio, mu_static, mu_kinetic;
} vx_plane;

/* SimConfig (physics.hpp:16-29) */
typedef struct {
    double gravity, dt, duration, actuation_frequency;
    int32_t enable_gravity, enable_contact;
} vx_sim;

/* TrajectorySummary (physics.hpp:31-37) + exact work audit */
typedef struct {
    double com_start[3];
    double com_end[3];
    double horizontal_displacement;
    double max_speed;
    int32_t diverged;
    int32_t status;          /* 0 simulated, 1 gated empty, 2 gated no muscle */
    int64_t steps;           /* step() calls made (incl. a diverging one) */
    uint64_t spring_updates; /* SimWorkspace::spring_updates (physics.hpp:212) */
} vx_summary;

/* HyperParams (evolution.hpp:22-38) */
typedef struct {
    double mutation_rate, mutation_scale, crossover_rate, elite_fraction;
    double material_multipliers[3];
} vx_hyper;

/* EvolutionConfig (evolution.hpp:40-64) */
typedef struct {
    int32_t population, generations, grid_w, grid_h, grid_d, tournament_size, threads;
    uint64_t seed;
    vx_arch arch;
    vx_hyper initial_params;
    vx_materials materials;
    vx_plane plane;
    vx_sim sim;
} vx_evo_config;

/* GenerationReport (evolution.hpp:75-84) */
typedef struct {
    int32_t generation;
    int32_t evaluations;
    vx_hyper params;
    double best, mean, stddev, diversity, wall_time;
    uint64_t spring_updates; /* exact, summed over this generation's simulations */
} vx_report;

/* ------------------------------------------------------------ library ---- */
int32_t vx_abi_version(void);
const char* vx_last_error(void);
/* Reference defaults (struct initializers in the headers above). */
void vx_default_arch(vx_arch* a);
void vx_default_materials(vx_materials* m);
void vx_default_plane(vx_plane* p);
void vx_default_sim(vx_sim* s);
void vx_default_hyper(vx_hyper* h);
void vx_default_evo_config(vx_evo_config* c);
/* Genome::parameter_count (genome.hpp:83-87); -1 on invalid arch */
int64_t vx_param_count(const vx_arch* a);
/* detail::elite_count (evolution.hpp:131-136) */
int32_t vx_elite_count(double elite_fraction, int32_t population);
/* HyperParams::clamp (evolution.hpp:29-35) */
void vx_hyper_clamp(vx_hyper* h);

/* ------------------------------------------------------------ context ---- */
vx_status vx_create(int32_t device, vx_ctx** out);
vx_status vx_destroy(vx_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 * NULL restores the context's own stream. */
vx_status vx_set_stream(vx_ctx* ctx, void* cuda_stream);
void* vx_get_stream(vx_ctx* ctx);
vx_status vx_synchronize(vx_ctx* ctx);
/* Number of this library's kernel launches issued on ctx so far. */
uint64_t vx_launch_count(vx_ctx* ctx);
/* 10^3 cluster integrator: a persistent one-SM streaming filler on the SMs no
 * 4-CTA cluster can be placed on (robots claimed from one shared counter).
 * mode -1: from the VX_FILLER environment variable (default 1), 0 off,
 * 1 on for batches large enough to keep the clusters busy, 2 on at any batch
 * size (tests).  vx_last_filler_ctas: filler CTAs of the last launch. */
vx_status vx_set_filler(vx_ctx* ctx, int32_t mode);
int32_t vx_last_filler_ctas(vx_ctx* ctx);
/* SM count / clock / name of the context device. */
vx_status vx_device_info(vx_ctx* ctx, int32_t* sm_count, int32_t* clock_khz, char* name, int32_t name_cap);

/* ------------------------------------------------ genome / decode (K1-K4) */
/* sample_genome for P seeds (genome.hpp:146-166): one mt19937_64 per genome
 * on device.  W is bit-exact (uniform draws); B uses device log/cos (ulp-level
 * vs glibc).  params: P x param_count, bmat: P x 3m (device pointers). */
vx_status vx_sample_genomes_dev(vx_ctx* ctx, const vx_arch* a, int32_t P, const uint64_t* d_seeds, double* d_params,
                                double* d_bmat);
/* gaussian_encode (genome.hpp:168-179) of one point v[3] with the m x 3
 * encoding matrix: out[r] = cos(2 pi B_r . v), out[m + r] = sin(...); host
 * libm, bit-identical to the reference on the same machine. */
vx_status vx_gaussian_encode(const double* v, const double* bmat, int32_t m, double* out);
/* Host-pointer variant: seeds (P), params (P x param_count), bmat (P x 3m). */
vx_status vx_sample_genomes(vx_ctx* ctx, const vx_arch* a, int32_t P, const uint64_t* seeds, double* params,
                            double* bmat);
/* forward (genome.hpp:187-211), the pure spatial query, for P genomes x
 * n_points points each (host pointers): points [P][n_points][3] in the unit
 * cube frame, probs [P][n_points][5] (max-subtracted softmax of the material
 * head), weight [P][n_points] (stable sigmoid of the weight head, unclamped).
 * Device tanh/exp: rtol ~1e-13 against glibc. */
vx_status vx_forward(vx_ctx* ctx, const vx_arch* a, int32_t P, const double* params, const double* bmat,
                     int32_t n_points, const double* points, double* probs, double* weight);
/* decode for P genomes (morphology.hpp:141-157 over forward, genome.hpp:187-211):
 * materials (u8, argmax strict-> ties low) and clamped weights per cell,
 * cells in x-fastest order.  The MLP layers run on the FP64 tensor pipe (DMMA);
 * a genome with any voxel whose top-2 probability gap is < 1e-8 (relative) is
 * re-decoded in the reference's sequential order, so materials equal the exact
 * path's (VX_DECODE=exact in the environment forces the exact path).  d_guard
 * (optional, 1 u32) counts voxels whose top-2 softmax gap is < 1e-12 (argmax
 * could differ from glibc's). */
vx_status vx_decode_dev(vx_ctx* ctx, const vx_arch* a, int32_t P, const double* d_params, const double* d_bmat,
                        int32_t w, int32_t h, int32_t d, uint8_t* d_mat, double* d_weight, uint32_t* d_guard);
vx_status vx_decode(vx_ctx* ctx, const vx_arch* a, int32_t P, const double* params, const double* bmat, int32_t w,
                    int32_t h, int32_t d, uint8_t* mat, double* weight);
/* How many genomes of the context's LAST decode launch were re-decoded on the
 * exact path (-1: that decode ran on the exact path only).  Synchronises the
 * context stream. */
vx_status vx_decode_refined(vx_ctx* ctx, int64_t* n_refined);
/* largest_component for P grids (morphology.hpp:162-208) */
vx_status vx_largest_component_dev(vx_ctx* ctx, int32_t P, int32_t w, int32_t h, int32_t d, const uint8_t* d_in,
                                   uint8_t* d_out);
vx_status vx_largest_component(vx_ctx* ctx, int32_t P, int32_t w, int32_t h, int32_t d, const uint8_t* in,
                               uint8_t* out);

/* ------------------------------------------- mass-spring batches (K5-K6) */
/* build_mass_spring for P body grids (morphology.hpp:217-299) on device.
 * Empty grids become zero-mass robots (the reference throws empty_robot;
 * vx_batch_robot_sizes reports nm = 0 for them). */
vx_status vx_batch_build_dev(vx_ctx* ctx, int32_t P, int32_t w, int32_t h, int32_t d, const uint8_t* d_mat,
                             const double* d_weight, const vx_materials* table, const vx_plane* plane,
                             vx_batch** out);
vx_status vx_batch_build(vx_ctx* ctx, int32_t P, int32_t w, int32_t h, int32_t d, const uint8_t* mat,
                         const double* weight, const vx_materials* table, const vx_plane* plane, vx_batch** out);
/* Upload n host-assembled systems (e.g. the reference tests' dumbbells,
 * test_physics.cpp:13-27).  Offsets are n+1 prefix sums; spring endpoints are
 * robot-local.  pos/vel are nm x 3 row-major.  act arrays may be NULL. */
vx_status vx_batch_upload(vx_ctx* ctx, int32_t n, const int64_t* mass_off, const int64_t* spring_off,
                          const double* pos, const double* vel, const double* mass, const int32_t* si,
                          const int32_t* sj, const double* k, const double* rest0, const double* zeta,
                          const uint8_t* has_act, const double* sign, const double* amp, const double* phase,
                          const vx_plane* plane, vx_batch** out);
vx_status vx_batch_free(vx_batch* b);
int32_t vx_batch_count(const vx_batch* b);
/* mass_off/spring_off: n+1 each (host). */
vx_status vx_batch_offsets(const vx_batch* b, int64_t* mass_off, int64_t* spring_off);
/* Download topology + current state (any pointer may be NULL). */
vx_status vx_batch_download(vx_batch* b, double* pos, double* vel, double* mass, int32_t* si, int32_t* sj, double* k,
                            double* rest0, double* zeta, uint8_t* has_act, double* sign, double* amp, double* phase);
/* Overwrite the current state (pos/vel nm x 3). */
vx_status vx_batch_set_state(vx_batch* b, const double* pos, const double* vel);
/* SimWorkspace-derived arrays (physics.hpp:140-185): damp_coef, amp_rest,
 * sin/cos(phase), ground_damp, CSR incidence (inc_off: per robot nm+1 local
 * offsets concatenated; inc_spring robot-local; inc_sign +-1). */
vx_status vx_batch_workspace(vx_batch* b, double* damp_coef, double* amp_rest, double* sin_phase, double* cos_phase,
                             double* ground_damp, int32_t* inc_off, int32_t* inc_spring, double* inc_sign);
/* Parity mode: replace device-computed sin/cos(phase) with host values
 * (glibc's), making the integrator bit-exact on identical inputs. */
vx_status vx_batch_override_phase(vx_batch* b, const double* sin_phase, const double* cos_phase);

/* ------------------------------------------------ integrator (K7-K9) ---- */
/* step() (physics.hpp:191-264) for k = k0 .. k0+n_steps-1 on every robot,
 * t = k*dt; MUTATES the batch state; each robot stops at its first diverged
 * step.  summaries (host, n entries, optional) report COM before/after,
 * max_speed, steps and exact spring updates of THIS call. */
vx_status vx_batch_step(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, int64_t k0, int64_t n_steps,
                        vx_summary* summaries);
/* step(sys, t, cfg, ws) (physics.hpp:191-264) once on every robot at an
 * arbitrary time t (drive sin/cos((2 pi f) t) with the host libm); MUTATES
 * the batch state; summaries as vx_batch_step (steps = 1 unless diverged,
 * spring_updates = springs when phase 1 completed). */
vx_status vx_batch_step_at(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, double t, vx_summary* summaries);
/* simulate() (physics.hpp:287-311) for every robot: llround(duration/dt)
 * steps from t = 0 on a private copy of the state (the batch is not
 * modified, like the reference's by-value argument). */
vx_status vx_batch_simulate(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, vx_summary* summaries);
/* simulate() with its trajectory dump (physics.hpp:280-311): for each robot
 * the (t, com x, com y, com z) rows the reference pushes — one every `stride`
 * steps before that step (stride <= 0: none) while the robot has not
 * diverged, then the final row at t = n_steps*dt — written to samples
 * (host, n x cap x 4 doubles; rows beyond cap are counted, not written) with
 * the per-robot row count in counts (host, n).  cap for no truncation:
 * ceil(n_steps / stride) + 1.  A robot without masses gets no rows and a
 * zero summary.  The batch is not modified.  Bit-identical to the
 * reference's simulate(sys, cfg, &dump, stride) on identical systems. */
vx_status vx_batch_simulate_dump(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, int32_t stride, int64_t cap,
                                 double* samples, int64_t* counts, vx_summary* summaries);
/* Device-pointer variant: summaries written to d_summaries (n entries). */
vx_status vx_batch_simulate_dev(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, vx_summary* d_summaries);

/* ------------------------------------------------ fitness (K4-K10 fused) */
/* evaluate_fitness (evolution.hpp:110-119) for P raw grids: largest
 * component -> gates (empty / no muscle -> 0) -> build -> simulate ->
 * diverged -> 0 else horizontal displacement.  table is the (already
 * scaled) material table.  d_todo (optional) selects n_todo grid indices;
 * fitness is written at those indices only.  d_summaries optional (P). */
vx_status vx_evaluate_dev(vx_ctx* ctx, int32_t P, int32_t w, int32_t h, int32_t d, const uint8_t* d_mat,
                          const double* d_weight, const vx_materials* table, const vx_plane* plane, const vx_sim* sim,
                          const int32_t* d_todo, int32_t n_todo, double* d_fitness, vx_summary* d_summaries);
vx_status vx_evaluate(vx_ctx* ctx, int32_t P, int32_t w, int32_t h, int32_t d, const uint8_t* mat,
                      const double* weight, const vx_materials* table, const vx_plane* plane, const vx_sim* sim,
                      double* fitness, vx_summary* summaries);

/* ------------------------------------------------- population stats (K11-K12) */
/* population_diversity (evolution.hpp:89-105) over P grids of `cells`
 * materials (0..4), in the given order: the reference's double BIT FOR BIT
 * (pair differ counts, then its ordered running sum of differ/cells
 * reproduced in parallel, diversity.cu). */
vx_status vx_population_diversity_dev(vx_ctx* ctx, int32_t P, int32_t cells, const uint8_t* d_mat, double* d_out);
vx_status vx_population_diversity(vx_ctx* ctx, int32_t P, int32_t cells, const uint8_t* mat, double* out);
/* Per-cell material counts (cells x 5 int64) and the O(P cells) diversity
 * from a (reduced) histogram: exact pair counts, within 1e-15 relative of the
 * reference (its rounding sequence is not reproduced; the evolution path uses
 * the bit-exact form above). */
vx_status vx_material_histogram_dev(vx_ctx* ctx, int32_t P, int32_t cells, const uint8_t* d_mat,
                                    int64_t* d_hist, int32_t accumulate);
vx_status vx_diversity_from_histogram_dev(vx_ctx* ctx, int32_t P, int32_t cells, const int64_t* d_hist,
                                          double* d_out);

/* ------------------------------------------------------- evolution (K11-K14) */
/* init_evolution (evolution.hpp:197-211) with genomes sampled on device. */
vx_status vx_evo_create(vx_ctx* ctx, const vx_evo_config* cfg, vx_evo** out);
vx_status vx_evo_free(vx_evo* e);
/* evolve_generation (evolution.hpp:217-293), advisor off (the shim calls the
 * advisor between generations and applies vx_evo_set_params). */
vx_status vx_evo_generation(vx_evo* e, vx_report* rep);
/* Sharded form: begin() decodes and evaluates the children
 * assigned to `rank` of `world` (strided over the todo list; no grid ever
 * moves: every rank derives the same owner map) and writes this rank's part
 * of the exchange buffer; the caller then all-reduces (sum) the buffer
 * (device, vx_evo_exchange_buffer) across ranks; finish() sorts, reports and
 * breeds (replicated, identical on every rank). */
vx_status vx_evo_begin(vx_evo* e, int32_t rank, int32_t world);
/* d_buf: P doubles (fitness of locally evaluated children, 0 elsewhere),
 * P doubles of per-robot spring updates, then cells x 5 material counts over
 * the individuals whose grid this rank owns (the population diversity is a
 * function of the summed counts); n_doubles = 2P + 5 cells. */
vx_status vx_evo_exchange_buffer(vx_evo* e, double** d_buf, int64_t* n_doubles);
/* Use a caller-owned device buffer of n_doubles (vx_evo_exchange_buffer; e.g.
 * a torch tensor that torch.distributed all-reduces over NCCL) as the
 * exchange buffer. */
vx_status vx_evo_set_exchange_buffer(vx_evo* e, double* d_buf);
/* Generation-0 reset from DEVICE arrays (P x np params, P x 3m B): fitness,
 * evaluated flags and cached grids are cleared (init_evolution state). */
vx_status vx_evo_load_population_dev(vx_evo* e, const double* d_params, const double* d_bmat);
vx_status vx_evo_finish(vx_evo* e, vx_report* rep);
vx_status vx_evo_get_population(vx_evo* e, double* params, double* bmat, double* fitness, uint8_t* evaluated,
                                uint8_t* grids, double* grid_w);
/* Replace the population (host arrays).  grids NULL => not decoded yet; with
 * grids, an individual whose first cell holds material 255 (the marker
 * vx_evo_get_population writes) is not decoded yet either. */
vx_status vx_evo_set_population(vx_evo* e, const double* params, const double* bmat, const double* fitness,
                                const uint8_t* evaluated, const uint8_t* grids, const double* grid_w);
/* Device views of the population genomes (P x np, P x 3m), valid until the
 * next vx_evo_* call. */
vx_status vx_evo_population_dev(vx_evo* e, double** d_params, double** d_bmat, double** d_fitness);
/* -------------------------------------- population sharding
 * Replaces the CPU parallel_for over children (evolution.hpp:237-241,
 * parallel.hpp:17-51) across GPUs: GA state replicated, children sharded,
 * ONE sum all-reduce of the exchange buffer per generation; results are
 * bit-identical for any world size (the reference's thread-count invariance,
 * test_evolution.cpp:196-215).  NCCL is loaded at run time (libnccl.so.2). */
#define VX_COMM_ID_BYTES 128
vx_status vx_comm_available(void);                            /* VX_OK when NCCL is loadable */
vx_status vx_comm_unique_id(uint8_t id[VX_COMM_ID_BYTES]);    /* rank 0 creates, the caller distributes */
/* One process per GPU (ncclCommInitRank; collective over the `world` ranks). */
vx_status vx_comm_create(vx_ctx* ctx, int32_t world, int32_t rank, const uint8_t id[VX_COMM_ID_BYTES],
                         vx_comm** out);
/* One process driving n GPUs (ncclCommInitAll over the contexts' devices). */
vx_status vx_comm_create_all(int32_t n, vx_ctx* const* ctxs, vx_comm** comms);
vx_status vx_comm_destroy(vx_comm* c);
vx_status vx_comm_rank(const vx_comm* c, int32_t* rank, int32_t* world);
/* Sum all-reduce of n device doubles on the communicator's context stream. */
vx_status vx_comm_allreduce_sum_dev(vx_comm* c, double* d_buf, int64_t n);
/* Attach a communicator: vx_evo_generation then runs begin(rank, world) ->
 * all-reduce of the exchange buffer -> finish.  NULL detaches. */
vx_status vx_evo_set_comm(vx_evo* e, vx_comm* c);
/* Any other transport (MPI, gloo, host copies): vx_evo_generation calls
 * fn(d_buf, n_doubles, user) between begin and finish; fn must leave the
 * element-wise SUM over all ranks in d_buf (device memory, context stream
 * synchronised before the call).  NULL detaches. */
typedef vx_status (*vx_exchange_fn)(double* d_buf, int64_t n_doubles, void* user);
vx_status vx_evo_set_exchange(vx_evo* e, int32_t rank, int32_t world, vx_exchange_fn fn, void* user);
/* One host thread, n GPUs: every evo has a communicator from ONE
 * vx_comm_create_all; begins all, all-reduces as one NCCL group, finishes
 * all.  reps may be NULL. */
vx_status vx_evo_generation_group(int32_t n, vx_evo* const* evos, vx_report* reps);

/* Rng::state / set_state text form of the GA stream (rng.hpp:41-50). */
int64_t vx_evo_rng_state(vx_evo* e, char* buf, int64_t cap);
vx_status vx_evo_set_rng_state(vx_evo* e, const char* state);
vx_status vx_evo_get_params(vx_evo* e, vx_hyper* h);
vx_status vx_evo_set_params(vx_evo* e, const vx_hyper* h); /* clamped like the advisor path */
int32_t vx_evo_generation_index(vx_evo* e);
/* best_fitness / best_genome (evolution.hpp:246-249); returns 1 if set. */
int32_t vx_evo_best(vx_evo* e, double* best_fitness, double* best_params);
/* The same plus the best genome's frozen B matrix (3m doubles): the
 * best_genome of a checkpoint (serialize.hpp:227-231). */
int32_t vx_evo_best_genome(vx_evo* e, double* best_fitness, double* best_params, double* best_bmat);
/* Resume support (evolution_state_from_json, serialize.hpp:235-262): set the
 * generation counter and best_fitness / best_genome (params and B both NULL =
 * no best genome yet).  Together with vx_evo_set_population (grids NULL),
 * vx_evo_set_params and vx_evo_set_rng_state this restores a checkpoint so
 * that the resumed run is identical to an uninterrupted one
 * (test_serialize.cpp:105-131). */
vx_status vx_evo_set_progress(vx_evo* e, int32_t generation, double best_fitness, const double* best_params,
                              const double* best_bmat);

/* ------------------------------------------------------- file formats --- */
/* Host only.  The JSON text of n doubles, separated by `sep`, exactly as the
 * reference's checkpoints print them (nlohmann::json dump(): Grisu2 digits,
 * "1.0", "1e-05"), so checkpoint checksums (serialize.hpp:264-292) and
 * curves.csv (serialize.hpp:321-343) are byte-identical.  Returns the text
 * length (written NUL-terminated into out when cap allows), -1 on bad args. */
int64_t vx_format_doubles(const double* v, int64_t n, char sep, char* out, int64_t cap);
/* Host only.  FNV-1a 64 of n bytes: the checkpoint checksum (serialize.hpp:23-28). */
uint64_t vx_fnv1a64(const char* data, int64_t n);

/* ------------------------------------------------------- measurement ---- */
/* Which integrator kernel the last simulate/step/evaluate launch used:
 * generic (any uploaded system), lattice (one CTA per robot, <= 351 masses),
 * cluster (one thread-block cluster per robot, 7^3..10^3 grids), stream
 * (per-slot arrays through L2/HBM, larger grids).  -1 before any launch. */
enum { VX_KERNEL_GENERIC = 0, VX_KERNEL_LATTICE = 1, VX_KERNEL_CLUSTER = 2, VX_KERNEL_STREAM = 3 };
int32_t vx_last_integrator(vx_ctx* ctx);
/* Live CUDA-event timing of every integrator launch on the context stream
 * (roofline reporting): enable, run, then read (and optionally reset) the
 * summed device time and launch count. */
vx_status vx_timing_enable(vx_ctx* ctx, int32_t on);
vx_status vx_integrator_timing(vx_ctx* ctx, double* total_ms, int64_t* n_launches, int32_t reset);
/* Measured FP64 FMA throughput of the device (TFLOP/s, 2 flops per DFMA),
 * the denominator for the FP64-issue-bound integrator's roofline. */
vx_status vx_fp64_peak(vx_ctx* ctx, double* tflops);
/* Summed device time (CUDA events on the context stream, while timing is
 * enabled) of every decode launch (tensor-pipe kernel + exact fix-up) and the
 * voxels those launches decoded; optionally reset. */
vx_status vx_decode_timing(vx_ctx* ctx, double* total_ms, int64_t* voxels, int32_t reset);
/* Measured FP64 tensor-pipe throughput (TFLOP/s, mma.sync m8n8k4 .f64 at 2 x
 * 8 x 8 x 4 flop), the decode MLP's roofline denominator. */
vx_status vx_dmma_peak(vx_ctx* ctx, double* tflops);
/* Self-check of the integrator's branch-free sqrt / reciprocal against the
 * IEEE sqrt(x) and 1.0/x over n pseudo-random inputs spanning the ranges the
 * integrator feeds them (plus powers of two and a few ulps around them);
 * mismatches[0] = sqrt, mismatches[1] = rcp, mismatches[2] = the fused
 * sqrt + reciprocal (sqrt(s) and 1.0/sqrt(s) from one refined rsqrt). */
vx_status vx_fastmath_check(vx_ctx* ctx, int64_t n, uint64_t seed, int64_t* mismatches);

/* ------------------------------------------------------------- bench ---- */
/* ------------------------------------------------ Rng + GA operators (host) */
/* Rng (rng.hpp:15-56): std::mt19937_64 with the reference's uniform01,
 * Box-Muller normal (glibc log/cos, two fresh draws), unbiased index and
 * libstdc++ text state.  Host only; no device needed. */
typedef struct vx_rng vx_rng;
vx_status vx_rng_create(uint64_t seed, vx_rng** out);
void vx_rng_free(vx_rng* r);
uint64_t vx_rng_next_u64(vx_rng* r);
double vx_rng_uniform01(vx_rng* r);
double vx_rng_normal(vx_rng* r);
uint64_t vx_rng_index(vx_rng* r, uint64_t n);
/* state text into buf (cap bytes incl. NUL); returns its full length */
int64_t vx_rng_state(vx_rng* r, char* buf, int64_t cap);
vx_status vx_rng_set_state(vx_rng* r, const char* state);
/* crossover (evolution.hpp:143-155) on flat parameter vectors: child[i] =
 * b[i] where uniform01 < 0.5, else a[i] (the encoding matrix stays a's: the
 * caller copies it) */
vx_status vx_crossover(vx_rng* r, int64_t np, const double* a, const double* b, double* child);
/* mutate (evolution.hpp:160-165) in place: params[i] += normal*scale where
 * uniform01 < rate, draws in parameter order */
vx_status vx_mutate(vx_rng* r, int64_t np, double* params, double rate, double scale);
/* tournament_select (evolution.hpp:169-173): the lowest of `size` index(P)
 * draws — an index into the best-first sorted population */
int32_t vx_tournament_select(vx_rng* r, int32_t population, int32_t size);

/* run_bench (bench.hpp:50-86): `jobs` copies of bench_robot(grid) stepped
 * `steps` times on device.  out = springs_per_robot, spring_updates,
 * expected_updates, seconds (device time), updates_per_second, diverged. */
vx_status vx_run_bench(vx_ctx* ctx, int32_t jobs, int64_t steps, int32_t grid, double dt, double* out6);

#ifdef __cplusplus
}
#endif
#endif /* VOXEVO_B200_H */
