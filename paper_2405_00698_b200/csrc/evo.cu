// evo.cu — device-resident EvolutionState and evolve_generation
// (evolution.hpp:177-293), plus the fused evaluate pipeline.
//
// Per generation:
//   begin : decode the individuals without a cached grid (replicated on every
//           rank), evaluate this rank's shard of the not-yet-evaluated ones
//           (component -> build -> gates -> fused integrator), and START the
//           breeding-plan parse on a host thread: the mt19937_64 draw sequence
//           of a generation depends only on (RNG state, HyperParams, P), never
//           on fitness, so the sequential stream parse
//           overlaps the GPU simulation;
//   [caller all-reduces the exchange buffer when world > 1]
//   finish: merge fitness, stable sort (CUB), sequential stats, histogram
//           diversity, best genome, then apply the plan on device (elite copy,
//           tournament parents gathered by sorted rank, crossover masks,
//           mutation deltas) into the double-buffered population.
// All RNG consumption and every GA decision are bit-identical to the
// reference; mutation noise uses the host glibc normal() exactly as the
// reference does.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "vx_ga.cuh"
#include "vx_internal.cuh"

using namespace vx;

namespace vx {

namespace {
// Host-exact actuation phases: every actuated spring takes sin/cos(phase) of
// its actuating voxel (phase = weight * phase_max, morphology.hpp:274-275;
// SimWorkspace physics.hpp:154-155) from a per-cell table the host computed
// with glibc, replacing the device sincos of derive_kernel.
__global__ void phase_override_kernel(int n, const int64_t* spring_off, const int32_t* nspring, const int16_t* act_vox,
                                      const int32_t* d_todo, int cells, const double2* tab, double* sinph,
                                      double* cosph) {
    const int r = blockIdx.x;
    if (r >= n) return;
    const int64_t so = spring_off[r];
    const double2* t = tab + static_cast<int64_t>(d_todo ? d_todo[r] : r) * cells;
    for (int q = threadIdx.x; q < nspring[r]; q += blockDim.x) {
        const int v = act_vox[so + q];
        if (v >= 0) {
            sinph[so + q] = t[v].x;
            cosph[so + q] = t[v].y;
        }
    }
}
}  // namespace

// raw grids -> component -> build -> gates -> integrate -> fitness
vx_status evaluate_pipeline(vx_ctx* ctx, int P, int w, int h, int d, const uint8_t* d_mat, const double* d_weight,
                            const vx_materials* table, const vx_plane* plane, const vx_sim* sim, const int32_t* d_todo,
                            int n_todo, double* d_fitness, double* d_updates, vx_summary* d_summaries,
                            const double2* d_phase_sc) {
    const int n = d_todo ? n_todo : P;
    if (n <= 0) return VX_OK;
    if (!(sim->dt > 0.0)) return (set_error("SimConfig: dt must be > 0"), VX_EINVAL);
    if (!(sim->duration >= 0.0)) return (set_error("SimConfig: duration must be >= 0"), VX_EINVAL);
    if (!(sim->actuation_frequency > 0.0)) return (set_error("SimConfig: frequency must be > 0"), VX_EINVAL);
    const int cells = w * h * d;
    VX_TRY(ctx->eval_body.alloc(static_cast<size_t>(n) * cells));
    VX_TRY(ctx->eval_summ.alloc(n));
    VX_TRY(largest_component_dev(ctx, n, w, h, d, d_mat, ctx->eval_body.p, d_todo));
    if (!ctx->eval_batch) ctx->eval_batch = new vx_batch;
    vx_batch* b = ctx->eval_batch;
    VX_TRY(build_batch_into(ctx, b, n, w, h, d, ctx->eval_body.p, d_weight, d_todo, table, plane));
    VX_TRY(gate_dev(ctx, b));
    if (d_phase_sc) {
        phase_override_kernel<<<n, 256, 0, ctx->stream>>>(n, b->spring_off.p, b->nspring.p, b->act_vox.p, d_todo,
                                                         cells, d_phase_sc, b->sinph.p, b->cosph.p);
        ctx->launches++;
        VX_CUDA(cudaGetLastError());
    }
    const int64_t n_steps = std::llround(sim->duration / sim->dt);  // physics.hpp:295
    VX_TRY(integrate(ctx, b, sim, 0, n_steps, false, nullptr, 0, ctx->eval_summ.p, nullptr));
    return fitness_dev(ctx, n, d_todo, b->status.p, ctx->eval_summ.p, d_fitness, d_updates, d_summaries);
}

}  // namespace vx

namespace {
// MutStore chunk memory: pinned, so the per-generation mutation upload is an
// asynchronous DMA straight from the chunks the plan thread wrote
void* pinned_alloc(size_t n) {
    void* p = nullptr;
    return cudaMallocHost(&p, n) == cudaSuccess ? p : nullptr;
}
void pinned_free(void* p) { cudaFreeHost(p); }

// a grow-only pinned host array (staging for async uploads)
template <typename T>
struct PinnedBuf {
    T* p = nullptr;
    size_t n = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
    vx_status alloc(size_t count) {
        if (count <= n) return VX_OK;
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
        const size_t want = count + count / 4;  // headroom: cudaFreeHost on a regrow can wait for the device
        const cudaError_t err = cudaMallocHost(reinterpret_cast<void**>(&p), want * sizeof(T));
        if (err != cudaSuccess) {
            p = nullptr;
            return cuda_status(err, "cudaMallocHost");
        }
        n = want;
        return VX_OK;
    }
};
}  // namespace

struct vx_evo {
    vx_ctx* ctx = nullptr;
    vx_evo_config cfg{};
    vx_hyper params{};
    int P = 0, cells = 0;
    int64_t np = 0, nb = 0;
    int cur = 0;
    DevBuf<double> prm[2], bm[2], fit[2], gw[2];
    DevBuf<uint8_t> ev[2], grid[2];
    std::vector<uint8_t> h_eval, h_has_grid;
    // rank that holds an individual's decoded grid (sharded decode; -1: none)
    std::vector<int32_t> h_owner;
    DevBuf<int32_t> d_own;
    // generation scratch
    DevBuf<int32_t> d_todo, d_dec, perm, iota;
    DevBuf<double> xbuf, sorted, keys_tmp, stats, div;
    DevBuf<uint32_t> guard;
    // breeding plan (host parse -> device)
    DevBuf<ChildPlan> d_plan;
    DevBuf<uint32_t> d_masks;
    DevBuf<MutEntry> d_mut;
    std::vector<ChildPlan> h_plan;
    std::vector<uint32_t> h_masks;
    MutStore h_mut{pinned_alloc, pinned_free};
    // the plan thread uploads its own result on up_stream as soon as the
    // scan is done (overlapping the GPU evaluate); finish() only makes the
    // breeding wait for `mut_uploaded` on the device
    cudaStream_t up_stream = nullptr;
    cudaEvent_t mut_uploaded = nullptr;  // the plan's async upload has read h_mut / the pinned staging
    PinnedBuf<ChildPlan> hp_plan;        // pinned staging of h_plan / h_masks for that upload
    PinnedBuf<uint32_t> hp_masks;
    vx_status plan_upload_status = VX_OK;
    std::string plan_upload_error;
    int64_t mask_words = 0;
    int plan_elite = 0;
    std::thread plan_thread;
    bool plan_running = false;
    bool plan_failed = false;  // host allocation failed inside the plan thread
    std::mt19937_64 rng;
    // begin() snapshot for rolling a generation back
    std::mt19937_64 rng_at_begin;
    std::vector<uint8_t> has_grid_at_begin;
    std::vector<int32_t> owner_at_begin;
    int generation = 0;
    double best_fitness = 0.0;
    bool has_best = false;
    std::vector<double> best_genome, best_bmat;
    // begin/finish
    bool begun = false;
    std::vector<int32_t> todo;
    int rank = 0, world = 1;
    std::chrono::steady_clock::time_point t0;
    std::chrono::steady_clock::time_point t_plan_done;  // the plan thread's end (VX_EVO_TRACE)
    vx_materials table{};
    double* ext_xbuf = nullptr;  // caller-owned exchange buffer (NCCL all-reduce operand)
    double* xb() { return ext_xbuf ? ext_xbuf : xbuf.p; }
    // the exchange step of vx_evo_generation: an NCCL communicator, or a
    // caller transport (rank / world of the shard either way)
    vx_comm* comm = nullptr;
    vx_exchange_fn xfn = nullptr;
    void* xuser = nullptr;
    int x_rank = 0, x_world = 1;

    ~vx_evo() {
        if (plan_thread.joinable()) plan_thread.join();
        if (up_stream) cudaStreamSynchronize(up_stream);
        if (mut_uploaded) cudaEventDestroy(mut_uploaded);
        if (up_stream) cudaStreamDestroy(up_stream);
    }
};

namespace {

// exchange buffer: [fitness P | spring updates P | packed grids P x diversity_words(cells)]
size_t xbuf_doubles(const vx_evo* e) {
    return 2 * static_cast<size_t>(e->P) + static_cast<size_t>(e->P) * diversity_words(e->cells);
}

// The plan's device copy, issued by the plan thread on up_stream: rows and
// masks through pinned staging, mutation entries straight from MutStore's
// pinned slabs (one copy per run of chunks in one slab); mut_uploaded marks
// the end.  The device buffers only grow, and nothing reads them until the
// breeding of this generation (after the previous one's final sync).
vx_status upload_plan(vx_evo* e) {
    cudaStream_t s = e->up_stream;
    const int n_child = e->P - e->plan_elite;
    // grow with 25% headroom: a regrow's cudaFree would wait for the running
    // integrator, and the hit count varies a little from generation to generation
    auto grow = [](auto& buf, size_t need) { return need <= buf.n ? VX_OK : buf.alloc(need + need / 4); };
    VX_TRY(grow(e->d_plan, static_cast<size_t>(std::max(1, n_child))));
    VX_TRY(grow(e->d_masks, std::max<size_t>(1, e->h_masks.size())));
    VX_TRY(grow(e->d_mut, std::max<size_t>(1, e->h_mut.size())));
    if (n_child > 0) {
        VX_TRY(e->hp_plan.alloc(static_cast<size_t>(n_child)));
        std::memcpy(e->hp_plan.p, e->h_plan.data(), n_child * sizeof(ChildPlan));
        VX_CUDA(cudaMemcpyAsync(e->d_plan.p, e->hp_plan.p, n_child * sizeof(ChildPlan), cudaMemcpyHostToDevice, s));
    }
    if (!e->h_masks.empty()) {
        VX_TRY(e->hp_masks.alloc(e->h_masks.size()));
        std::memcpy(e->hp_masks.p, e->h_masks.data(), e->h_masks.size() * sizeof(uint32_t));
        VX_CUDA(cudaMemcpyAsync(e->d_masks.p, e->hp_masks.p, e->h_masks.size() * sizeof(uint32_t),
                                cudaMemcpyHostToDevice, s));
    }
    for (size_t j = 0, nch = e->h_mut.chunks(); j < nch;) {
        size_t k = j + 1;
        while (k < nch && e->h_mut.continues(k)) ++k;
        const size_t count = (k - 1 - j) * MutStore::kChunk + e->h_mut.chunk_size(k - 1);
        VX_CUDA(cudaMemcpyAsync(e->d_mut.p + j * MutStore::kChunk, e->h_mut.chunk(j), count * sizeof(MutEntry),
                                cudaMemcpyHostToDevice, s));
        j = k;
    }
    VX_CUDA(cudaEventRecord(e->mut_uploaded, s));
    return VX_OK;
}

// Breeding loop (evolution.hpp:267-289) in rank space: consumes the GA
// stream draw-for-draw like the reference (ga_plan.cpp).
void parse_plan(vx_evo* e) {
    const int n_elite = vx_elite_count(e->params.elite_fraction, e->P);
    e->plan_elite = n_elite;
    const PlanParams a{e->P, n_elite, e->cfg.tournament_size, e->np, e->mask_words, e->params.crossover_rate,
                       e->params.mutation_rate, e->params.mutation_scale};
    try {
        plan_scan(e->rng, a, e->h_plan, e->h_masks, e->h_mut);
    } catch (const std::bad_alloc&) {
        e->plan_failed = true;
        return;
    }
    e->plan_upload_status = upload_plan(e);
    if (e->plan_upload_status != VX_OK) e->plan_upload_error = vx_last_error();
}

vx_status validate_cfg(const vx_evo_config* c) {
    if (c->population < 2) return (set_error("EvolutionConfig: population must be >= 2"), VX_EINVAL);
    if (c->generations < 0) return (set_error("EvolutionConfig: generations must be >= 0"), VX_EINVAL);
    if (c->grid_w < 1 || c->grid_h < 1 || c->grid_d < 1)
        return (set_error("EvolutionConfig: grid dimensions must be >= 1"), VX_EINVAL);
    if (c->tournament_size < 1) return (set_error("EvolutionConfig: tournament size must be >= 1"), VX_EINVAL);
    if (c->arch.m < 1) return (set_error("EncodingSpec: m must be >= 1"), VX_EINVAL);
    if (!(c->arch.sigma > 0.0)) return (set_error("EncodingSpec: sigma must be > 0"), VX_EINVAL);
    if (param_count(&c->arch) < 0) return (set_error("sample_genome: hidden widths must be >= 1"), VX_EINVAL);
    if (!(c->sim.dt > 0.0)) return (set_error("SimConfig: dt must be > 0"), VX_EINVAL);
    if (!(c->sim.duration >= 0.0)) return (set_error("SimConfig: duration must be >= 0"), VX_EINVAL);
    if (!(c->sim.actuation_frequency > 0.0)) return (set_error("SimConfig: frequency must be > 0"), VX_EINVAL);
    return VX_OK;
}

vx_status alloc_evo(vx_evo* e) {
    const size_t P = static_cast<size_t>(e->P);
    for (int s = 0; s < 2; ++s) {
        VX_TRY(e->prm[s].alloc(P * e->np));
        VX_TRY(e->bm[s].alloc(P * e->nb));
        VX_TRY(e->fit[s].alloc(P));
        VX_TRY(e->gw[s].alloc(P * e->cells));
        VX_TRY(e->ev[s].alloc(P));
        VX_TRY(e->grid[s].alloc(P * e->cells));
    }
    VX_TRY(e->d_todo.alloc(P));
    VX_TRY(e->d_dec.alloc(P));
    VX_TRY(e->perm.alloc(P));
    VX_TRY(e->iota.alloc(P));
    VX_TRY(e->xbuf.alloc(xbuf_doubles(e)));
    VX_TRY(e->sorted.alloc(P));
    VX_TRY(e->keys_tmp.alloc(P));
    VX_TRY(e->stats.alloc(4));
    VX_TRY(e->div.alloc(1));
    VX_TRY(e->guard.alloc(1));
    VX_TRY(e->d_plan.alloc(P));
    e->mask_words = (e->np + 31) / 32;
    e->h_eval.assign(P, 0);
    e->h_has_grid.assign(P, 0);
    e->h_owner.assign(P, -1);
    VX_TRY(e->d_own.alloc(P));
    return VX_OK;
}

void start_plan(vx_evo* e) {
    // the previous plan's upload reads h_mut and the staging asynchronously
    if (e->mut_uploaded) cudaEventSynchronize(e->mut_uploaded);
    e->plan_upload_status = VX_OK;
    e->plan_running = true;
    e->plan_failed = false;
    const int device = e->ctx->device;
    e->plan_thread = std::thread([e, device] {
        // the thread's pinned allocations must land in this rank's context,
        // not in a fresh one on device 0 (a new host thread starts there)
        cudaSetDevice(device);
        parse_plan(e);
        e->t_plan_done = std::chrono::steady_clock::now();
    });
}

void join_plan(vx_evo* e) {
    if (e->plan_thread.joinable()) e->plan_thread.join();
    e->plan_running = false;
}

// a begun generation whose exchange failed: join the plan and restore the
// state begin() found (RNG position, grid ownership)
void abandon_generation(vx_evo* e) {
    join_plan(e);
    cudaStreamSynchronize(e->ctx->stream);
    e->rng = e->rng_at_begin;
    e->h_has_grid = e->has_grid_at_begin;
    e->h_owner = e->owner_at_begin;
    e->begun = false;
}

}  // namespace

extern "C" {

vx_status vx_evo_create(vx_ctx* ctx, const vx_evo_config* cfg, vx_evo** out) {
    if (!ctx || !cfg || !out) return VX_EINVAL;
    VX_TRY(validate_cfg(cfg));
    VX_TRY(decode_feasible(ctx, &cfg->arch));  // fail up front, not in a later generation
    auto e = std::make_unique<vx_evo>();
    e->ctx = ctx;
    e->cfg = *cfg;
    e->params = cfg->initial_params;
    vx_hyper_clamp(&e->params);
    e->P = cfg->population;
    e->cells = cfg->grid_w * cfg->grid_h * cfg->grid_d;
    e->np = param_count(&cfg->arch);
    e->nb = 3LL * cfg->arch.m;
    VX_TRY(alloc_evo(e.get()));
    VX_CUDA(cudaStreamCreateWithFlags(&e->up_stream, cudaStreamNonBlocking));
    VX_CUDA(cudaEventCreateWithFlags(&e->mut_uploaded, cudaEventDisableTiming));
    // init_evolution (evolution.hpp:197-211): per-genome seeds from the master
    // stream, genomes sampled on device (K14)
    e->rng.seed(cfg->seed);
    std::vector<uint64_t> seeds(e->P);
    for (auto& s : seeds) s = e->rng();
    DevBuf<uint64_t> d_seeds;
    VX_TRY(d_seeds.alloc(e->P));
    VX_CUDA(cudaMemcpyAsync(d_seeds.p, seeds.data(), e->P * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
    VX_TRY(sample_genomes_dev(ctx, &cfg->arch, e->P, d_seeds.p, e->prm[0].p, e->bm[0].p));
    {  // B with the host glibc Box-Muller (bit-exact), over the device's
        std::vector<double> hb(static_cast<size_t>(e->P) * e->nb);
        host_sample_bmat(cfg->arch.m, cfg->arch.sigma, e->P, seeds.data(), hb.data());
        VX_CUDA(cudaMemcpyAsync(e->bm[0].p, hb.data(), hb.size() * sizeof(double), cudaMemcpyHostToDevice,
                                ctx->stream));
        VX_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    VX_CUDA(cudaMemsetAsync(e->fit[0].p, 0, e->P * sizeof(double), ctx->stream));
    VX_CUDA(cudaMemsetAsync(e->ev[0].p, 0, e->P, ctx->stream));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = e.release();
    return VX_OK;
}

vx_status vx_evo_free(vx_evo* e) {
    if (e) {
        join_plan(e);
        if (e->ctx) cudaStreamSynchronize(e->ctx->stream);
        delete e;
    }
    return VX_OK;
}

namespace {
vx_status evo_begin_body(vx_evo* e, int32_t rank, int32_t world);
}

vx_status vx_evo_begin(vx_evo* e, int32_t rank, int32_t world) {
    if (!e || world < 1 || rank < 0 || rank >= world) return VX_EINVAL;
    if (e->begun) return (set_error("vx_evo_begin: generation already begun"), VX_ESTATE);
    join_plan(e);  // never assign a new plan thread over a joinable one
    // a failed begin leaves the state as it found it: RNG position, grid
    // ownership and the plan thread (joined) all rolled back
    e->rng_at_begin = e->rng;
    e->has_grid_at_begin = e->h_has_grid;
    e->owner_at_begin = e->h_owner;
    const vx_status s = evo_begin_body(e, rank, world);
    if (s != VX_OK) abandon_generation(e);
    return s;
}

}  // extern "C"

namespace {
vx_status evo_begin_body(vx_evo* e, int32_t rank, int32_t world) {
    vx_ctx* ctx = e->ctx;
    e->t0 = std::chrono::steady_clock::now();
    e->rank = rank;
    e->world = world;
    const int c = e->cur;
    // detail::scaled_materials (evolution.hpp:123-129, 229)
    e->table = e->cfg.materials;
    e->table.k_muscle *= e->params.material_multipliers[0];
    e->table.k_soft *= e->params.material_multipliers[1];
    e->table.k_bone *= e->params.material_multipliers[2];
    // breeding plan parse overlaps everything below
    start_plan(e);
    // decode individuals without a cached grid (evolution.hpp:230-236),
    // sharded: an individual to evaluate is decoded by the rank that evaluates
    // it (strided over the todo list); grids needed only for the diversity
    // (elites restored without one) are striped over the remaining list.
    // Every rank derives the same owner map, so no grid ever moves.
    std::vector<int32_t> dec_rest;
    e->todo.clear();
    for (int a = 0; a < e->P; ++a) {
        if (!e->h_eval[a]) e->todo.push_back(a);
        else if (!e->h_has_grid[a]) dec_rest.push_back(a);
    }
    std::vector<int32_t> dec, mine;
    for (size_t q = 0; q < e->todo.size(); ++q) {
        const int a = e->todo[q];
        const int owner = static_cast<int>(q % static_cast<size_t>(world));
        if (owner == rank) mine.push_back(a);  // this rank's shard of the evaluations
        if (!e->h_has_grid[a]) {
            e->h_owner[a] = owner;
            e->h_has_grid[a] = 1;
            if (owner == rank) dec.push_back(a);
        }
    }
    for (size_t q = 0; q < dec_rest.size(); ++q) {
        const int a = dec_rest[q];
        const int owner = static_cast<int>(q % static_cast<size_t>(world));
        e->h_owner[a] = owner;
        e->h_has_grid[a] = 1;
        if (owner == rank) dec.push_back(a);
    }
    if (!dec.empty()) {
        VX_CUDA(cudaMemcpyAsync(e->d_dec.p, dec.data(), dec.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                                ctx->stream));
        VX_TRY(decode_dev(ctx, &e->cfg.arch, e->P, e->prm[c].p, e->bm[c].p, e->cfg.grid_w, e->cfg.grid_h,
                          e->cfg.grid_d, e->grid[c].p, e->gw[c].p, nullptr, e->d_dec.p, static_cast<int>(dec.size())));
    }
    VX_CUDA(cudaMemsetAsync(e->xb(), 0, xbuf_doubles(e) * sizeof(double), ctx->stream));
    if (!mine.empty()) {
        VX_CUDA(cudaMemcpyAsync(e->d_todo.p, mine.data(), mine.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                                ctx->stream));
        VX_TRY(evaluate_pipeline(ctx, e->P, e->cfg.grid_w, e->cfg.grid_h, e->cfg.grid_d, e->grid[c].p, e->gw[c].p,
                                 &e->table, &e->cfg.plane, &e->cfg.sim, e->d_todo.p, static_cast<int>(mine.size()),
                                 e->xb(), e->xb() + e->P, nullptr));
    }
    // the grids this rank holds, packed into the exchange buffer (zeros for
    // the others): the all-reduce gathers every grid for the exact
    // population_diversity (evolution.hpp:89-105) in finish
    {
        std::vector<int32_t> own;
        for (int a = 0; a < e->P; ++a)
            if (e->h_owner[a] == rank) own.push_back(a);
        if (!own.empty())
            VX_CUDA(cudaMemcpyAsync(e->d_own.p, own.data(), own.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                                    ctx->stream));
        VX_TRY(diversity_pack_dev(ctx, static_cast<int>(own.size()), e->d_own.p, e->cells, e->grid[c].p,
                                  e->xb() + 2 * e->P));
    }
    // the todo list (all ranks) goes to the device for the merge
    if (!e->todo.empty())
        VX_CUDA(cudaMemcpyAsync(e->d_todo.p, e->todo.data(), e->todo.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                                ctx->stream));
    e->begun = true;
    return VX_OK;
}
}  // namespace

extern "C" {

vx_status vx_evo_exchange_buffer(vx_evo* e, double** d_buf, int64_t* n_doubles) {
    if (!e || !d_buf) return VX_EINVAL;
    *d_buf = e->xb();
    if (n_doubles) *n_doubles = static_cast<int64_t>(xbuf_doubles(e));
    return VX_OK;
}

vx_status vx_evo_set_exchange_buffer(vx_evo* e, double* d_buf) {
    if (!e) return VX_EINVAL;
    if (e->begun) return (set_error("exchange buffer change mid-generation"), VX_ESTATE);
    e->ext_xbuf = d_buf;
    return VX_OK;
}

vx_status vx_evo_load_population_dev(vx_evo* e, const double* d_params, const double* d_bmat) {
    if (!e || !d_params || !d_bmat) return VX_EINVAL;
    if (e->begun) return (set_error("population is mid-generation"), VX_ESTATE);
    cudaStream_t s = e->ctx->stream;
    const int c = e->cur;
    const size_t P = e->P;
    VX_CUDA(cudaMemcpyAsync(e->prm[c].p, d_params, P * e->np * sizeof(double), cudaMemcpyDeviceToDevice, s));
    VX_CUDA(cudaMemcpyAsync(e->bm[c].p, d_bmat, P * e->nb * sizeof(double), cudaMemcpyDeviceToDevice, s));
    VX_CUDA(cudaMemsetAsync(e->fit[c].p, 0, P * sizeof(double), s));
    VX_CUDA(cudaMemsetAsync(e->ev[c].p, 0, P, s));
    std::fill(e->h_eval.begin(), e->h_eval.end(), 0);
    std::fill(e->h_has_grid.begin(), e->h_has_grid.end(), 0);
    std::fill(e->h_owner.begin(), e->h_owner.end(), -1);
    return VX_OK;
}

vx_status vx_evo_finish(vx_evo* e, vx_report* rep) {
    if (!e) return VX_EINVAL;
    if (!e->begun) return (set_error("vx_evo_finish without vx_evo_begin"), VX_ESTATE);
    vx_ctx* ctx = e->ctx;
    const int c = e->cur, nx = 1 - c, P = e->P;
    const auto t_fin0 = std::chrono::steady_clock::now();
    VX_TRY(merge_dev(ctx, static_cast<int>(e->todo.size()), e->d_todo.p, e->xb(), e->fit[c].p, e->ev[c].p));
    VX_TRY(sort_stats_dev(ctx, P, e->fit[c].p, e->perm.p, e->sorted.p, e->iota.p, e->keys_tmp.p, e->stats.p));
    // population_diversity over the sorted population (evolution.hpp:265), bit-exact
    VX_TRY(diversity_exact_dev(ctx, P, e->cells, e->xb() + 2 * P, e->perm.p, e->div.p));
    double st[3], div = 0.0;
    std::vector<double> upd(e->todo.empty() ? 0 : P);
    VX_CUDA(cudaMemcpyAsync(st, e->stats.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    VX_CUDA(cudaMemcpyAsync(&div, e->div.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (!upd.empty())
        VX_CUDA(cudaMemcpyAsync(upd.data(), e->xb() + P, P * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    int32_t top = 0;
    VX_CUDA(cudaMemcpyAsync(&top, e->perm.p, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));
    // best_fitness / best_genome (evolution.hpp:246-249)
    if (!e->has_best || st[0] > e->best_fitness) {
        e->best_fitness = st[0];
        e->best_genome.resize(e->np);
        VX_CUDA(cudaMemcpy(e->best_genome.data(), e->prm[c].p + static_cast<size_t>(top) * e->np,
                           e->np * sizeof(double), cudaMemcpyDeviceToHost));
        e->best_bmat.resize(e->nb);
        VX_CUDA(cudaMemcpy(e->best_bmat.data(), e->bm[c].p + static_cast<size_t>(top) * e->nb,
                           e->nb * sizeof(double), cudaMemcpyDeviceToHost));
        e->has_best = true;
    }
    vx_report r{};
    r.generation = e->generation;
    r.params = e->params;
    r.best = st[0];
    r.mean = st[1];
    r.stddev = st[2];
    r.diversity = div;
    r.evaluations = static_cast<int32_t>(e->todo.size());
    uint64_t total = 0;
    for (int32_t a : e->todo) total += static_cast<uint64_t>(upd[a]);
    r.spring_updates = total;
    // breed (evolution.hpp:267-289)
    static const bool trace = [] {
        const char* v = std::getenv("VX_EVO_TRACE");  // development aid: where finish() waits
        return v && *v == '1';
    }();
    const auto t_join0 = std::chrono::steady_clock::now();
    join_plan(e);
    const auto t_join1 = std::chrono::steady_clock::now();
    if (e->plan_failed) return (set_error("breeding plan: host allocation failed"), VX_EOOM);
    if (e->plan_upload_status != VX_OK) {
        set_error(e->plan_upload_error.c_str());
        return e->plan_upload_status;
    }
    const int n_elite = e->plan_elite;
    // the plan thread's upload (up_stream) before the breeding reads it
    VX_CUDA(cudaStreamWaitEvent(ctx->stream, e->mut_uploaded, 0));
    std::chrono::steady_clock::time_point t_up = t_join1, t_br = t_join1;
    if (trace) {  // attribute the wait: uploads drained
        VX_CUDA(cudaStreamSynchronize(ctx->stream));
        t_up = std::chrono::steady_clock::now();
    }
    BreedArgs A{};
    A.n_elite = n_elite;
    A.np = e->np;
    A.nb = e->nb;
    A.cells = e->cells;
    A.mask_words = e->mask_words;
    A.perm = e->perm.p;
    A.plan = e->d_plan.p;
    A.masks = e->d_masks.p;
    A.src_params = e->prm[c].p;
    A.src_bmat = e->bm[c].p;
    A.src_fit = e->fit[c].p;
    A.src_eval = e->ev[c].p;
    A.src_grid = e->grid[c].p;
    A.src_gridw = e->gw[c].p;
    A.dst_params = e->prm[nx].p;
    A.dst_bmat = e->bm[nx].p;
    A.dst_fit = e->fit[nx].p;
    A.dst_eval = e->ev[nx].p;
    A.dst_grid = e->grid[nx].p;
    A.dst_gridw = e->gw[nx].p;
    VX_TRY(breed_dev(ctx, A, P, e->d_mut.p, static_cast<int64_t>(e->h_mut.size())));
    if (trace) {
        VX_CUDA(cudaStreamSynchronize(ctx->stream));
        t_br = std::chrono::steady_clock::now();
    }
    // host mirrors: elites are evaluated and keep their grids (and owners);
    // children are fresh
    std::vector<int32_t> elite_src(static_cast<size_t>(n_elite));
    if (n_elite > 0)
        VX_CUDA(cudaMemcpyAsync(elite_src.data(), e->perm.p, n_elite * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                ctx->stream));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));
    std::vector<int32_t> owner_next(static_cast<size_t>(P), -1);
    for (int a = 0; a < n_elite; ++a) owner_next[a] = e->h_owner[elite_src[a]];
    e->h_owner.swap(owner_next);
    for (int a = 0; a < P; ++a) {
        e->h_eval[a] = a < n_elite ? 1 : 0;
        e->h_has_grid[a] = a < n_elite ? 1 : 0;
    }
    e->cur = nx;
    ++e->generation;
    e->begun = false;
    VX_CUDA(cudaStreamSynchronize(ctx->stream));  // host plan buffers are reused next generation
    if (trace) {
        const auto t_end = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "[evo] gen %lld: plan ready %.3f ms after begin, finish: stats %.3f ms, plan wait %.3f ms, "
                             "upload %.3f ms, breed %.3f ms, host tail %.3f ms, mutations %zu\n",
                     static_cast<long long>(e->generation - 1), ms(e->t0, e->t_plan_done), ms(t_fin0, t_join0),
                     ms(t_join0, t_join1), ms(t_join1, t_up), ms(t_up, t_br), ms(t_br, t_end), e->h_mut.size());
    }
    r.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - e->t0).count();
    if (rep) *rep = r;
    return VX_OK;
}

vx_status vx_evo_generation(vx_evo* e, vx_report* rep) {
    if (!e) return VX_EINVAL;
    if (e->comm) {  // sharded over the communicator's ranks
        VX_TRY(vx_evo_begin(e, comm_rank(e->comm), comm_world(e->comm)));
        const vx_status s = comm_exchange(e->comm, e->xb(), static_cast<int64_t>(xbuf_doubles(e)));
        if (s != VX_OK) {
            abandon_generation(e);
            return s;
        }
        return vx_evo_finish(e, rep);
    }
    if (e->xfn) {
        VX_TRY(vx_evo_begin(e, e->x_rank, e->x_world));
        cudaError_t ce = cudaStreamSynchronize(e->ctx->stream);
        const vx_status s = ce != cudaSuccess ? cuda_status(ce, "exchange")
                                              : e->xfn(e->xb(), static_cast<int64_t>(xbuf_doubles(e)), e->xuser);
        if (s != VX_OK) {
            abandon_generation(e);
            return s;
        }
        return vx_evo_finish(e, rep);
    }
    VX_TRY(vx_evo_begin(e, 0, 1));
    return vx_evo_finish(e, rep);
}

vx_status vx_evo_set_comm(vx_evo* e, vx_comm* c) {
    if (!e) return VX_EINVAL;
    if (e->begun) return (set_error("communicator change mid-generation"), VX_ESTATE);
    if (c && comm_ctx(c)->device != e->ctx->device)
        return (set_error("vx_evo_set_comm: communicator and evolution state are on different devices"), VX_EINVAL);
    e->comm = c;
    return VX_OK;
}

vx_status vx_evo_set_exchange(vx_evo* e, int32_t rank, int32_t world, vx_exchange_fn fn, void* user) {
    if (!e || (fn && (world < 1 || rank < 0 || rank >= world))) return VX_EINVAL;
    if (e->begun) return (set_error("exchange change mid-generation"), VX_ESTATE);
    e->xfn = fn;
    e->xuser = user;
    e->x_rank = fn ? rank : 0;
    e->x_world = fn ? world : 1;
    return VX_OK;
}

vx_status vx_evo_generation_group(int32_t n, vx_evo* const* evos, vx_report* reps) {
    if (n < 1 || !evos) return VX_EINVAL;
    std::vector<vx_comm*> cs(static_cast<size_t>(n));
    std::vector<double*> bufs(static_cast<size_t>(n));
    std::vector<int64_t> counts(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        if (!evos[i] || !evos[i]->comm || comm_world(evos[i]->comm) != n)
            return (set_error("vx_evo_generation_group: every state needs a communicator of this group"), VX_EINVAL);
        cs[static_cast<size_t>(i)] = evos[i]->comm;
    }
    int begun = 0;
    vx_status s = VX_OK;
    for (; begun < n && s == VX_OK; ++begun) {
        vx_evo* e = evos[begun];
        s = vx_evo_begin(e, comm_rank(e->comm), n);
        if (s != VX_OK) break;
        bufs[static_cast<size_t>(begun)] = e->xb();
        counts[static_cast<size_t>(begun)] = static_cast<int64_t>(xbuf_doubles(e));
    }
    if (s == VX_OK) s = comm_exchange_group(n, cs.data(), bufs.data(), counts.data());
    if (s != VX_OK) {
        for (int i = 0; i < begun; ++i) abandon_generation(evos[i]);
        return s;
    }
    for (int i = 0; i < n; ++i) VX_TRY(vx_evo_finish(evos[i], reps ? reps + i : nullptr));
    return VX_OK;
}

vx_status vx_evo_get_population(vx_evo* e, double* params, double* bmat, double* fitness, uint8_t* evaluated,
                                uint8_t* grids, double* grid_w) {
    if (!e) return VX_EINVAL;
    if (e->begun) return (set_error("population is mid-generation"), VX_ESTATE);
    const int c = e->cur;
    const size_t P = e->P;
    cudaStream_t s = e->ctx->stream;
    if (params) VX_CUDA(cudaMemcpyAsync(params, e->prm[c].p, P * e->np * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (bmat) VX_CUDA(cudaMemcpyAsync(bmat, e->bm[c].p, P * e->nb * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (fitness) VX_CUDA(cudaMemcpyAsync(fitness, e->fit[c].p, P * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (evaluated) VX_CUDA(cudaMemcpyAsync(evaluated, e->ev[c].p, P, cudaMemcpyDeviceToHost, s));
    if (grids) VX_CUDA(cudaMemcpyAsync(grids, e->grid[c].p, P * e->cells, cudaMemcpyDeviceToHost, s));
    if (grid_w) VX_CUDA(cudaMemcpyAsync(grid_w, e->gw[c].p, P * e->cells * sizeof(double), cudaMemcpyDeviceToHost, s));
    VX_CUDA(cudaStreamSynchronize(s));
    for (size_t a = 0; a < P; ++a)
        if (!e->h_has_grid[a]) {
            if (grids) std::memset(grids + a * e->cells, 255, e->cells);
            if (grid_w) std::fill(grid_w + a * e->cells, grid_w + (a + 1) * e->cells, 0.0);
        }
    return VX_OK;
}

vx_status vx_evo_set_population(vx_evo* e, const double* params, const double* bmat, const double* fitness,
                                const uint8_t* evaluated, const uint8_t* grids, const double* grid_w) {
    if (!e || !params || !bmat) return VX_EINVAL;
    if (e->begun) return (set_error("population is mid-generation"), VX_ESTATE);
    const int c = e->cur;
    const size_t P = e->P;
    cudaStream_t s = e->ctx->stream;
    VX_CUDA(cudaMemcpyAsync(e->prm[c].p, params, P * e->np * sizeof(double), cudaMemcpyHostToDevice, s));
    VX_CUDA(cudaMemcpyAsync(e->bm[c].p, bmat, P * e->nb * sizeof(double), cudaMemcpyHostToDevice, s));
    std::vector<double> f(P, 0.0);
    std::vector<uint8_t> ev(P, 0);
    if (fitness) std::copy(fitness, fitness + P, f.begin());
    if (evaluated) std::copy(evaluated, evaluated + P, ev.begin());
    VX_CUDA(cudaMemcpyAsync(e->fit[c].p, f.data(), P * sizeof(double), cudaMemcpyHostToDevice, s));
    VX_CUDA(cudaMemcpyAsync(e->ev[c].p, ev.data(), P, cudaMemcpyHostToDevice, s));
    std::vector<double> gw;
    if (grids) {
        VX_CUDA(cudaMemcpyAsync(e->grid[c].p, grids, P * e->cells, cudaMemcpyHostToDevice, s));
        if (!grid_w) gw.assign(P * e->cells, 1.0);
        VX_CUDA(cudaMemcpyAsync(e->gw[c].p, grid_w ? grid_w : gw.data(), P * e->cells * sizeof(double),
                                cudaMemcpyHostToDevice, s));
    }
    VX_CUDA(cudaStreamSynchronize(s));
    for (size_t a = 0; a < P; ++a) {
        // material 255 in a row's first cell: no grid for that individual
        // (vx_evo_get_population's marker), it is decoded when needed
        const bool has = grids && grids[a * e->cells] != 255;
        e->h_eval[a] = ev[a] ? 1 : 0;
        e->h_has_grid[a] = has ? 1 : 0;
        e->h_owner[a] = has ? 0 : -1;  // host-provided grids: rank 0's copy counts
    }
    return VX_OK;
}

vx_status vx_evo_population_dev(vx_evo* e, double** d_params, double** d_bmat, double** d_fitness) {
    if (!e) return VX_EINVAL;
    if (d_params) *d_params = e->prm[e->cur].p;
    if (d_bmat) *d_bmat = e->bm[e->cur].p;
    if (d_fitness) *d_fitness = e->fit[e->cur].p;
    return VX_OK;
}

int64_t vx_evo_rng_state(vx_evo* e, char* buf, int64_t cap) {
    if (!e) return -1;
    if (e->plan_running) join_plan(e);
    std::ostringstream os;
    os << e->rng;
    const std::string s = os.str();
    if (buf && cap > 0) {
        std::strncpy(buf, s.c_str(), static_cast<size_t>(cap - 1));
        buf[cap - 1] = 0;
    }
    return static_cast<int64_t>(s.size());
}

vx_status vx_evo_set_rng_state(vx_evo* e, const char* state) {
    if (!e || !state) return VX_EINVAL;
    if (e->begun) return (set_error("rng state change mid-generation"), VX_ESTATE);
    std::istringstream is(state);
    std::mt19937_64 r;
    is >> r;
    if (is.fail()) return (set_error("invalid mt19937_64 state text"), VX_EINVAL);
    e->rng = r;
    return VX_OK;
}

vx_status vx_evo_get_params(vx_evo* e, vx_hyper* h) {
    if (!e || !h) return VX_EINVAL;
    *h = e->params;
    return VX_OK;
}

vx_status vx_evo_set_params(vx_evo* e, const vx_hyper* h) {
    if (!e || !h) return VX_EINVAL;
    if (e->begun) return (set_error("params change mid-generation"), VX_ESTATE);
    e->params = *h;
    vx_hyper_clamp(&e->params);  // evolution.hpp:224-225
    return VX_OK;
}

int32_t vx_evo_generation_index(vx_evo* e) { return e ? e->generation : -1; }

int32_t vx_evo_best(vx_evo* e, double* best_fitness, double* best_params) {
    if (!e) return 0;
    if (best_fitness) *best_fitness = e->best_fitness;
    if (!e->has_best) return 0;
    if (best_params) std::copy(e->best_genome.begin(), e->best_genome.end(), best_params);
    return 1;
}

int32_t vx_evo_best_genome(vx_evo* e, double* best_fitness, double* best_params, double* best_bmat) {
    const int32_t has = vx_evo_best(e, best_fitness, best_params);
    if (has && best_bmat) std::copy(e->best_bmat.begin(), e->best_bmat.end(), best_bmat);
    return has;
}

vx_status vx_evo_set_progress(vx_evo* e, int32_t generation, double best_fitness, const double* best_params,
                              const double* best_bmat) {
    if (!e || generation < 0 || (best_params == nullptr) != (best_bmat == nullptr)) return VX_EINVAL;
    if (e->begun) return (set_error("progress change mid-generation"), VX_ESTATE);
    e->generation = generation;
    e->best_fitness = best_fitness;
    e->has_best = best_params != nullptr;
    if (best_params) {
        e->best_genome.assign(best_params, best_params + e->np);
        e->best_bmat.assign(best_bmat, best_bmat + e->nb);
    } else {
        e->best_genome.clear();
        e->best_bmat.clear();
    }
    return VX_OK;
}

}  // extern "C"
