// api_core.cu — C ABI: library, context, batches, integrator, bench.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "vx_internal.cuh"

namespace vx {

thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

vx_status cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return VX_OK;
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    if (e == cudaErrorMemoryAllocation) return VX_EOOM;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return VX_ENODEV;
    return VX_ECUDA;
}

}  // namespace vx

using namespace vx;

namespace {

// Upload n robots from host SoA (pos/vel nm x 3 row-major) into a new batch.
vx_status upload_impl(vx_ctx* ctx, int32_t n, const int64_t* mass_off, const int64_t* spring_off, const double* pos,
                      const double* vel, const double* mass, const int32_t* si, const int32_t* sj, const double* k,
                      const double* rest0, const double* zeta, const uint8_t* has_act, const double* sign,
                      const double* amp, const double* phase, const vx_plane* plane, vx_batch** out) {
    if (!ctx || !out || n < 0 || !mass_off || !spring_off) return (set_error("vx_batch_upload: bad arguments"), VX_EINVAL);
    auto* b = new vx_batch;
    b->ctx = ctx;
    b->plane = plane ? *plane : vx_plane{1e5, 0.1, 0.6, 1.0};
    const int64_t M = mass_off[n], S = spring_off[n];
    b->h_mass_off.assign(mass_off, mass_off + n + 1);
    b->h_spring_off.assign(spring_off, spring_off + n + 1);
    for (int r = 0; r < n; ++r) {
        const int64_t nm = mass_off[r + 1] - mass_off[r], ns = spring_off[r + 1] - spring_off[r];
        if (nm < 0 || ns < 0 || nm > 65535) {
            delete b;
            set_error("vx_batch_upload: robot " + std::to_string(r) + " has invalid size");
            return VX_EINVAL;
        }
        b->nm_max = std::max<int>(b->nm_max, static_cast<int>(nm));
        b->ns_max = std::max<int>(b->ns_max, static_cast<int>(ns));
    }
    vx_status st = batch_alloc(b, n, M, S);
    if (st != VX_OK) {
        delete b;
        return st;
    }
    // host-side SoA repack
    std::vector<double> hpos(3 * M), hvel(3 * M);
    for (int64_t a = 0; a < M; ++a)
        for (int c = 0; c < 3; ++c) {
            hpos[c * M + a] = pos[3 * a + c];
            hvel[c * M + a] = vel ? vel[3 * a + c] : 0.0;
        }
    b->h_nmass.resize(n);
    b->h_nspring.resize(n);
    for (int r = 0; r < n; ++r) {
        b->h_nmass[r] = static_cast<int32_t>(mass_off[r + 1] - mass_off[r]);
        b->h_nspring[r] = static_cast<int32_t>(spring_off[r + 1] - spring_off[r]);
    }
    b->counts_on_host = true;
    std::vector<uint32_t> hij(S);
    std::vector<uint8_t> hact(S, 0);
    std::vector<double> hsign(S, 0.0), hamp(S, 0.0), hphase(S, 0.0);
    for (int r = 0; r < n; ++r) {
        const int64_t nm = mass_off[r + 1] - mass_off[r];
        for (int64_t q = spring_off[r]; q < spring_off[r + 1]; ++q) {
            if (si[q] < 0 || sj[q] < 0 || si[q] >= nm || sj[q] >= nm) {
                delete b;
                set_error("vx_batch_upload: spring endpoint out of range");
                return VX_EINVAL;
            }
            hij[q] = static_cast<uint32_t>(si[q]) | (static_cast<uint32_t>(sj[q]) << 16);
            if (has_act && has_act[q]) {
                hact[q] = 1;
                hsign[q] = sign[q];
                hamp[q] = amp[q];
                hphase[q] = phase[q];
            }
        }
    }
    cudaStream_t s = ctx->stream;
    auto h2d = [&](void* d, const void* h, size_t bytes) { return cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s); };
    cudaError_t e = cudaSuccess;
    auto chk = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
    chk(h2d(b->mass_off.p, mass_off, (n + 1) * sizeof(int64_t)));
    chk(h2d(b->spring_off.p, spring_off, (n + 1) * sizeof(int64_t)));
    if (n > 0) {
        chk(h2d(b->nmass.p, b->h_nmass.data(), n * sizeof(int32_t)));
        chk(h2d(b->nspring.p, b->h_nspring.data(), n * sizeof(int32_t)));
    }
    chk(h2d(b->pos.p, hpos.data(), hpos.size() * sizeof(double)));
    chk(h2d(b->vel.p, hvel.data(), hvel.size() * sizeof(double)));
    chk(h2d(b->mass.p, mass, M * sizeof(double)));
    chk(h2d(b->ij.p, hij.data(), S * sizeof(uint32_t)));
    chk(h2d(b->k.p, k, S * sizeof(double)));
    chk(h2d(b->rest0.p, rest0, S * sizeof(double)));
    chk(h2d(b->zeta.p, zeta, S * sizeof(double)));
    chk(h2d(b->has_act.p, hact.data(), S));
    chk(h2d(b->sign.p, hsign.data(), S * sizeof(double)));
    chk(h2d(b->amp.p, hamp.data(), S * sizeof(double)));
    chk(h2d(b->phase.p, hphase.data(), S * sizeof(double)));
    if (e != cudaSuccess) {
        delete b;
        return cuda_status(e, "vx_batch_upload copy");
    }
    st = batch_derive_workspace(ctx, b);
    if (st == VX_OK) st = cuda_status(cudaStreamSynchronize(s), "vx_batch_upload sync");
    if (st != VX_OK) {
        delete b;
        return st;
    }
    *out = b;
    return VX_OK;
}

vx_status simulate_impl(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, int64_t k0, int64_t n_steps, bool write_back,
                        vx_summary* h_out, vx_summary* d_out) {
    if (!ctx || !b || !sim) return VX_EINVAL;
    if (!(sim->dt > 0.0)) return (set_error("SimConfig: dt must be > 0"), VX_EINVAL);
    if (!(sim->duration >= 0.0)) return (set_error("SimConfig: duration must be >= 0"), VX_EINVAL);
    if (!(sim->actuation_frequency > 0.0)) return (set_error("SimConfig: frequency must be > 0"), VX_EINVAL);
    DevBuf<vx_summary> tmp;
    vx_summary* d = d_out;
    if (!d) {
        VX_TRY(tmp.alloc(std::max(1, b->n)));
        d = tmp.p;
    }
    VX_TRY(integrate(ctx, b, sim, k0, n_steps, write_back, nullptr, 0, d, nullptr));
    if (h_out) {
        VX_CUDA(cudaMemcpyAsync(h_out, d, b->n * sizeof(vx_summary), cudaMemcpyDeviceToHost, ctx->stream));
        VX_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int r = 0; r < b->n; ++r) h_out[r].status = 0;
    }
    return VX_OK;
}

// center_of_mass (physics.hpp:265-277), one thread per robot walking its
// masses in index order: the reference's sequential sums, bit for bit.
__global__ void com_kernel(int n, const int64_t* __restrict__ mass_off, const int32_t* __restrict__ nmass,
                           const double* __restrict__ pos, const double* __restrict__ mass, int64_t M,
                           double* __restrict__ com) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int64_t o = mass_off[r];
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, total = 0.0;
    for (int i = 0; i < nmass[r]; ++i) {
        const double m = mass[o + i];
        c0 += m * pos[o + i];
        c1 += m * pos[M + o + i];
        c2 += m * pos[2 * M + o + i];
        total += m;
    }
    if (total > 0.0) {
        c0 /= total;
        c1 /= total;
        c2 /= total;
    }
    com[3 * r] = c0;
    com[3 * r + 1] = c1;
    com[3 * r + 2] = c2;
}

// simulate() with its COM dump (physics.hpp:285-311): the integrator runs in
// chunks of `stride` steps on the batch's own state (restored afterwards:
// simulate takes the system by value), sampling the COM of every still-live
// robot at each chunk start; a robot leaves the sampling at its first
// diverged step (the fused kernels stop it there), like the reference's
// break.  Chunked stepping is bit-identical to one launch (t = k*dt from the
// global step index).
vx_status simulate_dump_impl(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, int32_t stride, int64_t cap,
                             double* samples, int64_t* counts, vx_summary* h_out) {
    const int n = b->n;
    const int64_t n_steps = std::llround(sim->duration / sim->dt);  // physics.hpp:295
    cudaStream_t s = ctx->stream;
    const size_t sb = 3 * static_cast<size_t>(b->M) * sizeof(double);
    DevBuf<double> save_pos, save_vel, d_com;
    DevBuf<vx_summary> d_summ;
    VX_TRY(save_pos.alloc(3 * b->M));
    VX_TRY(save_vel.alloc(3 * b->M));
    VX_TRY(d_com.alloc(3 * static_cast<size_t>(n)));
    VX_TRY(d_summ.alloc(n));
    VX_CUDA(cudaMemcpyAsync(save_pos.p, b->pos.p, sb, cudaMemcpyDeviceToDevice, s));
    VX_CUDA(cudaMemcpyAsync(save_vel.p, b->vel.p, sb, cudaMemcpyDeviceToDevice, s));
    std::vector<int32_t> nm(n);
    VX_CUDA(cudaMemcpyAsync(nm.data(), b->nmass.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    std::vector<double> com(3 * static_cast<size_t>(n));
    auto get_com = [&]() -> vx_status {
        com_kernel<<<(n + 127) / 128, 128, 0, s>>>(n, b->mass_off.p, b->nmass.p, b->pos.p, b->mass.p, b->M, d_com.p);
        VX_CUDA(cudaGetLastError());
        VX_CUDA(cudaMemcpyAsync(com.data(), d_com.p, com.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
        VX_CUDA(cudaStreamSynchronize(s));
        return VX_OK;
    };
    std::vector<vx_summary> acc(n), part(n);
    std::vector<uint8_t> live(n);
    std::vector<double> max_speed(n, 0.0);
    for (int r = 0; r < n; ++r) {
        std::memset(&acc[r], 0, sizeof(vx_summary));
        counts[r] = 0;
        live[r] = nm[r] > 0;  // an empty system returns the default summary, no samples (:291)
    }
    auto push = [&](int r, double t) {
        if (counts[r] < cap) {
            double* row = samples + (static_cast<size_t>(r) * cap + counts[r]) * 4;
            row[0] = t;
            row[1] = com[3 * r];
            row[2] = com[3 * r + 1];
            row[3] = com[3 * r + 2];
        }
        ++counts[r];
    };
    vx_status st = get_com();
    if (st != VX_OK) return st;
    for (int r = 0; r < n; ++r)
        if (nm[r] > 0)
            for (int c = 0; c < 3; ++c) acc[r].com_start[c] = com[3 * r + c];
    const int64_t chunk = stride > 0 ? stride : std::max<int64_t>(1, n_steps);
    for (int64_t k = 0; k < n_steps && st == VX_OK; k += chunk) {
        if (stride > 0) {
            if (k > 0) st = get_com();
            if (st != VX_OK) break;
            for (int r = 0; r < n; ++r)
                if (live[r]) push(r, static_cast<double>(k) * sim->dt);
        }
        const int64_t len = std::min(chunk, n_steps - k);
        st = integrate(ctx, b, sim, k, len, true, nullptr, 0, d_summ.p, nullptr);
        if (st != VX_OK) break;
        VX_CUDA(cudaMemcpyAsync(part.data(), d_summ.p, n * sizeof(vx_summary), cudaMemcpyDeviceToHost, s));
        VX_CUDA(cudaStreamSynchronize(s));
        bool any = false;
        for (int r = 0; r < n; ++r) {
            if (!live[r]) continue;
            acc[r].steps += part[r].steps;
            acc[r].spring_updates += part[r].spring_updates;
            if (part[r].max_speed > max_speed[r]) max_speed[r] = part[r].max_speed;
            for (int c = 0; c < 3; ++c) acc[r].com_end[c] = part[r].com_end[c];
            if (part[r].diverged) {
                acc[r].diverged = 1;
                live[r] = 0;
            }
            any = any || live[r];
        }
        if (!any) break;
    }
    if (st == VX_OK) {
        // final sample at t = n_steps*dt and the summary (:303-309); a robot
        // that diverged keeps the state of its diverging step (com_end of
        // that chunk), everyone else the final state
        for (int r = 0; r < n; ++r) {
            if (nm[r] <= 0) continue;
            if (n_steps == 0)
                for (int c = 0; c < 3; ++c) acc[r].com_end[c] = acc[r].com_start[c];
            for (int c = 0; c < 3; ++c) com[3 * r + c] = acc[r].com_end[c];
            push(r, static_cast<double>(n_steps) * sim->dt);
            const double dx = acc[r].com_end[0] - acc[r].com_start[0];
            const double dy = acc[r].com_end[1] - acc[r].com_start[1];
            acc[r].horizontal_displacement = std::sqrt(dx * dx + dy * dy);
            acc[r].max_speed = max_speed[r];
        }
        if (h_out) std::memcpy(h_out, acc.data(), n * sizeof(vx_summary));
    }
    // simulate() never modifies the caller's system
    VX_CUDA(cudaMemcpyAsync(b->pos.p, save_pos.p, sb, cudaMemcpyDeviceToDevice, s));
    VX_CUDA(cudaMemcpyAsync(b->vel.p, save_vel.p, sb, cudaMemcpyDeviceToDevice, s));
    VX_CUDA(cudaStreamSynchronize(s));
    return st;
}

}  // namespace

extern "C" {

int32_t vx_abi_version(void) { return VX_ABI_VERSION; }
const char* vx_last_error(void) { return vx::g_last_error.c_str(); }

void vx_default_arch(vx_arch* a) {
    std::memset(a, 0, sizeof(*a));
    a->m = 32;  // EncodingSpec (genome.hpp:26-28), hidden {64,64} (evolution.hpp:44)
    a->n_hidden = 2;
    a->hidden[0] = 64;
    a->hidden[1] = 64;
    a->sigma = 1.0;
}
void vx_default_materials(vx_materials* m) { *m = vx_materials{2e3, 1e3, 1e4, 0.1, 0.25, M_PI, 0.1, 0.1}; }
void vx_default_plane(vx_plane* p) { *p = vx_plane{1e5, 0.1, 0.6, 1.0}; }
void vx_default_sim(vx_sim* s) { *s = vx_sim{9.81, 1e-5, 2.0, 2.0, 1, 1}; }
void vx_default_hyper(vx_hyper* h) { *h = vx_hyper{0.1, 0.1, 0.4, 0.3, {1.0, 1.0, 1.0}}; }
void vx_default_evo_config(vx_evo_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->population = 30;  // EvolutionConfig (evolution.hpp:40-53)
    c->generations = 100;
    c->grid_w = c->grid_h = c->grid_d = 5;
    c->tournament_size = 3;
    c->threads = 1;
    c->seed = 0;
    vx_default_arch(&c->arch);
    vx_default_hyper(&c->initial_params);
    vx_default_materials(&c->materials);
    vx_default_plane(&c->plane);
    vx_default_sim(&c->sim);
}

int64_t vx_param_count(const vx_arch* a) { return vx::param_count(a); }

int32_t vx_elite_count(double elite_fraction, int32_t population) {
    const int n = static_cast<int>(std::ceil(elite_fraction * population - 1e-9));
    return std::clamp(n, 1, std::max(1, population));
}

void vx_hyper_clamp(vx_hyper* h) {
    h->mutation_rate = std::clamp(h->mutation_rate, 0.001, 1.0);
    h->mutation_scale = std::clamp(h->mutation_scale, 0.001, 1.0);
    h->crossover_rate = std::clamp(h->crossover_rate, 0.0, 1.0);
    h->elite_fraction = std::clamp(h->elite_fraction, 0.05, 0.9);
    for (double& m : h->material_multipliers) m = std::clamp(m, 0.1, 10.0);
}

// ------------------------------------------------------------------ context
vx_status vx_create(int32_t device, vx_ctx** out) {
    if (!out) return VX_EINVAL;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        set_error(std::string("no CUDA device: ") + cudaGetErrorString(e));
        return VX_ENODEV;
    }
    if (device < 0 || device >= count) return (set_error("vx_create: bad device index"), VX_EINVAL);
    VX_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    VX_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) {
        set_error(std::string("libvoxevo_b200 is built for sm_100a; device is ") + prop.name);
        return VX_ENODEV;
    }
    auto* c = new vx_ctx;
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
    c->clock_khz = clk;
    std::strncpy(c->name, prop.name, sizeof(c->name) - 1);
    c->smem_optin = prop.sharedMemPerBlockOptin;
    e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return cuda_status(e, "cudaStreamCreate");
    }
    c->stream = c->own_stream;
    *out = c;
    return VX_OK;
}

vx_status vx_destroy(vx_ctx* ctx) {
    if (!ctx) return VX_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx->eval_batch;
    delete ctx;
    return VX_OK;
}

vx_status vx_set_stream(vx_ctx* ctx, void* s) {
    if (!ctx) return VX_EINVAL;
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
    return VX_OK;
}
void* vx_get_stream(vx_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
vx_status vx_synchronize(vx_ctx* ctx) {
    if (!ctx) return VX_EINVAL;
    VX_CUDA(cudaStreamSynchronize(ctx->stream));
    return VX_OK;
}
uint64_t vx_launch_count(vx_ctx* ctx) { return ctx ? ctx->launches : 0; }
int32_t vx_last_integrator(vx_ctx* ctx) { return ctx ? ctx->last_integrator : -1; }
vx_status vx_set_filler(vx_ctx* ctx, int32_t mode) {
    if (!ctx || mode < -1 || mode > 2) return VX_EINVAL;
    ctx->filler_mode = mode;
    return VX_OK;
}
int32_t vx_last_filler_ctas(vx_ctx* ctx) { return ctx ? ctx->filler_ctas : 0; }
vx_status vx_device_info(vx_ctx* ctx, int32_t* sm_count, int32_t* clock_khz, char* name, int32_t name_cap) {
    if (!ctx) return VX_EINVAL;
    if (sm_count) *sm_count = ctx->sm_count;
    if (clock_khz) *clock_khz = ctx->clock_khz;
    if (name && name_cap > 0) {
        std::strncpy(name, ctx->name, name_cap - 1);
        name[name_cap - 1] = 0;
    }
    return VX_OK;
}

// ------------------------------------------------------------------ batches
vx_status vx_batch_upload(vx_ctx* ctx, int32_t n, const int64_t* mass_off, const int64_t* spring_off,
                          const double* pos, const double* vel, const double* mass, const int32_t* si,
                          const int32_t* sj, const double* k, const double* rest0, const double* zeta,
                          const uint8_t* has_act, const double* sign, const double* amp, const double* phase,
                          const vx_plane* plane, vx_batch** out) {
    return upload_impl(ctx, n, mass_off, spring_off, pos, vel, mass, si, sj, k, rest0, zeta, has_act, sign, amp,
                       phase, plane, out);
}

vx_status vx_batch_free(vx_batch* b) {
    if (b) {
        if (b->ctx) cudaStreamSynchronize(b->ctx->stream);
        delete b;
    }
    return VX_OK;
}

int32_t vx_batch_count(const vx_batch* b) { return b ? b->n : 0; }

}  // extern "C"

// Host exchange is always COMPACT (robots back to back, offsets = prefix sums
// of the counts); device-built batches use a fixed per-robot stride.
namespace {
struct Layout {
    std::vector<int64_t> cm, cs;  // compact starts (n+1)
};
vx_status compact_layout(vx_batch* b, Layout& L) {
    VX_TRY(batch_sync_counts(b));
    L.cm.assign(b->n + 1, 0);
    L.cs.assign(b->n + 1, 0);
    for (int r = 0; r < b->n; ++r) {
        L.cm[r + 1] = L.cm[r] + b->h_nmass[r];
        L.cs[r + 1] = L.cs[r] + b->h_nspring[r];
    }
    return VX_OK;
}
template <typename T>
vx_status d2h_compact(vx_batch* b, T* dst, const T* src, int64_t total_dev, const std::vector<int64_t>& dev_start,
                      const std::vector<int64_t>& host_start, const std::vector<int32_t>& count, int width = 1) {
    if (!dst) return VX_OK;
    std::vector<T> tmp(static_cast<size_t>(total_dev) * width);
    VX_CUDA(cudaMemcpyAsync(tmp.data(), src, tmp.size() * sizeof(T), cudaMemcpyDeviceToHost, b->ctx->stream));
    VX_CUDA(cudaStreamSynchronize(b->ctx->stream));
    // width > 1: SoA planes of total_dev each -> row-major [row][width]
    for (int r = 0; r < b->n; ++r)
        for (int64_t q = 0; q < count[r]; ++q)
            for (int c = 0; c < width; ++c)
                dst[(host_start[r] + q) * width + c] = tmp[c * total_dev + dev_start[r] + q];
    return VX_OK;
}
template <typename T>
vx_status h2d_strided(vx_batch* b, T* dst, const T* src, int64_t total_dev, const std::vector<int64_t>& dev_start,
                      const std::vector<int64_t>& host_start, const std::vector<int32_t>& count, int width = 1) {
    std::vector<T> tmp(static_cast<size_t>(total_dev) * width);
    VX_CUDA(cudaMemcpyAsync(tmp.data(), dst, tmp.size() * sizeof(T), cudaMemcpyDeviceToHost, b->ctx->stream));
    VX_CUDA(cudaStreamSynchronize(b->ctx->stream));
    for (int r = 0; r < b->n; ++r)
        for (int64_t q = 0; q < count[r]; ++q)
            for (int c = 0; c < width; ++c)
                tmp[c * total_dev + dev_start[r] + q] = src[(host_start[r] + q) * width + c];
    VX_CUDA(cudaMemcpyAsync(dst, tmp.data(), tmp.size() * sizeof(T), cudaMemcpyHostToDevice, b->ctx->stream));
    VX_CUDA(cudaStreamSynchronize(b->ctx->stream));
    return VX_OK;
}
}  // namespace

extern "C" {

vx_status vx_batch_offsets(const vx_batch* cb, int64_t* mass_off, int64_t* spring_off) {
    vx_batch* b = const_cast<vx_batch*>(cb);
    if (!b) return VX_EINVAL;
    Layout L;
    VX_TRY(compact_layout(b, L));
    if (mass_off) std::copy(L.cm.begin(), L.cm.end(), mass_off);
    if (spring_off) std::copy(L.cs.begin(), L.cs.end(), spring_off);
    return VX_OK;
}

vx_status vx_batch_download(vx_batch* b, double* pos, double* vel, double* mass, int32_t* si, int32_t* sj, double* k,
                            double* rest0, double* zeta, uint8_t* has_act, double* sign, double* amp, double* phase) {
    if (!b) return VX_EINVAL;
    Layout L;
    VX_TRY(compact_layout(b, L));
    const auto& MO = b->h_mass_off;
    const auto& SO = b->h_spring_off;
    VX_TRY(d2h_compact(b, pos, b->pos.p, b->M, MO, L.cm, b->h_nmass, 3));
    VX_TRY(d2h_compact(b, vel, b->vel.p, b->M, MO, L.cm, b->h_nmass, 3));
    VX_TRY(d2h_compact(b, mass, b->mass.p, b->M, MO, L.cm, b->h_nmass));
    if (si || sj) {
        std::vector<uint32_t> ij(static_cast<size_t>(L.cs[b->n]));
        VX_TRY(d2h_compact(b, ij.data(), b->ij.p, b->S, SO, L.cs, b->h_nspring));
        for (size_t q = 0; q < ij.size(); ++q) {
            if (si) si[q] = static_cast<int32_t>(ij[q] & 0xFFFFu);
            if (sj) sj[q] = static_cast<int32_t>(ij[q] >> 16);
        }
    }
    VX_TRY(d2h_compact(b, k, b->k.p, b->S, SO, L.cs, b->h_nspring));
    VX_TRY(d2h_compact(b, rest0, b->rest0.p, b->S, SO, L.cs, b->h_nspring));
    VX_TRY(d2h_compact(b, zeta, b->zeta.p, b->S, SO, L.cs, b->h_nspring));
    VX_TRY(d2h_compact(b, has_act, b->has_act.p, b->S, SO, L.cs, b->h_nspring));
    VX_TRY(d2h_compact(b, sign, b->sign.p, b->S, SO, L.cs, b->h_nspring));
    VX_TRY(d2h_compact(b, amp, b->amp.p, b->S, SO, L.cs, b->h_nspring));
    VX_TRY(d2h_compact(b, phase, b->phase.p, b->S, SO, L.cs, b->h_nspring));
    return VX_OK;
}

vx_status vx_batch_set_state(vx_batch* b, const double* pos, const double* vel) {
    if (!b || !pos) return VX_EINVAL;
    Layout L;
    VX_TRY(compact_layout(b, L));
    VX_TRY(h2d_strided(b, b->pos.p, pos, b->M, b->h_mass_off, L.cm, b->h_nmass, 3));
    if (vel) {
        VX_TRY(h2d_strided(b, b->vel.p, vel, b->M, b->h_mass_off, L.cm, b->h_nmass, 3));
    } else {
        std::vector<double> z(static_cast<size_t>(L.cm[b->n]) * 3, 0.0);
        VX_TRY(h2d_strided(b, b->vel.p, z.data(), b->M, b->h_mass_off, L.cm, b->h_nmass, 3));
    }
    return VX_OK;
}

vx_status vx_batch_workspace(vx_batch* b, double* damp_coef, double* amp_rest, double* sin_phase, double* cos_phase,
                             double* ground_damp, int32_t* inc_off, int32_t* inc_spring, double* inc_sign) {
    if (!b) return VX_EINVAL;
    Layout L;
    VX_TRY(compact_layout(b, L));
    const auto& MO = b->h_mass_off;
    const auto& SO = b->h_spring_off;
    VX_TRY(d2h_compact(b, damp_coef, b->c.p, b->S, SO, L.cs, b->h_nspring));
    VX_TRY(d2h_compact(b, amp_rest, b->amp_rest.p, b->S, SO, L.cs, b->h_nspring));
    VX_TRY(d2h_compact(b, sin_phase, b->sinph.p, b->S, SO, L.cs, b->h_nspring));
    VX_TRY(d2h_compact(b, cos_phase, b->cosph.p, b->S, SO, L.cs, b->h_nspring));
    VX_TRY(d2h_compact(b, ground_damp, b->gdamp.p, b->M, MO, L.cm, b->h_nmass));
    if (inc_off) {
        std::vector<int64_t> ds(b->n), hs(b->n);
        std::vector<int32_t> cnt(b->n);
        for (int r = 0; r < b->n; ++r) {
            ds[r] = MO[r] + r;
            hs[r] = L.cm[r] + r;
            cnt[r] = b->h_nmass[r] + 1;
        }
        VX_TRY(d2h_compact(b, inc_off, b->inc_off.p, b->M + b->n, ds, hs, cnt));
    }
    if (inc_spring || inc_sign) {
        std::vector<int64_t> ds(b->n), hs(b->n);
        std::vector<int32_t> cnt(b->n);
        for (int r = 0; r < b->n; ++r) {
            ds[r] = 2 * SO[r];
            hs[r] = 2 * L.cs[r];
            cnt[r] = 2 * b->h_nspring[r];
        }
        std::vector<uint32_t> inc(static_cast<size_t>(2 * L.cs[b->n]));
        VX_TRY(d2h_compact(b, inc.data(), b->inc.p, 2 * b->S, ds, hs, cnt));
        for (size_t e = 0; e < inc.size(); ++e) {
            if (inc_spring) inc_spring[e] = static_cast<int32_t>(inc[e] >> 1);
            if (inc_sign) inc_sign[e] = (inc[e] & 1u) ? -1.0 : 1.0;
        }
    }
    return VX_OK;
}

vx_status vx_batch_override_phase(vx_batch* b, const double* sin_phase, const double* cos_phase) {
    if (!b || !sin_phase || !cos_phase) return VX_EINVAL;
    Layout L;
    VX_TRY(compact_layout(b, L));
    VX_TRY(h2d_strided(b, b->sinph.p, sin_phase, b->S, b->h_spring_off, L.cs, b->h_nspring));
    VX_TRY(h2d_strided(b, b->cosph.p, cos_phase, b->S, b->h_spring_off, L.cs, b->h_nspring));
    return VX_OK;
}

// --------------------------------------------------------------- integrator
vx_status vx_batch_step(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, int64_t k0, int64_t n_steps,
                        vx_summary* summaries) {
    if (n_steps < 0 || k0 < 0) return VX_EINVAL;
    return simulate_impl(ctx, b, sim, k0, n_steps, true, summaries, nullptr);
}

vx_status vx_batch_step_at(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, double t, vx_summary* summaries) {
    if (!ctx || !b || !sim) return VX_EINVAL;
    // the drive of step(sys, t, ...) (physics.hpp:196-198) for this t alone
    const double wt = kTwoPi * sim->actuation_frequency * t;
    const double2 h = make_double2(std::sin(wt), std::cos(wt));
    VX_TRY(ctx->drive.alloc(1));
    VX_CUDA(cudaMemcpyAsync(ctx->drive.p, &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->drive_freq = -1.0;  // the cached k-indexed table is gone
    ctx->drive_pinned = true;
    const vx_status s = simulate_impl(ctx, b, sim, 0, 1, true, summaries, nullptr);
    ctx->drive_pinned = false;
    return s;
}

vx_status vx_batch_simulate(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, vx_summary* summaries) {
    if (!sim) return VX_EINVAL;
    const int64_t n_steps = std::llround(sim->duration / sim->dt);  // physics.hpp:295
    return simulate_impl(ctx, b, sim, 0, n_steps, false, summaries, nullptr);
}

vx_status vx_batch_simulate_dump(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, int32_t stride, int64_t cap,
                                 double* samples, int64_t* counts, vx_summary* summaries) {
    if (!ctx || !b || !sim || cap < 0 || (cap > 0 && !samples) || !counts) return VX_EINVAL;
    if (!(sim->dt > 0.0)) return (set_error("SimConfig: dt must be > 0"), VX_EINVAL);
    if (!(sim->duration >= 0.0)) return (set_error("SimConfig: duration must be >= 0"), VX_EINVAL);
    if (!(sim->actuation_frequency > 0.0)) return (set_error("SimConfig: frequency must be > 0"), VX_EINVAL);
    if (b->n <= 0) return VX_OK;
    return simulate_dump_impl(ctx, b, sim, stride, cap, samples, counts, summaries);
}

vx_status vx_batch_simulate_dev(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, vx_summary* d_summaries) {
    if (!sim || !d_summaries) return VX_EINVAL;
    const int64_t n_steps = std::llround(sim->duration / sim->dt);
    return simulate_impl(ctx, b, sim, 0, n_steps, false, nullptr, d_summaries);
}

// -------------------------------------------------------------------- bench
// run_bench (bench.hpp:50-86): `jobs` copies of bench_robot(grid) built on
// device, each stepped `steps` times from t = 0 in one fused launch; the
// update count is audited from the kernel's own per-robot counters.
vx_status vx_run_bench(vx_ctx* ctx, int32_t jobs, int64_t steps, int32_t grid, double dt, double* out6) {
    if (!ctx || jobs < 1 || steps < 0 || grid < 1 || !out6) return VX_EINVAL;
    const int cells = grid * grid * grid;
    std::vector<uint8_t> mat(static_cast<size_t>(jobs) * cells);
    std::vector<double> wt(static_cast<size_t>(jobs) * cells, 1.0);
    static const uint8_t cyc[4] = {1, 3, 2, 4};  // bench.hpp:38-39
    for (int j = 0; j < jobs; ++j)
        for (int z = 0; z < grid; ++z)
            for (int y = 0; y < grid; ++y)
                for (int x = 0; x < grid; ++x)
                    mat[static_cast<size_t>(j) * cells + x + grid * (y + grid * z)] = cyc[(x + 2 * y + 3 * z) % 4];
    vx_materials table;
    vx_default_materials(&table);
    vx_plane plane;
    vx_default_plane(&plane);
    vx_batch* b = nullptr;
    VX_TRY(vx_batch_build(ctx, jobs, grid, grid, grid, mat.data(), wt.data(), &table, &plane, &b));
    vx_sim sim;
    vx_default_sim(&sim);
    sim.dt = dt;
    std::vector<vx_summary> summ(jobs);
    DevBuf<vx_summary> d;
    vx_status st = d.alloc(jobs);
    // the integrator's per-launch state upload happens inside the kernel; the
    // drive table is prepared before the timed region like the CPU's setup
    if (st == VX_OK) st = ensure_drive(ctx, sim.actuation_frequency, sim.dt, 0, steps > 0 ? steps : 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, ctx->stream);
    if (st == VX_OK) st = integrate(ctx, b, &sim, 0, steps, true, nullptr, 0, d.p, nullptr);
    cudaEventRecord(e1, ctx->stream);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (st == VX_OK)
        st = cuda_status(cudaMemcpy(summ.data(), d.p, jobs * sizeof(vx_summary), cudaMemcpyDeviceToHost), "bench d2h");
    const int64_t springs = b->h_spring_off[1] - b->h_spring_off[0];
    uint64_t updates = 0;
    bool diverged = false;
    for (const auto& s : summ) {
        updates += s.spring_updates;
        diverged = diverged || s.diverged;
    }
    vx_batch_free(b);
    if (st != VX_OK) return st;
    out6[0] = static_cast<double>(springs);
    out6[1] = static_cast<double>(updates);
    out6[2] = static_cast<double>(jobs) * static_cast<double>(steps) * static_cast<double>(springs);
    out6[3] = ms * 1e-3;
    out6[4] = ms > 0 ? static_cast<double>(updates) / (ms * 1e-3) : 0.0;
    out6[5] = diverged ? 1.0 : 0.0;
    return VX_OK;
}

}  // extern "C"
