// integrator.cu — K7/K8/K9: the fused multi-step spring-mass integrator.
//
// Replaces step() (physics.hpp:191-264), simulate() (physics.hpp:287-311) and
// center_of_mass() (physics.hpp:266-278) for a whole batch of robots.
//
// Design:
//  * one CTA per robot, ALL timesteps of the call fused in one launch;
//  * the robot's mass state (pos/vel, 48 B/mass), per-spring force slots
//    (24 B/spring) and CSR incidence live in shared memory when they fit
//    (<= 6^3 robots; 10^3 keeps state + CSR on chip and streams force slots
//    through L2), spring parameters stream from L2 (coalesced SoA);
//  * phase 1 (per spring) and phase 2 (per mass, ordered CSR gather) are
//    separated by __syncthreads_or, which also carries the divergence flags;
//  * PARITY MODE: this file is compiled with --fmad=false and every
//    expression keeps the reference's evaluation order,
//    sqrt and / are IEEE correctly rounded, the phase-2 gather is in
//    ascending spring index (physics.hpp:166-184, 219-225) and sin/cos(wt)
//    come from a glibc-computed table, so on identical inputs the trajectory
//    is BIT-IDENTICAL to the reference CPU integrator.
#include <cmath>
#include <cstdlib>
#include <string>

#include "vx_internal.cuh"

namespace vx {
namespace {

constexpr int kThreads = 256;

struct KernelArgs {
    BatchView b;
    const double2* drive;  // sin/cos(wt) for k0 .. k0+n_steps-1
    SimParams sp;
    int64_t n_steps;
    int write_back;
    const int32_t* robot_list;
    vx_summary* out;
    const int32_t* out_slot;
    double* g_state;  // per-CTA scratch when state does not fit in smem
    double* g_force;  // per-CTA scratch when force slots do not fit in smem
    int nm_max, ns_max;
};

// center_of_mass (physics.hpp:266-278): sequential in mass order.
__device__ void com_of(const double* X, const double* mass, int nm, double* com) {
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, total = 0.0;
    for (int a = 0; a < nm; ++a) {
        const double m = mass[a];
        c0 += m * X[a];
        c1 += m * X[nm + a];
        c2 += m * X[2 * nm + a];
        total += m;
    }
    if (total > 0.0) {
        c0 /= total;
        c1 /= total;
        c2 /= total;
    }
    com[0] = c0;
    com[1] = c1;
    com[2] = c2;
}

template <bool kStateSmem, bool kForceSmem>
__global__ void __launch_bounds__(kThreads) integrate_kernel(KernelArgs A) {
    const int r = A.robot_list ? A.robot_list[blockIdx.x] : static_cast<int>(blockIdx.x);
    const BatchView& b = A.b;
    const int64_t mo = b.mass_off[r], so = b.spring_off[r];
    const int nm = b.nmass[r];
    const int ns = b.nspring[r];
    vx_summary* out = A.out ? A.out + (A.out_slot ? A.out_slot[blockIdx.x] : r) : nullptr;
    const int tid = threadIdx.x;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* sm = reinterpret_cast<double*>(smem_raw);
    double* X;  // [x(nm) y(nm) z(nm) vx(nm) vy(nm) vz(nm)]
    if (kStateSmem) {
        X = sm;
        sm += 6 * nm;
    } else {
        X = A.g_state + static_cast<size_t>(blockIdx.x) * 10 * A.nm_max;
    }
    double* F;  // [fx(ns) fy(ns) fz(ns)]
    if (kForceSmem) {
        F = sm;
        sm += 3 * ns;
    } else {
        F = A.g_force + static_cast<size_t>(blockIdx.x) * 3 * A.ns_max;
    }
    // per-mass constants (same bits as recomputing them every step)
    double* MC = kStateSmem ? sm : A.g_state + static_cast<size_t>(blockIdx.x) * 10 * A.nm_max + 6 * A.nm_max;
    double* MG = MC;           // m * g            (physics.hpp:226)
    double* IMDT = MC + nm;    // dt / m           (physics.hpp:249)
    double* GD = MC + 2 * nm;  // ground damping   (physics.hpp:163-164)
    double* MASS = MC + 3 * nm;
    if (kStateSmem) sm += 4 * nm;
    __shared__ int s_flag;
    __shared__ double s_maxsq[kThreads / 32];

    if (nm == 0) {
        if (out && tid == 0) {
            for (int c = 0; c < 3; ++c) out->com_start[c] = out->com_end[c] = 0.0;
            out->horizontal_displacement = 0.0;
            out->max_speed = 0.0;
            out->diverged = 0;
            out->steps = 0;
            out->spring_updates = 0;
        }
        return;
    }

    const double dt = A.sp.dt;
    for (int a = tid; a < nm; a += kThreads) {
        for (int c = 0; c < 3; ++c) {
            X[c * nm + a] = b.pos[c * b.M + mo + a];
            X[(3 + c) * nm + a] = b.vel[c * b.M + mo + a];
        }
        const double m = b.mass[mo + a];
        MASS[a] = m;
        MG[a] = m * A.sp.gravity;
        IMDT[a] = dt / m;
        GD[a] = b.gdamp[mo + a];
    }
    const int32_t* inc_off = b.inc_off + mo + r;
    const uint32_t* inc = b.inc + 2 * so;
    const uint32_t* ij = b.ij + so;
    const double* kk = b.k + so;
    const double* rest0 = b.rest0 + so;
    const double* cc = b.c + so;
    const double* amp_rest = b.amp_rest + so;
    const double* sinph = b.sinph + so;
    const double* cosph = b.cosph + so;
    __syncthreads();

    double com_start[3];
    if (out && tid == 0) com_of(X, MASS, nm, com_start);

    double* PX = X;
    double* PY = X + nm;
    double* PZ = X + 2 * nm;
    double* VX = X + 3 * nm;
    double* VY = X + 4 * nm;
    double* VZ = X + 5 * nm;
    double* FX = F;
    double* FY = F + ns;
    double* FZ = F + 2 * ns;

    const double plane_k = A.sp.plane_k, mu_s = A.sp.mu_s, mu_k = A.sp.mu_k;
    double max_sq = 0.0;
    int64_t steps = 0, ok_phase1 = 0;
    int diverged = 0;
    for (int64_t kstep = 0; kstep < A.n_steps; ++kstep) {
        const double2 drv = __ldg(A.drive + kstep);
        const double sin_wt = drv.x, cos_wt = drv.y;
        // ---- phase 1: per-spring force on endpoint i (physics.hpp:201-212, 55-64)
        int zero_len = 0;
        for (int s = tid; s < ns; s += kThreads) {
            const uint32_t e = __ldg(ij + s);
            const int i = static_cast<int>(e & 0xFFFFu), j = static_cast<int>(e >> 16);
            const double xi0 = PX[i], xi1 = PY[i], xi2 = PZ[i];
            const double xj0 = PX[j], xj1 = PY[j], xj2 = PZ[j];
            const double dx = xj0 - xi0, dy = xj1 - xi1, dz = xj2 - xi2;
            const double len = sqrt(dx * dx + dy * dy + dz * dz);
            if (len < kZeroLengthEps) zero_len = 1;
            const double rest = __ldg(rest0 + s) + __ldg(amp_rest + s) * (sin_wt * __ldg(cosph + s) + cos_wt * __ldg(sinph + s));
            const double inv_len = 1.0 / len;
            const double nx = dx * inv_len;
            const double ny = dy * inv_len;
            const double nz = dz * inv_len;
            const double rel = (VX[j] - VX[i]) * nx + (VY[j] - VY[i]) * ny + (VZ[j] - VZ[i]) * nz;
            const double mag = __ldg(kk + s) * (len - rest) + __ldg(cc + s) * rel;
            FX[s] = mag * nx;
            FY[s] = mag * ny;
            FZ[s] = mag * nz;
        }
        ++steps;
        if (__syncthreads_or(zero_len)) {  // step returns diverged, masses untouched
            diverged = 1;
            break;
        }
        ++ok_phase1;
        // ---- phase 2: ordered gather + gravity + contact + integrate (physics.hpp:214-263)
        int bad = 0;
        for (int a = tid; a < nm; a += kThreads) {
            double fx = 0.0, fy = 0.0, fz = 0.0;
            const int e1 = inc_off[a + 1];
            for (int e = inc_off[a]; e < e1; ++e) {
                const uint32_t v = inc[e];
                const int s = static_cast<int>(v >> 1);
                if (v & 1u) {  // sgn = -1: fx += (-1)*f == fx - f exactly
                    fx -= FX[s];
                    fy -= FY[s];
                    fz -= FZ[s];
                } else {
                    fx += FX[s];
                    fy += FY[s];
                    fz += FZ[s];
                }
            }
            double px = PX[a], py = PY[a], pz = PZ[a];
            double vx = VX[a], vy = VY[a], vz = VZ[a];
            if (A.sp.en_grav) fz -= MG[a];
            if (A.sp.en_contact && pz < 0.0) {
                const double penetration = -pz;
                double normal = plane_k * penetration - GD[a] * vz;
                if (normal < 0.0) normal = 0.0;
                const double ft_norm = sqrt(fx * fx + fy * fy);
                const double vt_norm = sqrt(vx * vx + vy * vy);
                if (vt_norm < kStickVelocity && ft_norm <= mu_s * normal) {
                    fx = 0.0;
                    fy = 0.0;
                } else if (vt_norm > 0.0) {
                    const double scale = mu_k * normal / vt_norm;
                    fx -= scale * vx;
                    fy -= scale * vy;
                } else if (ft_norm > 0.0) {
                    const double scale = mu_k * normal / ft_norm;
                    fx -= scale * fx;
                    fy -= scale * fy;
                }
                fz += normal;
            }
            const double imdt = IMDT[a];
            vx += fx * imdt;
            vy += fy * imdt;
            vz += fz * imdt;
            px += vx * dt;
            py += vy * dt;
            pz += vz * dt;
            VX[a] = vx;
            VY[a] = vy;
            VZ[a] = vz;
            PX[a] = px;
            PY[a] = py;
            PZ[a] = pz;
            const double speed_sq = vx * vx + vy * vy + vz * vz;
            if (speed_sq > max_sq) max_sq = speed_sq;
            if (!(fabs(px) <= kDivergenceBound) || !(fabs(py) <= kDivergenceBound) ||
                !(fabs(pz) <= kDivergenceBound))
                bad = 1;
        }
        if (__syncthreads_or(bad)) {
            diverged = 1;
            break;
        }
    }

    // max over threads (order-independent: max of non-NaN values)
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(0xffffffffu, max_sq, o);
        if (other > max_sq) max_sq = other;
    }
    if ((tid & 31) == 0) s_maxsq[tid >> 5] = max_sq;
    __syncthreads();
    if (A.write_back) {
        for (int a = tid; a < nm; a += kThreads) {
            for (int c = 0; c < 3; ++c) {
                b.pos[c * b.M + mo + a] = X[c * nm + a];
                b.vel[c * b.M + mo + a] = X[(3 + c) * nm + a];
            }
        }
    }
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < kThreads / 32; ++w)
            if (s_maxsq[w] > m) m = s_maxsq[w];
        if (out) {
            double com_end[3];
            com_of(X, MASS, nm, com_end);
            for (int c = 0; c < 3; ++c) {
                out->com_start[c] = com_start[c];
                out->com_end[c] = com_end[c];
            }
            const double dx = com_end[0] - com_start[0];
            const double dy = com_end[1] - com_start[1];
            out->horizontal_displacement = sqrt(dx * dx + dy * dy);
            out->max_speed = sqrt(m);
            out->diverged = diverged;
            out->steps = steps;
            out->spring_updates = static_cast<uint64_t>(ok_phase1) * static_cast<uint64_t>(ns);
        }
    }
    (void)s_flag;
}

}  // namespace

// Host-side drive table: sin/cos(kTwoPi * f * t), t = double(k) * dt, with the
// host libm — the very calls the reference makes (physics.hpp:196-198, 297),
// so the table is bit-identical to the reference's per-step values.
vx_status ensure_drive(vx_ctx* ctx, double freq, double dt, int64_t k0, int64_t n) {
    if (ctx->drive_pinned) return VX_OK;
    if (ctx->drive_freq == freq && ctx->drive_dt == dt && ctx->drive_k0 == k0 && ctx->drive_n >= n && ctx->drive.p)
        return VX_OK;
    std::vector<double2> h(static_cast<size_t>(n > 0 ? n : 1));
    for (int64_t q = 0; q < n; ++q) {
        const double t = static_cast<double>(k0 + q) * dt;
        const double wt = kTwoPi * freq * t;
        h[static_cast<size_t>(q)] = make_double2(std::sin(wt), std::cos(wt));
    }
    VX_TRY(ctx->drive.alloc(h.size()));
    VX_CUDA(cudaMemcpyAsync(ctx->drive.p, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));  // h is about to go out of scope
    ctx->drive_freq = freq;
    ctx->drive_dt = dt;
    ctx->drive_k0 = k0;
    ctx->drive_n = n;
    return VX_OK;
}

vx_status integrate(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, int64_t k0, int64_t n_steps, bool write_back,
                    const int32_t* d_robot_list, int n_list, vx_summary* d_summaries, const int32_t* d_summary_slot) {
    if (!b || !sim) return VX_EINVAL;
    const int grid = d_robot_list ? n_list : b->n;
    if (grid <= 0) return VX_OK;
    VX_TRY(ensure_drive(ctx, sim->actuation_frequency, sim->dt, k0, n_steps > 0 ? n_steps : 1));

    static const char* force = std::getenv("VX_INTEGRATOR");  // "generic" forces this file's kernel
    const bool generic = force && std::string(force) == "generic";
    const bool lat = !generic && !d_robot_list && !d_summary_slot && lattice_applicable(ctx, b);
    const bool clus = !generic && !lat && !d_robot_list && !d_summary_slot && cluster_applicable(ctx, b);
    const bool strm = !generic && !lat && !clus && !d_robot_list && !d_summary_slot && stream_applicable(ctx, b);
    if (lat || clus || strm) {
        const SimParams sp{sim->gravity, sim->dt, sim->enable_gravity, sim->enable_contact, b->plane.k,
                           b->plane.mu_static, b->plane.mu_kinetic};
        std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
        if (ctx->timing) {
            if (ctx->event_pool.empty()) {
                VX_CUDA(cudaEventCreate(&ev.first));
                VX_CUDA(cudaEventCreate(&ev.second));
            } else {
                ev = ctx->event_pool.back();
                ctx->event_pool.pop_back();
            }
            VX_CUDA(cudaEventRecord(ev.first, ctx->stream));
        }
        ctx->last_integrator = lat ? VX_KERNEL_LATTICE : clus ? VX_KERNEL_CLUSTER : VX_KERNEL_STREAM;
        if (lat) {
            VX_TRY(integrate_lattice(ctx, b, sim, n_steps, write_back, d_summaries, sp));
        } else if (clus) {
            VX_TRY(integrate_cluster(ctx, b, n_steps, write_back, d_summaries, sp, zero_len2_threshold()));
        } else {
            VX_TRY(integrate_stream(ctx, b, n_steps, write_back, d_summaries, sp, zero_len2_threshold()));
        }
        if (ctx->timing) {
            VX_CUDA(cudaEventRecord(ev.second, ctx->stream));
            ctx->pending.push_back(ev);
        }
        return VX_OK;
    }

    ctx->last_integrator = VX_KERNEL_GENERIC;
    KernelArgs A{};
    A.b = view_of(b);
    A.drive = ctx->drive.p;
    A.sp = SimParams{sim->gravity, sim->dt, sim->enable_gravity, sim->enable_contact, b->plane.k, b->plane.mu_static,
                     b->plane.mu_kinetic};
    A.n_steps = n_steps;
    A.write_back = write_back ? 1 : 0;
    A.robot_list = d_robot_list;
    A.out = d_summaries;
    A.out_slot = d_summary_slot;
    A.nm_max = b->nm_max;
    A.ns_max = b->ns_max;

    const size_t state_b = 6ull * b->nm_max * sizeof(double);
    const size_t force_b = 3ull * b->ns_max * sizeof(double);
    const size_t mconst_b = 4ull * b->nm_max * sizeof(double);
    const size_t budget = ctx->smem_optin ? ctx->smem_optin - 1024 : 48 * 1024;
    bool state_smem = true, force_smem = true;
    if (state_b + force_b + mconst_b > budget) force_smem = false;
    if (state_b + mconst_b > budget) state_smem = false;
    size_t smem = (state_smem ? state_b + mconst_b : 0) + (force_smem ? force_b : 0);
    if (!state_smem) {
        VX_TRY(ctx->scratch_state.alloc(static_cast<size_t>(grid) * 10 * b->nm_max));
        A.g_state = ctx->scratch_state.p;
    }
    if (!force_smem) {
        VX_TRY(ctx->scratch_force.alloc(static_cast<size_t>(grid) * 3 * b->ns_max));
        A.g_force = ctx->scratch_force.p;
    }
    auto launch = [&](auto kernel) -> vx_status {
        VX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
        if (ctx->timing) {
            if (ctx->event_pool.empty()) {
                VX_CUDA(cudaEventCreate(&ev.first));
                VX_CUDA(cudaEventCreate(&ev.second));
            } else {
                ev = ctx->event_pool.back();
                ctx->event_pool.pop_back();
            }
            VX_CUDA(cudaEventRecord(ev.first, ctx->stream));
        }
        kernel<<<grid, kThreads, smem, ctx->stream>>>(A);
        ctx->launches++;
        VX_CUDA(cudaGetLastError());
        if (ctx->timing) {
            VX_CUDA(cudaEventRecord(ev.second, ctx->stream));
            ctx->pending.push_back(ev);
        }
        return VX_OK;
    };
    if (state_smem && force_smem) return launch(integrate_kernel<true, true>);
    if (state_smem) return launch(integrate_kernel<true, false>);
    return launch(integrate_kernel<false, false>);
}

}  // namespace vx
