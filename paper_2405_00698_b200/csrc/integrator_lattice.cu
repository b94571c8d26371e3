// integrator_lattice.cu — K7/K8/K9 specialised for device-built lattice robots.
//
// Same semantics and bit-exact results as integrator.cu (step()
// physics.hpp:191-264, simulate() :287-311), re-laid-out for the SM:
//
//  * thread (g, a): g in {0,1} is a direction group, a a mass (lanes =
//    consecutive masses).  A lattice spring (i, j) joins vertex i to i + off_d
//    for one of 13 "forward" directions d (ascending key offset, == ascending
//    j, so == the reference's spring order).  Group 0 owns directions 0-6 of
//    mass a, group 1 directions 7-12.  Each thread keeps its springs'
//    k / rest0 / c / neighbour / actuating voxel in REGISTERS for the whole
//    launch and its own mass state in registers for the step;
//  * phase 1 writes the force on endpoint i of spring (a, a+off_d) to the
//    direction-major slot F[d][a] — neighbour loads and slot stores of a warp
//    touch consecutive addresses (no bank conflicts);
//  * phase 2 (group 0): mass a sums its backward slots F[d][b(a,d)] for d =
//    12..0 (ascending i) then its forward slots F[d][a] for d = 0..12
//    (ascending j): exactly the reference's ascending-spring-index CSR order
//    (physics.hpp:166-184, 219-225); group 1 meanwhile evaluates the per-voxel
//    drive D_v = sin(wt)cos(phi_v) + cos(wt)sin(phi_v) for the next step (every
//    spring actuated by voxel v shares it, so amp_rest*D_v is the reference's
//    amp_rest*(sin_wt*cos_phase + cos_wt*sin_phase) bit for bit);
//  * two __syncthreads_or per step carry the zero-length and divergence flags.
// Compiled with --fmad=false; all sums in reference order.
#include <cmath>
#include <cstdlib>
#include <string>

#include "vx_internal.cuh"

namespace vx {
namespace {

constexpr int kSlots = 7;  // directions per group (7 + 6)

struct LatArgs {
    BatchView b;
    const int32_t* vkey;
    const int16_t* act_vox;
    const double* sign;
    const double* amp;
    const double2* drive;
    SimParams sp;
    int64_t n_steps;
    int write_back;
    vx_summary* out;
    int nmp;  // masses per group, multiple of 32
    int vw, vh, nv, ncell;
};

__device__ void com_seq(const double* X, int nmp, const double* mass, int nm, double* com) {
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, total = 0.0;
    for (int a = 0; a < nm; ++a) {
        const double m = mass[a];
        c0 += m * X[a];
        c1 += m * X[nmp + a];
        c2 += m * X[2 * nmp + a];
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

template <int kMaxThreads>
__global__ void __launch_bounds__(kMaxThreads, 1) lattice_kernel(LatArgs A) {
    const int r = blockIdx.x;
    const BatchView& b = A.b;
    const int64_t mo = b.mass_off[r], so = b.spring_off[r];
    const int nm = b.nmass[r];
    const int NMP = A.nmp;
    const int tid = threadIdx.x;
    const int g = tid / NMP, a = tid - g * NMP;
    const bool live = a < nm;
    vx_summary* out = A.out ? A.out + r : nullptr;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* X = reinterpret_cast<double*>(smem_raw);     // [6][NMP]  x y z vx vy vz
    double* F = X + 6 * NMP;                              // [13*3][NMP]
    double* MASS = F + 39 * NMP;                          // [NMP]
    double* D = MASS + NMP;                               // [ncell] drive per voxel
    double* SA = D + A.ncell;                             // [ncell] sign*amplitude
    double* SPH = SA + A.ncell;                           // [ncell] sin(phase)
    double* CPH = SPH + A.ncell;                          // [ncell] cos(phase)
    double* PR = CPH + A.ncell;                           // [13][NMP] rest0 of slot (d, a)
    double* PC = PR + 13 * NMP;                           // [13][NMP] damping coefficient c
    uint16_t* BNB = reinterpret_cast<uint16_t*>(PC + 13 * NMP);  // [13][NMP] backward neighbour
    uint16_t* VMAP = BNB + 13 * NMP;                      // [nv] vertex -> mass
    __shared__ double s_maxsq[32];

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

    // ---------------------------------------------------------- prologue
    for (int v = tid; v < A.nv; v += blockDim.x) VMAP[v] = 0xFFFFu;
    for (int v = tid; v < A.ncell; v += blockDim.x) {
        SA[v] = 0.0;
        SPH[v] = 0.0;
        CPH[v] = 1.0;
    }
    __syncthreads();
    if (g == 0 && live) {
        VMAP[A.vkey[mo + a]] = static_cast<uint16_t>(a);
        for (int c = 0; c < 3; ++c) {
            X[c * NMP + a] = b.pos[c * b.M + mo + a];
            X[(3 + c) * NMP + a] = b.vel[c * b.M + mo + a];
        }
        MASS[a] = b.mass[mo + a];
    }
    // per-voxel actuation (every spring of a voxel carries identical values)
    const int ns = b.nspring[r];
    for (int s = tid; s < ns; s += blockDim.x) {
        const int v = A.act_vox[so + s];
        if (v >= 0) {
            SA[v] = A.sign[so + s] * A.amp[so + s];  // sign * amplitude (physics.hpp:153)
            SPH[v] = b.sinph[so + s];
            CPH[v] = b.cosph[so + s];
        }
    }
    // slot parameters (registers for the whole launch)
    double pk[kSlots];
    uint32_t pnb[kSlots];  // neighbour (16 bits) | (voxel + 1) << 16, 0 = no spring
    unsigned fmask = 0u, bmask = 0u;
    double mg = 0.0, imdt = 0.0, gdmp = 0.0;
#pragma unroll
    for (int q = 0; q < kSlots; ++q) {
        pk[q] = 0.0;
        pnb[q] = 0u;
    }
    if (live && g < 2) {
        const int ka = A.vkey[mo + a];
        const int xa = ka % A.vw, ya = (ka / A.vw) % A.vh, za = ka / (A.vw * A.vh);
        const int32_t* inc_off = b.inc_off + mo + r;
        const uint32_t* inc = b.inc + 2 * so;
        for (int e = inc_off[a]; e < inc_off[a + 1]; ++e) {
            const uint32_t iv = inc[e];
            const int s = static_cast<int>(iv >> 1);
            const uint32_t ij = b.ij[so + s];
            const int other = (iv & 1u) ? static_cast<int>(ij & 0xFFFFu) : static_cast<int>(ij >> 16);
            const int kb = A.vkey[mo + other];
            const int dx = kb % A.vw - xa, dy = (kb / A.vw) % A.vh - ya, dz = kb / (A.vw * A.vh) - za;
            const int L = 9 * dz + 3 * dy + dx;  // forward iff L > 0; direction d = |L| - 1
            const int d = (L > 0 ? L : -L) - 1;
            if (L > 0) {
                fmask |= 1u << d;
                const int q = d - g * kSlots;
                if (q >= 0 && q < kSlots) {
#pragma unroll
                    for (int qq = 0; qq < kSlots; ++qq) {
                        if (qq == q) {
                            pk[qq] = b.k[so + s];
                            PR[d * NMP + a] = b.rest0[so + s];
                            PC[d * NMP + a] = b.c[so + s];
                            pnb[qq] = static_cast<uint32_t>(other) |
                                      (static_cast<uint32_t>(A.act_vox[so + s] + 1) << 16) | 0x80000000u;
                        }
                    }
                }
            } else {
                bmask |= 1u << d;
                if (g == 0) BNB[d * NMP + a] = static_cast<uint16_t>(other);
            }
        }
        if (g == 0) {
            const double m = b.mass[mo + a];
            mg = m * A.sp.gravity;  // physics.hpp:226
            imdt = A.sp.dt / m;     // physics.hpp:249
            gdmp = b.gdamp[mo + a];
        }
    }
    __syncthreads();
    {
        const double2 drv = __ldg(A.drive);
        for (int v = tid; v < A.ncell; v += blockDim.x) D[v] = drv.x * CPH[v] + drv.y * SPH[v];
    }
    double com_start[3];
    if (out && tid == 0) com_seq(X, NMP, MASS, nm, com_start);
    __syncthreads();

    const double dt = A.sp.dt;
    const double plane_k = A.sp.plane_k, mu_s = A.sp.mu_s, mu_k = A.sp.mu_k;
    double max_sq = 0.0;
    int64_t steps = 0, ok_phase1 = 0;
    int diverged = 0;
    for (int64_t kstep = 0; kstep < A.n_steps; ++kstep) {
        // ---- phase 1: forward springs of (g, a), force on endpoint a -> F[d][a]
        double x0 = 0.0, x1 = 0.0, x2 = 0.0, v0 = 0.0, v1 = 0.0, v2 = 0.0;
        int zero_len = 0;
        if (live) {
            x0 = X[a];
            x1 = X[NMP + a];
            x2 = X[2 * NMP + a];
            v0 = X[3 * NMP + a];
            v1 = X[4 * NMP + a];
            v2 = X[5 * NMP + a];
#pragma unroll
            for (int q = 0; q < kSlots; ++q) {
                const uint32_t p = pnb[q];
                if (p & 0x80000000u) {
                    const int nb = static_cast<int>(p & 0xFFFFu);
                    const int vox = static_cast<int>((p >> 16) & 0x7FFFu) - 1;
                    const double dx = X[nb] - x0;
                    const double dy = X[NMP + nb] - x1;
                    const double dz = X[2 * NMP + nb] - x2;
                    const double len = sqrt(dx * dx + dy * dy + dz * dz);
                    if (len < kZeroLengthEps) zero_len = 1;
                    const int d = q + g * kSlots;
                    const double r0 = PR[d * NMP + a];
                    double rest = r0;
                    if (vox >= 0) rest = r0 + (SA[vox] * r0) * D[vox];
                    const double inv_len = 1.0 / len;
                    const double nx = dx * inv_len, ny = dy * inv_len, nz = dz * inv_len;
                    const double rel = (X[3 * NMP + nb] - v0) * nx + (X[4 * NMP + nb] - v1) * ny +
                                       (X[5 * NMP + nb] - v2) * nz;
                    const double mag = pk[q] * (len - rest) + PC[d * NMP + a] * rel;
                    F[(3 * d) * NMP + a] = mag * nx;
                    F[(3 * d + 1) * NMP + a] = mag * ny;
                    F[(3 * d + 2) * NMP + a] = mag * nz;
                }
            }
        }
        ++steps;
        if (__syncthreads_or(zero_len)) {
            diverged = 1;
            break;
        }
        ++ok_phase1;
        // ---- phase 2
        int bad = 0;
        if (g == 0 && live) {
            double fx = 0.0, fy = 0.0, fz = 0.0;
#pragma unroll
            for (int d = 12; d >= 0; --d) {
                if (bmask & (1u << d)) {
                    const int nb = BNB[d * NMP + a];
                    fx -= F[(3 * d) * NMP + nb];
                    fy -= F[(3 * d + 1) * NMP + nb];
                    fz -= F[(3 * d + 2) * NMP + nb];
                }
            }
#pragma unroll
            for (int d = 0; d < 13; ++d) {
                if (fmask & (1u << d)) {
                    fx += F[(3 * d) * NMP + a];
                    fy += F[(3 * d + 1) * NMP + a];
                    fz += F[(3 * d + 2) * NMP + a];
                }
            }
            if (A.sp.en_grav) fz -= mg;
            if (A.sp.en_contact && x2 < 0.0) {
                const double penetration = -x2;
                double normal = plane_k * penetration - gdmp * v2;
                if (normal < 0.0) normal = 0.0;
                const double ft_norm = sqrt(fx * fx + fy * fy);
                const double vt_norm = sqrt(v0 * v0 + v1 * v1);
                if (vt_norm < kStickVelocity && ft_norm <= mu_s * normal) {
                    fx = 0.0;
                    fy = 0.0;
                } else if (vt_norm > 0.0) {
                    const double scale = mu_k * normal / vt_norm;
                    fx -= scale * v0;
                    fy -= scale * v1;
                } else if (ft_norm > 0.0) {
                    const double scale = mu_k * normal / ft_norm;
                    fx -= scale * fx;
                    fy -= scale * fy;
                }
                fz += normal;
            }
            v0 += fx * imdt;
            v1 += fy * imdt;
            v2 += fz * imdt;
            x0 += v0 * dt;
            x1 += v1 * dt;
            x2 += v2 * dt;
            X[a] = x0;
            X[NMP + a] = x1;
            X[2 * NMP + a] = x2;
            X[3 * NMP + a] = v0;
            X[4 * NMP + a] = v1;
            X[5 * NMP + a] = v2;
            const double speed_sq = v0 * v0 + v1 * v1 + v2 * v2;
            if (speed_sq > max_sq) max_sq = speed_sq;
            if (!(fabs(x0) <= kDivergenceBound) || !(fabs(x1) <= kDivergenceBound) ||
                !(fabs(x2) <= kDivergenceBound))
                bad = 1;
        } else if (g == 1 && kstep + 1 < A.n_steps) {
            const double2 drv = __ldg(A.drive + kstep + 1);
            for (int v = a; v < A.ncell; v += NMP) D[v] = drv.x * CPH[v] + drv.y * SPH[v];
        }
        if (__syncthreads_or(bad)) {
            diverged = 1;
            break;
        }
    }

    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(0xffffffffu, max_sq, o);
        if (other > max_sq) max_sq = other;
    }
    if ((tid & 31) == 0) s_maxsq[tid >> 5] = max_sq;
    __syncthreads();
    if (A.write_back && g == 0 && live) {
        for (int c = 0; c < 3; ++c) {
            b.pos[c * b.M + mo + a] = X[c * NMP + a];
            b.vel[c * b.M + mo + a] = X[(3 + c) * NMP + a];
        }
    }
    if (tid == 0 && out) {
        double m = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w)
            if (s_maxsq[w] > m) m = s_maxsq[w];
        double com_end[3];
        com_seq(X, NMP, MASS, nm, com_end);
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
        out->spring_updates = static_cast<uint64_t>(ok_phase1) * static_cast<uint64_t>(b.nspring[r]);
    }
}

}  // namespace

// Returns VX_ENODEV-free "not applicable" (false) when the batch is not a
// lattice batch or too large; the caller then uses the generic kernel.
bool lattice_applicable(vx_ctx* ctx, vx_batch* b) {
    if (!b->lattice || !b->vkey.p || !b->act_vox.p) return false;
    static const char* force = std::getenv("VX_INTEGRATOR");  // "generic" forces integrator.cu's kernel
    if (force && std::string(force) == "generic") return false;
    const int nmp = (b->nm_max + 31) / 32 * 32;
    if (2 * nmp > 1024) return false;
    const int ncell = b->lw * b->lh * b->ld;
    const int nv = (b->lw + 1) * (b->lh + 1) * (b->ld + 1);
    const size_t smem = (72ull * nmp + 4ull * ncell) * sizeof(double) + (13ull * nmp + nv) * sizeof(uint16_t) + 64;
    return smem + 1024 <= ctx->smem_optin;
}

vx_status integrate_lattice(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, int64_t n_steps, bool write_back,
                            vx_summary* d_summaries, const SimParams& sp) {
    LatArgs A{};
    A.b = view_of(b);
    A.vkey = b->vkey.p;
    A.act_vox = b->act_vox.p;
    A.sign = b->sign.p;
    A.amp = b->amp.p;
    A.drive = ctx->drive.p;
    A.sp = sp;
    A.n_steps = n_steps;
    A.write_back = write_back ? 1 : 0;
    A.out = d_summaries;
    A.nmp = (b->nm_max + 31) / 32 * 32;
    A.vw = b->lw + 1;
    A.vh = b->lh + 1;
    A.nv = (b->lw + 1) * (b->lh + 1) * (b->ld + 1);
    A.ncell = b->lw * b->lh * b->ld;
    const int threads = 2 * A.nmp;
    const size_t smem =
        (72ull * A.nmp + 4ull * A.ncell) * sizeof(double) + (13ull * A.nmp + A.nv) * sizeof(uint16_t) + 64;
    auto launch = [&](auto kernel) -> vx_status {
        VX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        kernel<<<b->n, threads, smem, ctx->stream>>>(A);
        ctx->launches++;
        VX_CUDA(cudaGetLastError());
        return VX_OK;
    };
    if (threads <= 256) return launch(lattice_kernel<256>);
    if (threads <= 512) return launch(lattice_kernel<512>);
    if (threads <= 768) return launch(lattice_kernel<768>);
    return launch(lattice_kernel<1024>);
}

}  // namespace vx
