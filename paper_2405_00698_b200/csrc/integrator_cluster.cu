// integrator_cluster.cu — K7c: the on-chip lattice integrator for robots too
// big for one SM (352 .. 1,404 masses: 7^3 .. 10^3 grids, the robots of
// configs 3 and 4).
//
// Same algorithm and bit-exact results as integrator_lattice.cu (step()
// physics.hpp:191-264, simulate() :287-311): the higher endpoint of every
// lattice spring computes it in phase 1 for d = 12..0 (the head of the
// reference's ascending-spring-index gather, accumulated in registers), then
// phase 2 adds the forward terms d = 0..12 and integrates.  What changes is the
// placement: ONE THREAD-BLOCK CLUSTER PER ROBOT.
//
//  * The robot's masses (z-major index order) are split into CL contiguous
//    ranges of q masses, one per CTA of the cluster (CL = 2..4, q <= 351), one
//    thread per mass, everything (state, force slots, rest lengths, damping,
//    per-voxel drive) in that CTA's shared memory: nothing streams from HBM.
//  * Lattice springs reach at most H = vw*vh + vw + 1 mass indices back, so a
//    CTA needs the state of the previous CTA's last H masses: a HALO that the
//    previous CTA pushes into this CTA's shared memory with st.shared::cluster
//    right after it integrates them (phase 2).
//  * Force slots are indexed by the LOWER endpoint, F[d][i]: the higher
//    endpoint stores each force once, into its own CTA or — for the ~1.1k
//    springs that cross a range boundary — straight into the previous CTA's
//    shared memory (DSMEM stores, fire-and-forget, spread over phase 1).
//    Phase 2 then reads only local, contiguous slots.
//  * Two cluster barriers per step (barrier.cluster arrive.release /
//    wait.acquire) replace the two __syncthreads of the one-SM kernel; the
//    zero-length / divergence flags are broadcast to every CTA's flag word
//    before the barrier (rare path), tagged with the step so no reset is
//    needed.  The vertex-indexed kernel SPLITS them: every warp arrives after
//    its phase, but only the warps whose data crosses a CTA boundary wait
//    before their next phase (halo readers before phase 1, remote-force
//    receivers before phase 2); the others wait after computing it (+7.5%
//    at 10^3, profiles/r02_split_barrier.md).
// Compiled with --fmad=false; all sums in reference order.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

#include "stream_sym.cuh"
#include "vx_cluster.cuh"
#include "vx_internal.cuh"

#ifndef VX_CL_DRV_EARLY
#define VX_CL_DRV_EARLY 1  // next step's drive loaded before phase 2 (+1.1%, profiles/r02_split_barrier.md)
#endif

namespace vx {
namespace {

constexpr int kNmp = 352;              // threads per CTA; owned masses <= kNmp - 1
constexpr int kXS = 512;               // X row stride: [halo | own kNmp | ghost]
constexpr int kH0 = kXS - kNmp - 1;    // own mass a lives at X index kH0 + a; halo below
constexpr int kGhost = kXS - 1;        // far-away resting mass for missing springs
constexpr int kVpt = 3;                // voxels per thread (drive table rows kept in registers)
constexpr int kMaxCluster = 4;

struct ClArgs {
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
    double* xfinal;  // [6][M] final state, read back by rank 0 for the centre of mass
    int cl;          // CTAs per robot
    int halo;        // H: max backward mass-index offset of a lattice spring
    int vw, vh, ncell;
    double zero_len2;
    // persistent 10^3 mode (claim non-null): robots are claimed from claim[0],
    // shared with the one-SM filler the last cluster to start launches
    int32_t* claim;  // [0] next robot [1] filler robots [2] clusters started, [4..] u64 timestamps
    int n_robots;
    int n_clusters;  // co-resident clusters of this launch
    int n_fill;      // filler CTAs (0: none)
    int fill_stop;   // the filler claims no robot once claim[0] reaches this
    SymArgs fill;    // the filler's arguments (stream_sym.cuh)
};

__global__ void __launch_bounds__(kNmp, 1) cluster_kernel(ClArgs A) {
    const int cl = A.cl;
    const uint32_t rank = cluster_rank();
    const int r = blockIdx.x / cl;
    const BatchView& b = A.b;
    const int64_t mo = b.mass_off[r], so = b.spring_off[r];
    const int nm = b.nmass[r];
    const int a = threadIdx.x;
    vx_summary* out = (A.out && rank == 0) ? A.out + r : nullptr;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* X = reinterpret_cast<double*>(smem_raw);  // [6][kXS]  x y z vx vy vz
    double* F = X + 6 * kXS;                           // [13*3][kNmp] force on i of spring (i, i+off_d)
    double* PR = F + 39 * kNmp;                        // [13][kNmp] rest0 of backward slot (d, a)
    double* PC = PR + 13 * kNmp;                       // [13][kNmp] damping coefficient of slot (d, a)
    const int NT = A.ncell + 1;                        // voxel tables + dummy passive entry
    double* D = PC + 13 * kNmp;                        // [NT] drive per voxel
    double* SA = D + NT;                               // [NT] sign*amplitude (0 for the dummy)
    __shared__ double s_maxsq[kNmp / 32];
    __shared__ double s_cmax[kMaxCluster];
    __shared__ uint32_t s_flag;

    if (nm == 0) {  // uniform over the cluster: every CTA leaves, rank 0 reports
        if (out && a == 0) {
            for (int c = 0; c < 3; ++c) out->com_start[c] = out->com_end[c] = 0.0;
            out->horizontal_displacement = 0.0;
            out->max_speed = 0.0;
            out->diverged = 0;
            out->steps = 0;
            out->spring_updates = 0;
        }
        return;
    }

    // ---------------------------------------------------------- ranges
    const int H = A.halo;
    int q = (nm + cl - 1) / cl;
    if (q < H) q = H;  // a backward neighbour is never more than one CTA away
    const int lo = static_cast<int>(rank) * q;
    const int hi = min(nm, lo + q);
    const int nown = max(0, hi - lo);
    const bool live = a < nown;
    const int g = lo + a;                                    // global mass index of this thread
    const bool has_next = static_cast<int>(rank) + 1 < cl && lo + q < nm;
    const bool push_halo = live && has_next && g >= lo + q - H;  // next CTA reads this mass's state
    const bool warp_live = (a & ~31) < nown;

    // ---------------------------------------------------------- prologue
    // voxel tables: SA in place; sin/cos(phase) staged in the (still unused)
    // force area, then kept in registers (kVpt voxels per thread)
    double* SPH = F;
    double* CPH = F + NT;
    for (int v = a; v < NT; v += kNmp) {
        SA[v] = 0.0;
        SPH[v] = 0.0;
        CPH[v] = 1.0;
    }
    if (a == 0) s_flag = 0u;
    __syncthreads();
    const int ns = b.nspring[r];
    for (int s = a; s < ns; s += kNmp) {  // per-voxel actuation, identical for all its springs
        const int v = A.act_vox[so + s];
        if (v >= 0) {
            SA[v] = A.sign[so + s] * A.amp[so + s];  // sign * amplitude (physics.hpp:153)
            SPH[v] = b.sinph[so + s];
            CPH[v] = b.cosph[so + s];
        }
    }
    // state: own masses, the halo below them, the ghost
    for (int li = kH0 - H + a; li < kH0; li += kNmp) {
        const int gg = lo - kH0 + li;
        if (gg >= 0) {
            for (int c = 0; c < 3; ++c) {
                X[c * kXS + li] = b.pos[c * b.M + mo + gg];
                X[(3 + c) * kXS + li] = b.vel[c * b.M + mo + gg];
            }
        }
    }
    if (a == 0) {
        X[kGhost] = 1e3;
        X[kXS + kGhost] = 1e3;
        X[2 * kXS + kGhost] = 1e3;
        X[3 * kXS + kGhost] = 0.0;
        X[4 * kXS + kGhost] = 0.0;
        X[5 * kXS + kGhost] = 0.0;
    }
    double pk[13];
    uint32_t pnb[13];  // X index of the lower neighbour | voxel << 9 (ncell = passive/missing)
    unsigned fmask = 0u, bmask = 0u;
    double mg = 0.0, imdt = 0.0, gdmp = 0.0;
    double x0 = 0.0, x1 = 0.0, x2 = 0.0, v0 = 0.0, v1 = 0.0, v2 = 0.0;
#pragma unroll
    for (int d = 0; d < 13; ++d) {
        pk[d] = 0.0;
        pnb[d] = static_cast<uint32_t>(kGhost) | (static_cast<uint32_t>(A.ncell) << 9);
        PR[d * kNmp + a] = 1.0;
        PC[d * kNmp + a] = 0.0;
    }
    if (live) {
        x0 = b.pos[mo + g];
        x1 = b.pos[b.M + mo + g];
        x2 = b.pos[2 * b.M + mo + g];
        v0 = b.vel[mo + g];
        v1 = b.vel[b.M + mo + g];
        v2 = b.vel[2 * b.M + mo + g];
        X[kH0 + a] = x0;
        X[kXS + kH0 + a] = x1;
        X[2 * kXS + kH0 + a] = x2;
        X[3 * kXS + kH0 + a] = v0;
        X[4 * kXS + kH0 + a] = v1;
        X[5 * kXS + kH0 + a] = v2;
        const double m = b.mass[mo + g];
        mg = m * A.sp.gravity;  // physics.hpp:226
        imdt = A.sp.dt / m;     // physics.hpp:249
        gdmp = b.gdamp[mo + g];
        const int ka = A.vkey[mo + g];
        const int xa = ka % A.vw, ya = (ka / A.vw) % A.vh, za = ka / (A.vw * A.vh);
        const int32_t* inc_off = b.inc_off + mo + r;
        const uint32_t* inc = b.inc + 2 * so;
        for (int e = inc_off[g]; e < inc_off[g + 1]; ++e) {
            const uint32_t iv = inc[e];
            const int s = static_cast<int>(iv >> 1);
            const uint32_t ij = b.ij[so + s];
            const int other = (iv & 1u) ? static_cast<int>(ij & 0xFFFFu) : static_cast<int>(ij >> 16);
            const int kb = A.vkey[mo + other];
            const int dx = kb % A.vw - xa, dy = (kb / A.vw) % A.vh - ya, dz = kb / (A.vw * A.vh) - za;
            const int L = 9 * dz + 3 * dy + dx;  // forward iff L > 0; direction d = |L| - 1
            const int dd = (L > 0 ? L : -L) - 1;
#pragma unroll
            for (int d = 0; d < 13; ++d) {
                if (d == dd) {
                    if (L < 0) {  // spring (other, g): g is its higher endpoint and computes it
                        bmask |= 1u << d;
                        pk[d] = b.k[so + s];
                        PR[d * kNmp + a] = b.rest0[so + s];
                        PC[d * kNmp + a] = b.c[so + s];
                        const int av = A.act_vox[so + s];
                        pnb[d] = static_cast<uint32_t>(other - lo + kH0) |
                                 (static_cast<uint32_t>(av >= 0 ? av : A.ncell) << 9);
                    } else {  // spring (g, other): its force arrives in F[d][a]
                        fmask |= 1u << d;
                    }
                }
            }
        }
    }
    __syncthreads();
    double vsin[kVpt], vcos[kVpt];
    {
        const double2 drv = __ldg(A.drive);
#pragma unroll
        for (int j = 0; j < kVpt; ++j) {
            const int v = a + j * kNmp;
            vsin[j] = v < NT ? SPH[v] : 0.0;
            vcos[j] = v < NT ? CPH[v] : 1.0;
            if (v < NT) D[v] = drv.x * vcos[j] + drv.y * vsin[j];
        }
    }
    double com_start[3] = {0.0, 0.0, 0.0};
    if (out && a == 0) {  // center_of_mass (physics.hpp:266-278) of the initial state, in mass order
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, total = 0.0;
        for (int m = 0; m < nm; ++m) {
            const double w = b.mass[mo + m];
            c0 += w * b.pos[mo + m];
            c1 += w * b.pos[b.M + mo + m];
            c2 += w * b.pos[2 * b.M + mo + m];
            total += w;
        }
        if (total > 0.0) {
            c0 /= total;
            c1 /= total;
            c2 /= total;
        }
        com_start[0] = c0;
        com_start[1] = c1;
        com_start[2] = c2;
    }
    // DSMEM targets: the previous CTA's force slots, the next CTA's state rows,
    // every CTA's flag word
    const uint32_t f_prev = rank > 0 ? map_rank(smem_addr(F), rank - 1) : 0u;
    const uint32_t x_next = has_next ? map_rank(smem_addr(X), rank + 1) : 0u;
    const uint32_t flag_local = smem_addr(&s_flag);
    cluster_barrier();  // every CTA initialised before any remote store

    const double dt = A.sp.dt;
    const double plane_k = A.sp.plane_k, mu_s = A.sp.mu_s, mu_k = A.sp.mu_k;
    const bool en_grav = A.sp.en_grav, en_contact = A.sp.en_contact;
    double max_sq = 0.0;
    int64_t steps = 0, ok_phase1 = 0;
    int diverged = 0;
    auto raise_flag = [&](uint32_t tag) {  // rare: tell every CTA before the barrier
        for (int c = 0; c < cl; ++c) st_remote_u32(map_rank(flag_local, static_cast<uint32_t>(c)), tag);
    };
    for (int64_t kstep = 0; kstep < A.n_steps; ++kstep) {
        const uint32_t tag1 = static_cast<uint32_t>(2 * kstep + 1), tag2 = tag1 + 1u;
        // ---- phase 1: the backward springs of mass g, d = 12..0 (see integrator_lattice.cu)
        int zero_len = 0;
        double sx = 0.0, sy = 0.0, sz = 0.0;
        if (warp_live) {
            const double* __restrict__ Xr = X;
            constexpr int kChunk = 5;
#pragma unroll
            for (int c0 = 12; c0 >= 0; c0 -= kChunk) {
                double ofx[kChunk], ofy[kChunk], ofz[kChunk];
#pragma unroll
                for (int qq = 0; qq < kChunk; ++qq) {
                    const int d = c0 - qq;
                    if (d < 0) break;
                    const bool valid = (bmask >> d) & 1u;
                    const int nb = static_cast<int>(pnb[d] & 0x1FFu);
                    const int vox = static_cast<int>(pnb[d] >> 9);
                    VX_DCHECK(nb >= kH0 - H && nb < kXS && vox < NT);
                    // spring_force_on_i with i = nb, j = g (physics.hpp:55-64, 201-212)
                    double dx = x0 - Xr[nb];
                    double dy = x1 - Xr[kXS + nb];
                    double dz = x2 - Xr[2 * kXS + nb];
                    const double len2 = dx * dx + dy * dy + dz * dz;
                    const double len = sqrt_rn_fast(len2);
                    zero_len |= (valid && len2 < A.zero_len2) ? 1 : 0;
                    const double r0 = PR[d * kNmp + a];
                    const double rest = r0 + (SA[vox] * r0) * D[vox];
                    const double inv_len = rcp_rn_fast(len);
                    const double nx = dx * inv_len, ny = dy * inv_len, nz = dz * inv_len;
                    const double rel = (v0 - Xr[3 * kXS + nb]) * nx + (v1 - Xr[4 * kXS + nb]) * ny +
                                       (v2 - Xr[5 * kXS + nb]) * nz;
                    const double mag = pk[d] * (len - rest) + PC[d * kNmp + a] * rel;
                    ofx[qq] = mag * nx;
                    ofy[qq] = mag * ny;
                    ofz[qq] = mag * nz;
                }
#pragma unroll
                for (int qq = 0; qq < kChunk; ++qq) {
                    const int d = c0 - qq;
                    if (d < 0) break;
                    const bool valid = (bmask >> d) & 1u;
                    if (valid) {
                        sx -= ofx[qq];  // fx += (-1)*F == fx - F exactly
                        sy -= ofy[qq];
                        sz -= ofz[qq];
                    }
                    // lower endpoint in this CTA (X index >= kH0) or in the previous
                    // one, where its slot index is nb - kH0 + q: predicated, no branch
                    const int li = static_cast<int>(pnb[d] & 0x1FFu) - kH0;
                    const bool rem = li < 0;
                    VX_DCHECK(!valid || (rem ? (rank > 0 && li + q >= 0 && li + q < kNmp) : li < kNmp));
                    if (valid && !rem) {
                        F[(3 * d) * kNmp + li] = ofx[qq];
                        F[(3 * d + 1) * kNmp + li] = ofy[qq];
                        F[(3 * d + 2) * kNmp + li] = ofz[qq];
                    }
                    const uint32_t o = f_prev + 8u * static_cast<uint32_t>((3 * d) * kNmp + li + q);
                    st_remote_if(valid && rem, o, ofx[qq]);
                    st_remote_if(valid && rem, o + 8u * kNmp, ofy[qq]);
                    st_remote_if(valid && rem, o + 16u * kNmp, ofz[qq]);
                }
            }
        }
        ++steps;
        if (zero_len) raise_flag(tag1);
        cluster_barrier();
        if (*reinterpret_cast<volatile uint32_t*>(&s_flag) == tag1) {  // step() returns diverged
            diverged = 1;
            break;
        }
        ++ok_phase1;
        // ---- phase 2: ascending spring index = backward d = 12..0, forward d = 0..12
        int bad = 0;
        if (live) {
            double fx = sx, fy = sy, fz = sz;
#pragma unroll
            for (int d = 0; d < 13; ++d) {
                if (fmask & (1u << d)) {
                    fx += F[(3 * d) * kNmp + a];
                    fy += F[(3 * d + 1) * kNmp + a];
                    fz += F[(3 * d + 2) * kNmp + a];
                }
            }
            if (en_grav) fz -= mg;
            if (en_contact && x2 < 0.0) {
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
            X[kH0 + a] = x0;
            X[kXS + kH0 + a] = x1;
            X[2 * kXS + kH0 + a] = x2;
            X[3 * kXS + kH0 + a] = v0;
            X[4 * kXS + kH0 + a] = v1;
            X[5 * kXS + kH0 + a] = v2;
            if (push_halo) {  // the next CTA's halo copy of this mass
                VX_DCHECK(g - (lo + q) + kH0 >= kH0 - H && g - (lo + q) + kH0 < kH0);
                const uint32_t o = x_next + 8u * static_cast<uint32_t>(g - (lo + q) + kH0);
                st_remote(o, x0);
                st_remote(o + 8u * kXS, x1);
                st_remote(o + 16u * kXS, x2);
                st_remote(o + 24u * kXS, v0);
                st_remote(o + 32u * kXS, v1);
                st_remote(o + 40u * kXS, v2);
            }
            const double speed_sq = v0 * v0 + v1 * v1 + v2 * v2;
            if (speed_sq > max_sq) max_sq = speed_sq;
            if (!(fabs(x0) <= kDivergenceBound) || !(fabs(x1) <= kDivergenceBound) ||
                !(fabs(x2) <= kDivergenceBound))
                bad = 1;
        }
        if (kstep + 1 < A.n_steps) {  // drive of the next step, per voxel
            const double2 drv = __ldg(A.drive + kstep + 1);
#pragma unroll
            for (int j = 0; j < kVpt; ++j) {
                const int v = a + j * kNmp;
                if (v < NT) D[v] = drv.x * vcos[j] + drv.y * vsin[j];
            }
        }
        if (bad) raise_flag(tag2);
        cluster_barrier();
        if (*reinterpret_cast<volatile uint32_t*>(&s_flag) == tag2) {
            diverged = 1;
            break;
        }
    }

    // ---------------------------------------------------------- summary
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(0xffffffffu, max_sq, o);
        if (other > max_sq) max_sq = other;
    }
    if ((a & 31) == 0) s_maxsq[a >> 5] = max_sq;
    if (live) {
        for (int c = 0; c < 3; ++c) {
            A.xfinal[c * b.M + mo + g] = X[c * kXS + kH0 + a];
            A.xfinal[(3 + c) * b.M + mo + g] = X[(3 + c) * kXS + kH0 + a];
            if (A.write_back) {
                b.pos[c * b.M + mo + g] = X[c * kXS + kH0 + a];
                b.vel[c * b.M + mo + g] = X[(3 + c) * kXS + kH0 + a];
            }
        }
    }
    __syncthreads();
    if (a == 0) {
        double m = 0.0;
        for (int w = 0; w < kNmp / 32; ++w)
            if (s_maxsq[w] > m) m = s_maxsq[w];
        st_remote(map_rank(smem_addr(&s_cmax[rank]), 0u), m);
    }
    __threadfence();   // final state visible to rank 0 (global memory)
    cluster_barrier();
    if (out && a == 0) {
        double m = 0.0;
        for (int c = 0; c < cl; ++c)
            if (s_cmax[c] > m) m = s_cmax[c];
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, total = 0.0;
        for (int mm = 0; mm < nm; ++mm) {
            const double w = b.mass[mo + mm];
            c0 += w * A.xfinal[mo + mm];
            c1 += w * A.xfinal[b.M + mo + mm];
            c2 += w * A.xfinal[2 * b.M + mo + mm];
            total += w;
        }
        if (total > 0.0) {
            c0 /= total;
            c1 /= total;
            c2 /= total;
        }
        const double com_end[3] = {c0, c1, c2};
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

// ---------------------------------------------------------------------------
// cluster_vertex_kernel<N>: the same cluster algorithm for N^3 grids with
// threads indexed by LATTICE VERTEX KEY (see vertex_kernel in
// integrator_lattice.cu): CTA c owns keys [c q, c q + q), every neighbour is
// at a compile-time key offset (halo included: the state rows start PAD keys
// below the range), absent vertices are idle threads parked far away.
template <int N>
struct ClusterGeom {
    static constexpr int VW = N + 1;
    static constexpr int NV = VW * VW * VW;
    static constexpr int CL = (NV + kNmp - 2) / (kNmp - 1);     // CTAs per robot
    static constexpr int Q = (NV + CL - 1) / CL;                  // keys per CTA
    static constexpr int PAD = VW * VW + VW + 1;                  // largest backward key offset
    static constexpr int XS = (PAD + kNmp + 1) / 2 * 2;           // state row stride
    static constexpr int NCELL = N * N * N;
    static_assert(Q <= kNmp - 1 && Q >= PAD && CL <= kMaxCluster, "cluster geometry");
};

template <int N>
size_t cluster_vertex_smem() {
    using G = ClusterGeom<N>;
    return (6ull * G::XS + 65ull * kNmp + 2ull * (G::NCELL + 1)) * sizeof(double);
}

// one robot r on this cluster (every CTA of the cluster calls it with the same r)
template <int N>
__device__ __forceinline__ void cluster_vertex_robot(const ClArgs& A, const int r) {
    using G = ClusterGeom<N>;
    constexpr int CL = G::CL, Q = G::Q, PAD = G::PAD, XS = G::XS, VW = G::VW, NV = G::NV;
    constexpr int NTV = G::NCELL + 1;
    const uint32_t rank = cluster_rank();
    const BatchView& b = A.b;
    const int64_t mo = b.mass_off[r], so = b.spring_off[r];
    const int nm = b.nmass[r];
    const int a = threadIdx.x;
    vx_summary* out = (A.out && rank == 0) ? A.out + r : nullptr;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* X = reinterpret_cast<double*>(smem_raw);  // [6][XS]: keys lo - PAD .. lo + kNmp
    double* F = X + 6 * XS;                            // [13*3][kNmp] force on the lower endpoint
    double* PR = F + 39 * kNmp;                        // [13][kNmp] rest0 of backward slot (d, key)
    double* PC = PR + 13 * kNmp;                       // [13][kNmp] damping coefficient
    double* D = PC + 13 * kNmp;                        // [NTV] drive per voxel
    double* SA = D + NTV;                              // [NTV] sign*amplitude
    int* MAP = reinterpret_cast<int*>(F);              // prologue: key -> mass index (-1 absent)
    double* SPH = F + (NV + 1) / 2 + 8;                // prologue: sin/cos(phase) staging
    double* CPH = SPH + NTV;
    __shared__ double s_maxsq[kNmp / 32];
    __shared__ double s_cmax[kMaxCluster];
    __shared__ uint32_t s_flag;
    __shared__ uint32_t s_flags[4];  // split barriers: zero-length [step & 1], divergence [2 + (step & 1)]

    if (nm == 0) {  // uniform over the cluster: every CTA leaves, rank 0 reports
        if (out && a == 0) {
            for (int c = 0; c < 3; ++c) out->com_start[c] = out->com_end[c] = 0.0;
            out->horizontal_displacement = 0.0;
            out->max_speed = 0.0;
            out->diverged = 0;
            out->steps = 0;
            out->spring_updates = 0;
        }
        return;
    }
    const int lo = static_cast<int>(rank) * Q;
    const int g = lo + a;                               // vertex key of this thread
    const bool in_range = a < Q && g < NV;
    const bool has_next = static_cast<int>(rank) + 1 < CL;  // the next CTA owns keys (Q * CL >= NV)

    // ---------------------------------------------------------- prologue
    for (int v = a; v < NTV; v += kNmp) {
        SA[v] = 0.0;
        SPH[v] = 0.0;
        CPH[v] = 1.0;
    }
    for (int k = a; k < NV; k += kNmp) MAP[k] = -1;
    if (a < 5) (a == 0 ? s_flag : s_flags[a - 1]) = 0u;
    __syncthreads();
    for (int m = a; m < nm; m += kNmp) MAP[A.vkey[mo + m]] = m;
    const int ns = b.nspring[r];
    for (int s = a; s < ns; s += kNmp) {
        const int v = A.act_vox[so + s];
        if (v >= 0) {
            SA[v] = A.sign[so + s] * A.amp[so + s];  // sign * amplitude (physics.hpp:153)
            SPH[v] = b.sinph[so + s];
            CPH[v] = b.cosph[so + s];
        }
    }
    __syncthreads();
    // state rows: halo keys [lo - PAD, lo) and own keys; absent -> far away
    for (int li = a; li < PAD; li += kNmp) {
        const int k = lo - PAD + li;
        const int mm = k >= 0 ? MAP[k] : -1;
        for (int c = 0; c < 3; ++c) {
            X[c * XS + li] = mm >= 0 ? b.pos[c * b.M + mo + mm] : 1e3;
            X[(3 + c) * XS + li] = mm >= 0 ? b.vel[c * b.M + mo + mm] : 0.0;
        }
    }
    const int m = in_range ? MAP[g] : -1;
    const bool live = m >= 0;
    const bool push_halo = live && has_next && a >= Q - PAD;  // the next CTA's halo holds this key
    double pk[13];
    uint32_t pvox[7];
    unsigned fmask = 0u, bmask = 0u;
    double mg = 0.0, imdt = 0.0, gdmp = 0.0;
    double x0 = 1e3, x1 = 1e3, x2 = 1e3, v0 = 0.0, v1 = 0.0, v2 = 0.0;
#pragma unroll
    for (int d = 0; d < 13; ++d) {
        pk[d] = 0.0;
        PR[d * kNmp + a] = 1.0;
        PC[d * kNmp + a] = 0.0;
    }
#pragma unroll
    for (int qv = 0; qv < 7; ++qv) pvox[qv] = static_cast<uint32_t>(G::NCELL) * 0x10001u;
    if (live) {
        x0 = b.pos[mo + m];
        x1 = b.pos[b.M + mo + m];
        x2 = b.pos[2 * b.M + mo + m];
        v0 = b.vel[mo + m];
        v1 = b.vel[b.M + mo + m];
        v2 = b.vel[2 * b.M + mo + m];
        const double mm = b.mass[mo + m];
        mg = mm * A.sp.gravity;  // physics.hpp:226
        imdt = A.sp.dt / mm;     // physics.hpp:249
        gdmp = b.gdamp[mo + m];
        const int32_t* inc_off = b.inc_off + mo + r;
        const uint32_t* inc = b.inc + 2 * so;
        for (int e = inc_off[m]; e < inc_off[m + 1]; ++e) {
            const uint32_t iv = inc[e];
            const int sp = static_cast<int>(iv >> 1);
            const uint32_t ij = b.ij[so + sp];
            const int other = (iv & 1u) ? static_cast<int>(ij & 0xFFFFu) : static_cast<int>(ij >> 16);
            const int kb = A.vkey[mo + other];
            const int dx = kb % VW - g % VW, dy = (kb / VW) % VW - (g / VW) % VW, dz = kb / (VW * VW) - g / (VW * VW);
            const int L = 9 * dz + 3 * dy + dx;
            const int dd = (L > 0 ? L : -L) - 1;
#pragma unroll
            for (int d = 0; d < 13; ++d) {
                if (d == dd) {
                    if (L < 0) {
                        bmask |= 1u << d;
                        pk[d] = b.k[so + sp];
                        PR[d * kNmp + a] = b.rest0[so + sp];
                        PC[d * kNmp + a] = b.c[so + sp];
                        const int av = A.act_vox[so + sp];
                        const uint32_t vv = static_cast<uint32_t>(av >= 0 ? av : G::NCELL);
                        const int sh = 16 * (d & 1);
                        pvox[d >> 1] = (pvox[d >> 1] & ~(0xFFFFu << sh)) | (vv << sh);
                    } else {
                        fmask |= 1u << d;
                    }
                }
            }
        }
    }
    __syncthreads();
    double vsin[kVpt], vcos[kVpt];
    {
        const double2 drv = __ldg(A.drive);
#pragma unroll
        for (int j = 0; j < kVpt; ++j) {
            const int v = a + j * kNmp;
            vsin[j] = v < NTV ? SPH[v] : 0.0;
            vcos[j] = v < NTV ? CPH[v] : 1.0;
            if (v < NTV) D[v] = drv.x * vcos[j] + drv.y * vsin[j];
        }
    }
    X[PAD + a] = x0;  // own rows (absent / out-of-range keys: far away, at rest)
    X[XS + PAD + a] = x1;
    X[2 * XS + PAD + a] = x2;
    X[3 * XS + PAD + a] = v0;
    X[4 * XS + PAD + a] = v1;
    X[5 * XS + PAD + a] = v2;
    const unsigned wmask = __reduce_or_sync(0xffffffffu, bmask);
    double com_start[3] = {0.0, 0.0, 0.0};
    // center_of_mass sums (rank 0): the CTA stages (mass, x, y, z) in mass
    // order into the free part of the force-slot area with coalesced loads,
    // then one thread adds them in the reference's order from shared memory
    // instead of walking four global arrays serially
    double* CS = F + (NV + 1) / 2 + 8 + 2 * NTV;  // past the MAP / phase staging of the prologue
    static_assert((NV + 1) / 2 + 8 + 2 * NTV + 4 * NV <= 39 * kNmp, "COM staging fits the force slots");
    if (out) {  // CTA-uniform (rank 0)
        for (int q = a; q < nm; q += kNmp) {
            CS[q] = b.mass[mo + q];
            CS[NV + q] = b.pos[mo + q];
            CS[2 * NV + q] = b.pos[b.M + mo + q];
            CS[3 * NV + q] = b.pos[2 * b.M + mo + q];
        }
        __syncthreads();
    }
    if (out && a == 0) {  // center_of_mass (physics.hpp:266-278) of the initial state, in mass order
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, total = 0.0;
        for (int q = 0; q < nm; ++q) {
            const double w = CS[q];
            c0 += w * CS[NV + q];
            c1 += w * CS[2 * NV + q];
            c2 += w * CS[3 * NV + q];
            total += w;
        }
        if (total > 0.0) {
            c0 /= total;
            c1 /= total;
            c2 /= total;
        }
        com_start[0] = c0;
        com_start[1] = c1;
        com_start[2] = c2;
    }
#ifdef VX_CL_ASM_REMOTE
    const uint32_t f_prev = rank > 0 ? map_rank(smem_addr(F), rank - 1) : 0u;
    const uint32_t x_next = has_next ? map_rank(smem_addr(X), rank + 1) : 0u;
#else
    double* const Fprev = map_generic(F, rank > 0 ? rank - 1 : 0u);
    double* const Xnext = map_generic(X, has_next ? rank + 1 : rank);
#endif
    const uint32_t flag_local = smem_addr(&s_flag);
    cluster_barrier();  // every CTA initialised (MAP and staging in F are dead) before any remote store

    const double dt = A.sp.dt;
    const double plane_k = A.sp.plane_k, mu_s = A.sp.mu_s, mu_k = A.sp.mu_k;
    const bool en_grav = A.sp.en_grav, en_contact = A.sp.en_contact;
    double max_sq = 0.0;
    int64_t steps = 0, ok_phase1 = 0;
    int diverged = 0;
    auto raise_flag = [&](uint32_t tag) {
        for (int c = 0; c < CL; ++c) st_remote_u32(map_rank(flag_local, static_cast<uint32_t>(c)), tag);
    };
    const double* __restrict__ Xa = X + PAD + a;
#ifndef VX_CL_FULL_BARRIER
    // Split cluster barriers (arrive after a phase, wait only where the data
    // crosses a CTA boundary).  Per warp: H reads the halo and stores forces
    // into the previous CTA (keys < PAD), so it waits for barrier B before
    // phase 1; R receives the next CTA's forces and pushes the halo (keys >=
    // Q - PAD), so it waits for barrier A before phase 2.  Every other warp
    // waits after its phase (phase 2 results are committed only after the
    // wait, so a zero-length step of ANY CTA still leaves the state untouched).
    // CTA-local ordering stays with __syncthreads.  Flags live in per-step-
    // parity slots: a slot is rewritten two steps later, after a barrier every
    // reader has passed.
    const int wfirst = a & ~31;
    const bool wH = rank > 0 && wfirst < PAD;
    const bool wR = has_next && wfirst + 31 >= Q - PAD;
    bool pendB = false;
    auto flag_at = [&](int i) { return *reinterpret_cast<volatile uint32_t*>(&s_flags[i]); };
    auto raise_at = [&](int i, uint32_t tag) {
        const uint32_t fl = smem_addr(&s_flags[i]);
        for (int c = 0; c < CL; ++c) st_remote_u32(map_rank(fl, static_cast<uint32_t>(c)), tag);
    };
#endif
    for (int64_t kstep = 0; kstep < A.n_steps; ++kstep) {
        const uint32_t tag1 = static_cast<uint32_t>(2 * kstep + 1), tag2 = tag1 + 1u;
#ifndef VX_CL_FULL_BARRIER
        if (wH && pendB) {  // barrier B of the previous step: halo in, previous CTA done reading our stores
            cluster_wait();
            pendB = false;
            if (flag_at(2 + ((kstep - 1) & 1)) == tag1 - 1u) {
                diverged = 1;
                break;
            }
        }
#endif
        int zero_len = 0;
        double sx = 0.0, sy = 0.0, sz = 0.0;
#if VX_CL_DRV_EARLY == 2
        const double2 drv_pre = __ldg(A.drive + (kstep + 1 < A.n_steps ? kstep + 1 : kstep));
#endif
        {
            auto chunk = [&](auto c0_tag, auto n_tag) {
                constexpr int c0 = decltype(c0_tag)::value, n = decltype(n_tag)::value;
                double ofx[n], ofy[n], ofz[n];
#pragma unroll
                for (int qq = 0; qq < n; ++qq) {
                    const int d = c0 - qq;
                    const int off = key_off<VW>(d);
                    const bool valid = (bmask >> d) & 1u;
                    const int vox = static_cast<int>((pvox[d >> 1] >> (16 * (d & 1))) & 0xFFFFu);
                    double dx = x0 - Xa[-off];
                    double dy = x1 - Xa[XS - off];
                    double dz = x2 - Xa[2 * XS - off];
                    const double len2 = dx * dx + dy * dy + dz * dz;
#ifdef VX_CL_SPLIT_SQRT
                    const double len = sqrt_rn_fast(len2);
                    const double inv_len = rcp_rn_fast(len);
#else
                    double len, inv_len;  // RN(sqrt) and RN(1/len) from one refined rsqrt
                    sqrt_rcp_rn_fast(len2, len, inv_len);
#endif
                    zero_len |= (valid && len2 < A.zero_len2) ? 1 : 0;
                    const double r0 = PR[d * kNmp + a];
                    const double rest = r0 + (SA[vox] * r0) * D[vox];
                    const double nx = dx * inv_len, ny = dy * inv_len, nz = dz * inv_len;
                    const double rel = (v0 - Xa[3 * XS - off]) * nx + (v1 - Xa[4 * XS - off]) * ny +
                                       (v2 - Xa[5 * XS - off]) * nz;
                    const double mag = pk[d] * (len - rest) + PC[d * kNmp + a] * rel;
                    ofx[qq] = mag * nx;
                    ofy[qq] = mag * ny;
                    ofz[qq] = mag * nz;
                }
#pragma unroll
                for (int qq = 0; qq < n; ++qq) {
                    const int d = c0 - qq;
                    const int off = key_off<VW>(d);
                    const bool valid = (bmask >> d) & 1u;
                    if (valid) {
                        sx -= ofx[qq];
                        sy -= ofy[qq];
                        sz -= ofz[qq];
                    }
                    const int li = a - off;
                    const bool rem = li < 0;
                    if (valid && !rem) {
                        F[(3 * d) * kNmp + li] = ofx[qq];
                        F[(3 * d + 1) * kNmp + li] = ofy[qq];
                        F[(3 * d + 2) * kNmp + li] = ofz[qq];
                    }
#ifdef VX_CL_ASM_REMOTE
                    const uint32_t o = f_prev + 8u * static_cast<uint32_t>((3 * d) * kNmp + li + Q);
                    st_remote_if(valid && rem, o, ofx[qq]);
                    st_remote_if(valid && rem, o + 8u * kNmp, ofy[qq]);
                    st_remote_if(valid && rem, o + 16u * kNmp, ofz[qq]);
#else
                    if (valid && rem) {  // lower endpoint in the previous CTA: its slot, over DSMEM
                        double* o = Fprev + (3 * d) * kNmp + li + Q;
                        o[0] = ofx[qq];
                        o[kNmp] = ofy[qq];
                        o[2 * kNmp] = ofz[qq];
                    }
#endif
                }
            };
            // chunks 12..9 | 8..4 | 3..0, each skipped when no lane of the warp
            // has it (measured: +6% over unskipped 5-wide chunks)
            using I4 = std::integral_constant<int, 4>;
            using I5 = std::integral_constant<int, 5>;
            if (wmask & 0x1E00u) chunk(std::integral_constant<int, 12>{}, I4{});
            if (wmask & 0x01F0u) chunk(std::integral_constant<int, 8>{}, I5{});
            if (wmask & 0x000Fu) chunk(std::integral_constant<int, 3>{}, I4{});
        }
#ifndef VX_CL_FULL_BARRIER
        if (pendB) {  // the previous step's barrier B, after this warp's (discardable) phase 1
            cluster_wait();
            pendB = false;
            if (flag_at(2 + ((kstep - 1) & 1)) == tag1 - 1u) {
                diverged = 1;
                break;
            }
        }
        ++steps;
        if (zero_len) raise_at(kstep & 1, tag1);
        cluster_arrive();
        __syncthreads();
        if (wR) {
            cluster_wait();
            if (flag_at(kstep & 1) == tag1) {
                diverged = 1;
                break;
            }
        }
#else
        ++steps;
        if (zero_len) raise_flag(tag1);
#ifdef VX_CL_TIMING_NOSYNC  // timing-only bound (WRONG results): CTA barrier, no cluster sync, no exits
        __syncthreads();
        if (false) {
#else
        cluster_barrier();
        if (*reinterpret_cast<volatile uint32_t*>(&s_flag) == tag1) {
#endif
            diverged = 1;
            break;
        }
#endif
#if VX_CL_DRV_EARLY == 1
        // next step's drive, loaded before phase 2 so the L2 latency overlaps it
        const double2 drv_next = __ldg(A.drive + (kstep + 1 < A.n_steps ? kstep + 1 : kstep));
#endif
        int bad = 0;
        double speed_sq = 0.0;
        if (live) {
            double fx = sx, fy = sy, fz = sz;
#pragma unroll
            for (int d = 0; d < 13; ++d) {
                if (fmask & (1u << d)) {
                    fx += F[(3 * d) * kNmp + a];
                    fy += F[(3 * d + 1) * kNmp + a];
                    fz += F[(3 * d + 2) * kNmp + a];
                }
            }
            if (en_grav) fz -= mg;
            if (en_contact && x2 < 0.0) {
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
            speed_sq = v0 * v0 + v1 * v1 + v2 * v2;
            if (!(fabs(x0) <= kDivergenceBound) || !(fabs(x1) <= kDivergenceBound) ||
                !(fabs(x2) <= kDivergenceBound))
                bad = 1;
        }
#ifndef VX_CL_FULL_BARRIER
        if (!wR) {  // barrier A after computing (not committing) phase 2
            cluster_wait();
            if (flag_at(kstep & 1) == tag1) {
                diverged = 1;
                break;
            }
        }
#endif
        ++ok_phase1;
        if (live) {
            X[PAD + a] = x0;
            X[XS + PAD + a] = x1;
            X[2 * XS + PAD + a] = x2;
            X[3 * XS + PAD + a] = v0;
            X[4 * XS + PAD + a] = v1;
            X[5 * XS + PAD + a] = v2;
            if (push_halo) {  // the next CTA's halo copy of this key: row a - Q + PAD there
#ifdef VX_CL_ASM_REMOTE
                const uint32_t o = x_next + 8u * static_cast<uint32_t>(a - Q + PAD);
                st_remote(o, x0);
                st_remote(o + 8u * XS, x1);
                st_remote(o + 16u * XS, x2);
                st_remote(o + 24u * XS, v0);
                st_remote(o + 32u * XS, v1);
                st_remote(o + 40u * XS, v2);
#else
                double* o = Xnext + (a - Q + PAD);
                o[0] = x0;
                o[XS] = x1;
                o[2 * XS] = x2;
                o[3 * XS] = v0;
                o[4 * XS] = v1;
                o[5 * XS] = v2;
#endif
            }
            if (speed_sq > max_sq) max_sq = speed_sq;
        }
        if (kstep + 1 < A.n_steps) {
#if VX_CL_DRV_EARLY == 1
            const double2 drv = drv_next;
#elif VX_CL_DRV_EARLY == 2
            const double2 drv = drv_pre;
#else
            const double2 drv = __ldg(A.drive + kstep + 1);
#endif
#pragma unroll
            for (int j = 0; j < kVpt; ++j) {
                const int v = a + j * kNmp;
                if (v < NTV) D[v] = drv.x * vcos[j] + drv.y * vsin[j];
            }
        }
#ifndef VX_CL_FULL_BARRIER
        if (bad) raise_at(2 + (kstep & 1), tag2);
        cluster_arrive();
        __syncthreads();
        pendB = true;
    }
    if (pendB) {  // barrier B of the last step
        cluster_wait();
        if (flag_at(2 + ((A.n_steps - 1) & 1)) == static_cast<uint32_t>(2 * A.n_steps)) diverged = 1;
    }
#else
        if (bad) raise_flag(tag2);
#ifdef VX_CL_TIMING_NOSYNC
        __syncthreads();
        if (false) {
#else
        cluster_barrier();
        if (*reinterpret_cast<volatile uint32_t*>(&s_flag) == tag2) {
#endif
            diverged = 1;
            break;
        }
    }
#endif

    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(0xffffffffu, max_sq, o);
        if (other > max_sq) max_sq = other;
    }
    if ((a & 31) == 0) s_maxsq[a >> 5] = max_sq;
    if (live) {
        for (int c = 0; c < 3; ++c) {
            A.xfinal[c * b.M + mo + m] = X[c * XS + PAD + a];
            A.xfinal[(3 + c) * b.M + mo + m] = X[(3 + c) * XS + PAD + a];
            if (A.write_back) {
                b.pos[c * b.M + mo + m] = X[c * XS + PAD + a];
                b.vel[c * b.M + mo + m] = X[(3 + c) * XS + PAD + a];
            }
        }
    }
    __syncthreads();
    if (a == 0) {
        double mx = 0.0;
        for (int w = 0; w < kNmp / 32; ++w)
            if (s_maxsq[w] > mx) mx = s_maxsq[w];
        st_remote(map_rank(smem_addr(&s_cmax[rank]), 0u), mx);
    }
    __threadfence();
    cluster_barrier();
    if (out) {  // stage the final positions for the COM (no remote store reaches F any more)
        for (int q = a; q < nm; q += kNmp) {
            CS[q] = b.mass[mo + q];
            CS[NV + q] = A.xfinal[mo + q];
            CS[2 * NV + q] = A.xfinal[b.M + mo + q];
            CS[3 * NV + q] = A.xfinal[2 * b.M + mo + q];
        }
        __syncthreads();
    }
    if (out && a == 0) {
        double mx = 0.0;
        for (int c = 0; c < CL; ++c)
            if (s_cmax[c] > mx) mx = s_cmax[c];
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, total = 0.0;
        for (int q = 0; q < nm; ++q) {
            const double w = CS[q];
            c0 += w * CS[NV + q];
            c1 += w * CS[2 * NV + q];
            c2 += w * CS[3 * NV + q];
            total += w;
        }
        if (total > 0.0) {
            c0 /= total;
            c1 /= total;
            c2 /= total;
        }
        const double com_end[3] = {c0, c1, c2};
        for (int c = 0; c < 3; ++c) {
            out->com_start[c] = com_start[c];
            out->com_end[c] = com_end[c];
        }
        const double dx = com_end[0] - com_start[0];
        const double dy = com_end[1] - com_start[1];
        out->horizontal_displacement = sqrt(dx * dx + dy * dy);
        out->max_speed = sqrt(mx);
        out->diverged = diverged;
        out->steps = steps;
        out->spring_updates = static_cast<uint64_t>(ok_phase1) * static_cast<uint64_t>(b.nspring[r]);
    }
}

// Static: cluster blockIdx.x / CL integrates robot blockIdx.x / CL.
// Persistent (A.claim set, grid = the co-resident cluster count, 10^3): every
// cluster claims robots from the counter it shares with the one-SM filler
// (stream_sym.cuh, stream_sym_filler); rank 0 draws and broadcasts through
// DSMEM.  The last cluster to become resident launches the filler from the
// device (dynamic parallelism, fire-and-forget), so its CTAs can only land on
// the SMs no 4-CTA cluster was placed on; the cluster grid completes only
// after its child grid.
template <int N>
__global__ void __launch_bounds__(kNmp, 1) cluster_vertex_kernel(ClArgs A) {
    cluster_vertex_robot<N>(A, static_cast<int>(blockIdx.x) / ClusterGeom<N>::CL);
}

template <int N>
__global__ void __launch_bounds__(kNmp, 1) cluster_vertex_persistent(ClArgs A) {
    constexpr int CL = ClusterGeom<N>::CL;
    __shared__ int s_robot;
    const uint32_t rank = cluster_rank();
    unsigned long long* tstat = reinterpret_cast<unsigned long long*>(A.claim + 4);  // [0] min start [1] max start [2] max end
    if (rank == 0 && threadIdx.x == 0) {
        const unsigned long long t = globaltimer_ns();
        atomicMin(tstat, t);
        atomicMax(tstat + 1, t);
        if constexpr (N == 10) {
            if (atomicAdd(A.claim + 2, 1) == A.n_clusters - 1 && A.n_fill > 0)
                stream_sym_filler<10><<<A.n_fill, kStreamThreads, sym_filler_smem(), cudaStreamFireAndForget>>>(
                    A.fill, A.claim, A.n_robots, A.fill_stop);
        }
    }
    for (;;) {
        cluster_barrier();  // every CTA done with the previous s_robot / robot
        if (rank == 0 && threadIdx.x == 0) {
            const int c = atomicAdd(A.claim, 1);
            for (int q = 0; q < CL; ++q) st_remote_u32(map_rank(smem_addr(&s_robot), static_cast<uint32_t>(q)), c);
        }
        cluster_barrier();
        const int r = s_robot;
        if (r >= A.n_robots) {  // uniform over the cluster
            if (rank == 0 && threadIdx.x == 0) atomicMax(tstat + 2, globaltimer_ns());
            return;
        }
        cluster_vertex_robot<N>(A, r);
    }
}

size_t cluster_smem(int ncell) { return (6ull * kXS + 65ull * kNmp + 2ull * (ncell + 1)) * sizeof(double); }

int cluster_size_for(int nm_max) { return (nm_max + kNmp - 2) / (kNmp - 1); }

// cubic grids 7..10 run the vertex-indexed cluster kernel (VX_CLUSTER=rank
// forces the rank-indexed one, for A/B runs)
int cluster_vertex_grid(const vx_batch* b) {
    static const char* force = std::getenv("VX_CLUSTER");
    if (force && std::string(force) == "rank") return 0;
    if (b->lw != b->lh || b->lw != b->ld || b->lw < 7 || b->lw > 10) return 0;
    return b->lw;
}

}  // namespace

// false when the batch is not a device-built lattice batch of the size this
// kernel covers; the caller then uses the streaming kernel.
bool cluster_applicable(vx_ctx* ctx, vx_batch* b) {
    if (!b->lattice || !b->vkey.p || !b->act_vox.p) return false;
    static const char* force = std::getenv("VX_INTEGRATOR");  // "stream" / "generic" skip this kernel
    if (force && (std::string(force) == "stream" || std::string(force) == "generic")) return false;
    const int ncell = b->lw * b->lh * b->ld;
    const int halo = (b->lw + 1) * (b->lh + 1) + (b->lw + 1) + 1;
    const int cl = cluster_size_for(b->nm_max);
    if (cluster_vertex_grid(b) == 0) {
        if (cl < 2 || cl > kMaxCluster || halo > kH0 || ncell + 1 > kVpt * kNmp) return false;
        if (cluster_smem(ncell) + 1024 > ctx->smem_optin) return false;
    }
    if (ctx->cluster_ok < 0) {  // can a cluster of kMaxCluster such CTAs be co-scheduled?
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(kMaxCluster);
        cfg.blockDim = dim3(kNmp);
        cfg.dynamicSmemBytes = cluster_smem(kVpt * kNmp - 1);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kMaxCluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        const bool ok = cudaFuncSetAttribute(cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(cfg.dynamicSmemBytes)) == cudaSuccess &&
                        cudaOccupancyMaxActiveClusters(&n, cluster_kernel, &cfg) == cudaSuccess && n > 0;
        cudaGetLastError();
        ctx->cluster_ok = ok ? 1 : 0;
    }
    return ctx->cluster_ok == 1;
}

vx_status integrate_cluster(vx_ctx* ctx, vx_batch* b, int64_t n_steps, bool write_back, vx_summary* d_summaries,
                            const SimParams& sp, double zero_len2) {
    ClArgs A{};
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
    A.cl = cluster_size_for(b->nm_max);
    A.halo = (b->lw + 1) * (b->lh + 1) + (b->lw + 1) + 1;
    A.vw = b->lw + 1;
    A.vh = b->lh + 1;
    A.ncell = b->lw * b->lh * b->ld;
    A.zero_len2 = zero_len2;
    VX_TRY(ctx->cluster_state.alloc(6 * static_cast<size_t>(b->M)));
    A.xfinal = ctx->cluster_state.p;
    auto launch = [&](auto kernel, int cl, size_t smem) -> vx_status {
        VX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(b->n * cl));
        cfg.blockDim = dim3(kNmp);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(cl);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        VX_CUDA(cudaLaunchKernelEx(&cfg, kernel, A));
        ctx->launches++;
        return VX_OK;
    };
    if (cluster_vertex_grid(b) == 10) {
        ctx->filler_ctas = 0;
        using G = ClusterGeom<10>;
        const size_t smem = cluster_vertex_smem<10>();
        int mode = ctx->filler_mode;
        if (mode < 0) {
            static const char* env = std::getenv("VX_FILLER");
            mode = env ? std::atoi(env) : 1;
        }
        if (ctx->cluster_slots < 0) {  // co-resident 4-CTA clusters on this device
            VX_CUDA(cudaFuncSetAttribute(cluster_vertex_persistent<10>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(G::CL);
            cfg.blockDim = dim3(kNmp);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = G::CL;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, cluster_vertex_persistent<10>, &cfg) != cudaSuccess) n = 0;
            cudaGetLastError();
            ctx->cluster_slots = n;
        }
        const int slots = ctx->cluster_slots;
        const int idle = ctx->sm_count - slots * G::CL;
        // a filler robot takes ~kFillerRatio cluster-robot times: the filler
        // stops claiming while the clusters still have that much work left
        static const char* ratio_env = std::getenv("VX_FILLER_RATIO");
        const int ratio = ratio_env ? std::atoi(ratio_env) : 6;  // re-swept after the split barriers (profiles/r02_filler.md)
        const int64_t stop_at = static_cast<int64_t>(b->n) - static_cast<int64_t>(slots) * ratio;
        const bool use = slots > 0 && idle > 0 &&
                         ((mode == 1 && stop_at >= idle) || (mode == 2 && b->n > 0));
        if (use) {
            VX_TRY(ctx->claim.alloc(16));
            VX_CUDA(cudaMemsetAsync(ctx->claim.p, 0, 16 * sizeof(int32_t), ctx->stream));
            VX_CUDA(cudaMemsetAsync(ctx->claim.p + 4, 0xFF, sizeof(uint64_t), ctx->stream));   // min timestamps
            VX_CUDA(cudaMemsetAsync(ctx->claim.p + 10, 0xFF, sizeof(uint64_t), ctx->stream));
            static const char* ctas_env = std::getenv("VX_FILLER_CTAS");  // A/B: filler width (0: none)
            int nfill = mode == 2 ? std::min(idle, std::max(1, b->n / 2)) : idle;
            if (ctas_env) nfill = std::min(idle, std::max(0, std::atoi(ctas_env)));
            const int stop = mode == 2 ? b->n : static_cast<int>(stop_at);
            const int nclus = std::min(slots, b->n);
            A.claim = ctx->claim.p;
            A.n_robots = b->n;
            A.n_clusters = nclus;
            A.n_fill = nfill;
            A.fill_stop = stop;
            if (nfill > 0) {  // the filler's arguments and per-CTA scratch slots
                SymArgs& F = A.fill;
                F.b = A.b;
                F.vkey = b->vkey.p;
                F.act_vox = b->act_vox.p;
                F.sign = b->sign.p;
                F.amp = b->amp.p;
                F.drive = ctx->drive.p;
                F.sp = sp;
                F.n_steps = n_steps;
                F.write_back = write_back ? 1 : 0;
                F.out = d_summaries;
                F.zero_len2 = zero_len2;
                F.zeta2 = b->uniform_zeta * 2.0;
                F.mu = b->uniform_mass * b->uniform_mass / (b->uniform_mass + b->uniform_mass);
                F.L = sym_layout<10>();
                F.ntab_max = nullptr;
                VX_TRY(ctx->filler_scratch.alloc(F.L.per_robot * static_cast<size_t>(nfill)));
                F.scratch = ctx->filler_scratch.p;
                VX_CUDA(cudaFuncSetAttribute(stream_sym_filler<10>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(sym_filler_smem())));
            }
            VX_CUDA(cudaFuncSetAttribute(cluster_vertex_persistent<10>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(static_cast<unsigned>(nclus * G::CL));
            cfg.blockDim = dim3(kNmp);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = ctx->stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = G::CL;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            VX_CUDA(cudaLaunchKernelEx(&cfg, cluster_vertex_persistent<10>, A));
            ctx->launches += nfill > 0 ? 2 : 1;
            static const char* stats_env = std::getenv("VX_FILLER_STATS");
            if (stats_env && *stats_env == '1') {  // development aid: who did what, when
                int32_t h[16];
                VX_CUDA(cudaMemcpyAsync(h, ctx->claim.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
                VX_CUDA(cudaStreamSynchronize(ctx->stream));
                uint64_t t[6];
                std::memcpy(t, h + 4, sizeof(t));
                const uint64_t t0 = t[0];
                auto rel = [t0](uint64_t x) { return (x == ~0ull || x == 0) ? -1.0 : (static_cast<double>(x) - t0) * 1e-6; };
                std::fprintf(stderr,
                             "[filler] robots %d / %d, filler CTAs %d, stop_at %d | ms from first cluster start: "
                             "last cluster start %.3f, first filler start %.3f, filler end %.3f, cluster end %.3f\n",
                             h[1], b->n, nfill, stop, rel(t[1]), rel(t[3]), rel(t[4]), rel(t[2]));
            }
            ctx->filler_ctas = nfill;
            return VX_OK;
        }
    }
    switch (cluster_vertex_grid(b)) {
        case 7: return launch(cluster_vertex_kernel<7>, ClusterGeom<7>::CL, cluster_vertex_smem<7>());
        case 8: return launch(cluster_vertex_kernel<8>, ClusterGeom<8>::CL, cluster_vertex_smem<8>());
        case 9: return launch(cluster_vertex_kernel<9>, ClusterGeom<9>::CL, cluster_vertex_smem<9>());
        case 10: return launch(cluster_vertex_kernel<10>, ClusterGeom<10>::CL, cluster_vertex_smem<10>());
        default: return launch(cluster_kernel, A.cl, cluster_smem(A.ncell));
    }
}

}  // namespace vx
