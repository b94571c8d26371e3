// integrator_lattice.cu — K7/K8/K9 specialised for device-built lattice robots.
//
// Same semantics and bit-exact results as integrator.cu (step()
// physics.hpp:191-264, simulate() :287-311), re-laid-out for the SM:
//
//  * one thread per mass a (lanes = consecutive masses), padded mass count NMP
//    a compile-time constant so every shared-memory address is an immediate
//    offset.  A lattice spring (i, j) joins vertex i to i + off_d for one of 13
//    "forward" directions d (ascending key offset == ascending j, i.e. the
//    reference's (i, j) spring order).  Thread a owns the <= 13 BACKWARD
//    springs (a - off_d, a) of mass a (it is their higher endpoint) and keeps
//    their k / neighbour / actuating voxel and its per-mass constants in
//    REGISTERS for the whole launch (rest0 and c in direction-major shared
//    memory), its own mass state in registers;
//  * phase 1 computes those springs for d = 12..0 (= ascending i = ascending
//    spring index): the reference's ordered gather for mass a begins with
//    exactly these terms (fx = 0.0; fx += (-1)*F_s), so thread a accumulates
//    them in registers as it goes and stores each force ONCE, to the
//    direction-major slot F[d][i] of the LOWER endpoint i — neighbour loads
//    and slot stores of a warp touch consecutive addresses (no conflicts);
//    a chunk of directions no lane of the warp has is skipped;
//  * phase 2 continues mass a's sum with its forward springs d = 0..12
//    (ascending j), reading its own contiguous slots F[d][a] — completing the reference's
//    ascending-spring-index CSR order (physics.hpp:166-184, 219-225) — then
//    gravity / contact / integrate; the
//    per-voxel drive D_v = sin(wt)cos(phi_v) + cos(wt)sin(phi_v) of the next
//    step is evaluated once per voxel (every spring actuated by voxel v shares
//    it, so amp_rest*D_v is the reference's
//    amp_rest*(sin_wt*cos_phase + cos_wt*sin_phase) bit for bit);
//  * two __syncthreads_or per step carry the zero-length and divergence flags.
// Compiled with --fmad=false; all sums in reference order.
#include <cmath>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "vx_internal.cuh"

namespace vx {
namespace {



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
    double zero_len2;  // smallest len^2 whose IEEE sqrt is >= kZeroLengthEps
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

// One thread per mass (NMP = padded mass count, a compile-time constant so
// every shared-memory address is base + immediate).
template <int NMP>
__global__ void __launch_bounds__(NMP, 1) lattice_kernel(LatArgs A) {
    const int r = blockIdx.x;
    const BatchView& b = A.b;
    const int64_t mo = b.mass_off[r], so = b.spring_off[r];
    const int nm = b.nmass[r];
    const int a = threadIdx.x;
    const bool live = a < nm;
    vx_summary* out = A.out ? A.out + r : nullptr;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* X = reinterpret_cast<double*>(smem_raw);  // [6][NMP]  x y z vx vy vz
    double* F = X + 6 * NMP;                           // [13*3][NMP] force on i of spring (a, a+off_d)
    double* MASS = F + 39 * NMP;                       // [NMP]
    double* D = MASS + NMP;                            // [ncell] drive per voxel
    const int NT = A.ncell + 1;                        // voxel tables + dummy passive entry
    double* SA = D + NT;                               // [NT] sign*amplitude (0 for the dummy)
    double* SPH = SA + NT;                             // [NT] sin(phase)
    double* CPH = SPH + NT;                            // [NT] cos(phase)
    double* PR = CPH + NT;                             // [13][NMP] rest0 of slot (d, a)
    double* PC = PR + 13 * NMP;                        // [13][NMP] damping coefficient of slot (d, a)
    __shared__ double s_maxsq[NMP / 32];

    if (nm == 0) {
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

    // ---------------------------------------------------------- prologue
    for (int v = a; v < NT; v += NMP) {
        SA[v] = 0.0;
        SPH[v] = 0.0;
        CPH[v] = 1.0;
    }
    __syncthreads();
    const int ns = b.nspring[r];
    for (int s = a; s < ns; s += NMP) {  // per-voxel actuation, identical for all its springs
        const int v = A.act_vox[so + s];
        if (v >= 0) {
            SA[v] = A.sign[so + s] * A.amp[so + s];  // sign * amplitude (physics.hpp:153)
            SPH[v] = b.sinph[so + s];
            CPH[v] = b.cosph[so + s];
        }
    }
    double pk[13];
    uint32_t pnb[13];  // backward (lower) neighbour | actuating voxel << 16 (ncell = passive/missing)
    unsigned fmask = 0u, bmask = 0u;
    double mg = 0.0, imdt = 0.0, gdmp = 0.0;
    double x0 = 0.0, x1 = 0.0, x2 = 0.0, v0 = 0.0, v1 = 0.0, v2 = 0.0;
#pragma unroll
    for (int d = 0; d < 13; ++d) {
        pk[d] = 0.0;
        pnb[d] = static_cast<uint32_t>(NMP - 1) | (static_cast<uint32_t>(A.ncell) << 16);  // ghost
        PR[d * NMP + a] = 1.0;
        PC[d * NMP + a] = 0.0;
    }
    if (a == NMP - 1) {  // ghost mass: far from every real mass, at rest; missing
        X[a] = 1e3;      // springs point at it so every slot runs the same
        X[NMP + a] = 1e3;  // branch-free code on the sqrt/div fast paths
        X[2 * NMP + a] = 1e3;
        X[3 * NMP + a] = 0.0;
        X[4 * NMP + a] = 0.0;
        X[5 * NMP + a] = 0.0;
    }
    if (live) {
        x0 = b.pos[mo + a];
        x1 = b.pos[b.M + mo + a];
        x2 = b.pos[2 * b.M + mo + a];
        v0 = b.vel[mo + a];
        v1 = b.vel[b.M + mo + a];
        v2 = b.vel[2 * b.M + mo + a];
        X[a] = x0;
        X[NMP + a] = x1;
        X[2 * NMP + a] = x2;
        X[3 * NMP + a] = v0;
        X[4 * NMP + a] = v1;
        X[5 * NMP + a] = v2;
        const double m = b.mass[mo + a];
        MASS[a] = m;
        mg = m * A.sp.gravity;  // physics.hpp:226
        imdt = A.sp.dt / m;     // physics.hpp:249
        gdmp = b.gdamp[mo + a];
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
            const int dd = (L > 0 ? L : -L) - 1;
#pragma unroll
            for (int d = 0; d < 13; ++d) {
                if (d == dd) {
                    if (L < 0) {  // spring (other, a): a is its higher endpoint and computes it
                        bmask |= 1u << d;
                        pk[d] = b.k[so + s];
                        PR[d * NMP + a] = b.rest0[so + s];
                        PC[d * NMP + a] = b.c[so + s];
                        const int av = A.act_vox[so + s];
                        pnb[d] = static_cast<uint32_t>(other) | (static_cast<uint32_t>(av >= 0 ? av : A.ncell) << 16);
                    } else {      // spring (a, other): `other` computes it and stores F[d][a]
                        fmask |= 1u << d;
                    }
                }
            }
        }
    }
    const unsigned wmask = __reduce_or_sync(0xffffffffu, bmask);  // directions any lane of the warp has
    __syncthreads();
    {
        const double2 drv = __ldg(A.drive);
        for (int v = a; v < NT; v += NMP) D[v] = drv.x * CPH[v] + drv.y * SPH[v];
    }
    double com_start[3];
    if (out && a == 0) com_seq(X, NMP, MASS, nm, com_start);
    __syncthreads();

    const double dt = A.sp.dt;
    const double plane_k = A.sp.plane_k, mu_s = A.sp.mu_s, mu_k = A.sp.mu_k;
    const bool en_grav = A.sp.en_grav, en_contact = A.sp.en_contact;
    double max_sq = 0.0;
    int64_t steps = 0, ok_phase1 = 0;
    int diverged = 0;
    for (int64_t kstep = 0; kstep < A.n_steps; ++kstep) {
        // ---- phase 1: the 13 forward springs of mass a -> F[d][a]
        // Branch-free over the 13 slots so independent springs interleave (ILP):
        // a missing spring gets a unit offset (no special values on the
        // sqrt/div fast paths) and no store; a passive spring uses the dummy
        // voxel (SA = 0), so rest = rest0 + (0*rest0)*D == rest0 exactly, as in
        // the reference (amp_rest = 0, physics.hpp:157-159).
        // Thread a computes its BACKWARD springs (i = lower neighbour, j = a),
        // d = 12..0 = ascending i = ascending spring index, which is exactly
        // the head of the reference's ordered gather for mass a
        // (physics.hpp:219-225): fx starts at 0.0 and adds (-1)*F_s in that
        // order, so the partial sums are accumulated here, in registers, and
        // each force is stored once (slot F[d][a]) for its lower endpoint's
        // forward pass.  Chunks keep independent springs overlapping: results
        // stay in registers until the chunk's ordered adds and stores.
        int zero_len = 0;
        double sx = 0.0, sy = 0.0, sz = 0.0;
        const double* __restrict__ Xr = X;
        // direction chunks 12..10 | 9..7 | 6..4 | 3..0 (the last: in-plane); a
        // chunk no lane of the warp has a spring in is skipped (warp-uniform
        // branch): z = 0 plane warps skip three of four
        auto chunk = [&](auto c0_tag, auto n_tag) {
            constexpr int c0 = decltype(c0_tag)::value, n = decltype(n_tag)::value;
            double ofx[n], ofy[n], ofz[n];
#pragma unroll
            for (int qq = 0; qq < n; ++qq) {
                const int d = c0 - qq;
                const bool valid = (bmask >> d) & 1u;
                const int nb = static_cast<int>(pnb[d] & 0xFFFFu);
                const int vox = static_cast<int>(pnb[d] >> 16);
                VX_DCHECK(nb < NMP && vox < NT);
                // spring_force_on_i with i = nb, j = a (physics.hpp:55-64, 201-212)
                double dx = x0 - Xr[nb];
                double dy = x1 - Xr[NMP + nb];
                double dz = x2 - Xr[2 * NMP + nb];
                const double len2 = dx * dx + dy * dy + dz * dz;
                double len, inv_len;  // RN(sqrt(len2)), RN(1 / len) (vx_internal.cuh)
                    sqrt_rcp_rn_fast(len2, len, inv_len);
                zero_len |= (valid && len2 < A.zero_len2) ? 1 : 0;  // <=> sqrt(len2) < kZeroLengthEps
                const double r0 = PR[d * NMP + a];
                const double rest = r0 + (SA[vox] * r0) * D[vox];
                const double nx = dx * inv_len, ny = dy * inv_len, nz = dz * inv_len;
                const double rel = (v0 - Xr[3 * NMP + nb]) * nx + (v1 - Xr[4 * NMP + nb]) * ny +
                                   (v2 - Xr[5 * NMP + nb]) * nz;
                const double mag = pk[d] * (len - rest) + PC[d * NMP + a] * rel;
                ofx[qq] = mag * nx;
                ofy[qq] = mag * ny;
                ofz[qq] = mag * nz;
            }
#pragma unroll
            for (int qq = 0; qq < n; ++qq) {
                const int d = c0 - qq;
                if ((bmask >> d) & 1u) {
                    sx -= ofx[qq];  // fx += (-1)*F == fx - F exactly
                    sy -= ofy[qq];
                    sz -= ofz[qq];
                    const int nb = static_cast<int>(pnb[d] & 0xFFFFu);  // slot of the LOWER endpoint
                    F[(3 * d) * NMP + nb] = ofx[qq];
                    F[(3 * d + 1) * NMP + nb] = ofy[qq];
                    F[(3 * d + 2) * NMP + nb] = ofz[qq];
                }
            }
        };
        // chunk sizes 3-3-3-4 measured best (profiles/README.md: 9.5e10 vs 9.1e10
        // for 4-5-4 and 9.3e10 for 2-wide chunks); the in-plane directions 3..0
        // are one chunk, so z = 0 plane warps run a single chunk
        using I3 = std::integral_constant<int, 3>;
        using I4 = std::integral_constant<int, 4>;
        if (wmask & 0x1C00u) chunk(std::integral_constant<int, 12>{}, I3{});
        if (wmask & 0x0380u) chunk(std::integral_constant<int, 9>{}, I3{});
        if (wmask & 0x0070u) chunk(std::integral_constant<int, 6>{}, I3{});
        if (wmask & 0x000Fu) chunk(std::integral_constant<int, 3>{}, I4{});
        ++steps;
        if (__syncthreads_or(zero_len)) {  // step() returns diverged; masses untouched
            diverged = 1;
            break;
        }
        ++ok_phase1;
        // ---- phase 2: ascending spring index = backward d = 12..0, forward d = 0..12
        int bad = 0;
        if (live) {
            // continue the ordered sum with the forward springs d = 0..12
            // (ascending j), whose forces their higher endpoints stored
            double fx = sx, fy = sy, fz = sz;
#pragma unroll
            for (int d = 0; d < 13; ++d) {
                if (fmask & (1u << d)) {  // F[d][a]: force on a of spring (a, a + off_d)
                    fx += F[(3 * d) * NMP + a];
                    fy += F[(3 * d + 1) * NMP + a];
                    fz += F[(3 * d + 2) * NMP + a];
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
        }
        if (kstep + 1 < A.n_steps) {  // drive of the next step, per voxel
            const double2 drv = __ldg(A.drive + kstep + 1);
            for (int v = a; v < NT; v += NMP) D[v] = drv.x * CPH[v] + drv.y * SPH[v];
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
    if ((a & 31) == 0) s_maxsq[a >> 5] = max_sq;
    __syncthreads();
    if (A.write_back && live) {
        for (int c = 0; c < 3; ++c) {
            b.pos[c * b.M + mo + a] = X[c * NMP + a];
            b.vel[c * b.M + mo + a] = X[(3 + c) * NMP + a];
        }
    }
    if (a == 0 && out) {
        double m = 0.0;
        for (int w = 0; w < NMP / 32; ++w)
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

// ---------------------------------------------------------------------------
// vertex_kernel<N>: the same algorithm for robots of an N^3 voxel grid, with
// threads indexed by LATTICE VERTEX KEY (x + vw(y + vh z)) instead of mass
// rank.  Every neighbour is then at a compile-time key offset, so the 13
// neighbour gathers and force-slot stores of a warp are base + immediate and
// touch consecutive addresses — no per-slot neighbour registers, no bank
// conflicts from sparse morphologies (the rank-indexed kernel's gathers carry
// ~21% excess wavefronts).  Absent vertices are idle threads parked far away
// (like the ghost); the state rows carry PAD leading far-away entries so that
// key - offset never underflows.  Masses are still processed in mass order
// wherever order matters (centre of mass), via the key of each mass.
template <int N>
struct VertexGeom {
    static constexpr int VW = N + 1;
    static constexpr int NV = VW * VW * VW;                // vertices
    static constexpr int NT = (NV + 31) / 32 * 32;         // threads
    static constexpr int PAD = VW * VW + VW + 1;           // largest backward key offset
    static constexpr int XS = (PAD + NT + 1) / 2 * 2;      // state row stride
    static constexpr int NCELL = N * N * N;
};

template <int N>
size_t vertex_smem() {
    using G = VertexGeom<N>;
    return (6ull * G::XS + 65ull * G::NT + 4ull * (G::NCELL + 1)) * sizeof(double) + 64;
}

template <int N>
__global__ void __launch_bounds__(VertexGeom<N>::NT, 1) vertex_kernel(LatArgs A) {
    using G = VertexGeom<N>;
    constexpr int NT = G::NT, XS = G::XS, PAD = G::PAD, VW = G::VW, NV = G::NV;
    const int r = blockIdx.x;
    const BatchView& b = A.b;
    const int64_t mo = b.mass_off[r], so = b.spring_off[r];
    const int nm = b.nmass[r];
    const int a = threadIdx.x;  // vertex key
    vx_summary* out = A.out ? A.out + r : nullptr;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* X = reinterpret_cast<double*>(smem_raw);  // [6][XS]: PAD far entries, then key order
    double* F = X + 6 * XS;                            // [13*3][NT] force on the lower endpoint (key)
    double* PR = F + 39 * NT;                          // [13][NT] rest0 of backward slot (d, key)
    double* PC = PR + 13 * NT;                         // [13][NT] damping coefficient
    constexpr int NTV = G::NCELL + 1;                  // voxel tables + dummy passive entry
    double* D = PC + 13 * NT;
    double* SA = D + NTV;
    double* SPH = SA + NTV;
    double* CPH = SPH + NTV;
    int* MAP = reinterpret_cast<int*>(F);              // prologue only: key -> mass index (-1 absent)
    __shared__ double s_maxsq[NT / 32];

    if (nm == 0) {
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

    // ---------------------------------------------------------- prologue
    for (int v = a; v < NTV; v += NT) {
        SA[v] = 0.0;
        SPH[v] = 0.0;
        CPH[v] = 1.0;
    }
    for (int k = a; k < NV; k += NT) MAP[k] = -1;
    for (int q = a; q < PAD; q += NT) {  // the far-away padding rows
        X[q] = 1e3;
        X[XS + q] = 1e3;
        X[2 * XS + q] = 1e3;
        X[3 * XS + q] = 0.0;
        X[4 * XS + q] = 0.0;
        X[5 * XS + q] = 0.0;
    }
    __syncthreads();
    for (int m = a; m < nm; m += NT) MAP[A.vkey[mo + m]] = m;
    const int ns = b.nspring[r];
    for (int s = a; s < ns; s += NT) {  // per-voxel actuation, identical for all its springs
        const int v = A.act_vox[so + s];
        if (v >= 0) {
            SA[v] = A.sign[so + s] * A.amp[so + s];  // sign * amplitude (physics.hpp:153)
            SPH[v] = b.sinph[so + s];
            CPH[v] = b.cosph[so + s];
        }
    }
    __syncthreads();
    const int m = a < NV ? MAP[a] : -1;  // this vertex's mass index
    const bool live = m >= 0;
    double pk[13];
    uint32_t pvox[7];  // actuating voxel of backward slot d, two u16 per word (NCELL = passive/missing)
    unsigned fmask = 0u, bmask = 0u;
    double mg = 0.0, imdt = 0.0, gdmp = 0.0;
    double x0 = 1e3, x1 = 1e3, x2 = 1e3, v0 = 0.0, v1 = 0.0, v2 = 0.0;
#pragma unroll
    for (int d = 0; d < 13; ++d) {
        pk[d] = 0.0;
        PR[d * NT + a] = 1.0;
        PC[d * NT + a] = 0.0;
    }
#pragma unroll
    for (int q = 0; q < 7; ++q) pvox[q] = static_cast<uint32_t>(G::NCELL) * 0x10001u;
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
            const int dx = kb % VW - a % VW, dy = (kb / VW) % VW - (a / VW) % VW, dz = kb / (VW * VW) - a / (VW * VW);
            const int L = 9 * dz + 3 * dy + dx;  // forward iff L > 0; direction d = |L| - 1
            const int dd = (L > 0 ? L : -L) - 1;
#pragma unroll
            for (int d = 0; d < 13; ++d) {
                if (d == dd) {
                    if (L < 0) {  // spring (other, m): m is its higher endpoint and computes it
                        bmask |= 1u << d;
                        pk[d] = b.k[so + sp];
                        PR[d * NT + a] = b.rest0[so + sp];
                        PC[d * NT + a] = b.c[so + sp];
                        const int av = A.act_vox[so + sp];
                        const uint32_t vv = static_cast<uint32_t>(av >= 0 ? av : G::NCELL);
                        const int sh = 16 * (d & 1);
                        pvox[d >> 1] = (pvox[d >> 1] & ~(0xFFFFu << sh)) | (vv << sh);
                    } else {  // spring (m, other): `other` computes it and stores F[d][key]
                        fmask |= 1u << d;
                    }
                }
            }
        }
    }
    __syncthreads();  // MAP (aliasing F) is dead from here on
    if (a < NV) {
        X[PAD + a] = x0;
        X[XS + PAD + a] = x1;
        X[2 * XS + PAD + a] = x2;
        X[3 * XS + PAD + a] = v0;
        X[4 * XS + PAD + a] = v1;
        X[5 * XS + PAD + a] = v2;
    }
    const unsigned wmask = __reduce_or_sync(0xffffffffu, bmask);
    {
        const double2 drv = __ldg(A.drive);
        for (int v = a; v < NTV; v += NT) D[v] = drv.x * CPH[v] + drv.y * SPH[v];
    }
    __syncthreads();
    // centre of mass over the masses in mass order (physics.hpp:266-278)
    auto com = [&](double* c3) {
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, total = 0.0;
        for (int q = 0; q < nm; ++q) {
            const double w = b.mass[mo + q];
            const int k = PAD + A.vkey[mo + q];
            c0 += w * X[k];
            c1 += w * X[XS + k];
            c2 += w * X[2 * XS + k];
            total += w;
        }
        if (total > 0.0) {
            c0 /= total;
            c1 /= total;
            c2 /= total;
        }
        c3[0] = c0;
        c3[1] = c1;
        c3[2] = c2;
    };
    double com_start[3];
    if (out && a == 0) com(com_start);

    const double dt = A.sp.dt;
    const double plane_k = A.sp.plane_k, mu_s = A.sp.mu_s, mu_k = A.sp.mu_k;
    const bool en_grav = A.sp.en_grav, en_contact = A.sp.en_contact;
    double max_sq = 0.0;
    int64_t steps = 0, ok_phase1 = 0;
    int diverged = 0;
    const double* __restrict__ Xa = X + PAD + a;  // this vertex's state column
    double* Fa = F + a;
    for (int64_t kstep = 0; kstep < A.n_steps; ++kstep) {
        // ---- phase 1: backward springs d = 12..0 (see lattice_kernel)
        int zero_len = 0;
        double sx = 0.0, sy = 0.0, sz = 0.0;
        auto chunk = [&](auto c0_tag, auto n_tag) {
            constexpr int c0 = decltype(c0_tag)::value, n = decltype(n_tag)::value;
            double ofx[n], ofy[n], ofz[n];
#pragma unroll
            for (int qq = 0; qq < n; ++qq) {
                const int d = c0 - qq;
                constexpr int dummy = 0;
                (void)dummy;
                const int off = key_off<VW>(d);  // compile-time after unrolling
                const bool valid = (bmask >> d) & 1u;
                const int vox = static_cast<int>((pvox[d >> 1] >> (16 * (d & 1))) & 0xFFFFu);
                VX_DCHECK(vox < NTV);
                // spring_force_on_i with i = key - off, j = key (physics.hpp:55-64, 201-212)
                double dx = x0 - Xa[-off];
                double dy = x1 - Xa[XS - off];
                double dz = x2 - Xa[2 * XS - off];
                const double len2 = dx * dx + dy * dy + dz * dz;
                double len, inv_len;  // RN(sqrt(len2)), RN(1 / len) (vx_internal.cuh)
                    sqrt_rcp_rn_fast(len2, len, inv_len);
                zero_len |= (valid && len2 < A.zero_len2) ? 1 : 0;
                const double r0 = PR[d * NT + a];
                const double rest = r0 + (SA[vox] * r0) * D[vox];
                const double nx = dx * inv_len, ny = dy * inv_len, nz = dz * inv_len;
                const double rel = (v0 - Xa[3 * XS - off]) * nx + (v1 - Xa[4 * XS - off]) * ny +
                                   (v2 - Xa[5 * XS - off]) * nz;
                const double mag = pk[d] * (len - rest) + PC[d * NT + a] * rel;
                ofx[qq] = mag * nx;
                ofy[qq] = mag * ny;
                ofz[qq] = mag * nz;
            }
#pragma unroll
            for (int qq = 0; qq < n; ++qq) {
                const int d = c0 - qq;
                const int off = key_off<VW>(d);
                if ((bmask >> d) & 1u) {
                    sx -= ofx[qq];  // fx += (-1)*F == fx - F exactly
                    sy -= ofy[qq];
                    sz -= ofz[qq];
                    VX_DCHECK(a - off >= 0);
                    Fa[(3 * d) * NT - off] = ofx[qq];  // slot of the LOWER endpoint key - off
                    Fa[(3 * d + 1) * NT - off] = ofy[qq];
                    Fa[(3 * d + 2) * NT - off] = ofz[qq];
                }
            }
        };
        // chunks 12..9 | 8..4 | 3..0 measured best for this kernel (profiles/README.md)
        using I4 = std::integral_constant<int, 4>;
        using I5 = std::integral_constant<int, 5>;
        if (wmask & 0x1E00u) chunk(std::integral_constant<int, 12>{}, I4{});
        if (wmask & 0x01F0u) chunk(std::integral_constant<int, 8>{}, I5{});
        if (wmask & 0x000Fu) chunk(std::integral_constant<int, 3>{}, I4{});
        ++steps;
        if (__syncthreads_or(zero_len)) {  // step() returns diverged; masses untouched
            diverged = 1;
            break;
        }
        ++ok_phase1;
        // ---- phase 2: forward springs d = 0..12 from the own slots, then integrate
        int bad = 0;
        if (live) {
            double fx = sx, fy = sy, fz = sz;
#pragma unroll
            for (int d = 0; d < 13; ++d) {
                if (fmask & (1u << d)) {
                    fx += Fa[(3 * d) * NT];
                    fy += Fa[(3 * d + 1) * NT];
                    fz += Fa[(3 * d + 2) * NT];
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
            double* Xw = X + PAD + a;
            Xw[0] = x0;
            Xw[XS] = x1;
            Xw[2 * XS] = x2;
            Xw[3 * XS] = v0;
            Xw[4 * XS] = v1;
            Xw[5 * XS] = v2;
            const double speed_sq = v0 * v0 + v1 * v1 + v2 * v2;
            if (speed_sq > max_sq) max_sq = speed_sq;
            if (!(fabs(x0) <= kDivergenceBound) || !(fabs(x1) <= kDivergenceBound) ||
                !(fabs(x2) <= kDivergenceBound))
                bad = 1;
        }
        if (kstep + 1 < A.n_steps) {  // drive of the next step, per voxel
            const double2 drv = __ldg(A.drive + kstep + 1);
            for (int v = a; v < NTV; v += NT) D[v] = drv.x * CPH[v] + drv.y * SPH[v];
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
    if ((a & 31) == 0) s_maxsq[a >> 5] = max_sq;
    __syncthreads();
    if (A.write_back && live) {
        for (int c = 0; c < 3; ++c) {
            b.pos[c * b.M + mo + m] = X[c * XS + PAD + a];
            b.vel[c * b.M + mo + m] = X[(3 + c) * XS + PAD + a];
        }
    }
    if (a == 0 && out) {
        double mx = 0.0;
        for (int w = 0; w < NT / 32; ++w)
            if (s_maxsq[w] > mx) mx = s_maxsq[w];
        double com_end[3];
        com(com_end);
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

// NMP > max masses: slot NMP-1 is the ghost mass
constexpr int kNmpChoices[] = {64, 128, 160, 224, 256, 352, 384, 512, 544};

int pick_nmp(int nm_cap) {
    for (int c : kNmpChoices)
        if (nm_cap < c) return c;
    return -1;
}

size_t lattice_smem(int nmp, int ncell) { return (73ull * nmp + 4ull * (ncell + 1)) * sizeof(double) + 64; }

// cubic grids 3..6 run the vertex-indexed kernel (VX_LATTICE=rank forces the
// rank-indexed one, for A/B runs)
int vertex_grid(const vx_batch* b) {
    static const char* force = std::getenv("VX_LATTICE");
    if (force && std::string(force) == "rank") return 0;
    if (b->lw != b->lh || b->lw != b->ld || b->lw < 3 || b->lw > 6) return 0;
    return b->lw;
}

}  // namespace

// sqrt is monotone and correctly rounded (host and device alike), so
// len < eps  <=>  len^2 < T with T the smallest double whose sqrt >= eps
double zero_len2_threshold() {
    double t = kZeroLengthEps * kZeroLengthEps;
    while (std::sqrt(t) >= kZeroLengthEps) t = std::nextafter(t, 0.0);
    while (std::sqrt(t) < kZeroLengthEps) t = std::nextafter(t, 1.0);
    return t;
}

// false when the batch is not a device-built lattice batch or is too large;
// the caller then uses the generic kernel (integrator.cu).
bool lattice_applicable(vx_ctx* ctx, vx_batch* b) {
    if (!b->lattice || !b->vkey.p || !b->act_vox.p) return false;
    static const char* force = std::getenv("VX_INTEGRATOR");  // "generic" forces integrator.cu's kernel
    if (force && std::string(force) == "generic") return false;
    if (vertex_grid(b) > 0) return true;
    const int nmp = pick_nmp(b->nm_max);
    if (nmp < 0) return false;
    return lattice_smem(nmp, b->lw * b->lh * b->ld) + 1024 <= ctx->smem_optin;
}

vx_status integrate_lattice(vx_ctx* ctx, vx_batch* b, const vx_sim* sim, int64_t n_steps, bool write_back,
                            vx_summary* d_summaries, const SimParams& sp) {
    (void)sim;
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
    A.nmp = pick_nmp(b->nm_max);
    A.vw = b->lw + 1;
    A.vh = b->lh + 1;
    A.nv = (b->lw + 1) * (b->lh + 1) * (b->ld + 1);
    A.ncell = b->lw * b->lh * b->ld;
    A.zero_len2 = zero_len2_threshold();
    auto launch_v = [&](auto kernel, int threads, size_t smem) -> vx_status {
        VX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        kernel<<<b->n, threads, smem, ctx->stream>>>(A);
        ctx->launches++;
        VX_CUDA(cudaGetLastError());
        return VX_OK;
    };
    switch (vertex_grid(b)) {
        case 3: return launch_v(vertex_kernel<3>, VertexGeom<3>::NT, vertex_smem<3>());
        case 4: return launch_v(vertex_kernel<4>, VertexGeom<4>::NT, vertex_smem<4>());
        case 5: return launch_v(vertex_kernel<5>, VertexGeom<5>::NT, vertex_smem<5>());
        case 6: return launch_v(vertex_kernel<6>, VertexGeom<6>::NT, vertex_smem<6>());
        default: break;
    }
    const size_t smem = lattice_smem(A.nmp, A.ncell);
    auto launch = [&](auto kernel, int threads) -> vx_status {
        VX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        kernel<<<b->n, threads, smem, ctx->stream>>>(A);
        ctx->launches++;
        VX_CUDA(cudaGetLastError());
        return VX_OK;
    };
    switch (A.nmp) {
        case 64: return launch(lattice_kernel<64>, 64);
        case 128: return launch(lattice_kernel<128>, 128);
        case 160: return launch(lattice_kernel<160>, 160);
        case 224: return launch(lattice_kernel<224>, 224);
        case 256: return launch(lattice_kernel<256>, 256);
        case 352: return launch(lattice_kernel<352>, 352);
        case 384: return launch(lattice_kernel<384>, 384);
        case 512: return launch(lattice_kernel<512>, 512);
        default: return launch(lattice_kernel<544>, 544);
    }
}

}  // namespace vx
