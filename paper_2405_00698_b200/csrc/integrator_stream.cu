// integrator_stream.cu — K7s: the streaming lattice integrator for large
// morphologies (10^3 and 20^3 grids: up to 9,261 masses and 108,860 springs
// per robot; SURVEY.md §2.2 row K7s, §8(d) "streaming (config 5)").
//
// Same algorithm and bit-exact results as integrator_lattice.cu (the higher
// endpoint of each lattice spring computes it during phase 1 for d = 12..0,
// accumulating the head of the reference's ascending-spring-index gather in
// order and storing the force once for the lower endpoint; phase 2 adds the
// forward terms d = 0..12, then gravity / contact / integrate), but a robot no
// longer fits on chip, so:
//  * per-slot parameters (k, rest0, c, amp_rest, neighbour|voxel) live in a
//    per-robot scratch in HBM laid out [direction][mass] (a warp reads 32
//    consecutive doubles: fully coalesced), built once per launch by
//    stream_prep_kernel from the CSR;
//  * force slots F[d][mass] and the phase-1 partial sums stream through L2;
//  * the mass state stays in shared memory when it fits (10^3: 64 KB), else
//    streams from L2/HBM too (20^3: 445 KB);
//  * each thread owns MPT masses (a fixed count, so all threads do equal work).
// Per spring update the kernel moves ~36 B of parameters + 24 B force store +
// 24 B force load (+ 48 B neighbour state when the state is off chip): it is
// L2/HBM-bandwidth bound by design (bench/scale numbers in profiles/).
// Compiled with --fmad=false.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "vx_internal.cuh"
#include "stream_sym.cuh"

namespace vx {
namespace {

struct StreamLayout {
    int nmp, mpt, threads;
    size_t per_robot;  // bytes
    // offsets (bytes) inside a robot's scratch
    size_t k, r0, f, s, mc, x, pnb, fnb, mask, cph, sph, sa;
};

StreamLayout stream_layout(int nm_cap, int ncell) {
    StreamLayout L{};
    L.mpt = (nm_cap + 1 + kStreamThreads - 1) / kStreamThreads;  // masses per thread (ghost included)
    L.nmp = (nm_cap + 1 + 32 * L.mpt - 1) / (32 * L.mpt) * (32 * L.mpt);
    L.threads = L.nmp / L.mpt;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o += (bytes + 255) / 256 * 256;
        return at;
    };
    const size_t n = static_cast<size_t>(L.nmp);
    L.k = take(13 * n * 8);
    L.r0 = take(13 * n * 8);
    L.f = take(39 * n * 8);
    L.s = take(3 * n * 8);
    L.mc = take(3 * n * 8);
    L.x = take(6 * n * 8);
    L.pnb = take(13 * n * 4);
    L.fnb = take(7 * n * 4);
    L.mask = take(n * 4);
    L.cph = take((ncell + 1) * 8ull);
    L.sph = take((ncell + 1) * 8ull);
    L.sa = take((ncell + 1) * 8ull);
    L.per_robot = o;
    return L;
}

struct StreamArgs {
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
    unsigned char* scratch;
    StreamLayout L;
    int vw, vh, ncell;
    double zero_len2;
    bool x_in_smem;
    double zeta2, mu;  // damping: c = (zeta*2) * sqrt(k * mu); built robots have uniform masses
};

// Builds the per-slot arrays of one robot from its CSR incidence lists.
__global__ void __launch_bounds__(1024) stream_prep_kernel(StreamArgs A) {
    const int r = blockIdx.x;
    const BatchView& b = A.b;
    const StreamLayout& L = A.L;
    const int NMP = L.nmp;
    unsigned char* base = A.scratch + static_cast<size_t>(r) * L.per_robot;
    double* K = at<double>(base, L.k);
    double* R0 = at<double>(base, L.r0);
    double* MC = at<double>(base, L.mc);
    double* XG = at<double>(base, L.x);
    double* F = at<double>(base, L.f);
    double* SAG = at<double>(base, L.sa);
    uint32_t* PNB = at<uint32_t>(base, L.pnb);
    uint32_t* FNB = at<uint32_t>(base, L.fnb);
    uint32_t* MASK = at<uint32_t>(base, L.mask);
    double* CPH = at<double>(base, L.cph);
    double* SPH = at<double>(base, L.sph);
    const int64_t mo = b.mass_off[r], so = b.spring_off[r];
    const int nm = b.nmass[r], ns = b.nspring[r];
    const int GH = NMP - 1;
    for (int v = threadIdx.x; v <= A.ncell; v += blockDim.x) {
        CPH[v] = 1.0;  // dummy passive voxel: D = sin(wt), amp_rest = 0
        SPH[v] = 0.0;
        SAG[v] = 0.0;
    }
    __syncthreads();
    for (int s = threadIdx.x; s < ns; s += blockDim.x) {
        const int v = A.act_vox[so + s];
        if (v >= 0) {
            CPH[v] = b.cosph[so + s];
            SPH[v] = b.sinph[so + s];
            SAG[v] = A.sign[so + s] * A.amp[so + s];  // sign * amplitude (physics.hpp:153)
        }
    }
    for (int a = threadIdx.x; a < NMP; a += blockDim.x) {
        for (int d = 0; d < 13; ++d) {
            K[d * NMP + a] = 1.0;  // missing spring: any normal value (its result is discarded)
            R0[d * NMP + a] = 1.0;
            PNB[d * NMP + a] = static_cast<uint32_t>(GH) | (static_cast<uint32_t>(A.ncell) << 14);
        }
        for (int q = 0; q < 7; ++q) FNB[q * NMP + a] = 0u;
        for (int row = 0; row < 39; ++row) F[row * NMP + a] = 0.0;
        unsigned fmask = 0u, bmask = 0u;
        if (a == GH) {  // ghost mass: far away, at rest
            for (int c = 0; c < 3; ++c) {
                XG[c * NMP + a] = 1e3;
                XG[(3 + c) * NMP + a] = 0.0;
            }
        } else if (a < nm) {
            for (int c = 0; c < 3; ++c) {
                XG[c * NMP + a] = b.pos[c * b.M + mo + a];
                XG[(3 + c) * NMP + a] = b.vel[c * b.M + mo + a];
            }
            const double m = b.mass[mo + a];
            MC[a] = m * A.sp.gravity;      // physics.hpp:226
            MC[NMP + a] = A.sp.dt / m;     // physics.hpp:249
            MC[2 * NMP + a] = b.gdamp[mo + a];
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
                const int Lc = 9 * dz + 3 * dy + dx;
                const int d = (Lc > 0 ? Lc : -Lc) - 1;
                if (Lc < 0) {  // spring (other, a): a is the higher endpoint
                    bmask |= 1u << d;
                    K[d * NMP + a] = b.k[so + s];
                    R0[d * NMP + a] = b.rest0[so + s];
                    const int av = A.act_vox[so + s];
                    PNB[d * NMP + a] = static_cast<uint32_t>(other) |
                                       (static_cast<uint32_t>(av >= 0 ? av : A.ncell) << 14);
                } else {
                    fmask |= 1u << d;
                    FNB[(d >> 1) * NMP + a] |= static_cast<uint32_t>(other) << (16 * (d & 1));
                }
            }
        }
        MASK[a] = fmask | (bmask << 13);
    }
}

template <bool kXSmem>
__global__ void __launch_bounds__(kStreamThreads, 1) stream_kernel(StreamArgs A) {
    const int r = blockIdx.x;
    const BatchView& b = A.b;
    const StreamLayout& L = A.L;
    const int NMP = L.nmp, T = L.threads, MPT = L.mpt;
    const int t = threadIdx.x;
    unsigned char* base = A.scratch + static_cast<size_t>(r) * L.per_robot;
    const double* K = at<double>(base, L.k);
    const double* R0 = at<double>(base, L.r0);
    const double* MC = at<double>(base, L.mc);
    const double* SAG = at<double>(base, L.sa);
    double* F = at<double>(base, L.f);
    double* S = at<double>(base, L.s);
    double* XG = at<double>(base, L.x);
    const uint32_t* PNB = at<uint32_t>(base, L.pnb);
    const uint32_t* FNB = at<uint32_t>(base, L.fnb);
    const uint32_t* MASK = at<uint32_t>(base, L.mask);
    const double* CPH = at<double>(base, L.cph);
    const double* SPH = at<double>(base, L.sph);
    const int64_t mo = b.mass_off[r];
    const int nm = b.nmass[r];
    vx_summary* out = A.out ? A.out + r : nullptr;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* D = reinterpret_cast<double*>(smem_raw);  // [ncell + 1] drive per voxel
    double* SA = D + A.ncell + 1;                      // [ncell + 1] sign*amplitude per voxel
    double* X = kXSmem ? SA + A.ncell + 1 : XG;        // [6][NMP]
    __shared__ double s_maxsq[32];
    __shared__ double s_com[3];

    if (nm == 0) {
        if (out && t == 0) {
            for (int c = 0; c < 3; ++c) out->com_start[c] = out->com_end[c] = 0.0;
            out->horizontal_displacement = 0.0;
            out->max_speed = 0.0;
            out->diverged = 0;
            out->steps = 0;
            out->spring_updates = 0;
        }
        return;
    }
    if (kXSmem)
        for (int q = t; q < 6 * NMP; q += T) X[q] = XG[q];
    {
        const double2 drv = __ldg(A.drive);
        for (int v = t; v <= A.ncell; v += T) {
            D[v] = drv.x * CPH[v] + drv.y * SPH[v];
            SA[v] = SAG[v];
        }
    }
    __syncthreads();
    // center_of_mass (physics.hpp:266-278), sequential in mass order
    auto com = [&](double* o3) {
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, total = 0.0;
        for (int a = 0; a < nm; ++a) {
            const double m = b.mass[mo + a];
            c0 += m * X[a];
            c1 += m * X[NMP + a];
            c2 += m * X[2 * NMP + a];
            total += m;
        }
        if (total > 0.0) {
            c0 /= total;
            c1 /= total;
            c2 /= total;
        }
        o3[0] = c0;
        o3[1] = c1;
        o3[2] = c2;
    };
    double com_start[3];
    if (out && t == 0) com(com_start);

    const double dt = A.sp.dt;
    const double plane_k = A.sp.plane_k, mu_s = A.sp.mu_s, mu_k = A.sp.mu_k;
    double max_sq = 0.0;
    int64_t steps = 0, ok_phase1 = 0;
    int diverged = 0;
    for (int64_t kstep = 0; kstep < A.n_steps; ++kstep) {
        // ---- phase 1: backward springs of every owned mass (d = 12..0)
        int zero_len = 0;
        for (int j = 0; j < MPT; ++j) {
            const int a = t + j * T;
            if (a >= nm) break;
            const double x0 = X[a], x1 = X[NMP + a], x2 = X[2 * NMP + a];
            const double v0 = X[3 * NMP + a], v1 = X[4 * NMP + a], v2 = X[5 * NMP + a];
            const unsigned bmask = MASK[a] >> 13;
            double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
            for (int c0 = 12; c0 >= 0; c0 -= kStreamChunk) {
                double ofx[kStreamChunk], ofy[kStreamChunk], ofz[kStreamChunk];
#pragma unroll
                for (int q = 0; q < kStreamChunk; ++q) {
                    const int d = c0 - q;
                    if (d < 0) break;
                    const bool valid = (bmask >> d) & 1u;
                    const uint32_t w = PNB[d * NMP + a];
                    const int nb = static_cast<int>(w & 0x3FFFu);
                    const int vox = static_cast<int>(w >> 14);
                    VX_DCHECK(nb < NMP && vox <= A.ncell);
                    const double dx = x0 - X[nb];
                    const double dy = x1 - X[NMP + nb];
                    const double dz = x2 - X[2 * NMP + nb];
                    const double len2 = dx * dx + dy * dy + dz * dz;
                    const double len = sqrt_rn_fast(len2);
                    zero_len |= (valid && len2 < A.zero_len2) ? 1 : 0;
                    // amp_rest = (sign*amplitude)*rest0 (physics.hpp:153); passive -> 0
                    const double r0 = R0[d * NMP + a];
                    const double rest = r0 + (SA[vox] * r0) * D[vox];
                    const double inv_len = rcp_rn_fast(len);
                    const double nx = dx * inv_len, ny = dy * inv_len, nz = dz * inv_len;
                    const double rel = (v0 - X[3 * NMP + nb]) * nx + (v1 - X[4 * NMP + nb]) * ny +
                                       (v2 - X[5 * NMP + nb]) * nz;
                    // damping_coefficient (physics.hpp:66-71) recomputed: FP64 is idle in this
                    // bandwidth-bound kernel, bytes are not (uniform masses: mu per robot)
                    const double kk = K[d * NMP + a];
                    const double cc = A.zeta2 * sqrt_rn_fast(kk * A.mu);
                    const double mag = kk * (len - rest) + cc * rel;
                    ofx[q] = mag * nx;
                    ofy[q] = mag * ny;
                    ofz[q] = mag * nz;
                }
#pragma unroll
                for (int q = 0; q < kStreamChunk; ++q) {
                    const int d = c0 - q;
                    if (d < 0) break;
                    if ((bmask >> d) & 1u) {
                        sx -= ofx[q];
                        sy -= ofy[q];
                        sz -= ofz[q];
                        F[(3 * d) * NMP + a] = ofx[q];
                        F[(3 * d + 1) * NMP + a] = ofy[q];
                        F[(3 * d + 2) * NMP + a] = ofz[q];
                    }
                }
            }
            S[a] = sx;
            S[NMP + a] = sy;
            S[2 * NMP + a] = sz;
        }
        ++steps;
        if (__syncthreads_or(zero_len)) {
            diverged = 1;
            break;
        }
        ++ok_phase1;
        // ---- phase 2: forward terms d = 0..12, then gravity / contact / integrate
        int bad = 0;
        for (int j = 0; j < MPT; ++j) {
            const int a = t + j * T;
            if (a >= nm) break;
            const unsigned fmask = MASK[a] & 0x1FFFu;
            double fx = S[a], fy = S[NMP + a], fz = S[2 * NMP + a];
#pragma unroll
            for (int d = 0; d < 13; ++d) {
                if (fmask & (1u << d)) {
                    const int nb = static_cast<int>((FNB[(d >> 1) * NMP + a] >> (16 * (d & 1))) & 0xFFFFu);
                    VX_DCHECK(nb < NMP);
                    fx += F[(3 * d) * NMP + nb];
                    fy += F[(3 * d + 1) * NMP + nb];
                    fz += F[(3 * d + 2) * NMP + nb];
                }
            }
            double px = X[a], py = X[NMP + a], pz = X[2 * NMP + a];
            double vx = X[3 * NMP + a], vy = X[4 * NMP + a], vz = X[5 * NMP + a];
            if (A.sp.en_grav) fz -= MC[a];
            if (A.sp.en_contact && pz < 0.0) {
                const double penetration = -pz;
                double normal = plane_k * penetration - MC[2 * NMP + a] * vz;
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
            const double imdt = MC[NMP + a];
            vx += fx * imdt;
            vy += fy * imdt;
            vz += fz * imdt;
            px += vx * dt;
            py += vy * dt;
            pz += vz * dt;
            X[a] = px;
            X[NMP + a] = py;
            X[2 * NMP + a] = pz;
            X[3 * NMP + a] = vx;
            X[4 * NMP + a] = vy;
            X[5 * NMP + a] = vz;
            const double speed_sq = vx * vx + vy * vy + vz * vz;
            if (speed_sq > max_sq) max_sq = speed_sq;
            if (!(fabs(px) <= kDivergenceBound) || !(fabs(py) <= kDivergenceBound) ||
                !(fabs(pz) <= kDivergenceBound))
                bad = 1;
        }
        if (kstep + 1 < A.n_steps) {
            const double2 drv = __ldg(A.drive + kstep + 1);
            for (int v = t; v <= A.ncell; v += T) D[v] = drv.x * CPH[v] + drv.y * SPH[v];
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
    if ((t & 31) == 0) s_maxsq[t >> 5] = max_sq;
    __syncthreads();
    if (A.write_back) {
        for (int a = t; a < nm; a += T)
            for (int c = 0; c < 3; ++c) {
                b.pos[c * b.M + mo + a] = X[c * NMP + a];
                b.vel[c * b.M + mo + a] = X[(3 + c) * NMP + a];
            }
    }
    if (t == 0 && out) {
        double m = 0.0;
        for (int w = 0; w < T / 32; ++w)
            if (s_maxsq[w] > m) m = s_maxsq[w];
        double com_end[3];
        com(com_end);
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
    (void)s_com;
}

template <int N>
vx_status launch_stream_sym(vx_ctx* ctx, vx_batch* b, const StreamArgs& S) {
    SymArgs A{};
    A.b = S.b;
    A.vkey = S.vkey;
    A.act_vox = S.act_vox;
    A.sign = S.sign;
    A.amp = S.amp;
    A.drive = S.drive;
    A.sp = S.sp;
    A.n_steps = S.n_steps;
    A.write_back = S.write_back;
    A.out = S.out;
    A.zero_len2 = S.zero_len2;
    A.zeta2 = S.zeta2;
    A.mu = S.mu;
    // VX_STREAM_TMA=1: the bulk-copy-fed kernel (when its stage ring + the
    // batch's actuator tables fit shared memory).  Correct, but 17% slower
    // than the L1-fed default: the ring couples the warps stage by stage
    // (profiles/r02_stream_tma.md)
    const char* tma_env = std::getenv("VX_STREAM_TMA");
    bool tma = tma_env && *tma_env == '1' && kSymDBuf == 1;
    int32_t ntab = 0;  // shared memory sized for the batch's largest actuator table
    for (int pass = 0; pass < 2; ++pass) {
        A.L = tma ? sym_layout<N, kTmaT>() : sym_layout<N>();
        VX_TRY(ctx->stream_scratch.alloc(A.L.per_robot * static_cast<size_t>(b->n)));
        A.scratch = ctx->stream_scratch.p;
        VX_TRY(ctx->stream_ntab.alloc(1));
        VX_CUDA(cudaMemsetAsync(ctx->stream_ntab.p, 0, sizeof(int32_t), ctx->stream));
        A.ntab_max = ctx->stream_ntab.p;
        if (tma)
            stream_sym_prep_kernel<N, kTmaT><<<b->n, 1024, 0, ctx->stream>>>(A);
        else
            stream_sym_prep_kernel<N><<<b->n, 1024, 0, ctx->stream>>>(A);
        ctx->launches++;
        VX_CUDA(cudaGetLastError());
        VX_CUDA(cudaMemcpyAsync(&ntab, ctx->stream_ntab.p, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        VX_CUDA(cudaStreamSynchronize(ctx->stream));
        if (!tma) break;
        const size_t smem_t = static_cast<size_t>(kTmaNB) * kStageBytes + 2ull * std::max(1, ntab) * sizeof(double);
        if (smem_t + 2048 > ctx->smem_optin) {  // tables too large for the ring: the L1-fed kernel
            tma = false;
            continue;
        }
        VX_CUDA(cudaFuncSetAttribute(stream_sym_tma_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem_t)));
        stream_sym_tma_kernel<N><<<b->n, kTmaThreads, smem_t, ctx->stream>>>(A);
        ctx->launches++;
        VX_CUDA(cudaGetLastError());
        return VX_OK;
    }
    const size_t smem = (kSymDBuf + 1ull) * std::max(1, ntab) * sizeof(double);
    VX_CUDA(cudaFuncSetAttribute(stream_sym_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    {  // the smallest shared-memory carveout that holds the tables: the rest of
       // the unified L1 serves the neighbour-state reads (default 5.20e10,
       // minimal carveout 5.30e10, maximal 4.1e10: profiles/README.md)
        const char* co = std::getenv("VX_STREAM_CARVEOUT");  // A/B: a fixed percentage
        const int pct = co ? std::atoi(co)
                           : std::min(100, static_cast<int>((100 * (smem + 4096) + ctx->smem_optin - 1) /
                                                            ctx->smem_optin) + 2);
        VX_CUDA(cudaFuncSetAttribute(stream_sym_kernel<N>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
    }
    stream_sym_kernel<N><<<b->n, kStreamThreads, smem, ctx->stream>>>(A);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

}  // namespace

bool stream_applicable(vx_ctx* ctx, vx_batch* b) {
    if (!b->lattice || !b->vkey.p || !b->act_vox.p || !(b->uniform_mass > 0.0)) return false;
    const int ncell = b->lw * b->lh * b->ld;
    if (ncell + 1 >= (1 << 18)) return false;  // voxel id packed in 18 bits
    if (b->nm_max + 1 > (1 << 14)) return false;  // neighbour packed in 14 bits
    return 2ull * (ncell + 1) * sizeof(double) + 1024 <= ctx->smem_optin;
}

vx_status integrate_stream(vx_ctx* ctx, vx_batch* b, int64_t n_steps, bool write_back, vx_summary* d_summaries,
                           const SimParams& sp, double zero_len2) {
    StreamArgs A{};
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
    A.vw = b->lw + 1;
    A.vh = b->lh + 1;
    A.ncell = b->lw * b->lh * b->ld;
    A.zero_len2 = zero_len2;
    A.zeta2 = b->uniform_zeta * 2.0;
    A.mu = b->uniform_mass * b->uniform_mass / (b->uniform_mass + b->uniform_mass);
    {  // 20^3 grids: the symmetric vertex-indexed kernel (measured 5.0e10 vs 3.7e10 for the
       // force-slot rank kernel below); VX_STREAM=rank forces the latter for A/B runs
        static const char* force = std::getenv("VX_STREAM");
        const bool rank_only = force && std::string(force) == "rank";
        if (!rank_only && b->lw == 20 && b->lh == 20 && b->ld == 20) return launch_stream_sym<20>(ctx, b, A);
        if (!rank_only && b->lw == 10 && b->lh == 10 && b->ld == 10) return launch_stream_sym<10>(ctx, b, A);
    }
    A.L = stream_layout(b->nm_max, A.ncell);
    VX_TRY(ctx->stream_scratch.alloc(A.L.per_robot * static_cast<size_t>(b->n)));
    A.scratch = ctx->stream_scratch.p;
    const size_t smem_d = 2ull * (A.ncell + 1) * sizeof(double);
    const size_t smem_x = 6ull * A.L.nmp * sizeof(double);
    A.x_in_smem = smem_d + smem_x + 2048 <= ctx->smem_optin;
    stream_prep_kernel<<<b->n, 1024, 0, ctx->stream>>>(A);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    auto launch = [&](auto kernel, size_t smem) -> vx_status {
        VX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        kernel<<<b->n, A.L.threads, smem, ctx->stream>>>(A);
        ctx->launches++;
        VX_CUDA(cudaGetLastError());
        return VX_OK;
    };
    if (A.x_in_smem) return launch(stream_kernel<true>, smem_d + smem_x);
    return launch(stream_kernel<false>, smem_d);
}

}  // namespace vx
