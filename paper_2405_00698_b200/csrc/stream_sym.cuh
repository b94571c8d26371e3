// stream_sym.cuh — the symmetric vertex-indexed streaming integrator
// (stream_sym_kernel<N>, one robot per CTA, parameters and state in a
// per-robot HBM scratch) and its persistent one-SM form stream_sym_filler<N>.
// Shared by integrator_stream.cu (20^3 robots, and 10^3 under
// VX_INTEGRATOR=stream) and integrator_cluster.cu, whose persistent 10^3
// cluster kernel launches the filler from the device onto the SMs no 4-CTA
// cluster can use.  Compiled with --fmad=false.
#pragma once

#include "vx_cluster.cuh"
#include "vx_internal.cuh"

namespace vx {
namespace {

#ifndef VX_STREAM_THREADS
#define VX_STREAM_THREADS 1024
#endif
constexpr int kStreamThreads = VX_STREAM_THREADS;  // threads per robot: 1024 (64 registers) measured best
#ifndef VX_STREAM_CHUNK
#define VX_STREAM_CHUNK 2
#endif
constexpr int kStreamChunk = VX_STREAM_CHUNK;      // springs evaluated together: 2 measured best at 1024 threads

template <typename T>
__device__ __forceinline__ T* at(unsigned char* base, size_t off) {
    return reinterpret_cast<T*>(base + off);
}

// ---------------------------------------------------------------------------
// stream_sym_kernel<N>: SYMMETRIC vertex-indexed streaming integrator — each
// mass evaluates all of its springs itself in the reference's ascending
// spring-index order (backward d = 12..0: fx -= F_i(neighbour, key); forward
// d = 0..12: fx += F_i(key, neighbour)), so no force slots or partial sums
// are stored: per step it reads the per-slot parameters (k, rest0, voxel) of
// both sides — a forward slot is the neighbour's backward slot, at a
// compile-time key offset, so there is no dependent index load — and the
// double-buffered state.  One __syncthreads per step; a zero-length abort
// keeps X[k] (physics.hpp:205-207), a divergence keeps X[k+1] (:260-263).
template <int N, int TT = kStreamThreads>
struct SymGeom {
    static constexpr int VW = N + 1;
    static constexpr int NV = VW * VW * VW;
    static constexpr int T = TT;                      // keys per block (= computing threads)
    static constexpr int MPT = (NV + T - 1) / T;
    static constexpr int NVP = MPT * T;
    static constexpr int PAD = VW * VW + VW + 1;
    static constexpr int PC = (NVP + PAD + 7) / 8 * 8;  // parameter columns (forward reads reach key + PAD;
                                                         // rows 16-byte aligned for bulk copies)
    static constexpr int XS = PAD + NVP + PAD;        // state row stride: far entries on both sides
    // shared-memory state (the filler): rows cover the keys of warps that hold a vertex
    static constexpr int XSS = PAD + (NV + 31) / 32 * 32 + PAD;
    static constexpr int NCELL = N * N * N;
};

struct SymLayout {
    size_t per_robot, k, r0, vox, x0, x1, mc, mask, cph, sph, sa, amap;
};

// constexpr: the kernel folds every array of the per-robot scratch into one
// base register plus immediate offsets (ten 64-bit pointers would cost 20 of
// its 64 registers)
template <int N, int TT = kStreamThreads>
__host__ __device__ constexpr SymLayout sym_layout() {
    using G = SymGeom<N, TT>;
    SymLayout L{};
    size_t o = 0;
    auto take = [&o](size_t bytes) {
        const size_t at = o;
        o += (bytes + 255) / 256 * 256;
        return at;
    };
    L.k = take(13ull * G::PC * 8);
    L.r0 = take(13ull * G::PC * 8);
    L.vox = take(13ull * G::PC * 2);
    L.x0 = take(6ull * G::XS * 8);
    L.x1 = take(6ull * G::XS * 8);
    L.mc = take(3ull * G::NVP * 8);
    L.mask = take(G::NVP * 4ull);
    L.cph = take((G::NCELL + 1) * 8ull);
    L.sph = take((G::NCELL + 1) * 8ull);
    L.sa = take((G::NCELL + 1) * 8ull);
    L.amap = take((G::NCELL + 2) * 4ull);  // voxel -> actuator id, then [NCELL + 1] = table size
    L.per_robot = o;
    return L;
}

struct SymArgs {
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
    SymLayout L;
    double zero_len2;
    double zeta2, mu;
    int32_t* ntab_max;  // prep: max actuator-table size over the batch
};

// one robot's scratch (parameter columns, state, actuator tables) from the
// batch; the whole CTA (1024 threads) takes part
template <int N, int TT = kStreamThreads>
__device__ void sym_prep_robot(const SymArgs& A, int r, unsigned char* base) {
    using G = SymGeom<N, TT>;
    constexpr int PCOL = G::PC, NVP = G::NVP, XS = G::XS, PAD = G::PAD, VW = G::VW;
    const BatchView& b = A.b;
    const SymLayout& L = A.L;
    double* K = at<double>(base, L.k);
    double* R0 = at<double>(base, L.r0);
    uint16_t* VOX = at<uint16_t>(base, L.vox);
    double* X0 = at<double>(base, L.x0);
    double* X1 = at<double>(base, L.x1);
    double* MC = at<double>(base, L.mc);
    uint32_t* MASK = at<uint32_t>(base, L.mask);
    double* CPH = at<double>(base, L.cph);
    double* SPH = at<double>(base, L.sph);
    double* SAG = at<double>(base, L.sa);
    int32_t* AMAP = at<int32_t>(base, L.amap);
    const int64_t mo = b.mass_off[r], so = b.spring_off[r];
    const int nm = b.nmass[r], ns = b.nspring[r];
    // compact actuator tables: only the voxels that actuate a spring get a
    // row (ids in voxel order), the last row is the passive sentinel (sin 0,
    // cos 1, amplitude 0: rest = r0 + (0 * r0) * D = r0).  The kernel keeps
    // the drive and amplitude tables in shared memory, and the smaller they
    // are the more of the SM's unified L1 serves the neighbour reads.
#ifndef VX_SYM_COMPACT
#define VX_SYM_COMPACT 1
#endif
    for (int v = threadIdx.x; v < G::NCELL; v += blockDim.x) AMAP[v] = VX_SYM_COMPACT ? 0 : 1;
    __syncthreads();
    for (int s = threadIdx.x; s < ns && VX_SYM_COMPACT; s += blockDim.x) {
        const int v = A.act_vox[so + s];
        if (v >= 0) AMAP[v] = 1;
    }
    __syncthreads();
    {  // exclusive scan of the flags over NCELL voxels, 1024 threads x contiguous runs
        __shared__ int s_cnt[1024];
        constexpr int RUN = (G::NCELL + 1023) / 1024;
        const int lo = threadIdx.x * RUN, hi = min(G::NCELL, lo + RUN);
        int c = 0;
        for (int v = lo; v < hi; ++v) c += AMAP[v];
        s_cnt[threadIdx.x] = c;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
            const int add = threadIdx.x >= o ? s_cnt[threadIdx.x - o] : 0;
            __syncthreads();
            s_cnt[threadIdx.x] += add;
            __syncthreads();
        }
        int id = s_cnt[threadIdx.x] - c;
        for (int v = lo; v < hi; ++v) {
            const int f = AMAP[v];
            AMAP[v] = f ? id : -1;
            id += f;
        }
        if (threadIdx.x == 1023) {
            AMAP[G::NCELL] = s_cnt[1023];           // sentinel id
            AMAP[G::NCELL + 1] = s_cnt[1023] + 1;   // table size
            if (A.ntab_max) atomicMax(A.ntab_max, s_cnt[1023] + 1);
        }
    }
    __syncthreads();
    const int sentinel = AMAP[G::NCELL];
    if (threadIdx.x == 0) {
        CPH[sentinel] = 1.0;
        SPH[sentinel] = 0.0;
        SAG[sentinel] = 0.0;
    }
    for (int k = threadIdx.x; k < PCOL; k += blockDim.x)
        for (int d = 0; d < 13; ++d) {
            K[d * PCOL + k] = 1.0;
            R0[d * PCOL + k] = 1.0;
            VOX[d * PCOL + k] = static_cast<uint16_t>(sentinel);
        }
    for (int k = threadIdx.x; k < NVP; k += blockDim.x) {
        MASK[k] = 0u;
        MC[k] = MC[NVP + k] = MC[2 * NVP + k] = 0.0;
    }
    for (int q = threadIdx.x; q < XS; q += blockDim.x)
        for (int c = 0; c < 6; ++c) X0[c * XS + q] = X1[c * XS + q] = c < 3 ? 1e3 : 0.0;
    __syncthreads();
    for (int s = threadIdx.x; s < ns; s += blockDim.x) {
        const int v = A.act_vox[so + s];
        if (v >= 0) {
            const int id = AMAP[v];
            CPH[id] = b.cosph[so + s];
            SPH[id] = b.sinph[so + s];
            SAG[id] = A.sign[so + s] * A.amp[so + s];  // sign * amplitude (physics.hpp:153)
        }
    }
    for (int m = threadIdx.x; m < nm; m += blockDim.x) {
        const int key = A.vkey[mo + m];
        for (int c = 0; c < 3; ++c) {
            X0[c * XS + PAD + key] = b.pos[c * b.M + mo + m];
            X0[(3 + c) * XS + PAD + key] = b.vel[c * b.M + mo + m];
        }
        const double mm = b.mass[mo + m];
        MC[key] = mm * A.sp.gravity;      // physics.hpp:226
        MC[NVP + key] = A.sp.dt / mm;     // physics.hpp:249
        MC[2 * NVP + key] = b.gdamp[mo + m];
        const int32_t* inc_off = b.inc_off + mo + r;
        const uint32_t* inc = b.inc + 2 * so;
        unsigned fmask = 0u, bmask = 0u;
        for (int e = inc_off[m]; e < inc_off[m + 1]; ++e) {
            const uint32_t iv = inc[e];
            const int sp = static_cast<int>(iv >> 1);
            const uint32_t ij = b.ij[so + sp];
            const int other = (iv & 1u) ? static_cast<int>(ij & 0xFFFFu) : static_cast<int>(ij >> 16);
            const int kb = A.vkey[mo + other];
            const int dx = kb % VW - key % VW, dy = (kb / VW) % VW - (key / VW) % VW,
                      dz = kb / (VW * VW) - key / (VW * VW);
            const int Lc = 9 * dz + 3 * dy + dx;
            const int d = (Lc > 0 ? Lc : -Lc) - 1;
            if (Lc < 0) {
                bmask |= 1u << d;
                K[d * PCOL + key] = b.k[so + sp];
                R0[d * PCOL + key] = b.rest0[so + sp];
                const int av = A.act_vox[so + sp];
                VOX[d * PCOL + key] = static_cast<uint16_t>(av >= 0 ? AMAP[av] : sentinel);
            } else {
                fmask |= 1u << d;
            }
        }
        MASK[key] = bmask | (fmask << 13) | (1u << 26);
    }
}

template <int N, int TT = kStreamThreads>
__global__ void __launch_bounds__(1024) stream_sym_prep_kernel(SymArgs A) {
    sym_prep_robot<N, TT>(A, blockIdx.x, A.scratch + static_cast<size_t>(blockIdx.x) * A.L.per_robot);
}

// The per-actuator drive table D is single-buffered (a second barrier per
// step rewrites it) unless VX_SYM_DBUF: shared memory taken by tables is L1
// the neighbour state / forward-slot reads do not get.
#ifndef VX_SYM_DBUF
#define VX_SYM_DBUF 0
#endif
constexpr int kSymDBuf = VX_SYM_DBUF ? 2 : 1;

// one robot's n_steps from its prepared scratch; kSmemX: the double-buffered
// state lives in shared memory (rows of XSS) instead of the HBM scratch
template <int N, bool kSmemX = false>
__device__ void sym_robot(const SymArgs& A, int r, unsigned char* base) {
    using G = SymGeom<N>;
    constexpr int PCOL = G::PC, NVP = G::NVP, XS = kSmemX ? G::XSS : G::XS, PAD = G::PAD, VW = G::VW, T = G::T,
                  MPT = G::MPT;
    constexpr int NV = G::NV;
    const BatchView& b = A.b;
    constexpr SymLayout L = sym_layout<N>();
    const int t = threadIdx.x;
    const int NT = at<int32_t>(base, L.amap)[G::NCELL + 1];  // this robot's actuator rows + sentinel
    const double* __restrict__ K = at<double>(base, L.k);
    const double* __restrict__ R0 = at<double>(base, L.r0);
    const uint16_t* __restrict__ VOX = at<uint16_t>(base, L.vox);
    const double* __restrict__ MC = at<double>(base, L.mc);
    const uint32_t* __restrict__ MASK = at<uint32_t>(base, L.mask);
    const double* SAG = at<double>(base, L.sa);
    const double* CPH = at<double>(base, L.cph);
    const double* SPH = at<double>(base, L.sph);
    double* Xc = at<double>(base, L.x0);
    double* Xn = at<double>(base, L.x1);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if constexpr (kSmemX) {  // both buffers from the prepared (far-initialised) HBM state
        double* S = reinterpret_cast<double*>(smem_raw);
        for (int q = t; q < 6 * XS; q += T) {
            const int c = q / XS, k = q - c * XS;
            S[q] = S[6 * XS + q] = Xc[c * G::XS + k];
        }
        Xc = S;
        Xn = S + 6 * XS;
        __syncthreads();
    }
    const int64_t mo = b.mass_off[r];
    const int nm = b.nmass[r];
    vx_summary* out = A.out ? A.out + r : nullptr;

    double* D = reinterpret_cast<double*>(smem_raw) + (kSmemX ? 12 * XS : 0);  // [kSymDBuf][NT] drive per actuator row
    double* SA = D + kSymDBuf * NT;                    // [NT]
    __shared__ double s_maxsq[32];

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
    {
        const double2 drv = __ldg(A.drive);
        for (int v = t; v < NT; v += T) {
            D[v] = drv.x * CPH[v] + drv.y * SPH[v];
            SA[v] = SAG[v];
        }
    }
    __syncthreads();
    auto com = [&](const double* X, double* o3) {
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
        o3[0] = c0;
        o3[1] = c1;
        o3[2] = c2;
    };
    double com_start[3];
    if (out && t == 0) com(Xc, com_start);

    const double dt = A.sp.dt;
    const double plane_k = A.sp.plane_k, mu_s = A.sp.mu_s, mu_k = A.sp.mu_k;
    double max_sq = 0.0;
    int64_t steps = 0, ok_phase1 = 0;
    int diverged = 0;
    for (int64_t kstep = 0; kstep < A.n_steps; ++kstep) {
        const double* Dc = D + (kSymDBuf == 2 ? (kstep & 1) * NT : 0);
        int zero_len = 0, bad = 0;
        double step_max = 0.0;
        for (int j = 0; j < MPT; ++j) {
            const int key = t + j * T;
            const unsigned msk = key < NV ? MASK[key] : 0u;
            if (__all_sync(0xffffffffu, !(msk >> 26))) continue;  // no mass in this warp's keys
            const double* Xk = Xc + PAD + key;
            const double x0 = Xk[0], x1 = Xk[XS], x2 = Xk[2 * XS];
            const double v0 = Xk[3 * XS], v1 = Xk[4 * XS], v2 = Xk[5 * XS];
            const unsigned bmask = msk & 0x1FFFu, fmask = (msk >> 13) & 0x1FFFu;
            double fx = 0.0, fy = 0.0, fz = 0.0;
            // spring_force_on_i (physics.hpp:55-64): F_i for the spring (i, j) with
            // i's state (xi, vi) and j's state at Xj
            auto force = [&](double xi0, double xi1, double xi2, double vi0, double vi1, double vi2, const double* Xj,
                             double kk, double r0, int vox, bool valid, double* f) {
                const double dx = Xj[0] - xi0;
                const double dy = Xj[XS] - xi1;
                const double dz = Xj[2 * XS] - xi2;
                const double len2 = dx * dx + dy * dy + dz * dz;
#ifdef VX_SYM_SPLIT_SQRT
                const double len = sqrt_rn_fast(len2);
                const double inv_len = rcp_rn_fast(len);
#else
                double len, inv_len;  // RN(sqrt) and RN(1/len) from one refined rsqrt
                sqrt_rcp_rn_fast(len2, len, inv_len);
#endif
                zero_len |= (valid && len2 < A.zero_len2) ? 1 : 0;
                const double rest = r0 + (SA[vox] * r0) * Dc[vox];
                const double nx = dx * inv_len, ny = dy * inv_len, nz = dz * inv_len;
                const double rel = (Xj[3 * XS] - vi0) * nx + (Xj[4 * XS] - vi1) * ny + (Xj[5 * XS] - vi2) * nz;
                const double cc = A.zeta2 * sqrt_rn_fast(kk * A.mu);  // damping_coefficient (physics.hpp:66-71)
                const double mag = kk * (len - rest) + cc * rel;
                f[0] = mag * nx;
                f[1] = mag * ny;
                f[2] = mag * nz;
            };
            // backward springs (i = key - off, j = key), d = 12..0: fx += (-1) * F_i
#pragma unroll
            for (int c0 = 12; c0 >= 0; c0 -= kStreamChunk) {
                double of[kStreamChunk][3];
#pragma unroll
                for (int q = 0; q < kStreamChunk; ++q) {
                    const int d = c0 - q;
                    if (d < 0) break;
                    const int off = key_off<VW>(d);
                    const double* Xi = Xk - off;
                    VX_DCHECK(PAD + key - off >= 0 && VOX[d * PCOL + key] < NT);
#ifdef VX_SYM_TIMING_NOPARAM  // timing-only bound (WRONG results): no per-slot parameter loads
                    force(Xi[0], Xi[XS], Xi[2 * XS], Xi[3 * XS], Xi[4 * XS], Xi[5 * XS], Xk, 1e4 + d, 0.1, NT - 1,
                          (bmask >> d) & 1u, of[q]);
#else
                    force(Xi[0], Xi[XS], Xi[2 * XS], Xi[3 * XS], Xi[4 * XS], Xi[5 * XS], Xk, K[d * PCOL + key],
                          R0[d * PCOL + key], VOX[d * PCOL + key], (bmask >> d) & 1u, of[q]);
#endif
                }
#pragma unroll
                for (int q = 0; q < kStreamChunk; ++q) {
                    const int d = c0 - q;
                    if (d < 0) break;
                    if ((bmask >> d) & 1u) {
                        fx -= of[q][0];
                        fy -= of[q][1];
                        fz -= of[q][2];
                    }
                }
            }
            // forward springs (i = key, j = key + off), d = 0..12: fx += F_i; the
            // parameters are the neighbour's backward slot d
#pragma unroll
            for (int c0 = 0; c0 <= 12; c0 += kStreamChunk) {
                double of[kStreamChunk][3];
#pragma unroll
                for (int q = 0; q < kStreamChunk; ++q) {
                    const int d = c0 + q;
                    if (d > 12) break;
                    const int off = key_off<VW>(d);
                    VX_DCHECK(key + off < PCOL && PAD + key + off < XS && VOX[d * PCOL + key + off] < NT);
#ifdef VX_SYM_TIMING_NOPARAM
                    force(x0, x1, x2, v0, v1, v2, Xk + off, 1e4 + d, 0.1, NT - 1, (fmask >> d) & 1u, of[q]);
#else
                    force(x0, x1, x2, v0, v1, v2, Xk + off, K[d * PCOL + key + off], R0[d * PCOL + key + off],
                          VOX[d * PCOL + key + off], (fmask >> d) & 1u, of[q]);
#endif
                }
#pragma unroll
                for (int q = 0; q < kStreamChunk; ++q) {
                    const int d = c0 + q;
                    if (d > 12) break;
                    if ((fmask >> d) & 1u) {
                        fx += of[q][0];
                        fy += of[q][1];
                        fz += of[q][2];
                    }
                }
            }
            if (!(msk >> 26)) continue;  // not a mass: nothing to integrate
            double px = x0, py = x1, pz = x2, vx = v0, vy = v1, vz = v2;
            if (A.sp.en_grav) fz -= MC[key];
            if (A.sp.en_contact && pz < 0.0) {
                const double penetration = -pz;
                double normal = plane_k * penetration - MC[2 * NVP + key] * vz;
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
            const double imdt = MC[NVP + key];
            vx += fx * imdt;
            vy += fy * imdt;
            vz += fz * imdt;
            px += vx * dt;
            py += vy * dt;
            pz += vz * dt;
            double* Xw = Xn + PAD + key;
            Xw[0] = px;
            Xw[XS] = py;
            Xw[2 * XS] = pz;
            Xw[3 * XS] = vx;
            Xw[4 * XS] = vy;
            Xw[5 * XS] = vz;
            const double speed_sq = vx * vx + vy * vy + vz * vz;
            if (speed_sq > step_max) step_max = speed_sq;
            if (!(fabs(px) <= kDivergenceBound) || !(fabs(py) <= kDivergenceBound) ||
                !(fabs(pz) <= kDivergenceBound))
                bad = 1;
        }
        if (kSymDBuf == 2 && kstep + 1 < A.n_steps) {  // next drive into the other buffer
            const double2 drv = __ldg(A.drive + kstep + 1);
            double* Dn = D + ((kstep + 1) & 1) * NT;
            for (int v = t; v < NT; v += T) Dn[v] = drv.x * CPH[v] + drv.y * SPH[v];
        }
#ifdef VX_SYM_TIMING_NOPARAM
        const int flags = __syncthreads_or(0) & 0 & (zero_len | bad);
#else
        const int flags = __syncthreads_or(zero_len | (bad << 1));
#endif
        if (kSymDBuf == 1 && !(flags & 3) && kstep + 1 < A.n_steps) {  // every read of D[k] is behind the barrier
            const double2 drv = __ldg(A.drive + kstep + 1);
            for (int v = t; v < NT; v += T) D[v] = drv.x * CPH[v] + drv.y * SPH[v];
            __syncthreads();
        }
        ++steps;
        if (flags & 1) {  // step() returned before touching any mass: keep X[k]
            diverged = 1;
            break;
        }
        ++ok_phase1;
        if (step_max > max_sq) max_sq = step_max;
        double* tmp = Xc;
        Xc = Xn;
        Xn = tmp;
        if (flags & 2) {
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
        for (int q = t; q < nm; q += T) {
            const int k = PAD + A.vkey[mo + q];
            for (int c = 0; c < 3; ++c) {
                b.pos[c * b.M + mo + q] = Xc[c * XS + k];
                b.vel[c * b.M + mo + q] = Xc[(3 + c) * XS + k];
            }
        }
    }
    if (t == 0 && out) {
        double m = 0.0;
        for (int w = 0; w < T / 32; ++w)
            if (s_maxsq[w] > m) m = s_maxsq[w];
        double com_end[3];
        com(Xc, com_end);
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

template <int N>
__global__ void __launch_bounds__(kStreamThreads, 1) stream_sym_kernel(SymArgs A) {
    sym_robot<N>(A, blockIdx.x, A.scratch + static_cast<size_t>(blockIdx.x) * A.L.per_robot);
}

// ---------------------------------------------------------------------------
// stream_sym_tma_kernel<N>: the symmetric streaming integrator with its
// per-slot parameters fed by a bulk-copy (TMA) pipeline.  Warp-specialised:
// 31 consumer warps own 992 keys per block (one key per thread, the order and
// arithmetic of sym_robot unchanged); one producer lane streams, for every
// (block, direction, backward|forward) stage, the block's K / rest0 / actuator
// row segments into a ring of kTmaNB shared-memory stages with
// cp.async.bulk + mbarrier complete_tx, running ahead across blocks and steps
// (the parameters never change during a launch).  Consumers wait on the
// stage's full barrier, copy the three values to registers, and release the
// slot on its empty barrier; the neighbour state is still read through L1.
// The timing-only bound with every parameter load removed was +49%
// (profiles/r02_stream_tma.md).
constexpr int kTmaT = 992;                 // consumer threads = keys per block (31 warps)
constexpr int kTmaWarps = kTmaT / 32;
constexpr int kTmaThreads = kTmaT + 32;    // + the producer warp
#ifndef VX_TMA_NB
#define VX_TMA_NB 4
#endif
constexpr int kTmaNB = VX_TMA_NB;          // stage ring depth (a power of two)
constexpr int kStageKeys = kTmaT + 8;      // a block's 992 keys, the segment start rounded down to 8
constexpr int kStageBytes = kStageKeys * (8 + 8 + 2);  // K, rest0, actuator row: 18000 B (16-byte multiple)
static_assert((kTmaNB & (kTmaNB - 1)) == 0 && kTmaT % 32 == 0 && kTmaT % 8 == 0, "stage ring");

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    return ok != 0;
}
// blocking wait: the warp is suspended in hardware (time hint) instead of spinning
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}
// OR of v over the 992 consumer threads (named barrier 1; the producer warp is not in it)
__device__ __forceinline__ int consumers_or(int v) {
    int r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.s32 p, %1, 0;\n\tbar.red.or.pred q, 1, %2, p;\n\tselp.s32 %0, 1, 0, q;\n\t}"
        : "=r"(r)
        : "r"(v), "n"(kTmaT)
        : "memory");
    return r;
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kTmaT) : "memory"); }

// stage i of a block (0..25): backward d = 12 - i for i < 13, forward d = i - 13
__host__ __device__ constexpr int stage_dir(int i) { return i < 13 ? 12 - i : i - 13; }

template <int N>
__device__ void sym_robot_tma(const SymArgs& A, int r, unsigned char* base) {
    using G = SymGeom<N, kTmaT>;
    constexpr int PCOL = G::PC, NVP = G::NVP, XS = G::XS, PAD = G::PAD, VW = G::VW, T = G::T, MPT = G::MPT;
    constexpr int NV = G::NV;
    constexpr SymLayout L = sym_layout<N, kTmaT>();
    const BatchView& b = A.b;
    const int t = threadIdx.x, wid = t >> 5, lane = t & 31;
    const bool producer = wid == kTmaWarps;
    const int NT = at<int32_t>(base, L.amap)[G::NCELL + 1];
    const double* __restrict__ MC = at<double>(base, L.mc);
    const uint32_t* __restrict__ MASK = at<uint32_t>(base, L.mask);
    const double* SAG = at<double>(base, L.sa);
    const double* CPH = at<double>(base, L.cph);
    const double* SPH = at<double>(base, L.sph);
    double* Xc = at<double>(base, L.x0);
    double* Xn = at<double>(base, L.x1);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* stages = smem_raw;                                       // [kTmaNB][kStageBytes]
    double* D = reinterpret_cast<double*>(smem_raw + kTmaNB * kStageBytes);  // [NT] drive per actuator row
    double* SA = D + NT;                                                     // [NT]
    __shared__ __align__(8) uint64_t s_full[kTmaNB], s_empty[kTmaNB];
    __shared__ double s_maxsq[32];
    __shared__ int s_stop;
    const int64_t mo = b.mass_off[r];
    const int nm = b.nmass[r];
    vx_summary* out = A.out ? A.out + r : nullptr;
    if (nm == 0) {  // uniform over the CTA: nothing issued yet
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
    const uint32_t full0 = smem_addr(&s_full[0]), empty0 = smem_addr(&s_empty[0]);
    if (t == 0) {
        for (int q = 0; q < kTmaNB; ++q) {
            mbar_init(full0 + 8u * q, 1u);
            mbar_init(empty0 + 8u * q, static_cast<uint32_t>(kTmaWarps));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_stop = 0;
    }
    if (!producer) {
        const double2 drv = __ldg(A.drive);
        for (int v = t; v < NT; v += T) {
            D[v] = drv.x * CPH[v] + drv.y * SPH[v];
            SA[v] = SAG[v];
        }
    }
    __syncthreads();

    if (producer) {
        // ------------------------------------------------------ producer lane
        if (lane == 0) {
            const unsigned char* gK = base + L.k;
            const unsigned char* gR = base + L.r0;
            const unsigned char* gV = base + L.vox;
            const uint32_t st0 = smem_addr(stages);
            const int64_t total = A.n_steps * MPT * 26;
            int64_t issued = 0;
            for (int64_t s = 0; s < total; ++s) {
                const int q = static_cast<int>(s & (kTmaNB - 1));
                const uint32_t use = static_cast<uint32_t>(s / kTmaNB);
                if (s >= kTmaNB) {  // the slot's previous stage consumed by every consumer warp
                    bool stop = false;
                    while (!mbar_try(empty0 + 8u * q, (use - 1u) & 1u))
                        if (*reinterpret_cast<volatile int*>(&s_stop)) {
                            stop = true;
                            break;
                        }
                    if (stop) break;
                }
                if (*reinterpret_cast<volatile int*>(&s_stop)) break;
                const int i = static_cast<int>(s % 26);
                const int j = static_cast<int>((s / 26) % MPT);
                const int d = stage_dir(i);
                const int off = i < 13 ? 0 : kOffDz(d) * VW * VW + kOffDy(d) * VW + kOffDx(d);
                const int k0 = (j * T + off) & ~7;
                int k1 = (j * T + T + off + 7) & ~7;
                if (k1 > PCOL) k1 = PCOL;
                const uint32_t nk = static_cast<uint32_t>(k1 - k0);
                VX_DCHECK(k0 >= 0 && k1 <= PCOL && nk <= static_cast<uint32_t>(kStageKeys) && nk % 8 == 0);
                const uint32_t dst = st0 + static_cast<uint32_t>(q) * kStageBytes;
                const uint32_t fb = full0 + 8u * q;
                mbar_expect_tx(fb, nk * 18u);
                const size_t col = static_cast<size_t>(d) * PCOL + k0;
                bulk_g2s(dst, gK + col * 8, nk * 8u, fb);
                bulk_g2s(dst + kStageKeys * 8u, gR + col * 8, nk * 8u, fb);
                bulk_g2s(dst + kStageKeys * 16u, gV + col * 2, nk * 2u, fb);
                issued = s + 1;
            }
            // no copy may still be in flight into this CTA's shared memory when it exits
            for (int64_t s = issued > kTmaNB ? issued - kTmaNB : 0; s < issued; ++s)
                mbar_wait(full0 + 8u * static_cast<uint32_t>(s & (kTmaNB - 1)),
                          static_cast<uint32_t>(s / kTmaNB) & 1u);
        }
        __syncwarp();
        __syncthreads();  // pairs with the consumers' final barrier
        return;
    }

    // ---------------------------------------------------------- consumers
    auto com = [&](const double* X, double* o3) {
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
        o3[0] = c0;
        o3[1] = c1;
        o3[2] = c2;
    };
    double com_start[3];
    if (out && t == 0) com(Xc, com_start);
    // stage s: wait until its copy landed, take the thread's three values, release the slot
    auto take = [&](int64_t s, int li, double& kk, double& r0, int& vox) {
        const int q = static_cast<int>(s & (kTmaNB - 1));
        mbar_wait(full0 + 8u * q, static_cast<uint32_t>(s / kTmaNB) & 1u);
        const unsigned char* st = stages + q * kStageBytes;
        VX_DCHECK(li >= 0 && li < kStageKeys);
        kk = reinterpret_cast<const double*>(st)[li];
        r0 = reinterpret_cast<const double*>(st + kStageKeys * 8)[li];
        vox = reinterpret_cast<const uint16_t*>(st + kStageKeys * 16)[li];
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8u * q);
    };
    auto skip = [&](int64_t s) {  // a stage this warp has no mass for: still consumed in order
        const int q = static_cast<int>(s & (kTmaNB - 1));
        mbar_wait(full0 + 8u * q, static_cast<uint32_t>(s / kTmaNB) & 1u);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8u * q);
    };

    const double dt = A.sp.dt;
    const double plane_k = A.sp.plane_k, mu_s = A.sp.mu_s, mu_k = A.sp.mu_k;
    double max_sq = 0.0;
    int64_t steps = 0, ok_phase1 = 0;
    int diverged = 0;
    for (int64_t kstep = 0; kstep < A.n_steps; ++kstep) {
        int zero_len = 0, bad = 0;
        double step_max = 0.0;
        for (int j = 0; j < MPT; ++j) {
            const int64_t s0 = (kstep * MPT + j) * 26;
            const int key = t + j * T;
            const unsigned msk = key < NV ? MASK[key] : 0u;
            if (__all_sync(0xffffffffu, !(msk >> 26))) {  // no mass in this warp's keys
                for (int i = 0; i < 26; ++i) skip(s0 + i);
                continue;
            }
            const double* Xk = Xc + PAD + key;
            const double x0 = Xk[0], x1 = Xk[XS], x2 = Xk[2 * XS];
            const double v0 = Xk[3 * XS], v1 = Xk[4 * XS], v2 = Xk[5 * XS];
            const unsigned bmask = msk & 0x1FFFu, fmask = (msk >> 13) & 0x1FFFu;
            double fx = 0.0, fy = 0.0, fz = 0.0;
            auto force = [&](double xi0, double xi1, double xi2, double vi0, double vi1, double vi2, const double* Xj,
                             double kk, double r0, int vox, bool valid, double* f) {  // physics.hpp:55-64
                const double dx = Xj[0] - xi0;
                const double dy = Xj[XS] - xi1;
                const double dz = Xj[2 * XS] - xi2;
                const double len2 = dx * dx + dy * dy + dz * dz;
                double len, inv_len;
                sqrt_rcp_rn_fast(len2, len, inv_len);
                zero_len |= (valid && len2 < A.zero_len2) ? 1 : 0;
                const double rest = r0 + (SA[vox] * r0) * D[vox];
                const double nx = dx * inv_len, ny = dy * inv_len, nz = dz * inv_len;
                const double rel = (Xj[3 * XS] - vi0) * nx + (Xj[4 * XS] - vi1) * ny + (Xj[5 * XS] - vi2) * nz;
                const double cc = A.zeta2 * sqrt_rn_fast(kk * A.mu);  // damping_coefficient (physics.hpp:66-71)
                const double mag = kk * (len - rest) + cc * rel;
                f[0] = mag * nx;
                f[1] = mag * ny;
                f[2] = mag * nz;
            };
            // backward springs, d = 12..0 (stages 0..12): fx += (-1) * F_i
#pragma unroll
            for (int c0 = 12; c0 >= 0; c0 -= 2) {
                double of[2][3], kk[2], r0[2];
                int vx_[2];
#pragma unroll
                for (int q = 0; q < 2; ++q)
                    if (c0 - q >= 0) take(s0 + 12 - (c0 - q), t, kk[q], r0[q], vx_[q]);
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int d = c0 - q;
                    if (d < 0) break;
                    const double* Xi = Xk - key_off<VW>(d);
                    force(Xi[0], Xi[XS], Xi[2 * XS], Xi[3 * XS], Xi[4 * XS], Xi[5 * XS], Xk, kk[q], r0[q], vx_[q],
                          (bmask >> d) & 1u, of[q]);
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int d = c0 - q;
                    if (d < 0) break;
                    if ((bmask >> d) & 1u) {
                        fx -= of[q][0];
                        fy -= of[q][1];
                        fz -= of[q][2];
                    }
                }
            }
            // forward springs, d = 0..12 (stages 13..25): the neighbour's backward slot
#pragma unroll
            for (int c0 = 0; c0 <= 12; c0 += 2) {
                double of[2][3], kk[2], r0[2];
                int vx_[2];
#pragma unroll
                for (int q = 0; q < 2; ++q)
                    if (c0 + q <= 12) take(s0 + 13 + c0 + q, t + (key_off<VW>(c0 + q) & 7), kk[q], r0[q], vx_[q]);
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int d = c0 + q;
                    if (d > 12) break;
                    force(x0, x1, x2, v0, v1, v2, Xk + key_off<VW>(d), kk[q], r0[q], vx_[q], (fmask >> d) & 1u, of[q]);
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int d = c0 + q;
                    if (d > 12) break;
                    if ((fmask >> d) & 1u) {
                        fx += of[q][0];
                        fy += of[q][1];
                        fz += of[q][2];
                    }
                }
            }
            if (!(msk >> 26)) continue;  // not a mass: nothing to integrate
            double px = x0, py = x1, pz = x2, vx = v0, vy = v1, vz = v2;
            if (A.sp.en_grav) fz -= MC[key];
            if (A.sp.en_contact && pz < 0.0) {
                const double penetration = -pz;
                double normal = plane_k * penetration - MC[2 * NVP + key] * vz;
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
            const double imdt = MC[NVP + key];
            vx += fx * imdt;
            vy += fy * imdt;
            vz += fz * imdt;
            px += vx * dt;
            py += vy * dt;
            pz += vz * dt;
            double* Xw = Xn + PAD + key;
            Xw[0] = px;
            Xw[XS] = py;
            Xw[2 * XS] = pz;
            Xw[3 * XS] = vx;
            Xw[4 * XS] = vy;
            Xw[5 * XS] = vz;
            const double speed_sq = vx * vx + vy * vy + vz * vz;
            if (speed_sq > step_max) step_max = speed_sq;
            if (!(fabs(px) <= kDivergenceBound) || !(fabs(py) <= kDivergenceBound) ||
                !(fabs(pz) <= kDivergenceBound))
                bad = 1;
        }
        int flags = 0;
        if (consumers_or(zero_len | bad)) flags = consumers_or(zero_len) | (consumers_or(bad) << 1);
        if (!(flags & 3) && kstep + 1 < A.n_steps) {  // every read of D[k] is behind the barrier
            const double2 drv = __ldg(A.drive + kstep + 1);
            for (int v = t; v < NT; v += T) D[v] = drv.x * CPH[v] + drv.y * SPH[v];
            consumers_sync();
        }
        ++steps;
        if (flags & 1) {  // step() returned before touching any mass: keep X[k]
            diverged = 1;
            break;
        }
        ++ok_phase1;
        if (step_max > max_sq) max_sq = step_max;
        double* tmp = Xc;
        Xc = Xn;
        Xn = tmp;
        if (flags & 2) {
            diverged = 1;
            break;
        }
    }
    if (t == 0) *reinterpret_cast<volatile int*>(&s_stop) = 1;  // the producer stops issuing and drains
    __syncthreads();                                           // pairs with the producer's

    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(0xffffffffu, max_sq, o);
        if (other > max_sq) max_sq = other;
    }
    if (lane == 0) s_maxsq[wid] = max_sq;
    consumers_sync();
    if (A.write_back) {
        for (int q = t; q < nm; q += T) {
            const int k = PAD + A.vkey[mo + q];
            for (int c = 0; c < 3; ++c) {
                b.pos[c * b.M + mo + q] = Xc[c * XS + k];
                b.vel[c * b.M + mo + q] = Xc[(3 + c) * XS + k];
            }
        }
    }
    if (t == 0 && out) {
        double m = 0.0;
        for (int w = 0; w < kTmaWarps; ++w)
            if (s_maxsq[w] > m) m = s_maxsq[w];
        double com_end[3];
        com(Xc, com_end);
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

template <int N>
__global__ void __launch_bounds__(kTmaThreads, 1) stream_sym_tma_kernel(SymArgs A) {
    sym_robot_tma<N>(A, blockIdx.x, A.scratch + static_cast<size_t>(blockIdx.x) * A.L.per_robot);
}

// dynamic shared memory of the filler: single- or double-buffered drive table
// plus the amplitude table, sized for any actuator count
// plus (VX_FILLER_SMEMX, default on) the double-buffered state
#ifndef VX_FILLER_SMEMX
#define VX_FILLER_SMEMX 1
#endif
constexpr bool kFillerSmemX = VX_FILLER_SMEMX != 0;
__host__ __device__ constexpr size_t sym_filler_smem() {
    return ((kFillerSmemX ? 12ull * SymGeom<10>::XSS : 0ull) + (kSymDBuf + 1ull) * (SymGeom<10>::NCELL + 1)) *
           sizeof(double);
}

// Persistent filler: robots claimed one at a time from the counter the
// persistent 10^3 cluster kernel also draws from (integrator_cluster.cu, which
// launches this grid from the device once every cluster is resident), each
// prepared into this CTA's own scratch slot and simulated; no new claims once
// `stop_at` robots are taken, so the slower one-SM robots do not stretch the
// tail.  claim[1] counts the robots it integrated, claim[6..9] (as u64) keep
// its first start / last end time for the VX_FILLER_STATS report.
template <int N>
__global__ void __launch_bounds__(kStreamThreads, 1) stream_sym_filler(SymArgs A, int32_t* claim, int n,
                                                                        int stop_at) {
    __shared__ int s_r;
    unsigned char* base = A.scratch + static_cast<size_t>(blockIdx.x) * A.L.per_robot;
    unsigned long long* tstat = reinterpret_cast<unsigned long long*>(claim + 4);
    if (threadIdx.x == 0) atomicMin(tstat + 3, globaltimer_ns());
    for (;;) {
        if (threadIdx.x == 0) {
            const int c = *reinterpret_cast<volatile int32_t*>(claim);
            s_r = c >= stop_at ? n : atomicAdd(claim, 1);
        }
        __syncthreads();
        const int r = s_r;
        __syncthreads();
        if (r >= n) break;
        if (threadIdx.x == 0) atomicAdd(claim + 1, 1);
        sym_prep_robot<N>(A, r, base);
        __syncthreads();
        sym_robot<N, kFillerSmemX>(A, r, base);
        __syncthreads();
    }
    if (threadIdx.x == 0) atomicMax(tstat + 4, globaltimer_ns());
}

}  // namespace
}  // namespace vx
