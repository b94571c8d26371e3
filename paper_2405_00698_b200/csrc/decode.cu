// decode.cu — K1-K3 (decode) and K14 (genome sampling) on device.
//
// K1-K3 replace decode (morphology.hpp:141-157) over forward
// (genome.hpp:187-211), gaussian_encode (:169-179), affine (:118-126) and
// stable_sigmoid (:128-138) for a whole population:
//  * one CTA per genome keeps the genome's parameters resident in shared
//    memory (8710 FP64 = 68 KB for the default architecture) and sweeps the
//    robot's voxels in tiles of 32 (one voxel per lane);
//  * every affine keeps the reference's sequential order acc = b; acc +=
//    w*x (c ascending) with separately rounded mul/add (compiled --fmad=false),
//    so pre-activations are bit-identical given identical inputs; the
//    activations are stored [feature][voxel] so W rows are warp broadcasts and
//    activations are conflict-free;
//  * epilogue: softmax (first max, ordered sum), strict-> argmax (ties to the
//    lowest material), stable sigmoid + both clamps, and a guard counter for
//    voxels whose top-2 probability gap is < 1e-12 (where device vs glibc
//    transcendentals could flip the argmax — never observed).
// This exact-order kernel serves forward() point queries, VX_DECODE=exact, the
// fix-up of near-tie genomes and architectures too large for the tensor path;
// decode() runs decode_mma_kernel (below: the MLP layers on DMMA) first.
//
// K14 replaces sample_genome (genome.hpp:146-166): one warp per genome runs
// its own mt19937_64 (warp-parallel twist, smem state), W entries are exact
// uniform draws; B uses device log/cos (ulp-level vs glibc).
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "vx_internal.cuh"

namespace vx {

int64_t param_count(const vx_arch* a) {
    if (!a || a->m < 1 || a->n_hidden < 0 || a->n_hidden > VX_MAX_HIDDEN) return -1;
    int64_t n = 0;
    int64_t in = 2LL * a->m;
    for (int l = 0; l < a->n_hidden; ++l) {
        if (a->hidden[l] < 1) return -1;
        n += in * a->hidden[l] + a->hidden[l];
        in = a->hidden[l];
    }
    n += in * VX_NMAT + VX_NMAT;
    n += in + 1;
    return n;
}

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTile = 32;

struct DecodeArgs {
    int m, nh;
    int widths[VX_MAX_HIDDEN];
    int64_t np;
    int max_width;  // max(2m, hidden...)
    int w, h, d;
    const double* params;
    const double* bmat;
    const int32_t* select;
    uint8_t* mat;
    double* weight;
    uint32_t* guard;
    bool params_in_smem;
    int tile;  // voxels per tile (<= 32, one per lane of warp-wide rows; smaller for very wide networks)
    // forward() point queries instead of voxel centres (genome.hpp:187-211):
    // points [genome][n_points][3]; probs [genome][n_points][5] and the
    // unclamped weight head into `weight`
    const double* points;
    double* probs;
    int n_points;
    // fix-up launch after decode_mma_kernel: only CTAs whose flag is set run
    const uint8_t* fix_only;
};

__device__ __forceinline__ double stable_sigmoid(double z) {
    double s;
    if (z >= 0.0) {
        s = 1.0 / (1.0 + exp(-z));
    } else {
        const double e = exp(z);
        s = e / (1.0 + e);
    }
    if (s < 1e-12) s = 1e-12;
    if (s > 1.0 - 1e-12) s = 1.0 - 1e-12;
    return s;
}

__global__ void __launch_bounds__(kThreads) decode_kernel(DecodeArgs A) {
    if (A.fix_only && !A.fix_only[blockIdx.x]) return;
    const int g = A.select ? A.select[blockIdx.x] : static_cast<int>(blockIdx.x);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* sm = reinterpret_cast<double*>(smem_raw);
    const double* gp = A.params + static_cast<size_t>(g) * A.np;
    const double* P;
    if (A.params_in_smem) {
        double* sp = sm;
        for (int64_t q = threadIdx.x; q < A.np; q += kThreads) sp[q] = gp[q];
        P = sp;
        sm += A.np;
    } else {
        P = gp;
    }
    double* Bm = sm;  // 3m
    sm += 3 * A.m;
    const int T = A.tile;
    double* X = sm;  // [feature][T]
    double* Y = sm + static_cast<size_t>(A.max_width) * T;
    double* L = Y + static_cast<size_t>(A.max_width) * T;  // logits [6][T]
    for (int q = threadIdx.x; q < 3 * A.m; q += kThreads) Bm[q] = A.bmat[static_cast<size_t>(g) * 3 * A.m + q];
    __syncthreads();

    const int ncell = A.points ? A.n_points : A.w * A.h * A.d;
    const int m = A.m;
    const bool lane_in = lane < T;
    for (int t0 = 0; t0 < ncell; t0 += T) {
        const int cell = t0 + lane;
        const bool live = lane_in && cell < ncell;
        double v0 = 0.0, v1 = 0.0, v2 = 0.0;
        if (live && A.points) {
            const double* pt = A.points + (static_cast<size_t>(g) * ncell + cell) * 3;
            v0 = pt[0];
            v1 = pt[1];
            v2 = pt[2];
        } else if (live) {
            const int x = cell % A.w, y = (cell / A.w) % A.h, z = cell / (A.w * A.h);
            v0 = (x + 0.5) / A.w;  // morphology.hpp:147
            v1 = (y + 0.5) / A.h;
            v2 = (z + 0.5) / A.d;
        }
        // gaussian_encode (genome.hpp:169-179)
        for (int r = wid; r < m; r += kWarps) {
            const double phase = kTwoPi * (Bm[3 * r] * v0 + Bm[3 * r + 1] * v1 + Bm[3 * r + 2] * v2);
            double sn, cs;
            sincos(phase, &sn, &cs);
            if (lane_in) {
                X[r * T + lane] = cs;
                X[(m + r) * T + lane] = sn;
            }
        }
        __syncthreads();
        // hidden layers: affine (genome.hpp:118-126) + tanh (:192)
        int in = 2 * m;
        const double* lp = P;
        for (int l = 0; l < A.nh; ++l) {
            const int out = A.widths[l];
            const double* W = lp;
            const double* b = lp + static_cast<int64_t>(in) * out;
            for (int r = wid; r < out; r += kWarps) {
                const double* wr = W + static_cast<int64_t>(r) * in;
                double acc = b[r];
                if (!lane_in) continue;
                for (int c = 0; c < in; ++c) acc += wr[c] * X[c * T + lane];
                Y[r * T + lane] = tanh(acc);
            }
            __syncthreads();
            double* t = X;
            X = Y;
            Y = t;
            lp = b + out;
            in = out;
        }
        // heads: 5 material logits then 1 weight logit
        {
            const double* Wm = lp;
            const double* bm = lp + static_cast<int64_t>(in) * VX_NMAT;
            const double* Ww = bm + VX_NMAT;
            const double* bw = Ww + in;
            for (int r = wid; r < VX_NMAT + 1; r += kWarps) {
                const double* wr = r < VX_NMAT ? Wm + static_cast<int64_t>(r) * in : Ww;
                double acc = r < VX_NMAT ? bm[r] : bw[0];
                if (!lane_in) continue;
                for (int c = 0; c < in; ++c) acc += wr[c] * X[c * T + lane];
                L[r * T + lane] = acc;
            }
        }
        __syncthreads();
        if (wid == 0 && live) {
            double lg[VX_NMAT];
            for (int i = 0; i < VX_NMAT; ++i) lg[i] = L[i * T + lane];
            double mx = lg[0];  // std::max_element: first maximal
            for (int i = 1; i < VX_NMAT; ++i)
                if (mx < lg[i]) mx = lg[i];
            double p[VX_NMAT];
            double sum = 0.0;
            for (int i = 0; i < VX_NMAT; ++i) {
                p[i] = exp(lg[i] - mx);
                sum += p[i];
            }
            for (int i = 0; i < VX_NMAT; ++i) p[i] /= sum;
            const size_t o = static_cast<size_t>(g) * ncell + cell;
            const double wgt = stable_sigmoid(L[VX_NMAT * T + lane]);
            if (A.probs) {  // forward(): MaterialQuery{probs, weight}
                for (int i = 0; i < VX_NMAT; ++i) A.probs[o * VX_NMAT + i] = p[i];
                A.weight[o] = wgt;
            } else {  // decode(): argmax material, clamped weight
                int best = 0;
                for (int i = 1; i < VX_NMAT; ++i)
                    if (p[i] > p[best]) best = i;
                if (A.guard) {
                    double second = -1.0;
                    for (int i = 0; i < VX_NMAT; ++i)
                        if (i != best && p[i] > second) second = p[i];
                    if (p[best] - second < 1e-12 * p[best]) atomicAdd(A.guard, 1u);
                }
                A.mat[o] = static_cast<uint8_t>(best);
                A.weight[o] = wgt < kMinVoxelWeight ? kMinVoxelWeight : (wgt > 1.0 ? 1.0 : wgt);  // morphology.hpp:154
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------- K2 on the FP64 tensor pipe
// decode_mma_kernel: the same decode with every affine layer (genome.hpp:118-126)
// as a [voxels x in] x [in x out] product on DMMA (mma.sync m8n8k4 .f64 —
// tcgen05 has no f64 kind, so this is sm_100a's FP64 tensor path).
//  * weights are re-laid into shared memory in FRAGMENT order (layer, n-tile,
//    k-step, lane), zero-padded to 8-column / 4-deep tiles, so every B load is
//    one conflict-free 256 B wavefront pair; biases seed the accumulators;
//  * activations stay [feature][voxel] with a 36-double row stride (32 voxels
//    + 4): A loads and C stores hit every bank pair exactly twice;
//  * padded output columns come out exactly 0 (zero weights, zero bias,
//    tanh(0) = 0), which is the next layer's zero K padding.
// DMMA accumulates in a different order than the reference's sequential
// acc += w*x, so logits differ by ulps.  Materials are made bit-identical to
// the exact kernel BY CONSTRUCTION: a voxel whose top-2 probability gap is
// below kFixGap (orders of magnitude above any DMMA-vs-sequential logit
// difference) flags its genome, and decode_kernel re-decodes flagged genomes
// with the exact sequential order (a fix-up launch whose unflagged CTAs exit).
#ifndef VX_MMA_MT
#define VX_MMA_MT 4
#endif
constexpr int kMmaMT = VX_MMA_MT;             // m-tiles of 8 voxels per tile
constexpr int kMmaTile = kMmaMT * 8;         // 32 voxels per tile (default)
static_assert(kMmaTile <= kThreads && kMmaTile % 32 == 0, "one epilogue thread per voxel of a tile");
constexpr int kXS = kMmaTile + 4;            // activation row stride (doubles)
constexpr double kFixGap = 1e-8;             // relative top-2 gap that forces the exact path

struct MmaLayout {  // shared-memory offsets (doubles), host-computed
    int nl;                                  // nh hidden layers + 1 head
    int in[VX_MAX_HIDDEN + 1], out[VX_MAX_HIDDEN + 1];
    int64_t src_w[VX_MAX_HIDDEN + 1], src_b[VX_MAX_HIDDEN + 1];  // offsets into the genome
    int wf[VX_MAX_HIDDEN + 1], bias[VX_MAX_HIDDEN + 1];          // offsets in smem
    int total_w;                                                 // weights + biases (doubles)
    int rows;                                                    // activation rows (>= every padded width)
};

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// One warp: output n-tile `nt`, m-tiles [mt0, mt1) of the 32-voxel tile.
template <bool kTanh>
__device__ __forceinline__ void mma_tile(const double* __restrict__ WF, const double* __restrict__ bias,
                                         const double* __restrict__ X, double* __restrict__ Y, int KS, int nt,
                                         int mt0, int mt1, int lane) {
    double acc[kMmaMT][2];
    const double b0 = bias[nt * 8 + 2 * (lane & 3)], b1 = bias[nt * 8 + 2 * (lane & 3) + 1];
#pragma unroll
    for (int mt = 0; mt < kMmaMT; ++mt) {
        acc[mt][0] = b0;
        acc[mt][1] = b1;
    }
    const double* wf = WF + static_cast<size_t>(nt) * KS * 32 + lane;
    const double* xa = X + (lane & 3) * kXS + (lane >> 2);
    for (int ks = 0; ks < KS; ++ks) {
        const double b = wf[ks * 32];
#pragma unroll
        for (int mt = 0; mt < kMmaMT; ++mt)
            if (mt >= mt0 && mt < mt1) dmma884(acc[mt], xa[ks * 4 * kXS + mt * 8], b);
    }
#pragma unroll
    for (int mt = 0; mt < kMmaMT; ++mt) {
        if (mt < mt0 || mt >= mt1) continue;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int n = nt * 8 + 2 * (lane & 3) + i;
            Y[n * kXS + mt * 8 + (lane >> 2)] = kTanh ? tanh(acc[mt][i]) : acc[mt][i];
        }
    }
}

template <bool kTanh>
__device__ __forceinline__ void mma_layer(const double* WF, const double* bias, const double* X, double* Y, int in,
                                          int out, int wid, int lane, int rows_x, int rows_y) {
    const int NT = (out + 7) / 8, KS = (in + 3) / 4;
    VX_DCHECK(KS * 4 <= rows_x && NT * 8 <= rows_y);  // activation rows cover the padded K and N
    if (NT >= kWarps) {
        for (int nt = wid; nt < NT; nt += kWarps) mma_tile<kTanh>(WF, bias, X, Y, KS, nt, 0, kMmaMT, lane);
    } else {
        const int wpn = kWarps / NT;  // warps per n-tile split the m-tiles
        if (wid < NT * wpn) {
            const int nt = wid / wpn, part = wid % wpn;
            const int mt0 = part * kMmaMT / wpn, mt1 = (part + 1) * kMmaMT / wpn;
            if (mt0 < mt1) mma_tile<kTanh>(WF, bias, X, Y, KS, nt, mt0, mt1, lane);
        }
    }
}

__global__ void __launch_bounds__(kThreads) decode_mma_kernel(DecodeArgs A, MmaLayout Lo, uint8_t* fix) {
    const int g = A.select ? A.select[blockIdx.x] : static_cast<int>(blockIdx.x);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* sm = reinterpret_cast<double*>(smem_raw);
    const double* gp = A.params + static_cast<size_t>(g) * A.np;
    // weights in fragment order + padded biases
    for (int l = 0; l < Lo.nl; ++l) {
        const int in = Lo.in[l], out = Lo.out[l], KS = (in + 3) / 4, NT = (out + 7) / 8;
        const bool head = l == Lo.nl - 1;
        const int nfrag = NT * KS * 32;
        double* wf = sm + Lo.wf[l];
        for (int q = threadIdx.x; q < nfrag; q += kThreads) {
            const int ln = q & 31, ks = (q >> 5) % KS, nt = (q >> 5) / KS;
            const int n = nt * 8 + (ln >> 2), k = ks * 4 + (ln & 3);
            double v = 0.0;
            if (k < in && n < out) {
                // head: material rows 0..4 (Wm) then the weight row (Ww, after bm)
                const int64_t src = head && n == VX_NMAT ? Lo.src_w[l] + static_cast<int64_t>(VX_NMAT) * in + VX_NMAT + k
                                                         : Lo.src_w[l] + static_cast<int64_t>(n) * in + k;
                v = gp[src];
            }
            wf[q] = v;
        }
        double* bs = sm + Lo.bias[l];
        for (int n = threadIdx.x; n < NT * 8; n += kThreads) {
            double v = 0.0;
            if (n < out) v = head && n == VX_NMAT ? gp[Lo.src_b[l] + VX_NMAT + in] : gp[Lo.src_b[l] + n];
            bs[n] = v;
        }
    }
    double* Bm = sm + Lo.total_w;  // 3m
    double* X = Bm + 3 * A.m;      // [rows][kXS]
    double* Y = X + Lo.rows * kXS;
    double* L = Y + Lo.rows * kXS;  // logits [8][kXS]
    for (int q = threadIdx.x; q < 3 * A.m; q += kThreads) Bm[q] = A.bmat[static_cast<size_t>(g) * 3 * A.m + q];
    __syncthreads();

    const int ncell = A.w * A.h * A.d;
    const int m = A.m, in0 = 2 * m, in0p = ((in0 + 3) / 4) * 4;
    __shared__ int s_fix;
    if (threadIdx.x == 0) s_fix = 0;
    for (int t0 = 0; t0 < ncell; t0 += kMmaTile) {
        // gaussian_encode (genome.hpp:169-179) for 32 voxels; K padding zeroed
        for (int q = threadIdx.x; q < m * kMmaTile; q += kThreads) {
            const int r = q / kMmaTile, vx_ = q % kMmaTile, cell = t0 + vx_;
            double sn = 0.0, cs = 0.0;
            if (cell < ncell) {
                const int x = cell % A.w, y = (cell / A.w) % A.h, z = cell / (A.w * A.h);
                const double v0 = (x + 0.5) / A.w, v1 = (y + 0.5) / A.h, v2 = (z + 0.5) / A.d;  // morphology.hpp:147
                const double phase = kTwoPi * (Bm[3 * r] * v0 + Bm[3 * r + 1] * v1 + Bm[3 * r + 2] * v2);
                sincos(phase, &sn, &cs);
            }
            X[r * kXS + vx_] = cs;
            X[(m + r) * kXS + vx_] = sn;
        }
        for (int q = threadIdx.x; q < (in0p - in0) * kMmaTile; q += kThreads)
            X[(in0 + q / kMmaTile) * kXS + q % kMmaTile] = 0.0;
        __syncthreads();
        for (int l = 0; l + 1 < Lo.nl; ++l) {  // hidden: affine + tanh (genome.hpp:192)
            mma_layer<true>(sm + Lo.wf[l], sm + Lo.bias[l], X, Y, Lo.in[l], Lo.out[l], wid, lane, Lo.rows, Lo.rows);
            __syncthreads();
            double* t = X;
            X = Y;
            Y = t;
        }
        mma_layer<false>(sm + Lo.wf[Lo.nl - 1], sm + Lo.bias[Lo.nl - 1], X, L, Lo.in[Lo.nl - 1], VX_NMAT + 1, wid,
                         lane, Lo.rows, 8);
        __syncthreads();
        if (threadIdx.x < kMmaTile && t0 + static_cast<int>(threadIdx.x) < ncell) {
            const int vl = threadIdx.x, cell = t0 + vl;
            double lg[VX_NMAT];
            for (int i = 0; i < VX_NMAT; ++i) lg[i] = L[i * kXS + vl];
            double mx = lg[0];  // std::max_element: first maximal
            for (int i = 1; i < VX_NMAT; ++i)
                if (mx < lg[i]) mx = lg[i];
            double p[VX_NMAT];
            double sum = 0.0;
            for (int i = 0; i < VX_NMAT; ++i) {
                p[i] = exp(lg[i] - mx);
                sum += p[i];
            }
            for (int i = 0; i < VX_NMAT; ++i) p[i] /= sum;
            int best = 0;
            for (int i = 1; i < VX_NMAT; ++i)
                if (p[i] > p[best]) best = i;
            double second = -1.0;
            for (int i = 0; i < VX_NMAT; ++i)
                if (i != best && p[i] > second) second = p[i];
            if (p[best] - second < kFixGap * p[best]) s_fix = 1;
            const size_t o = static_cast<size_t>(g) * ncell + cell;
            const double wgt = stable_sigmoid(L[VX_NMAT * kXS + vl]);
            A.mat[o] = static_cast<uint8_t>(best);
            A.weight[o] = wgt < kMinVoxelWeight ? kMinVoxelWeight : (wgt > 1.0 ? 1.0 : wgt);  // morphology.hpp:154
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) fix[blockIdx.x] = s_fix ? 1 : 0;  // the tile loop ends with a barrier
}

// ------------------------------------------------------------ K14: mt19937_64
constexpr int kMtN = 312, kMtM = 156;
constexpr int kSampleWarps = 4;  // 4 x 7.3 KB of mt19937_64 state per CTA
constexpr uint64_t kUM = 0xFFFFFFFF80000000ULL, kLM = 0x7FFFFFFFULL, kMatA = 0xB5026F5AA96619E9ULL;

__device__ __forceinline__ uint64_t mt_mix(uint64_t cur, uint64_t nxt, uint64_t far) {
    const uint64_t y = (cur & kUM) | (nxt & kLM);
    return far ^ (y >> 1) ^ ((y & 1ULL) ? kMatA : 0ULL);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

// Warp-parallel twist: old state in A, new state written to B (2 phases + tail).
__device__ void warp_twist(const uint64_t* A, uint64_t* B, int lane) {
    for (int i = lane; i < kMtN - kMtM; i += 32) B[i] = mt_mix(A[i], A[i + 1], A[i + kMtM]);
    __syncwarp();
    for (int i = kMtN - kMtM + lane; i < kMtN - 1; i += 32) B[i] = mt_mix(A[i], A[i + 1], B[i - (kMtN - kMtM)]);
    __syncwarp();
    if (lane == 0) B[kMtN - 1] = mt_mix(A[kMtN - 1], B[0], B[kMtM - 1]);
    __syncwarp();
}

struct SampleArgs {
    int m, nh;
    int widths[VX_MAX_HIDDEN];
    int64_t np;
    double sigma;
    int P;
    const uint64_t* seeds;
    double* params;
    double* bmat;
};

// One warp per genome.  Draw t of the genome stream is tempered word t % 312
// of twist t / 312 (the first twist happens before draw 0).
__global__ void __launch_bounds__(kSampleWarps * 32) sample_kernel(SampleArgs A) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = blockIdx.x * kSampleWarps + wid;
    __shared__ uint64_t s_state[kSampleWarps][2][kMtN];
    __shared__ uint64_t s_out[kSampleWarps][kMtN];
    if (g >= A.P) return;
    uint64_t* S0 = s_state[wid][0];
    uint64_t* S1 = s_state[wid][1];
    uint64_t* O = s_out[wid];
    double* params = A.params + static_cast<size_t>(g) * A.np;
    double* bmat = A.bmat + static_cast<size_t>(g) * 3 * A.m;
    // seeding (sequential recurrence, lane 0)
    if (lane == 0) {
        uint64_t x = A.seeds[g];
        S0[0] = x;
        for (int i = 1; i < kMtN; ++i) {
            x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
            S0[i] = x;
        }
    }
    __syncwarp();
    // zero biases; W filled from the stream below
    {
        int64_t off = 0;
        int in = 2 * A.m;
        for (int l = 0; l <= A.nh + 1; ++l) {
            const int out = l < A.nh ? A.widths[l] : (l == A.nh ? VX_NMAT : 1);
            off += static_cast<int64_t>(in) * out;
            for (int q = lane; q < out; q += 32) params[off + q] = 0.0;
            off += out;
            if (l < A.nh) in = out;
        }
    }
    const int64_t n_b_draws = 6LL * A.m;  // 3m normals, 2 draws each
    int64_t n_w = 0;
    {
        int in = 2 * A.m;
        for (int l = 0; l < A.nh; ++l) {
            n_w += static_cast<int64_t>(in) * A.widths[l];
            in = A.widths[l];
        }
        n_w += static_cast<int64_t>(in) * VX_NMAT + in;
    }
    const int64_t total = n_b_draws + n_w;
    uint64_t* cur = S0;
    uint64_t* nxt = S1;
    for (int64_t base = 0; base < total; base += kMtN) {
        warp_twist(cur, nxt, lane);
        uint64_t* t = cur;
        cur = nxt;
        nxt = t;
        for (int i = lane; i < kMtN; i += 32) O[i] = mt_temper(cur[i]);
        __syncwarp();
        for (int i = lane; i < kMtN; i += 32) {
            const int64_t dix = base + i;
            if (dix >= total) break;
            if (dix < n_b_draws) {
                if ((dix & 1) == 0) {  // Rng::normal (rng.hpp:26-30) on draws dix, dix+1
                    const double u1 = (static_cast<double>(O[i] >> 11) + 0.5) * 0x1.0p-53;
                    const double u2 = static_cast<double>(O[i + 1] >> 11) * 0x1.0p-53;
                    const double nrm = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
                    bmat[dix >> 1] = A.sigma * nrm;
                }
            } else {
                // uniform W entry: locate its tensor (init_layer, genome.hpp:106-115)
                int64_t q = dix - n_b_draws;
                int64_t off = 0;
                int in = 2 * A.m;
                for (int l = 0; l <= A.nh + 1; ++l) {
                    const int out = l < A.nh ? A.widths[l] : (l == A.nh ? VX_NMAT : 1);
                    const int64_t nw = static_cast<int64_t>(in) * out;
                    if (q < nw) {
                        const double limit = sqrt(6.0 / static_cast<double>(in + out));
                        const double u = static_cast<double>(O[i] >> 11) * 0x1.0p-53;
                        params[off + q] = (2.0 * u - 1.0) * limit;
                        break;
                    }
                    q -= nw;
                    off += nw + out;
                    if (l < A.nh) in = out;
                }
            }
        }
        __syncwarp();
    }
}

}  // namespace

vx_status launch_decode(vx_ctx* ctx, const vx_arch* a, int64_t np, int maxw, DecodeArgs& A, int n);

vx_status decode_dev(vx_ctx* ctx, const vx_arch* a, int P, const double* d_params, const double* d_bmat, int w, int h,
                     int d, uint8_t* d_mat, double* d_weight, uint32_t* d_guard, const int32_t* d_select,
                     int n_select) {
    const int64_t np = param_count(a);
    if (np < 0) return (set_error("invalid architecture"), VX_EINVAL);
    if (w < 1 || h < 1 || d < 1) return (set_error("decode: dims must be positive"), VX_EINVAL);
    const int n = d_select ? n_select : P;
    if (n <= 0) return VX_OK;
    DecodeArgs A{};
    A.m = a->m;
    A.nh = a->n_hidden;
    int maxw = 2 * a->m;
    for (int l = 0; l < a->n_hidden; ++l) {
        A.widths[l] = a->hidden[l];
        maxw = maxw > a->hidden[l] ? maxw : a->hidden[l];
    }
    A.np = np;
    A.max_width = maxw;
    A.w = w;
    A.h = h;
    A.d = d;
    A.params = d_params;
    A.bmat = d_bmat;
    A.select = d_select;
    A.mat = d_mat;
    A.weight = d_weight;
    A.guard = d_guard;
    return launch_decode(ctx, a, np, maxw, A, n);
}

vx_status forward_dev(vx_ctx* ctx, const vx_arch* a, int P, const double* d_params, const double* d_bmat,
                      int n_points, const double* d_points, double* d_probs, double* d_weight) {
    const int64_t np = param_count(a);
    if (np < 0) return (set_error("invalid architecture"), VX_EINVAL);
    if (P <= 0 || n_points <= 0) return VX_OK;
    DecodeArgs A{};
    A.m = a->m;
    A.nh = a->n_hidden;
    int maxw = 2 * a->m;
    for (int l = 0; l < a->n_hidden; ++l) {
        A.widths[l] = a->hidden[l];
        maxw = maxw > a->hidden[l] ? maxw : a->hidden[l];
    }
    A.np = np;
    A.max_width = maxw;
    A.params = d_params;
    A.bmat = d_bmat;
    A.points = d_points;
    A.probs = d_probs;
    A.n_points = n_points;
    A.weight = d_weight;
    return launch_decode(ctx, a, np, maxw, A, P);
}

// activation buffers of the exact kernel for a tile of `tile` voxels
static size_t exact_act_bytes(int maxw, int m, int tile) {
    return (2ull * maxw + VX_NMAT + 1) * tile * sizeof(double) + 3ull * m * sizeof(double);
}
// the widest voxel tile (32, 16, .., 1) whose activations fit shared memory; 0 if none
static int exact_tile(const vx_ctx* ctx, int maxw, int m) {
    for (int t = kTile; t >= 1; t /= 2)
        if (exact_act_bytes(maxw, m, t) + 1024 <= ctx->smem_optin) return t;
    return 0;
}

vx_status decode_feasible(vx_ctx* ctx, const vx_arch* a) {
    int maxw = 2 * a->m;
    for (int l = 0; l < a->n_hidden; ++l) maxw = maxw > a->hidden[l] ? maxw : a->hidden[l];
    if (exact_tile(ctx, maxw, a->m) == 0) return (set_error("decode: architecture too wide"), VX_EINVAL);
    return VX_OK;
}

// Tensor-pipe layout of the default decode (decode_mma_kernel); false when the
// architecture's weights do not fit shared memory next to the activations.
static bool mma_layout(const vx_ctx* ctx, const vx_arch* a, MmaLayout& Lo, size_t& smem) {
    Lo = MmaLayout{};
    Lo.nl = a->n_hidden + 1;
    int in = 2 * a->m, rows = ((2 * a->m + 3) / 4) * 4;
    int64_t src = 0;
    int off = 0;
    for (int l = 0; l < Lo.nl; ++l) {
        const bool head = l == a->n_hidden;
        const int out = head ? VX_NMAT + 1 : a->hidden[l];
        Lo.in[l] = in;
        Lo.out[l] = out;
        Lo.src_w[l] = src;
        Lo.src_b[l] = src + static_cast<int64_t>(head ? VX_NMAT : out) * in;
        const int NT = (out + 7) / 8, KS = (in + 3) / 4;
        Lo.wf[l] = off;
        off += NT * KS * 32;
        Lo.bias[l] = off;
        off += NT * 8;
        if (!head) {
            src += static_cast<int64_t>(in) * out + out;
            rows = rows > NT * 8 ? rows : NT * 8;
            in = out;
        }
    }
    Lo.total_w = off;
    Lo.rows = rows;
    smem = (static_cast<size_t>(off) + 3ull * a->m + (2ull * rows + 8) * kXS) * sizeof(double);
    return smem + 1024 <= ctx->smem_optin;
}

vx_status launch_decode(vx_ctx* ctx, const vx_arch* a, int64_t np, int maxw, DecodeArgs& A, int n) {
    // exact kernel: 32-voxel tiles with the genome in shared memory when it
    // fits, else the genome read from global memory, else narrower tiles
    // (very wide networks: the reference accepts any width)
    A.tile = exact_tile(ctx, maxw, a->m);
    if (A.tile == 0) return (set_error("decode: architecture too wide"), VX_EINVAL);
    const size_t act = exact_act_bytes(maxw, a->m, A.tile);
    size_t smem = act + static_cast<size_t>(np) * sizeof(double);
    A.params_in_smem = A.tile == kTile && smem + 1024 <= ctx->smem_optin;
    if (!A.params_in_smem) smem = act;
    // decode(): the MLP layers on the FP64 tensor pipe, exact re-decode of flagged
    // genomes; forward() point queries and VX_DECODE=exact keep the CUDA-core kernel
    std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
    if (ctx->timing && !A.points) {  // live decode timing (bench.py's decode roofline)
        if (ctx->event_pool.empty()) {
            VX_CUDA(cudaEventCreate(&ev.first));
            VX_CUDA(cudaEventCreate(&ev.second));
        } else {
            ev = ctx->event_pool.back();
            ctx->event_pool.pop_back();
        }
        VX_CUDA(cudaEventRecord(ev.first, ctx->stream));
        ctx->dec_voxels += static_cast<int64_t>(n) * A.w * A.h * A.d;
    }
    MmaLayout Lo;
    size_t smem_mma = 0;
    const char* mode = std::getenv("VX_DECODE");
    const bool exact = mode && std::strcmp(mode, "exact") == 0;
    if (!A.points && !exact && mma_layout(ctx, a, Lo, smem_mma)) {
        VX_TRY(ctx->decode_fix.alloc(static_cast<size_t>(n)));
        VX_CUDA(cudaFuncSetAttribute(decode_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem_mma)));
        decode_mma_kernel<<<n, kThreads, smem_mma, ctx->stream>>>(A, Lo, ctx->decode_fix.p);
        ctx->launches++;
        VX_CUDA(cudaGetLastError());
        A.fix_only = ctx->decode_fix.p;
        ctx->decode_fix_n = n;
    } else {
        ctx->decode_fix_n = -1;
    }
    VX_CUDA(cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    decode_kernel<<<n, kThreads, smem, ctx->stream>>>(A);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    if (ev.first) {
        VX_CUDA(cudaEventRecord(ev.second, ctx->stream));
        ctx->dec_pending.push_back(ev);
    }
    return VX_OK;
}

vx_status sample_genomes_dev(vx_ctx* ctx, const vx_arch* a, int P, const uint64_t* d_seeds, double* d_params,
                             double* d_bmat) {
    const int64_t np = param_count(a);
    if (np < 0) return (set_error("invalid architecture"), VX_EINVAL);
    if (!(a->sigma > 0.0)) return (set_error("EncodingSpec: sigma must be > 0"), VX_EINVAL);
    if (P <= 0) return VX_OK;
    SampleArgs A{};
    A.m = a->m;
    A.nh = a->n_hidden;
    for (int l = 0; l < a->n_hidden; ++l) A.widths[l] = a->hidden[l];
    A.np = np;
    A.sigma = a->sigma;
    A.P = P;
    A.seeds = d_seeds;
    A.params = d_params;
    A.bmat = d_bmat;
    sample_kernel<<<ceil_div(P, kSampleWarps), kSampleWarps * 32, 0, ctx->stream>>>(A);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

}  // namespace vx
