// diversity.cu — K12: population_diversity (evolution.hpp:89-105), bit-exact.
//
// The reference sums the pair terms t_ab = differ_ab / cells (a < b, in the
// population's order — after the stable sort in evolve_generation) one by one
// into a double and divides by the pair count.  Reproducing that rounding
// sequence needs every pair term in order, so:
//
//  * pack:   grids -> 4-bit cells, 12 per double (an integer < 2^48, exact in
//            FP64, so the exchange buffer's SUM all-reduce gathers the packed
//            grids of every rank's individuals: zeros elsewhere);
//  * unpack: into 3 material bit-planes of 32 cells per word, in population
//            (sorted) order;
//  * count:  differ_ab for a tile of 32 x 32 pairs per CTA (2 x 2 per thread),
//            planes staged in shared memory: a cell differs iff any plane
//            does, so 3 XOR/OR + one POPC per 32 cells; written to a
//            pair-ordered count array (chunks of row tiles);
//  * sum:    the ordered, correctly rounded sequential sum, in parallel.  While
//            the running sum s stays in one binade [2^e, 2^e+1) every partial
//            sum is a multiple of u = ulp(s), so RN(s + t) = s + u * rint(t / u)
//            EXACTLY unless t / u is a tie (x.5, where round-to-even looks at
//            s) — the rounding no longer depends on s.  A cooperative grid
//            scans windows of terms with integer prefix sums of rint(t / u);
//            the first term that would leave the binade (or is a tie) is found
//            with a grid-wide min, applied with one ordinary double addition
//            (s is known exactly there), and the scan restarts after it.  The
//            running sum crosses a binade ~log2(pairs) times, so almost every
//            window is a single parallel pass.  Result: the reference's double,
//            bit for bit, in O(P^2 cells / bandwidth) + O(pairs / throughput).
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "vx_internal.cuh"

namespace cg = cooperative_groups;

namespace vx {
namespace {

constexpr int kCellsPerWord = 12;  // 4 bits each: 48-bit integers, exact as doubles
constexpr int kTile = 32;          // pair tile: 32 x 32 rows
constexpr int kKW = 32;            // 32-cell words per staging step (1024 cells)
constexpr int kPlanes = 3;         // material bit-planes (materials 0..4)
constexpr int kSumThreads = 1024;
constexpr int kTermsPerThread = 8;
constexpr uint64_t kNone = ~0ull;

__global__ void pack_kernel(int n, const int32_t* __restrict__ sel, int cells, int W, const uint8_t* __restrict__ mat,
                            double* __restrict__ out) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= static_cast<int64_t>(n) * W) return;
    const int r = static_cast<int>(q / W), w = static_cast<int>(q % W);
    const int ind = sel ? sel[r] : r;
    const uint8_t* g = mat + static_cast<size_t>(ind) * cells;
    uint64_t v = 0;
    for (int k = 0; k < kCellsPerWord; ++k) {
        const int c = w * kCellsPerWord + k;
        if (c < cells) v |= static_cast<uint64_t>(g[c] & 0xF) << (4 * k);
    }
    out[static_cast<size_t>(ind) * W + w] = static_cast<double>(v);
}

// packed doubles (population order via perm) -> 3 bit-planes of 32 cells per
// u32 word: planes[r][p][w], bit k of plane p = bit p of cell 32w + k's material
__global__ void unpack_kernel(int P, int cells, int W48, int W32, const int32_t* __restrict__ perm,
                              const double* __restrict__ packed, uint32_t* __restrict__ planes) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= static_cast<int64_t>(P) * W32) return;
    const int r = static_cast<int>(q / W32), w = static_cast<int>(q % W32);
    const int ind = perm ? perm[r] : r;
    const double* src = packed + static_cast<size_t>(ind) * W48;
    uint32_t b0 = 0, b1 = 0, b2 = 0;
    for (int k = 0; k < 32; ++k) {
        const int c = w * 32 + k;
        if (c >= cells) break;
        const uint32_t m = static_cast<uint32_t>(static_cast<uint64_t>(src[c / kCellsPerWord]) >> (4 * (c % kCellsPerWord))) & 7u;
        b0 |= (m & 1u) << k;
        b1 |= ((m >> 1) & 1u) << k;
        b2 |= ((m >> 2) & 1u) << k;
    }
    uint32_t* dst = planes + static_cast<size_t>(r) * kPlanes * W32 + w;
    dst[0] = b0;
    dst[W32] = b1;
    dst[2 * W32] = b2;
}

// index of pair (a, b), a < b, in the reference's loop order
__device__ __host__ __forceinline__ int64_t pair_index(int64_t P, int64_t a, int64_t b) {
    return a * (2 * P - a - 1) / 2 + (b - a - 1);
}

// one CTA per (row tile ta, column tile tb >= ta), ta from ta0: 32 x 32
// pairs, 256 threads x 2 x 2 pairs in registers; a cell differs when any of
// its 3 material bit-planes differs: 3 LOP3 + POPC per 32 cells and pair
__global__ void __launch_bounds__(256) count_kernel(int P, int W32, const uint32_t* __restrict__ planes, int ta0,
                                                    int ntile, int64_t n_base, int64_t cap,
                                                    uint32_t* __restrict__ cnt) {
    int64_t rem = blockIdx.x;
    int ta = ta0;
    while (rem >= ntile - ta) {
        rem -= ntile - ta;
        ++ta;
    }
    const int tb = ta + static_cast<int>(rem);
    __shared__ uint32_t sA[kPlanes * kKW][kTile + 1];
    __shared__ uint32_t sB[kPlanes * kKW][kTile + 1];
    const int ti = threadIdx.x >> 4, tj = threadIdx.x & 15;
    uint32_t c00 = 0, c01 = 0, c10 = 0, c11 = 0;
    for (int k0 = 0; k0 < W32; k0 += kKW) {
        const int kn = min(kKW, W32 - k0);
        for (int q = threadIdx.x; q < kTile * kPlanes * kKW; q += 256) {
            const int k = q % kKW, pr = q / kKW, pl = pr % kPlanes, row = pr / kPlanes;
            const int ra = ta * kTile + row, rb = tb * kTile + row;
            const bool ok = k < kn;
            sA[pl * kKW + k][row] = (ok && ra < P) ? planes[(static_cast<size_t>(ra) * kPlanes + pl) * W32 + k0 + k] : 0u;
            sB[pl * kKW + k][row] = (ok && rb < P) ? planes[(static_cast<size_t>(rb) * kPlanes + pl) * W32 + k0 + k] : 0u;
        }
        __syncthreads();
        for (int k = 0; k < kn; ++k) {
            const uint32_t a00 = sA[k][ti], a01 = sA[kKW + k][ti], a02 = sA[2 * kKW + k][ti];
            const uint32_t a10 = sA[k][ti + 16], a11 = sA[kKW + k][ti + 16], a12 = sA[2 * kKW + k][ti + 16];
            const uint32_t b00 = sB[k][tj], b01 = sB[kKW + k][tj], b02 = sB[2 * kKW + k][tj];
            const uint32_t b10 = sB[k][tj + 16], b11 = sB[kKW + k][tj + 16], b12 = sB[2 * kKW + k][tj + 16];
            c00 += __popc((a00 ^ b00) | (a01 ^ b01) | (a02 ^ b02));
            c01 += __popc((a00 ^ b10) | (a01 ^ b11) | (a02 ^ b12));
            c10 += __popc((a10 ^ b00) | (a11 ^ b01) | (a12 ^ b02));
            c11 += __popc((a10 ^ b10) | (a11 ^ b11) | (a12 ^ b12));
        }
        __syncthreads();
    }
    const int a0 = ta * kTile + ti, b0 = tb * kTile + tj;
    auto put = [&](int a, int b, uint32_t v) {
        if (a < b && b < P) {
            VX_DCHECK(pair_index(P, a, b) >= n_base && pair_index(P, a, b) - n_base < cap);
            cnt[pair_index(P, a, b) - n_base] = v;
        }
    };
    put(a0, b0, c00);
    put(a0, b0 + 16, c01);
    put(a0 + 16, b0, c10);
    put(a0 + 16, b0 + 16, c11);
}

struct SumScratch {
    double s;              // running sum (in/out across chunks)
    uint64_t first[2];     // grid-wide first stop index of the window (by window parity)
    uint64_t before_first; // integer prefix (units of u) before that term
    uint64_t tot[1];       // per-CTA window totals (gridDim.x entries)
};

// The running sum over n_terms counts (the chunk), in order, starting from
// scratch->s.  Cooperative launch, one 1024-thread CTA per SM.
__global__ void __launch_bounds__(kSumThreads) ordered_sum_kernel(int64_t n_terms, const uint32_t* __restrict__ cnt,
                                                                  double cells_d, SumScratch* sc) {
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int G = gridDim.x;
    const int64_t per_cta = static_cast<int64_t>(kSumThreads) * kTermsPerThread;
    const int64_t T = per_cta * G;
    __shared__ uint64_t s_warp[kSumThreads / 32];
    __shared__ uint64_t s_first;
    __shared__ uint64_t s_cta_off, s_total;
    volatile double* vs = &sc->s;
    double s = *vs;
    int64_t base = 0;
    int parity = 0;
    if (blockIdx.x == 0 && tid == 0) sc->first[0] = sc->first[1] = kNone;
    grid.sync();
    while (base < n_terms) {
        // this thread's terms: base + blockIdx * per_cta + tid * K + k
        const int64_t n0 = base + blockIdx.x * per_cta + static_cast<int64_t>(tid) * kTermsPerThread;
        double t[kTermsPerThread];
#pragma unroll
        for (int k = 0; k < kTermsPerThread; ++k) {
            const int64_t n = n0 + k;
            t[k] = n < n_terms ? static_cast<double>(cnt[n]) / cells_d : 0.0;  // evolution.hpp:100
        }
        if (tid == 0) s_first = kNone;
        uint64_t local_first = kNone;
        if (s == 0.0) {  // 0 + t = t exactly: the first nonzero term starts the sum
#pragma unroll
            for (int k = 0; k < kTermsPerThread; ++k)
                if (local_first == kNone && t[k] != 0.0 && n0 + k < n_terms) local_first = static_cast<uint64_t>(n0 + k);
            __syncthreads();
            if (local_first != kNone) atomicMin(reinterpret_cast<unsigned long long*>(&s_first), local_first);
            __syncthreads();
            if (tid == 0 && s_first != kNone)
                atomicMin(reinterpret_cast<unsigned long long*>(&sc->first[parity]), s_first);
            grid.sync();
            const uint64_t j = sc->first[parity];
            grid.sync();  // everyone read it before it is reset for the window after next
            if (blockIdx.x == 0 && tid == 0) sc->first[parity] = kNone;
            parity ^= 1;
            if (j == kNone) {
                base += T;
            } else {
                s = static_cast<double>(cnt[j]) / cells_d;
                base = static_cast<int64_t>(j) + 1;
            }
            continue;
        }
        int ex;
        frexp(s, &ex);                          // s = m 2^ex, m in [0.5, 1): binade 2^(ex-1)
        const double inv_u = ldexp(1.0, 53 - ex);  // 1 / ulp(s)
        const double u = ldexp(1.0, ex - 53);
        const uint64_t S = static_cast<uint64_t>(s * inv_u);  // in [2^52, 2^53)
        const double two53 = 9007199254740992.0;
        uint64_t r[kTermsPerThread];
        uint64_t mine = 0;
#pragma unroll
        for (int k = 0; k < kTermsPerThread; ++k) {
            const double q = t[k] * inv_u;  // exact: a power-of-two scaling
            const double rq = q < two53 ? rint(q) : two53;
            r[k] = static_cast<uint64_t>(rq);
            mine += r[k];
        }
        // CTA exclusive scan of the per-thread sums (wrapping uint64: only
        // prefixes before the first stop are ever used, and those are < 2^53)
        uint64_t incl = mine;
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) s_warp[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            uint64_t w = s_warp[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t v = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += v;
            }
            s_warp[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        const uint64_t thread_excl = (wid ? s_warp[wid - 1] : 0ull) + incl - mine;
        if (tid == 0) sc->tot[blockIdx.x] = s_warp[31];
        grid.sync();
        if (tid < 32) {  // this CTA's offset in the window and the window total
            uint64_t off = 0, tot = 0;
            for (int c = lane; c < G; c += 32) {
                const uint64_t v = *reinterpret_cast<volatile uint64_t*>(&sc->tot[c]);
                tot += v;
                if (c < static_cast<int>(blockIdx.x)) off += v;
            }
            for (int o = 16; o > 0; o >>= 1) {
                off += __shfl_xor_sync(0xffffffffu, off, o);
                tot += __shfl_xor_sync(0xffffffffu, tot, o);
            }
            if (lane == 0) {
                s_cta_off = off;
                s_total = tot;
            }
        }
        __syncthreads();
        // first term that leaves the binade (exact sum reaches 2^(ex)) or is a tie
        uint64_t before = S + s_cta_off + thread_excl;
#pragma unroll
        for (int k = 0; k < kTermsPerThread; ++k) {
            const int64_t n = n0 + k;
            if (n < n_terms && local_first == kNone) {
                const double room = two53 - static_cast<double>(before);  // exact: before < 2^53 here
                const double q = t[k] * inv_u;
                const bool tie = q - floor(q) == 0.5;
                if (q >= room || static_cast<double>(r[k]) >= room || tie) local_first = static_cast<uint64_t>(n);
                before += r[k];
            }
        }
        if (local_first != kNone) atomicMin(reinterpret_cast<unsigned long long*>(&s_first), local_first);
        __syncthreads();
        if (tid == 0 && s_first != kNone) atomicMin(reinterpret_cast<unsigned long long*>(&sc->first[parity]), s_first);
        grid.sync();
        const uint64_t j = *reinterpret_cast<volatile uint64_t*>(&sc->first[parity]);
        if (j != kNone && local_first == j) {
            // the owner of the stop term publishes the prefix before it
            uint64_t b2 = S + s_cta_off + thread_excl;
            for (int k = 0; k < kTermsPerThread; ++k) {
                if (static_cast<uint64_t>(n0 + k) == j) break;
                b2 += r[k];
            }
            sc->before_first = b2;
        }
        grid.sync();
        if (blockIdx.x == 0 && tid == 0) sc->first[parity] = kNone;  // read by all before the sync above
        parity ^= 1;
        if (j == kNone) {
            s = static_cast<double>(S + s_total) * u;  // exact (<= 2^53 units)
            base += T;
        } else {
            const uint64_t b2 = *reinterpret_cast<volatile uint64_t*>(&sc->before_first);
            const double sj = static_cast<double>(b2) * u;          // the running sum before term j, exact
            s = sj + static_cast<double>(cnt[j]) / cells_d;           // the reference's addition, as is
            base = static_cast<int64_t>(j) + 1;
        }
        grid.sync();  // before_first / tot are rewritten next window
    }
    if (blockIdx.x == 0 && tid == 0) *vs = s;
}

__global__ void finish_div_kernel(const double* s, double pairs, double* out) { *out = *s / pairs; }  // :104

}  // namespace

int diversity_words(int cells) { return (cells + kCellsPerWord - 1) / kCellsPerWord; }

// grids of the listed individuals (or all P when sel is null) -> packed doubles
vx_status diversity_pack_dev(vx_ctx* ctx, int n, const int32_t* d_sel, int cells, const uint8_t* d_mat,
                             double* d_packed) {
    if (n <= 0 || cells <= 0) return VX_OK;
    const int W = diversity_words(cells);
    const int64_t total = static_cast<int64_t>(n) * W;
    pack_kernel<<<ceil_div(total, 256), 256, 0, ctx->stream>>>(n, d_sel, cells, W, d_mat, d_packed);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

// population_diversity of P packed grids taken in the order perm (rank ->
// packed row; null: row order) -> *d_out
vx_status diversity_exact_dev(vx_ctx* ctx, int P, int cells, const double* d_packed, const int32_t* d_perm,
                              double* d_out) {
    if (P < 2 || cells <= 0) {
        VX_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), ctx->stream));
        return VX_OK;
    }
    const int W48 = diversity_words(cells), W32 = (cells + 31) / 32;
    VX_TRY(ctx->div_words.alloc(static_cast<size_t>(P) * kPlanes * W32));
    unpack_kernel<<<ceil_div(static_cast<int64_t>(P) * W32, 256), 256, 0, ctx->stream>>>(P, cells, W48, W32, d_perm,
                                                                                        d_packed, ctx->div_words.p);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    // cooperative grid for the ordered sum: one CTA per SM
    if (ctx->div_coop_ctas < 0) {
        int per_sm = 0;
        VX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ordered_sum_kernel, kSumThreads, 0));
        ctx->div_coop_ctas = per_sm > 0 ? ctx->sm_count : 0;
    }
    if (ctx->div_coop_ctas == 0) return (set_error("diversity: ordered-sum kernel cannot be co-resident"), VX_ECUDA);
    const int G = ctx->div_coop_ctas;
    VX_TRY(ctx->div_scratch.alloc((sizeof(SumScratch) + G * sizeof(uint64_t) + 7) / 8));
    SumScratch* sc = reinterpret_cast<SumScratch*>(ctx->div_scratch.p);
    VX_CUDA(cudaMemsetAsync(sc, 0, sizeof(double), ctx->stream));  // s = 0
    // pair counts in chunks of whole row tiles, <= ~2^28 pairs each
    const int ntile = (P + kTile - 1) / kTile;
    int64_t max_chunk = int64_t{1} << 28;  // pairs per count chunk (u32 counts: 1 GB)
    if (const char* env = std::getenv("VX_DIV_CHUNK")) max_chunk = std::max<int64_t>(1, std::atoll(env));  // tests
    VX_TRY(ctx->div_counts.alloc(static_cast<size_t>(std::min<int64_t>(
        max_chunk + static_cast<int64_t>(kTile) * P, static_cast<int64_t>(P) * (P - 1) / 2))));
    const double cells_d = static_cast<double>(cells);
    for (int ta0 = 0; ta0 < ntile;) {
        // rows [ta0 * 32, ta1 * 32): as many row tiles as fit the chunk
        int ta1 = ta0;
        int64_t n_tiles_pairs = 0;
        const int64_t a_lo = static_cast<int64_t>(ta0) * kTile;
        while (ta1 < ntile) {
            const int64_t a_hi = std::min<int64_t>(P - 1, static_cast<int64_t>(ta1 + 1) * kTile);
            const int64_t np = pair_index(P, a_hi, a_hi + 1) - pair_index(P, a_lo, a_lo + 1);
            if (ta1 > ta0 && np > max_chunk) break;
            n_tiles_pairs += ntile - ta1;
            ++ta1;
        }
        const int64_t a_hi = std::min<int64_t>(P - 1, static_cast<int64_t>(ta1) * kTile);
        const int64_t n_base = pair_index(P, a_lo, a_lo + 1);
        const int64_t n_terms = pair_index(P, a_hi, a_hi + 1) - n_base;
        VX_DCHECK_HOST(n_terms <= static_cast<int64_t>(ctx->div_counts.n));
        count_kernel<<<static_cast<unsigned>(n_tiles_pairs), 256, 0, ctx->stream>>>(
            P, W32, ctx->div_words.p, ta0, ntile, n_base, static_cast<int64_t>(ctx->div_counts.n), ctx->div_counts.p);
        ctx->launches++;
        VX_CUDA(cudaGetLastError());
        if (n_terms > 0) {
            const uint32_t* cp = ctx->div_counts.p;
            int64_t nt = n_terms;
            void* args[] = {&nt, &cp, const_cast<double*>(&cells_d), &sc};
            VX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(ordered_sum_kernel), dim3(G), dim3(kSumThreads),
                                                args, 0, ctx->stream));
            ctx->launches++;
        }
        ta0 = ta1;
    }
    const double pairs = static_cast<double>(static_cast<int64_t>(P) * (P - 1) / 2);
    finish_div_kernel<<<1, 1, 0, ctx->stream>>>(&sc->s, pairs, d_out);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

}  // namespace vx
