// ga.cu — K10-K13 on device: fitness gating, stable fitness sort, population
// statistics, diversity and the breeding gather/apply.
//
//  * gate_kernel / fitness_kernel: evaluate_fitness gates
//    (evolution.hpp:110-119): empty -> 0, no muscle -> 0 (and not simulated),
//    diverged -> 0, else horizontal displacement;
//  * sort: std::stable_sort by fitness descending (evolution.hpp:243-244) as
//    a CUB stable radix sort on the (non-negative, NaN-free) fitness keys;
//  * stats_kernel: best / mean / stddev with the reference's sequential sums
//    in sorted order (evolution.hpp:255-263) -> bit-identical;
//  * diversity: population_diversity (evolution.hpp:89-105) as per-cell
//    material histograms: sum_{a<b} differ_ab = sum_c [C(P,2) - sum_k C(n_ck,2)]
//    (exact integers, O(P*cells) instead of O(P^2*cells)); the final
//    division differs from the reference's pairwise running sum by rounding
//    only (<= 1e-15 relative);
//  * breed kernels: elites copied, children = crossover(sorted[pa],
//    sorted[pb], mask) then + mutation deltas (evolution.hpp:143-165,
//    267-289) from the host-parsed mt19937_64 plan (evo.cu).
#include <cub/cub.cuh>

#include "vx_internal.cuh"
#include "vx_ga.cuh"

namespace vx {
namespace {

constexpr int kThreads = 256;

// per-cell material counts over P grids: blocks tile (cell range x slice of
// the population), one integer atomic per (cell, material) and block
__global__ void hist_kernel(int P, int cells, const uint8_t* __restrict__ mat, int64_t* __restrict__ hist) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cells) return;
    const int per = (P + gridDim.y - 1) / gridDim.y;
    const int a0 = blockIdx.y * per, a1 = min(P, a0 + per);
    if (a0 >= a1) return;
    int n[VX_NMAT] = {0, 0, 0, 0, 0};
    for (int a = a0; a < a1; ++a) {
        const int m = mat[static_cast<size_t>(a) * cells + c];
        if (m < VX_NMAT) n[m] += 1;
    }
    for (int k = 0; k < VX_NMAT; ++k)
        if (n[k])
            atomicAdd(reinterpret_cast<unsigned long long*>(hist + c * VX_NMAT + k),
                      static_cast<unsigned long long>(n[k]));
}

// counts over a list of individuals (this rank's share), as doubles for the
// exchange-buffer all-reduce: blocks tile (cell range x slice of the list),
// each adds its slice's integer counts with one atomic per (cell, material)
// (exact and order-free: counts < 2^53); `out` is zeroed first
__global__ void hist_sel_kernel(int n, const int32_t* __restrict__ sel, int cells, const uint8_t* __restrict__ mat,
                                double* __restrict__ out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cells) return;
    const int per = (n + gridDim.y - 1) / gridDim.y;
    const int q0 = blockIdx.y * per, q1 = min(n, q0 + per);
    if (q0 >= q1) return;
    int cnt[VX_NMAT] = {0, 0, 0, 0, 0};
    for (int q = q0; q < q1; ++q) {
        const int m = mat[static_cast<size_t>(sel[q]) * cells + c];
        if (m < VX_NMAT) cnt[m] += 1;
    }
    for (int k = 0; k < VX_NMAT; ++k)
        if (cnt[k]) atomicAdd(out + c * VX_NMAT + k, static_cast<double>(cnt[k]));
}

__global__ void hist_from_doubles_kernel(int n, const double* __restrict__ in, int64_t* __restrict__ out) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < n) out[q] = static_cast<int64_t>(in[q]);
}

__global__ void diversity_kernel(int P, int cells, const int64_t* __restrict__ hist, double* out) {
    __shared__ unsigned long long s_tot;
    if (threadIdx.x == 0) s_tot = 0ull;
    __syncthreads();
    const unsigned long long pairs = static_cast<unsigned long long>(P) * (P - 1) / 2;
    unsigned long long local = 0;
    for (int c = threadIdx.x; c < cells; c += blockDim.x) {
        unsigned long long same = 0;
        for (int k = 0; k < VX_NMAT; ++k) {
            const unsigned long long n = static_cast<unsigned long long>(hist[c * VX_NMAT + k]);
            same += n * (n - (n > 0)) / 2;
        }
        local += pairs - same;
    }
    atomicAdd(&s_tot, local);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (P < 2 || cells == 0) {
            *out = 0.0;
        } else {
            *out = (static_cast<double>(s_tot) / static_cast<double>(cells)) / static_cast<double>(pairs);
        }
    }
}

}  // namespace

vx_status histogram_dev(vx_ctx* ctx, int P, int cells, const uint8_t* d_mat, int64_t* d_hist, bool accumulate) {
    if (cells <= 0) return VX_OK;
    if (!accumulate)
        VX_CUDA(cudaMemsetAsync(d_hist, 0, static_cast<size_t>(cells) * VX_NMAT * sizeof(int64_t), ctx->stream));
    if (P <= 0) return VX_OK;
    const int bx = ceil_div(cells, kThreads);
    const int by = std::max(1, std::min(ceil_div(P, 16), ceil_div(2 * ctx->sm_count * 8, bx)));
    hist_kernel<<<dim3(bx, by), kThreads, 0, ctx->stream>>>(P, cells, d_mat, d_hist);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

vx_status histogram_sel_dev(vx_ctx* ctx, int n_sel, const int32_t* d_sel, int cells, const uint8_t* d_mat,
                            double* d_out) {
    if (cells <= 0) return VX_OK;
    VX_CUDA(cudaMemsetAsync(d_out, 0, static_cast<size_t>(cells) * VX_NMAT * sizeof(double), ctx->stream));
    if (n_sel <= 0) return VX_OK;
    // ~2 waves of 256-thread blocks, >= 16 individuals per slice
    const int bx = ceil_div(cells, kThreads);
    const int by = std::max(1, std::min(ceil_div(n_sel, 16), ceil_div(2 * ctx->sm_count * 8, bx)));
    hist_sel_kernel<<<dim3(bx, by), kThreads, 0, ctx->stream>>>(n_sel, d_sel, cells, d_mat, d_out);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

vx_status hist_from_doubles_dev(vx_ctx* ctx, int cells, const double* d_in, int64_t* d_out) {
    const int n = cells * VX_NMAT;
    if (n <= 0) return VX_OK;
    hist_from_doubles_kernel<<<ceil_div(n, kThreads), kThreads, 0, ctx->stream>>>(n, d_in, d_out);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

vx_status diversity_from_hist_dev(vx_ctx* ctx, int P, int cells, const int64_t* d_hist, double* d_out) {
    diversity_kernel<<<1, 1024, 0, ctx->stream>>>(P, cells, d_hist, d_out);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

namespace {

// evaluate_fitness gates after build: gated robots are not simulated.
__global__ void gate_kernel(int n, const int32_t* status, int32_t* nmass, int32_t* nspring) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n && status[r] != 0) {
        nmass[r] = 0;
        nspring[r] = 0;
    }
}

__global__ void fitness_kernel(int n, const int32_t* todo, const int32_t* status, vx_summary* summ,
                               double* fitness, double* updates_out, vx_summary* summ_out) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int g = todo ? todo[q] : q;
    vx_summary& s = summ[q];
    s.status = status[q];
    const double f = (s.status != 0 || s.diverged) ? 0.0 : s.horizontal_displacement;
    if (fitness) fitness[g] = f;
    if (updates_out) updates_out[g] = static_cast<double>(s.spring_updates);
    if (summ_out) summ_out[g] = s;
}

__global__ void merge_kernel(int n, const int32_t* todo, const double* xbuf, double* fitness, uint8_t* evaluated) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int g = todo[q];
    fitness[g] = xbuf[g];
    evaluated[g] = 1;
}

__global__ void iota_kernel(int n, int32_t* v) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < n) v[q] = q;
}

// Sequential sums in sorted order (evolution.hpp:246-263): one thread, so the
// rounding sequence is the reference's.
__global__ void stats_kernel(int P, const double* sorted_fit, double* out3) {
    if (threadIdx.x != 0) return;
    double sum = 0.0;
    for (int a = 0; a < P; ++a) sum += sorted_fit[a];
    const double mean = sum / static_cast<double>(P);
    double var = 0.0;
    for (int a = 0; a < P; ++a) {
        const double d = sorted_fit[a] - mean;
        var += d * d;
    }
    out3[0] = sorted_fit[0];
    out3[1] = mean;
    out3[2] = sqrt(var / static_cast<double>(P));
}

// next[c] for every slot: elites copy sorted[c]; children copy sorted[pa],
// overwritten by sorted[pb] where the crossover mask bit is set.
__global__ void breed_kernel(BreedArgs A) {
    const int c = blockIdx.x;  // child slot (gridDim.x: up to 2^31-1 individuals)
    const int64_t i0 = static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x;
    int src_a, src_b = -1;
    const uint32_t* mask = nullptr;
    if (c < A.n_elite) {
        src_a = A.perm[c];
    } else {
        const ChildPlan& p = A.plan[c - A.n_elite];
        src_a = A.perm[p.pa];
        if (p.pb >= 0) {
            src_b = A.perm[p.pb];
            mask = A.masks + static_cast<int64_t>(p.mask_slot) * A.mask_words;
        }
    }
    for (int64_t i = i0; i < A.np; i += static_cast<int64_t>(gridDim.y) * blockDim.x) {
        double v = A.src_params[static_cast<int64_t>(src_a) * A.np + i];
        if (mask && ((mask[i >> 5] >> (i & 31)) & 1u)) v = A.src_params[static_cast<int64_t>(src_b) * A.np + i];
        A.dst_params[static_cast<int64_t>(c) * A.np + i] = v;
    }
    for (int64_t i = i0; i < A.nb; i += static_cast<int64_t>(gridDim.y) * blockDim.x)
        A.dst_bmat[static_cast<int64_t>(c) * A.nb + i] = A.src_bmat[static_cast<int64_t>(src_a) * A.nb + i];
    if (c < A.n_elite) {
        // elites keep fitness, evaluated flag and cached raw grid
        for (int64_t i = i0; i < A.cells; i += static_cast<int64_t>(gridDim.y) * blockDim.x) {
            A.dst_grid[static_cast<int64_t>(c) * A.cells + i] = A.src_grid[static_cast<int64_t>(src_a) * A.cells + i];
            A.dst_gridw[static_cast<int64_t>(c) * A.cells + i] =
                A.src_gridw[static_cast<int64_t>(src_a) * A.cells + i];
        }
        if (i0 == 0) {
            A.dst_fit[c] = A.src_fit[src_a];
            A.dst_eval[c] = A.src_eval[src_a];
        }
    } else if (i0 == 0) {
        A.dst_fit[c] = 0.0;
        A.dst_eval[c] = 0;
    }
}

// v = v + (normal * scale), one entry per mutated parameter (evolution.hpp:164)
__global__ void mutate_kernel(int64_t n, const MutEntry* __restrict__ e, int64_t np, double* dst_params) {
    const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const MutEntry m = e[q];
    double* p = dst_params + static_cast<int64_t>(m.child) * np + m.index;
    *p = *p + m.delta;
}

__global__ void gather_sorted_kernel(int P, const int32_t* perm, const double* fit, double* sorted) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < P) sorted[q] = fit[perm[q]];
}

}  // namespace

vx_status gate_dev(vx_ctx* ctx, vx_batch* b) {
    if (b->n == 0) return VX_OK;
    gate_kernel<<<ceil_div(b->n, kThreads), kThreads, 0, ctx->stream>>>(b->n, b->status.p, b->nmass.p, b->nspring.p);
    ctx->launches++;
    b->counts_on_host = false;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

vx_status fitness_dev(vx_ctx* ctx, int n, const int32_t* d_todo, const int32_t* d_status, vx_summary* d_summ,
                      double* d_fitness, double* d_updates, vx_summary* d_summ_out) {
    if (n == 0) return VX_OK;
    fitness_kernel<<<ceil_div(n, kThreads), kThreads, 0, ctx->stream>>>(n, d_todo, d_status, d_summ, d_fitness,
                                                                        d_updates, d_summ_out);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

vx_status merge_dev(vx_ctx* ctx, int n, const int32_t* d_todo, const double* d_xbuf, double* d_fitness,
                    uint8_t* d_eval) {
    if (n == 0) return VX_OK;
    merge_kernel<<<ceil_div(n, kThreads), kThreads, 0, ctx->stream>>>(n, d_todo, d_xbuf, d_fitness, d_eval);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

// Stable descending sort of P fitness values -> perm (sorted position ->
// population index) and the sorted fitness vector; then the stats.
vx_status sort_stats_dev(vx_ctx* ctx, int P, const double* d_fit, int32_t* d_perm, double* d_sorted, int32_t* d_iota,
                         double* d_keys_tmp, double* d_stats3) {
    iota_kernel<<<ceil_div(P, kThreads), kThreads, 0, ctx->stream>>>(P, d_iota);
    ctx->launches++;
    size_t bytes = 0;
    VX_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, d_fit, d_keys_tmp, d_iota, d_perm, P, 0, 64,
                                                      ctx->stream));
    VX_TRY(ctx->tmp.alloc(bytes + 16));
    VX_CUDA(cub::DeviceRadixSort::SortPairsDescending(ctx->tmp.p, bytes, d_fit, d_keys_tmp, d_iota, d_perm, P, 0, 64,
                                                      ctx->stream));
    ctx->launches += 4;  // CUB's onesweep passes (library kernels)
    gather_sorted_kernel<<<ceil_div(P, kThreads), kThreads, 0, ctx->stream>>>(P, d_perm, d_fit, d_sorted);
    ctx->launches++;
    stats_kernel<<<1, 32, 0, ctx->stream>>>(P, d_sorted, d_stats3);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

vx_status breed_dev(vx_ctx* ctx, const BreedArgs& A, int P, const MutEntry* d_mut, int64_t n_mut) {
    dim3 grid(P, ceil_div(A.np, kThreads) < 64 ? ceil_div(A.np, kThreads) : 64);
    breed_kernel<<<grid, kThreads, 0, ctx->stream>>>(A);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    if (n_mut > 0) {
        mutate_kernel<<<ceil_div(n_mut, kThreads), kThreads, 0, ctx->stream>>>(n_mut, d_mut, A.np, A.dst_params);
        ctx->launches++;
        VX_CUDA(cudaGetLastError());
    }
    return VX_OK;
}

}  // namespace vx
