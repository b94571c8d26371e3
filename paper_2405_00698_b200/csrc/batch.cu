// batch.cu — device-resident MassSpringSystem batches and K6, the
// SimWorkspace derivation (physics.hpp:140-185) on device.
#include <cmath>

#include "vx_internal.cuh"

namespace vx {
namespace {

constexpr int kThreads = 256;

struct DeriveArgs {
    int n;
    const int64_t* mass_off;
    const int64_t* spring_off;
    const int32_t* nmass;
    const int32_t* nspring;
    const uint32_t* ij;
    const double* mass;
    const double* k;
    const double* rest0;
    const double* zeta;
    const uint8_t* has_act;
    const double* sign;
    const double* amp;
    const double* phase;
    double* c;
    double* amp_rest;
    double* sinph;
    double* cosph;
    double* gdamp;
    int32_t* any_act;
    int32_t* inc_off;
    uint32_t* inc;
    double plane_k, plane_zeta;
};

// One CTA per robot.  Per spring: damping_coefficient (physics.hpp:66-71),
// amp_rest / sin / cos of the actuation phase (physics.hpp:151-160); per mass:
// ground damping (physics.hpp:163-164); then the CSR incidence lists sorted
// by spring index (physics.hpp:166-184) built with atomics + a per-mass sort,
// so the result is deterministic and identical to the reference's lists.
__global__ void __launch_bounds__(kThreads) derive_kernel(DeriveArgs A) {
    const int r = blockIdx.x;
    const int64_t mo = A.mass_off[r], so = A.spring_off[r];
    const int nm = A.nmass[r];
    const int ns = A.nspring[r];
    __shared__ int s_any;
    if (threadIdx.x == 0) s_any = 0;
    int32_t* off = A.inc_off + mo + r;  // nm + 1 entries
    for (int a = threadIdx.x; a <= nm; a += kThreads) off[a] = 0;
    __syncthreads();
    int any = 0;
    for (int q = threadIdx.x; q < ns; q += kThreads) {
        const int64_t g = so + q;
        const uint32_t e = A.ij[g];
        const int i = static_cast<int>(e & 0xFFFFu), j = static_cast<int>(e >> 16);
        const double mi = A.mass[mo + i], mj = A.mass[mo + j];
        const double mu = mi * mj / (mi + mj);
        A.c[g] = A.zeta[g] * 2.0 * sqrt(A.k[g] * mu);
        if (A.has_act[g]) {
            any = 1;
            A.amp_rest[g] = A.sign[g] * A.amp[g] * A.rest0[g];
            double sp, cp;
            sincos(A.phase[g], &sp, &cp);
            A.sinph[g] = sp;
            A.cosph[g] = cp;
        } else {
            A.amp_rest[g] = 0.0;
            A.sinph[g] = 0.0;
            A.cosph[g] = 1.0;
        }
        atomicAdd(&off[i + 1], 1);
        atomicAdd(&off[j + 1], 1);
    }
    if (any) atomicOr(&s_any, 1);
    for (int a = threadIdx.x; a < nm; a += kThreads)
        A.gdamp[mo + a] = A.plane_zeta * 2.0 * sqrt(A.plane_k * A.mass[mo + a]);
    __syncthreads();
    if (threadIdx.x == 0) {
        A.any_act[r] = s_any;
        for (int a = 0; a < nm; ++a) off[a + 1] += off[a];
    }
    __syncthreads();
    // scatter with per-mass cursors (smem atomics), then sort each list
    uint32_t* inc = A.inc + 2 * so;
    extern __shared__ int32_t cursor_sm[];
    const bool cursor_in_smem = nm <= 12288;
    if (cursor_in_smem) {
        int32_t* cursor = cursor_sm;
        for (int a = threadIdx.x; a < nm; a += kThreads) cursor[a] = off[a];
        __syncthreads();
        for (int q = threadIdx.x; q < ns; q += kThreads) {
            const uint32_t e = A.ij[so + q];
            const int i = static_cast<int>(e & 0xFFFFu), j = static_cast<int>(e >> 16);
            inc[atomicAdd(&cursor[i], 1)] = static_cast<uint32_t>(q) << 1;
            inc[atomicAdd(&cursor[j], 1)] = (static_cast<uint32_t>(q) << 1) | 1u;
        }
    }
    __syncthreads();
    if (!cursor_in_smem) {
        // very large robots: one thread fills in ascending spring order (lists
        // come out sorted); off[] doubles as the cursor and is restored after
        if (threadIdx.x == 0) {
            for (int q = 0; q < ns; ++q) {
                const uint32_t e = A.ij[so + q];
                const int i = static_cast<int>(e & 0xFFFFu), j = static_cast<int>(e >> 16);
                inc[off[i]++] = static_cast<uint32_t>(q) << 1;
                inc[off[j]++] = (static_cast<uint32_t>(q) << 1) | 1u;
            }
            for (int a = nm; a > 0; --a) off[a] = off[a - 1];
            off[0] = 0;
        }
        return;
    }
    // per-mass insertion sort by spring index (== by value, one entry per s)
    for (int a = threadIdx.x; a < nm; a += kThreads) {
        const int e0 = off[a], e1 = off[a + 1];
        for (int x = e0 + 1; x < e1; ++x) {
            const uint32_t v = inc[x];
            int y = x - 1;
            while (y >= e0 && inc[y] > v) {
                inc[y + 1] = inc[y];
                --y;
            }
            inc[y + 1] = v;
        }
    }
}

}  // namespace

vx_status batch_alloc(vx_batch* b, int n, int64_t M, int64_t S) {
    b->n = n;
    b->M = M;
    b->S = S;
    VX_TRY(b->mass_off.alloc(n + 1));
    VX_TRY(b->spring_off.alloc(n + 1));
    VX_TRY(b->nmass.alloc(n + 1));
    VX_TRY(b->nspring.alloc(n + 1));
    VX_TRY(b->status.alloc(n + 1));
    VX_TRY(b->pos.alloc(3 * M));
    VX_TRY(b->vel.alloc(3 * M));
    VX_TRY(b->mass.alloc(M));
    VX_TRY(b->gdamp.alloc(M));
    VX_TRY(b->ij.alloc(S));
    VX_TRY(b->k.alloc(S));
    VX_TRY(b->rest0.alloc(S));
    VX_TRY(b->zeta.alloc(S));
    VX_TRY(b->c.alloc(S));
    VX_TRY(b->amp_rest.alloc(S));
    VX_TRY(b->sinph.alloc(S));
    VX_TRY(b->cosph.alloc(S));
    VX_TRY(b->has_act.alloc(S));
    VX_TRY(b->sign.alloc(S));
    VX_TRY(b->amp.alloc(S));
    VX_TRY(b->phase.alloc(S));
    VX_TRY(b->inc_off.alloc(M + n));
    VX_TRY(b->inc.alloc(2 * S));
    VX_TRY(b->any_act.alloc(n));
    return VX_OK;
}

vx_status batch_derive_workspace(vx_ctx* ctx, vx_batch* b) {
    if (b->n == 0) return VX_OK;
    DeriveArgs A{};
    A.n = b->n;
    A.mass_off = b->mass_off.p;
    A.spring_off = b->spring_off.p;
    A.nmass = b->nmass.p;
    A.nspring = b->nspring.p;
    A.ij = b->ij.p;
    A.mass = b->mass.p;
    A.k = b->k.p;
    A.rest0 = b->rest0.p;
    A.zeta = b->zeta.p;
    A.has_act = b->has_act.p;
    A.sign = b->sign.p;
    A.amp = b->amp.p;
    A.phase = b->phase.p;
    A.c = b->c.p;
    A.amp_rest = b->amp_rest.p;
    A.sinph = b->sinph.p;
    A.cosph = b->cosph.p;
    A.gdamp = b->gdamp.p;
    A.any_act = b->any_act.p;
    A.inc_off = b->inc_off.p;
    A.inc = b->inc.p;
    A.plane_k = b->plane.k;
    A.plane_zeta = b->plane.damping_ratio;
    const size_t smem = static_cast<size_t>(b->nm_max <= 12288 ? b->nm_max : 0) * sizeof(int32_t) + 16;
    VX_CUDA(cudaFuncSetAttribute(derive_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    derive_kernel<<<b->n, kThreads, smem, ctx->stream>>>(A);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

vx_status batch_sync_counts(vx_batch* b) {
    if (b->counts_on_host) return VX_OK;
    b->h_nmass.resize(b->n);
    b->h_nspring.resize(b->n);
    if (b->n > 0) {
        VX_CUDA(cudaMemcpyAsync(b->h_nmass.data(), b->nmass.p, b->n * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                b->ctx->stream));
        VX_CUDA(cudaMemcpyAsync(b->h_nspring.data(), b->nspring.p, b->n * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                b->ctx->stream));
        VX_CUDA(cudaStreamSynchronize(b->ctx->stream));
    }
    b->counts_on_host = true;
    return VX_OK;
}

}  // namespace vx
