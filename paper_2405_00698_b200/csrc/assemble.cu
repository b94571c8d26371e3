// assemble.cu — K4 largest_component and K5 build_mass_spring on device.
//
// K4 replaces largest_component (morphology.hpp:162-208): per grid, one CTA
// runs min-label propagation with pointer jumping in shared memory; labels
// converge to each component's lowest linear index (= the reference's DFS
// seed), and the winner is max size with ties to the lowest seed.
//
// K5 replaces build_mass_spring (morphology.hpp:217-299): per robot, one CTA
//  * marks occupied lattice vertices; mass index = exclusive warp-scan of the
//    occupancy in vertex-key order (== sort+unique of keys, :232-235);
//  * emits springs in lexicographic (i, j) order: for every mass (ascending)
//    its up-to-13 "forward" lattice neighbours in ascending key offset, the
//    spring existing iff a voxel contains both endpoints; k = ordered mean of
//    the contributing voxels' weight*base_k in ascending voxel index
//    (:256-278, 289), actuation from the lowest-index muscle contributor,
//    rest0 from the grounded positions (:280-293).
// Output uses a fixed per-robot stride (no host round trip); the integer
// topology and every double (only + - * / sqrt) are bit-identical to the
// reference's.
#include <cmath>

#include "vx_internal.cuh"

namespace vx {
namespace {

constexpr int kThreads = 256;

// ------------------------------------------------------------------ K4 ----
__global__ void __launch_bounds__(kThreads) component_kernel(int w, int h, int d, const uint8_t* __restrict__ in,
                                                             uint8_t* __restrict__ out, const int32_t* select) {
    const int n = w * h * d;
    const int g = select ? select[blockIdx.x] : static_cast<int>(blockIdx.x);
    const uint8_t* src = in + static_cast<size_t>(g) * n;
    uint8_t* dst = out + static_cast<size_t>(blockIdx.x) * n;
    extern __shared__ int sm_i[];
    int* label = sm_i;      // n
    int* count = sm_i + n;  // n
    __shared__ unsigned long long s_best;
    for (int c = threadIdx.x; c < n; c += kThreads) {
        label[c] = src[c] ? c : -1;
        count[c] = 0;
    }
    if (threadIdx.x == 0) s_best = 0ull;
    __syncthreads();
    for (;;) {
        int changed = 0;
        for (int c = threadIdx.x; c < n; c += kThreads) {
            int l = label[c];
            if (l < 0) continue;
            const int x = c % w, y = (c / w) % h, z = c / (w * h);
            int m = l;
            if (x > 0 && label[c - 1] >= 0) m = min(m, label[c - 1]);
            if (x + 1 < w && label[c + 1] >= 0) m = min(m, label[c + 1]);
            if (y > 0 && label[c - w] >= 0) m = min(m, label[c - w]);
            if (y + 1 < h && label[c + w] >= 0) m = min(m, label[c + w]);
            if (z > 0 && label[c - w * h] >= 0) m = min(m, label[c - w * h]);
            if (z + 1 < d && label[c + w * h] >= 0) m = min(m, label[c + w * h]);
            if (m < l) {
                // hook: the old root adopts the smaller label too (both are
                // cells of this component), then jump
                atomicMin(&label[l], m);
                atomicMin(&label[c], m);
                changed = 1;
            }
        }
        __syncthreads();
        for (int c = threadIdx.x; c < n; c += kThreads) {
            int l = label[c];
            if (l < 0) continue;
            int ll = label[l];
            while (ll < l) {
                l = ll;
                ll = label[l];
            }
            label[c] = l;
        }
        if (!__syncthreads_or(changed)) break;
    }
    for (int c = threadIdx.x; c < n; c += kThreads)
        if (label[c] >= 0) atomicAdd(&count[label[c]], 1);
    __syncthreads();
    for (int c = threadIdx.x; c < n; c += kThreads) {
        if (label[c] == c) {  // root = lowest index of its component
            const unsigned long long key =
                (static_cast<unsigned long long>(count[c]) << 32) | static_cast<unsigned>(0x7FFFFFFF - c);
            atomicMax(&s_best, key);
        }
    }
    __syncthreads();
    const int best = s_best ? 0x7FFFFFFF - static_cast<int>(s_best & 0xFFFFFFFFull) : -1;
    for (int c = threadIdx.x; c < n; c += kThreads) dst[c] = (src[c] != 0 && label[c] == best) ? src[c] : 0;
}

// ------------------------------------------------------------------ K5 ----
struct BuildArgs {
    int w, h, d;
    const uint8_t* mat;
    const double* wt;
    const int32_t* select;  // optional: robot r uses grid select[r]
    vx_materials table;
    int nm_cap, ns_cap;
    int64_t M;
    // outputs (batch arrays)
    int32_t* nmass;
    int32_t* nspring;
    int32_t* status;
    double* pos;
    double* vel;
    double* mass;
    uint32_t* ij;
    double* k;
    double* rest0;
    double* zeta;
    uint8_t* has_act;
    double* sign;
    double* amp;
    double* phase;
    int32_t* vkey;     // per mass: vertex key x + vw*(y + vh*z)
    int16_t* act_vox;  // per spring: actuating voxel (lowest-index muscle) or -1
};

// forward lattice offsets (dz, dy, dx), ascending key offset (see header)
__constant__ int8_t c_fwd[13][3] = {{0, 0, 1},   {0, 1, -1},  {0, 1, 0},  {0, 1, 1},  {1, -1, -1},
                                    {1, -1, 0},  {1, -1, 1},  {1, 0, -1}, {1, 0, 0},  {1, 0, 1},
                                    {1, 1, -1},  {1, 1, 0},   {1, 1, 1}};

__device__ __forceinline__ double base_stiffness(const vx_materials& t, int m) {
    return (m == 1 || m == 2) ? t.k_muscle : (m == 3 ? t.k_soft : (m == 4 ? t.k_bone : 0.0));
}

// Block-wide exclusive scan of v[0..n) in place (int), returns the total.
__device__ int block_exclusive_scan(int* v, int n, int* warp_tot) {
    const int per = (n + kThreads - 1) / kThreads;
    const int b0 = threadIdx.x * per, b1 = min(n, b0 + per);
    int local = 0;
    for (int i = b0; i < b1; ++i) local += v[i];
    // warp inclusive scan
    int x = local;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int q = 0; q < kThreads / 32; ++q) {
            const int t = warp_tot[q];
            warp_tot[q] = acc;
            acc += t;
        }
        warp_tot[kThreads / 32] = acc;
    }
    __syncthreads();
    int run = warp_tot[wid] + x - local;
    for (int i = b0; i < b1; ++i) {
        const int t = v[i];
        v[i] = run;
        run += t;
    }
    const int total = warp_tot[kThreads / 32];
    __syncthreads();
    return total;
}

__global__ void __launch_bounds__(kThreads) build_kernel(BuildArgs A) {
    const int r = blockIdx.x;
    const int g = A.select ? A.select[r] : r;  // weight grid of robot r
    const int w = A.w, h = A.h, d = A.d;
    const int vw = w + 1, vh = h + 1, vd = d + 1;
    const int ncell = w * h * d, nv = vw * vh * vd;
    const uint8_t* mat = A.mat + static_cast<size_t>(r) * ncell;  // compact body grids
    const double* wt = A.wt + static_cast<size_t>(g) * ncell;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* s_wt = reinterpret_cast<double*>(smem_raw);                 // ncell
    int* s_massid = reinterpret_cast<int*>(s_wt + ncell);                // nv (occupancy -> mass index)
    int* s_soff = s_massid + nv;                                         // nv (spring count -> offset)
    uint8_t* s_mat = reinterpret_cast<uint8_t*>(s_soff + nv);            // ncell
    __shared__ int s_warp[kThreads / 32 + 1];
    __shared__ int s_minz, s_muscle, s_any;

    if (threadIdx.x == 0) {
        s_minz = 0x7FFFFFFF;
        s_muscle = 0;
        s_any = 0;
    }
    for (int c = threadIdx.x; c < ncell; c += kThreads) {
        s_mat[c] = mat[c];
        s_wt[c] = wt[c];
    }
    __syncthreads();
    // occupancy of lattice vertices
    int muscle = 0, any = 0;
    for (int c = threadIdx.x; c < ncell; c += kThreads) {
        any |= s_mat[c] != 0;
        muscle |= (s_mat[c] == 1 || s_mat[c] == 2);
    }
    if (any) atomicOr(&s_any, 1);
    if (muscle) atomicOr(&s_muscle, 1);
    for (int v = threadIdx.x; v < nv; v += kThreads) {
        const int x = v % vw, y = (v / vw) % vh, z = v / (vw * vh);
        int occ = 0;
        for (int cz = z - 1; cz <= z && !occ; ++cz)
            for (int cy = y - 1; cy <= y && !occ; ++cy)
                for (int cx = x - 1; cx <= x && !occ; ++cx)
                    if (cx >= 0 && cy >= 0 && cz >= 0 && cx < w && cy < h && cz < d && s_mat[cx + w * (cy + h * cz)])
                        occ = 1;
        s_massid[v] = occ;
        if (occ) atomicMin(&s_minz, z);
    }
    __syncthreads();
    const int nm = block_exclusive_scan(s_massid, nv, s_warp);
    // s_massid[v] is now the mass index for occupied v (ranks in key order)
    const double edge = A.table.voxel_edge;
    // min over masses of z*edge; z*edge is monotone in z, so it is the
    // lowest occupied layer's value (morphology.hpp:280-281)
    const double min_z = nm > 0 ? s_minz * edge : 0.0;
    const int64_t mo = static_cast<int64_t>(r) * A.nm_cap;
    const int64_t so = static_cast<int64_t>(r) * A.ns_cap;

    // masses + per-mass forward-spring counts
    for (int v = threadIdx.x; v < nv; v += kThreads) {
        const int x = v % vw, y = (v / vw) % vh, z = v / (vw * vh);
        const bool occ = (v + 1 < nv ? s_massid[v + 1] : nm) != s_massid[v];
        int cnt = 0;
        if (occ) {
            const int a = s_massid[v];
            A.pos[0 * A.M + mo + a] = x * edge;
            A.pos[1 * A.M + mo + a] = y * edge;
            A.pos[2 * A.M + mo + a] = z * edge - min_z;
            A.vel[0 * A.M + mo + a] = 0.0;
            A.vel[1 * A.M + mo + a] = 0.0;
            A.vel[2 * A.M + mo + a] = 0.0;
            A.mass[mo + a] = A.table.mass_per_vertex;
            A.vkey[mo + a] = v;
            for (int q = 0; q < 13; ++q) {
                const int dz = c_fwd[q][0], dy = c_fwd[q][1], dx = c_fwd[q][2];
                const int ux = x + dx, uy = y + dy, uz = z + dz;
                if (ux < 0 || uy < 0 || uz < 0 || ux >= vw || uy >= vh || uz >= vd) continue;
                // candidate voxels containing both endpoints
                const int x0 = dx == 0 ? x - 1 : (dx > 0 ? x : x - 1), x1 = dx == 0 ? x : x0;
                const int y0 = dy == 0 ? y - 1 : (dy > 0 ? y : y - 1), y1 = dy == 0 ? y : y0;
                const int z0 = dz == 0 ? z - 1 : (dz > 0 ? z : z - 1), z1 = dz == 0 ? z : z0;
                bool found = false;
                for (int cz = z0; cz <= z1 && !found; ++cz)
                    for (int cy = y0; cy <= y1 && !found; ++cy)
                        for (int cx = x0; cx <= x1 && !found; ++cx)
                            if (cx >= 0 && cy >= 0 && cz >= 0 && cx < w && cy < h && cz < d &&
                                s_mat[cx + w * (cy + h * cz)])
                                found = true;
                cnt += found;
            }
        }
        s_soff[v] = cnt;
    }
    __syncthreads();
    const int ns = block_exclusive_scan(s_soff, nv, s_warp);
    // springs
    for (int v = threadIdx.x; v < nv; v += kThreads) {
        const bool occ = (v + 1 < nv ? s_massid[v + 1] : nm) != s_massid[v];
        if (!occ) continue;
        const int x = v % vw, y = (v / vw) % vh, z = v / (vw * vh);
        const int a = s_massid[v];
        int64_t q_out = so + s_soff[v];
        const double ax = x * edge, ay = y * edge, az = z * edge - min_z;
        for (int q = 0; q < 13; ++q) {
            const int dz = c_fwd[q][0], dy = c_fwd[q][1], dx = c_fwd[q][2];
            const int ux = x + dx, uy = y + dy, uz = z + dz;
            if (ux < 0 || uy < 0 || uz < 0 || ux >= vw || uy >= vh || uz >= vd) continue;
            const int x0 = dx == 0 ? x - 1 : (dx > 0 ? x : x - 1), x1 = dx == 0 ? x : x0;
            const int y0 = dy == 0 ? y - 1 : (dy > 0 ? y : y - 1), y1 = dy == 0 ? y : y0;
            const int z0 = dz == 0 ? z - 1 : (dz > 0 ? z : z - 1), z1 = dz == 0 ? z : z0;
            double k_sum = 0.0;
            int count = 0;
            int act_mat = 0, act_ci = -1;
            double act_w = 0.0;
            // ascending voxel linear index: z, then y, then x
            for (int cz = z0; cz <= z1; ++cz)
                for (int cy = y0; cy <= y1; ++cy)
                    for (int cx = x0; cx <= x1; ++cx) {
                        if (cx < 0 || cy < 0 || cz < 0 || cx >= w || cy >= h || cz >= d) continue;
                        const int ci = cx + w * (cy + h * cz);
                        const int m = s_mat[ci];
                        if (!m) continue;
                        k_sum += s_wt[ci] * base_stiffness(A.table, m);
                        count += 1;
                        if ((m == 1 || m == 2) && act_mat == 0) {
                            act_mat = m;
                            act_w = s_wt[ci];
                            act_ci = ci;
                        }
                    }
            if (count == 0) continue;
            const int u = ux + vw * (uy + vh * uz);
            const int b_ = s_massid[u];
            const double bx = ux * edge, by = uy * edge, bz = uz * edge - min_z;
            A.ij[q_out] = static_cast<uint32_t>(a) | (static_cast<uint32_t>(b_) << 16);
            A.k[q_out] = k_sum / count;
            A.rest0[q_out] = sqrt((bx - ax) * (bx - ax) + (by - ay) * (by - ay) + (bz - az) * (bz - az));
            A.zeta[q_out] = A.table.damping_ratio;
            A.has_act[q_out] = act_mat != 0;
            A.sign[q_out] = act_mat == 1 ? 1.0 : (act_mat == 2 ? -1.0 : 0.0);
            A.amp[q_out] = act_mat ? act_w * A.table.amp_max : 0.0;
            A.phase[q_out] = act_mat ? act_w * A.table.phase_max : 0.0;
            A.act_vox[q_out] = static_cast<int16_t>(act_ci);
            ++q_out;
        }
    }
    if (threadIdx.x == 0) {
        A.nmass[r] = nm;
        A.nspring[r] = ns;
        A.status[r] = !s_any ? 1 : (!s_muscle ? 2 : 0);
    }
}

}  // namespace

vx_status largest_component_dev(vx_ctx* ctx, int n, int w, int h, int d, const uint8_t* d_in, uint8_t* d_out,
                                const int32_t* d_select) {
    if (n <= 0) return VX_OK;
    const int cells = w * h * d;
    const size_t smem = 2ull * cells * sizeof(int);
    if (smem > ctx->smem_optin) return (set_error("largest_component: grid too large"), VX_EINVAL);
    VX_CUDA(cudaFuncSetAttribute(component_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    component_kernel<<<n, kThreads, smem, ctx->stream>>>(w, h, d, d_in, d_out, d_select);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return VX_OK;
}

static int64_t lattice_spring_cap(int w, int h, int d) {
    const int64_t W = w, H = h, D = d;
    return W * (H + 1) * (D + 1) + (W + 1) * H * (D + 1) + (W + 1) * (H + 1) * D  // edges
           + 2 * (W * H * (D + 1) + W * (H + 1) * D + (W + 1) * H * D)           // face diagonals
           + 4 * W * H * D;                                                      // body diagonals
}

vx_status build_batch_into(vx_ctx* ctx, vx_batch* b, int n, int w, int h, int d, const uint8_t* d_body,
                           const double* d_weight, const int32_t* d_wsel, const vx_materials* table,
                           const vx_plane* plane) {
    if (w < 1 || h < 1 || d < 1) return (set_error("decode: dims must be positive"), VX_EINVAL);
    const int nm_cap = (w + 1) * (h + 1) * (d + 1);
    const int64_t ns_cap = lattice_spring_cap(w, h, d);
    if (nm_cap > 65535) return (set_error("build: lattice too large (> 65535 vertices)"), VX_EINVAL);
    b->ctx = ctx;
    b->plane = *plane;
    b->nm_max = nm_cap;
    b->ns_max = static_cast<int>(ns_cap);
    VX_TRY(batch_alloc(b, n, static_cast<int64_t>(n) * nm_cap, static_cast<int64_t>(n) * ns_cap));
    if (static_cast<int>(b->h_mass_off.size()) != n + 1 || (n > 0 && b->h_mass_off[1] != nm_cap)) {
        b->h_mass_off.resize(n + 1);
        b->h_spring_off.resize(n + 1);
        for (int r = 0; r <= n; ++r) {
            b->h_mass_off[r] = static_cast<int64_t>(r) * nm_cap;
            b->h_spring_off[r] = static_cast<int64_t>(r) * ns_cap;
        }
        VX_CUDA(cudaMemcpyAsync(b->mass_off.p, b->h_mass_off.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice,
                                ctx->stream));
        VX_CUDA(cudaMemcpyAsync(b->spring_off.p, b->h_spring_off.data(), (n + 1) * sizeof(int64_t),
                                cudaMemcpyHostToDevice, ctx->stream));
        VX_CUDA(cudaStreamSynchronize(ctx->stream));  // host offsets are staged from pageable memory
    }
    b->counts_on_host = false;
    if (n == 0) return VX_OK;
    BuildArgs A{};
    A.w = w;
    A.h = h;
    A.d = d;
    A.mat = d_body;
    A.wt = d_weight;
    A.select = d_wsel;
    A.table = *table;
    A.nm_cap = nm_cap;
    A.ns_cap = static_cast<int>(ns_cap);
    A.M = b->M;
    A.nmass = b->nmass.p;
    A.nspring = b->nspring.p;
    A.status = b->status.p;
    A.pos = b->pos.p;
    A.vel = b->vel.p;
    A.mass = b->mass.p;
    A.ij = b->ij.p;
    A.k = b->k.p;
    A.rest0 = b->rest0.p;
    A.zeta = b->zeta.p;
    A.has_act = b->has_act.p;
    A.sign = b->sign.p;
    A.amp = b->amp.p;
    A.phase = b->phase.p;
    VX_TRY(b->vkey.alloc(b->M));
    VX_TRY(b->act_vox.alloc(b->S));
    A.vkey = b->vkey.p;
    A.act_vox = b->act_vox.p;
    b->lattice = true;
    b->uniform_mass = table->mass_per_vertex;
    b->uniform_zeta = table->damping_ratio;
    b->lw = w;
    b->lh = h;
    b->ld = d;
    const int ncell = w * h * d;
    const size_t smem = static_cast<size_t>(ncell) * (sizeof(double) + 1) + 2ull * nm_cap * sizeof(int) + 16;
    if (smem > ctx->smem_optin) return (set_error("build: grid too large for one CTA"), VX_EINVAL);
    VX_CUDA(cudaFuncSetAttribute(build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    build_kernel<<<n, kThreads, smem, ctx->stream>>>(A);
    ctx->launches++;
    VX_CUDA(cudaGetLastError());
    return batch_derive_workspace(ctx, b);
}

}  // namespace vx
