// api_ops.cu — C ABI: genome sampling, decode, component, build, evaluate,
// diversity (host- and device-pointer entry points).
#include <vector>

#include "vx_ga.cuh"
#include "vx_internal.cuh"

using namespace vx;

namespace {

template <typename T>
vx_status upload(DevBuf<T>& buf, const T* h, size_t n, cudaStream_t s) {
    VX_TRY(buf.alloc(n));
    VX_CUDA(cudaMemcpyAsync(buf.p, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
    return VX_OK;
}

}  // namespace

extern "C" {

vx_status vx_sample_genomes_dev(vx_ctx* ctx, const vx_arch* a, int32_t P, const uint64_t* d_seeds, double* d_params,
                                double* d_bmat) {
    if (!ctx || !a || P < 0) return VX_EINVAL;
    return sample_genomes_dev(ctx, a, P, d_seeds, d_params, d_bmat);
}

vx_status vx_sample_genomes(vx_ctx* ctx, const vx_arch* a, int32_t P, const uint64_t* seeds, double* params,
                            double* bmat) {
    if (!ctx || !a || P < 0 || (P > 0 && (!seeds || !params || !bmat))) return VX_EINVAL;
    const int64_t np = param_count(a);
    if (np < 0) return (set_error("invalid architecture"), VX_EINVAL);
    if (P == 0) return VX_OK;
    DevBuf<uint64_t> ds;
    DevBuf<double> dp, db;
    VX_TRY(upload(ds, seeds, static_cast<size_t>(P), ctx->stream));
    VX_TRY(dp.alloc(P * static_cast<size_t>(np)));
    VX_TRY(db.alloc(P * 3ull * a->m));
    VX_TRY(sample_genomes_dev(ctx, a, P, ds.p, dp.p, db.p));
    VX_CUDA(cudaMemcpyAsync(params, dp.p, P * static_cast<size_t>(np) * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));
    host_sample_bmat(a->m, a->sigma, P, seeds, bmat);  // glibc Box-Muller: bit-exact B
    return VX_OK;
}

vx_status vx_forward(vx_ctx* ctx, const vx_arch* a, int32_t P, const double* params, const double* bmat,
                     int32_t n_points, const double* points, double* probs, double* weight) {
    if (!ctx || !a || P < 0 || n_points < 0) return VX_EINVAL;
    if (P == 0 || n_points == 0) return VX_OK;
    if (!params || !bmat || !points || !probs || !weight) return VX_EINVAL;
    const int64_t np = param_count(a);
    if (np < 0) return (set_error("invalid architecture"), VX_EINVAL);
    const size_t nq = static_cast<size_t>(P) * n_points;
    DevBuf<double> dp, db, dq, dpr, dw;
    VX_TRY(upload(dp, params, P * static_cast<size_t>(np), ctx->stream));
    VX_TRY(upload(db, bmat, P * 3ull * a->m, ctx->stream));
    VX_TRY(upload(dq, points, 3 * nq, ctx->stream));
    VX_TRY(dpr.alloc(VX_NMAT * nq));
    VX_TRY(dw.alloc(nq));
    VX_TRY(forward_dev(ctx, a, P, dp.p, db.p, n_points, dq.p, dpr.p, dw.p));
    VX_CUDA(cudaMemcpyAsync(probs, dpr.p, VX_NMAT * nq * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    VX_CUDA(cudaMemcpyAsync(weight, dw.p, nq * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));
    return VX_OK;
}

vx_status vx_decode_dev(vx_ctx* ctx, const vx_arch* a, int32_t P, const double* d_params, const double* d_bmat,
                        int32_t w, int32_t h, int32_t d, uint8_t* d_mat, double* d_weight, uint32_t* d_guard) {
    if (!ctx || !a || P < 0) return VX_EINVAL;
    return decode_dev(ctx, a, P, d_params, d_bmat, w, h, d, d_mat, d_weight, d_guard, nullptr, 0);
}

vx_status vx_decode(vx_ctx* ctx, const vx_arch* a, int32_t P, const double* params, const double* bmat, int32_t w,
                    int32_t h, int32_t d, uint8_t* mat, double* weight) {
    if (!ctx || !a || P < 0 || !params || !bmat) return VX_EINVAL;
    if (w < 1 || h < 1 || d < 1) return (set_error("decode: dims must be positive"), VX_EINVAL);
    const int64_t np = param_count(a);
    if (np < 0) return (set_error("invalid architecture"), VX_EINVAL);
    const size_t cells = static_cast<size_t>(w) * h * d;
    DevBuf<double> dp, db, dw;
    DevBuf<uint8_t> dm;
    VX_TRY(upload(dp, params, P * static_cast<size_t>(np), ctx->stream));
    VX_TRY(upload(db, bmat, P * 3ull * a->m, ctx->stream));
    VX_TRY(dm.alloc(P * cells));
    VX_TRY(dw.alloc(P * cells));
    VX_TRY(decode_dev(ctx, a, P, dp.p, db.p, w, h, d, dm.p, dw.p, nullptr, nullptr, 0));
    VX_CUDA(cudaMemcpyAsync(mat, dm.p, P * cells, cudaMemcpyDeviceToHost, ctx->stream));
    VX_CUDA(cudaMemcpyAsync(weight, dw.p, P * cells * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));
    return VX_OK;
}

vx_status vx_decode_refined(vx_ctx* ctx, int64_t* n_refined) {
    if (!ctx || !n_refined) return VX_EINVAL;
    *n_refined = -1;
    if (ctx->decode_fix_n < 0) return VX_OK;
    std::vector<uint8_t> f(static_cast<size_t>(ctx->decode_fix_n));
    if (!f.empty())
        VX_CUDA(cudaMemcpyAsync(f.data(), ctx->decode_fix.p, f.size(), cudaMemcpyDeviceToHost, ctx->stream));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));
    int64_t n = 0;
    for (uint8_t v : f) n += v != 0;
    *n_refined = n;
    return VX_OK;
}

vx_status vx_largest_component_dev(vx_ctx* ctx, int32_t P, int32_t w, int32_t h, int32_t d, const uint8_t* d_in,
                                   uint8_t* d_out) {
    if (!ctx || P < 0 || w < 1 || h < 1 || d < 1) return VX_EINVAL;
    return largest_component_dev(ctx, P, w, h, d, d_in, d_out, nullptr);
}

vx_status vx_largest_component(vx_ctx* ctx, int32_t P, int32_t w, int32_t h, int32_t d, const uint8_t* in,
                               uint8_t* out) {
    if (!ctx || P < 0 || w < 1 || h < 1 || d < 1 || !in || !out) return VX_EINVAL;
    const size_t cells = static_cast<size_t>(w) * h * d;
    DevBuf<uint8_t> di, dout;
    VX_TRY(upload(di, in, P * cells, ctx->stream));
    VX_TRY(dout.alloc(P * cells));
    VX_TRY(largest_component_dev(ctx, P, w, h, d, di.p, dout.p, nullptr));
    VX_CUDA(cudaMemcpyAsync(out, dout.p, P * cells, cudaMemcpyDeviceToHost, ctx->stream));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));
    return VX_OK;
}

vx_status vx_batch_build_dev(vx_ctx* ctx, int32_t P, int32_t w, int32_t h, int32_t d, const uint8_t* d_mat,
                             const double* d_weight, const vx_materials* table, const vx_plane* plane,
                             vx_batch** out) {
    if (!ctx || !table || !plane || !out || P < 0) return VX_EINVAL;
    auto* b = new vx_batch;
    vx_status st = build_batch_into(ctx, b, P, w, h, d, d_mat, d_weight, nullptr, table, plane);
    if (st != VX_OK) {
        delete b;
        return st;
    }
    *out = b;
    return VX_OK;
}

vx_status vx_batch_build(vx_ctx* ctx, int32_t P, int32_t w, int32_t h, int32_t d, const uint8_t* mat,
                         const double* weight, const vx_materials* table, const vx_plane* plane, vx_batch** out) {
    if (!ctx || !mat || !weight || P < 0) return VX_EINVAL;
    if (w < 1 || h < 1 || d < 1) return (set_error("dims must be positive"), VX_EINVAL);
    const size_t cells = static_cast<size_t>(w) * h * d;
    DevBuf<uint8_t> dm;
    DevBuf<double> dw;
    VX_TRY(upload(dm, mat, P * cells, ctx->stream));
    VX_TRY(upload(dw, weight, P * cells, ctx->stream));
    VX_TRY(vx_batch_build_dev(ctx, P, w, h, d, dm.p, dw.p, table, plane, out));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));
    return VX_OK;
}

vx_status vx_evaluate_dev(vx_ctx* ctx, int32_t P, int32_t w, int32_t h, int32_t d, const uint8_t* d_mat,
                          const double* d_weight, const vx_materials* table, const vx_plane* plane, const vx_sim* sim,
                          const int32_t* d_todo, int32_t n_todo, double* d_fitness, vx_summary* d_summaries) {
    if (!ctx || !table || !plane || !sim || P < 0) return VX_EINVAL;
    if (w < 1 || h < 1 || d < 1) return (set_error("dims must be positive"), VX_EINVAL);
    return evaluate_pipeline(ctx, P, w, h, d, d_mat, d_weight, table, plane, sim, d_todo, n_todo, d_fitness, nullptr,
                             d_summaries);
}

vx_status vx_evaluate(vx_ctx* ctx, int32_t P, int32_t w, int32_t h, int32_t d, const uint8_t* mat,
                      const double* weight, const vx_materials* table, const vx_plane* plane, const vx_sim* sim,
                      double* fitness, vx_summary* summaries) {
    if (!ctx || !mat || !weight || !fitness || P < 0) return VX_EINVAL;
    if (w < 1 || h < 1 || d < 1) return (set_error("dims must be positive"), VX_EINVAL);
    const size_t cells = static_cast<size_t>(w) * h * d;
    DevBuf<uint8_t> dm;
    DevBuf<double> dw, df;
    DevBuf<vx_summary> ds;
    VX_TRY(upload(dm, mat, P * cells, ctx->stream));
    VX_TRY(upload(dw, weight, P * cells, ctx->stream));
    VX_TRY(df.alloc(P));
    if (summaries) VX_TRY(ds.alloc(P));
    // the weights are on the host: sin/cos of every cell's actuation phase
    // with the host glibc, as the reference's SimWorkspace computes them
    // (physics.hpp:154-155), so fitness is bit-identical to the reference's
    std::vector<double2> sc(P * cells);
    for (size_t q = 0; q < sc.size(); ++q) {
        const double phase = weight[q] * table->phase_max;  // morphology.hpp:275
        sc[q] = make_double2(std::sin(phase), std::cos(phase));
    }
    DevBuf<double2> dsc;
    VX_TRY(upload(dsc, sc.data(), sc.size(), ctx->stream));
    VX_TRY(evaluate_pipeline(ctx, P, w, h, d, dm.p, dw.p, table, plane, sim, nullptr, P, df.p, nullptr,
                             summaries ? ds.p : nullptr, dsc.p));
    VX_CUDA(cudaMemcpyAsync(fitness, df.p, P * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (summaries)
        VX_CUDA(cudaMemcpyAsync(summaries, ds.p, P * sizeof(vx_summary), cudaMemcpyDeviceToHost, ctx->stream));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));
    return VX_OK;
}

vx_status vx_material_histogram_dev(vx_ctx* ctx, int32_t P, int32_t cells, const uint8_t* d_mat, int64_t* d_hist,
                                    int32_t accumulate) {
    if (!ctx || P < 0 || cells < 0) return VX_EINVAL;
    return histogram_dev(ctx, P, cells, d_mat, d_hist, accumulate != 0);
}

vx_status vx_diversity_from_histogram_dev(vx_ctx* ctx, int32_t P, int32_t cells, const int64_t* d_hist,
                                          double* d_out) {
    if (!ctx || P < 0 || cells < 0) return VX_EINVAL;
    return diversity_from_hist_dev(ctx, P, cells, d_hist, d_out);
}

vx_status vx_population_diversity_dev(vx_ctx* ctx, int32_t P, int32_t cells, const uint8_t* d_mat, double* d_out) {
    if (!ctx || P < 0 || cells < 0) return VX_EINVAL;
    // bit-exact: the reference's ordered pairwise sum (diversity.cu)
    DevBuf<double> packed;
    VX_TRY(packed.alloc(static_cast<size_t>(P) * diversity_words(cells) + 1));
    VX_TRY(diversity_pack_dev(ctx, P, nullptr, cells, d_mat, packed.p));
    VX_TRY(diversity_exact_dev(ctx, P, cells, packed.p, nullptr, d_out));
    VX_CUDA(cudaStreamSynchronize(ctx->stream));  // packed is freed on return
    return VX_OK;
}

vx_status vx_population_diversity(vx_ctx* ctx, int32_t P, int32_t cells, const uint8_t* mat, double* out) {
    if (!ctx || P < 0 || cells < 0 || !out) return VX_EINVAL;
    DevBuf<uint8_t> dm;
    DevBuf<double> dd;
    VX_TRY(upload(dm, mat, static_cast<size_t>(P) * cells, ctx->stream));
    VX_TRY(dd.alloc(1));
    VX_TRY(vx_population_diversity_dev(ctx, P, cells, dm.p, dd.p));
    VX_CUDA(cudaMemcpy(out, dd.p, sizeof(double), cudaMemcpyDeviceToHost));
    return VX_OK;
}

}  // extern "C"
