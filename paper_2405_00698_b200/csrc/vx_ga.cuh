// vx_ga.cuh — GA plan structures shared by ga.cu (device apply) and evo.cu
// (host plan parse + driver).
#pragma once

#include <cstdint>

#include "ga_plan.hpp"
#include "vx_internal.cuh"

namespace vx {

struct BreedArgs {
    int n_elite;
    int64_t np, nb, cells;
    int64_t mask_words;
    const int32_t* perm;  // sorted position -> population index
    const ChildPlan* plan;
    const uint32_t* masks;
    const double* src_params;
    const double* src_bmat;
    const double* src_fit;
    const uint8_t* src_eval;
    const uint8_t* src_grid;
    const double* src_gridw;
    double* dst_params;
    double* dst_bmat;
    double* dst_fit;
    uint8_t* dst_eval;
    uint8_t* dst_grid;
    double* dst_gridw;
};

vx_status gate_dev(vx_ctx* ctx, vx_batch* b);
vx_status fitness_dev(vx_ctx* ctx, int n, const int32_t* d_todo, const int32_t* d_status, vx_summary* d_summ,
                      double* d_fitness, double* d_updates, vx_summary* d_summ_out);
vx_status merge_dev(vx_ctx* ctx, int n, const int32_t* d_todo, const double* d_xbuf, double* d_fitness,
                    uint8_t* d_eval);
vx_status sort_stats_dev(vx_ctx* ctx, int P, const double* d_fit, int32_t* d_perm, double* d_sorted, int32_t* d_iota,
                         double* d_keys_tmp, double* d_stats3);
vx_status breed_dev(vx_ctx* ctx, const BreedArgs& A, int P, const MutEntry* d_mut, int64_t n_mut);

// evaluate pipeline shared by the ABI and the evolution driver:
// raw grids (selected) -> component -> build -> gates -> integrate -> fitness.
vx_status evaluate_pipeline(vx_ctx* ctx, int P, int w, int h, int d, const uint8_t* d_mat, const double* d_weight,
                            const vx_materials* table, const vx_plane* plane, const vx_sim* sim, const int32_t* d_todo,
                            int n_todo, double* d_fitness, double* d_updates, vx_summary* d_summaries,
                            const double2* d_phase_sc = nullptr);

}  // namespace vx
