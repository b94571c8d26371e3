// ga_plan.hpp — the host-side breeding plan: structures shared with the
// device apply (ga.cu) and the scan that fills them (ga_plan.cpp, plain C++
// compiled by the host compiler).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <random>
#include <vector>

namespace vx {

// One child's breeding decisions in SORTED-rank space (evolution.hpp:274-282).
struct ChildPlan {
    int32_t pa;         // tournament winner rank (tournament_select, :169-173)
    int32_t pb;         // second parent rank or -1 (no crossover)
    int32_t mask_slot;  // crossover mask row (valid when pb >= 0)
    int32_t pad;
};

// A mutated parameter: child slot, flat parameter index, delta = normal*scale.
struct MutEntry {
    int32_t child;
    int32_t index;
    double delta;
};

struct PlanParams {
    int P;                // population
    int n_elite;          // children 0..n_elite-1 are elite copies (no draws)
    int tournament_size;  // EvolutionConfig::tournament_size
    int64_t np;           // controller parameter count
    int64_t mask_words;   // ceil(np / 32)
    double crossover_rate, mutation_rate, mutation_scale;
};

// The mutation list of one generation, in fixed-size chunks that never move
// once written (the deltas are filled by worker threads while the scan is
// still appending).  Chunk memory is kept across generations; the entry
// arrays come from `host_alloc` (pinned memory in the library, so the upload
// is a true async copy) or operator new.
class MutStore {
public:
    static constexpr size_t kChunk = size_t(1) << 14;
    using AllocFn = void* (*)(size_t);
    using FreeFn = void (*)(void*);

    explicit MutStore(AllocFn alloc = nullptr, FreeFn free = nullptr) : alloc_(alloc), free_(free) {}
    ~MutStore();
    MutStore(const MutStore&) = delete;
    MutStore& operator=(const MutStore&) = delete;

    size_t size() const { return n_; }
    size_t chunks() const { return (n_ + kChunk - 1) / kChunk; }
    const MutEntry* chunk(size_t j) const { return e_[j]; }
    size_t chunk_size(size_t j) const { return std::min(kChunk, n_ - j * kChunk); }
    // chunk j continues chunk j-1 inside the same allocation (one copy may span both)
    bool continues(size_t j) const { return j > 0 && slab_of_[j] == slab_of_[j - 1]; }
    void flatten(std::vector<MutEntry>& out) const;
    void clear() { n_ = 0; }

private:
    friend struct MutWriter;
    std::vector<MutEntry*> e_;  // per chunk; delta holds the first raw word until its normal is computed
    std::vector<uint64_t*> r2_;
    std::vector<void*> slabs_;           // e_ chunks come in slabs (geometric growth, few pinned allocations)
    std::vector<uint64_t*> r2_slabs_;
    std::vector<uint32_t> slab_of_;
    size_t n_ = 0;
    AllocFn alloc_;
    FreeFn free_;
};

// The breeding loop (evolution.hpp:267-289) for children n_elite..P-1 in
// rank space, consuming `rng` draw-for-draw like the reference (rng.hpp:23-39,
// crossover :143-155, mutate :160-165).  On return `rng` is the reference's
// post-generation GA stream state.  plan has max(1, P - n_elite) rows, masks
// mask_words words per crossover child, mut every (child, index, delta)
// in scan order.
void plan_scan(std::mt19937_64& rng, const PlanParams& a, std::vector<ChildPlan>& plan, std::vector<uint32_t>& masks,
               MutStore& mut);

}  // namespace vx
