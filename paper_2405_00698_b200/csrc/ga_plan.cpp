// ga_plan.cpp — the breeding-plan scan (evolution.hpp:267-289 in rank
// space), written for throughput.  The GA stream is ONE sequential
// mt19937_64 (rng.hpp:15-39), and a generation of P children consumes about
// P * (1 + crossover_rate) * n_params draws: ~14k per child for the default
// 8710-parameter controller, ~27M at P = 2048 (8 ranks x 256), replayed on
// every rank and overlapped with the GPU evaluate.  Per draw the naive loop
// pays a branchy twist/temper call plus a double compare; here:
//
//  * Stream — mt19937_64 generated a buffer of 32 blocks at a time: each
//    312-word twist writes the next state to its own slot and the tempered
//    outputs beside it, so both loops vectorise (AVX-512 or AVX2 when the host
//    has it, picked at run time; integer work only).  Outputs are identical to
//    std::mt19937_64, and the state round-trips through the libstdc++ text
//    format (312 words, then the position), so checkpoints and
//    vx_evo_rng_state are untouched;
//  * uniform01(r) < p is the integer test (r >> 11) < ceil(p * 2^53) (exact:
//    scaling by a power of two and the ceiling of a double below 2^53 are
//    both exact); for p = 1/2 it is "top bit clear", so a crossover mask
//    word is 32 sign bits;
//  * the mutation loop jumps from hit to hit (5% of draws at the default
//    rate) instead of testing parameter by parameter, and each mutation's
//    Box-Muller normal (rng.hpp:29-33) is DEFERRED: the scan records its two
//    raw words and the glibc sqrt/log/cos run afterwards on worker threads,
//    in generic (no-FMA) code — same expression, same libm, same bits.
#include "ga_plan.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <sstream>
#include <condition_variable>
#include <mutex>
#include <new>
#include <thread>

#include <immintrin.h>

namespace vx {
namespace {

constexpr int kN = 312, kM = 156;
constexpr int kBlocks = 32;
constexpr size_t kBuf = static_cast<size_t>(kBlocks) * kN;

__attribute__((always_inline)) inline uint64_t mix(uint64_t hi, uint64_t lo, uint64_t far) {
    const uint64_t y = (hi & 0xFFFFFFFF80000000ull) | (lo & 0x7FFFFFFFull);
    return far ^ (y >> 1) ^ ((0ull - (y & 1ull)) & 0xB5026F5AA96619E9ull);
}
__attribute__((always_inline)) inline uint64_t temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    return y ^ (y >> 43);
}

// libstdc++ _M_gen_rand with the old state in `x` and the new one in `y`
// (in the in-place original, x[k+M-N] and x[0] are already new).
__attribute__((always_inline)) inline void twist(const uint64_t* __restrict__ x, uint64_t* __restrict__ y,
                                                 uint64_t* __restrict__ out) {
    for (int k = 0; k < kN - kM; ++k) y[k] = mix(x[k], x[k + 1], x[k + kM]);
    for (int k = kN - kM; k < kN - 1; ++k) y[k] = mix(x[k], x[k + 1], y[k + kM - kN]);
    y[kN - 1] = mix(x[kN - 1], y[0], y[kM - 1]);
    for (int k = 0; k < kN; ++k) out[k] = temper(y[k]);
}

struct Stream {
    alignas(64) uint64_t raw[kBuf];  // state after each block's twist
    alignas(64) uint64_t out[kBuf];  // tempered outputs of that block
    size_t pos = 0;                  // next output
};

// blocks first..kBlocks-1; block 0 (when first == 0) twists from `prev`
__attribute__((always_inline)) inline void fill_blocks(Stream& s, const uint64_t* prev, int first) {
    for (int j = first; j < kBlocks; ++j) {
        twist(j == 0 ? prev : s.raw + static_cast<size_t>(j - 1) * kN, s.raw + static_cast<size_t>(j) * kN,
              s.out + static_cast<size_t>(j) * kN);
    }
}
void fill_generic(Stream& s, const uint64_t* prev, int first) { fill_blocks(s, prev, first); }
__attribute__((target("avx2"))) void fill_avx2(Stream& s, const uint64_t* prev, int first) {
    fill_blocks(s, prev, first);
}
__attribute__((target("avx512f,avx512vl"))) void fill_avx512(Stream& s, const uint64_t* prev, int first) {
    fill_blocks(s, prev, first);
}
using FillFn = void (*)(Stream&, const uint64_t*, int);

// bit k of the result: q[k] is a hit, i.e. uniform01(q[k]) < p <=> (q[k] >> 11) < t
uint64_t hits64_generic(const uint64_t* q, uint64_t t) {
    uint64_t m = 0;
    for (int k = 0; k < 64; ++k) m |= static_cast<uint64_t>((q[k] >> 11) < t) << k;
    return m;
}
__attribute__((target("avx2"))) uint64_t hits64_avx2(const uint64_t* q, uint64_t t) {
    const __m256i vt = _mm256_set1_epi64x(static_cast<long long>(t));  // t <= 2^53: signed compare is exact
    uint64_t m = 0;
    for (int k = 0; k < 64; k += 4) {
        const __m256i v = _mm256_srli_epi64(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(q + k)), 11);
        const int b = _mm256_movemask_pd(_mm256_castsi256_pd(_mm256_cmpgt_epi64(vt, v)));
        m |= static_cast<uint64_t>(b) << k;
    }
    return m;
}
__attribute__((target("avx512f"))) uint64_t hits64_avx512(const uint64_t* q, uint64_t t) {
    const __m512i vt = _mm512_set1_epi64(static_cast<long long>(t));
    uint64_t m = 0;
    for (int k = 0; k < 64; k += 8) {
        const __m512i v = _mm512_srli_epi64(_mm512_loadu_si512(q + k), 11);
        m |= static_cast<uint64_t>(_mm512_cmplt_epu64_mask(v, vt)) << k;
    }
    return m;
}
// bit k: top bit of q[k] clear, i.e. uniform01(q[k]) < 0.5 (crossover mask)
uint32_t half32_generic(const uint64_t* q) {
    uint32_t w = 0;
    for (int k = 0; k < 32; ++k) w |= static_cast<uint32_t>(~q[k] >> 63) << k;
    return w;
}
__attribute__((target("avx2"))) uint32_t half32_avx2(const uint64_t* q) {
    uint32_t w = 0;
    for (int k = 0; k < 32; k += 4)
        w |= static_cast<uint32_t>(_mm256_movemask_pd(_mm256_loadu_pd(reinterpret_cast<const double*>(q + k)))) << k;
    return ~w;
}

struct Kernels {
    FillFn fill;
    uint64_t (*hits64)(const uint64_t*, uint64_t);
    uint32_t (*half32)(const uint64_t*);
};

void load(Stream& s, const std::mt19937_64& r) {
    std::stringstream ss;
    ss << r;
    uint64_t* x = s.raw;
    for (int i = 0; i < kN; ++i) ss >> x[i];
    size_t p = 0;
    ss >> p;
    for (int i = 0; i < kN; ++i) s.out[i] = temper(x[i]);
    s.pos = p;  // p == 312: block 0 is used up, the next output opens block 1
}

void store(const Stream& s, std::mt19937_64& r) {
    // libstdc++ never rests at position 0 (it twists on demand), so a block
    // boundary is written as (previous block, 312) like std::mt19937_64
    // would hold it — the text state then matches the reference byte for byte.
    // s.pos >= 1 here: a refill is only ever followed by a draw.
    const size_t blk = (s.pos - 1) / kN;
    const size_t off = s.pos - blk * kN;  // 1..312
    std::stringstream ss;
    for (int i = 0; i < kN; ++i) ss << s.raw[blk * kN + i] << ' ';
    ss << off;
    ss >> r;
}

// Box-Muller from the two raw words of Rng::normal (rng.hpp:29-33); generic
// target so no FMA contraction can change a rounding.
double box_muller(uint64_t r1, uint64_t r2) {
    const double u1 = (static_cast<double>(r1 >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = static_cast<double>(r2 >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

// uniform01(r) < p <=> (r >> 11) < u01_threshold(p)
uint64_t u01_threshold(double p) {
    if (!(p > 0.0)) return 0;
    if (p >= 1.0) return uint64_t(1) << 53;
    return static_cast<uint64_t>(std::ceil(p * 0x1.0p53));
}

// Normals of full chunks, computed by a small pool while the scan runs on.
// Workers see a chunk only through the job copied out under `mu`: the scan
// thread keeps growing MutStore's vectors (which may reallocate) and its
// entry count, so no worker ever reads MutStore's members.
struct NormalJob {
    MutEntry* e;
    const uint64_t* r2;
    size_t count;
};
struct NormalPool {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<NormalJob> jobs;  // published chunks, in order
    size_t claimed = 0;           // jobs taken
    bool done = false;
    std::vector<std::thread> threads;
};

}  // namespace

struct MutWriter {
    MutStore& st;
    NormalPool& pool;
    double scale;

    void fill_chunk(const NormalJob& job) {
        MutEntry* e = job.e;
        const uint64_t* r2 = job.r2;
        for (size_t q = 0; q < job.count; ++q) {
            uint64_t r1;
            std::memcpy(&r1, &e[q].delta, sizeof(r1));
            e[q].delta = box_muller(r1, r2[q]) * scale;
        }
    }
    // claim chunks until the scan is over and every chunk is taken
    void work() {
        for (;;) {
            NormalJob job;
            {
                std::unique_lock<std::mutex> lk(pool.mu);
                pool.cv.wait(lk, [&] { return pool.claimed < pool.jobs.size() || pool.done; });
                if (pool.claimed >= pool.jobs.size()) return;  // done
                job = pool.jobs[pool.claimed++];
            }
            fill_chunk(job);
        }
    }
    inline void append(int32_t c, int32_t i, uint64_t r1, uint64_t r2) {
        const size_t j = st.n_ / MutStore::kChunk, k = st.n_ % MutStore::kChunk;
        if (k == 0 && j == st.e_.size()) grow();
        MutEntry& m = st.e_[j][k];
        m.child = c;
        m.index = i;
        std::memcpy(&m.delta, &r1, sizeof(r1));
        st.r2_[j][k] = r2;
        ++st.n_;
        if (k + 1 == MutStore::kChunk) publish(j);
    }
    // hand chunk j (complete: no more appends to it) to the workers
    void publish(size_t j) {
        const NormalJob job{st.e_[j], st.r2_[j], st.chunk_size(j)};
        {
            std::lock_guard<std::mutex> lk(pool.mu);
            pool.jobs.push_back(job);
        }
        pool.cv.notify_one();
    }
    void grow() {  // a slab as large as everything so far (1..256 chunks): few, large pinned allocations
        const size_t n = std::min<size_t>(256, std::max<size_t>(1, st.e_.size()));
        const size_t bytes = n * MutStore::kChunk * sizeof(MutEntry);
        void* p = st.alloc_ ? st.alloc_(bytes) : ::operator new(bytes, std::nothrow);
        if (!p) throw std::bad_alloc();
        st.slabs_.push_back(p);
        uint64_t* r2 = new uint64_t[n * MutStore::kChunk];
        st.r2_slabs_.push_back(r2);
        for (size_t c = 0; c < n; ++c) {
            st.e_.push_back(static_cast<MutEntry*>(p) + c * MutStore::kChunk);
            st.r2_.push_back(r2 + c * MutStore::kChunk);
            st.slab_of_.push_back(static_cast<uint32_t>(st.slabs_.size() - 1));
        }
    }
};

MutStore::~MutStore() {
    for (void* p : slabs_) {
        if (free_)
            free_(p);
        else
            ::operator delete(p);
    }
    for (uint64_t* p : r2_slabs_) delete[] p;
}

void MutStore::flatten(std::vector<MutEntry>& out) const {
    out.resize(n_);
    for (size_t j = 0; j < chunks(); ++j) std::memcpy(out.data() + j * kChunk, e_[j], chunk_size(j) * sizeof(MutEntry));
}

namespace {

struct ScanOut {
    std::vector<ChildPlan>* plan;
    std::vector<uint32_t>* masks;
    MutWriter* mut;
};

void scan_body(Stream& s, const Kernels& kern, const PlanParams& a, const ScanOut& o) {
    const FillFn fill = kern.fill;
    uint64_t tmp[kN];
    const size_t end = kBuf;
    fill(s, nullptr, 1);  // blocks 1.. from the loaded block 0
    auto refill = [&]() {
        std::memcpy(tmp, s.raw + kBuf - kN, sizeof(tmp));
        fill(s, tmp, 0);
        s.pos = 0;
    };
    auto next = [&]() -> uint64_t {
        if (s.pos == end) refill();
        return s.out[s.pos++];
    };
    const uint64_t uP = static_cast<uint64_t>(a.P), thrP = (0 - uP) % uP;
    auto index = [&]() -> uint64_t {  // Rng::index (rng.hpp:35-39)
        for (;;) {
            const uint64_t x = next();
            if (x >= thrP) return x % uP;
        }
    };
    auto tournament = [&]() -> int32_t {  // tournament_select (evolution.hpp:169-173)
        uint64_t w = index();
        for (int k = 1; k < a.tournament_size; ++k) w = std::min<uint64_t>(w, index());
        return static_cast<int32_t>(w);
    };
    const uint64_t t_cx = u01_threshold(a.crossover_rate), t_mut = u01_threshold(a.mutation_rate);
    const int64_t np = a.np;
    int slots = 0;
    for (int c = a.n_elite; c < a.P; ++c) {
        ChildPlan& p = (*o.plan)[c - a.n_elite];
        p.pa = tournament();
        p.pb = -1;
        p.mask_slot = -1;
        p.pad = 0;
        if ((next() >> 11) < t_cx) {  // crossover (evolution.hpp:143-155): bit = uniform01 < 0.5
            p.pb = tournament();
            p.mask_slot = slots++;
            const size_t base = o.masks->size();
            o.masks->resize(base + a.mask_words, 0u);
            uint32_t* m = o.masks->data() + base;
            for (int64_t w = 0; w * 32 < np; ++w) {
                const int nb = static_cast<int>(std::min<int64_t>(32, np - w * 32));
                uint32_t word = 0;
                if (nb == 32 && end - s.pos >= 32) {
                    word = kern.half32(s.out + s.pos);
                    s.pos += 32;
                } else {
                    for (int b = 0; b < nb; ++b) word |= static_cast<uint32_t>(~next() >> 63) << b;
                }
                m[w] = word;
            }
        }
        // mutate (evolution.hpp:160-165): a hit (uniform01 < rate) draws two
        // more words for its normal; walk 64-draw windows hit by hit
        int64_t i = 0;
        while (i < np) {
            if (end - s.pos < 64 + 2) {  // window would cross the buffer end: one parameter the slow way
                if ((next() >> 11) < t_mut) {
                    const uint64_t r1 = next();
                    o.mut->append(c, static_cast<int32_t>(i), r1, next());
                }
                ++i;
                continue;
            }
            const uint64_t* q = s.out + s.pos;
            const uint64_t m = kern.hits64(q, t_mut);
            int off = 0;  // window offset of the next parameter's draw (may end at 64..66)
            while (off < 64) {
                const uint64_t mm = m >> off;
                const int64_t left = np - i;
                if (mm == 0) {
                    const int64_t adv = std::min<int64_t>(64 - off, left);
                    i += adv;
                    off += static_cast<int>(adv);
                    break;
                }
                const int k = __builtin_ctzll(mm);
                if (k >= left) {  // this child's parameters end before the hit
                    i = np;
                    off += static_cast<int>(left);
                    break;
                }
                i += k;
                off += k;
                o.mut->append(c, static_cast<int32_t>(i), q[off + 1], q[off + 2]);
                off += 3;
                ++i;
                if (i >= np) break;
            }
            s.pos += off;
        }
    }
}

}  // namespace

void plan_scan(std::mt19937_64& rng, const PlanParams& a, std::vector<ChildPlan>& plan, std::vector<uint32_t>& masks,
               MutStore& mut) {
    plan.resize(std::max(1, a.P - a.n_elite));
    masks.clear();
    mut.clear();
    if (a.P - a.n_elite <= 0) return;  // no draws at all
    static const Kernels kern = __builtin_cpu_supports("avx512f") ? Kernels{fill_avx512, hits64_avx512, half32_avx2}
                                : __builtin_cpu_supports("avx2") ? Kernels{fill_avx2, hits64_avx2, half32_avx2}
                                                                 : Kernels{fill_generic, hits64_generic, half32_generic};
    NormalPool pool;
    MutWriter w{mut, pool, a.mutation_scale};
    // workers only when the generation will fill several chunks
    const double expect = std::max(0.0, std::min(1.0, a.mutation_rate)) * static_cast<double>(a.np) *
                          static_cast<double>(a.P - a.n_elite);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nw = expect >= 4.0 * MutStore::kChunk ? std::min<size_t>(hw > 1 ? hw - 1 : 1, 6) : 0;
    for (size_t t = 0; t < nw; ++t) pool.threads.emplace_back([&w] { w.work(); });
    {
        std::unique_ptr<Stream> s(new Stream);
        load(*s, rng);
        const ScanOut o{&plan, &masks, &w};
        scan_body(*s, kern, a, o);
        store(*s, rng);
    }
    if (mut.size() % MutStore::kChunk != 0) w.publish(mut.chunks() - 1);  // the partial tail chunk
    {
        std::lock_guard<std::mutex> lk(pool.mu);
        pool.done = true;
    }
    pool.cv.notify_all();
    w.work();  // the scan thread helps with the tail
    for (auto& th : pool.threads) th.join();
}

}  // namespace vx
