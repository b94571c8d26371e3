/* oracle/voxevo_oracle.c — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Plain-C restatement of the reference hot path (arXiv 2405.00698 `voxevo`,
 * /root/reference/proj/include/voxevo headers), written operation-for-operation
 * so that, built with -O2 -ffp-contract=off against the same glibc libm, it is
 * BIT-IDENTICAL to the compiled reference (oracle/_ref/libvoxevo_ref.so).
 * tests/test_oracle_pinning.py pins it against the reference itself and
 * against the golden vectors in tests/golden/ (reference KATs and outputs).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load this library — it is the checker, never the product.
 *
 * Parity notes: every sum keeps the reference's
 * left-to-right order with separately rounded mul/add; libm calls
 * (exp, tanh, sin, cos, log) go to the host glibc exactly as the reference's
 * do, so results are libm-variant dependent in the same way.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------ mt19937_64
 * std::mt19937_64 (rng.hpp:55), standard parameters. */
#define MT_N 312
#define MT_M 156
typedef struct {
    uint64_t mt[MT_N];
    int idx;
} orc_mt;

static void mt_seed(orc_mt* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
}

static void mt_twist(orc_mt* r) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    for (int i = 0; i < MT_N; ++i) {
        uint64_t y = (r->mt[i] & UM) | (r->mt[(i + 1) % MT_N] & LM);
        r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
    }
    r->idx = 0;
}

static uint64_t mt_next(orc_mt* r) {
    if (r->idx >= MT_N) mt_twist(r);
    uint64_t z = r->mt[r->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* Rng::uniform01 (rng.hpp:23) */
static double rng_uniform01(orc_mt* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }
/* Rng::normal (rng.hpp:26-30); 2.0 * M_PI * u2 evaluated left to right */
static double rng_normal(orc_mt* r) {
    double u1 = ((double)(mt_next(r) >> 11) + 0.5) * 0x1.0p-53;
    double u2 = (double)(mt_next(r) >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}
/* Rng::index (rng.hpp:33-39) */
static uint64_t rng_index(orc_mt* r, uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
        uint64_t x = mt_next(r);
        if (x >= threshold) return x % n;
    }
}

/* libstdc++ text form of the engine (rng.hpp:41-45): 312 words then index. */
static int64_t mt_state_text(const orc_mt* r, char* buf, int64_t cap) {
    char tmp[32];
    int64_t len = 0;
    for (int i = 0; i <= MT_N; ++i) {
        int n = (i < MT_N) ? snprintf(tmp, sizeof tmp, "%llu", (unsigned long long)r->mt[i])
                           : snprintf(tmp, sizeof tmp, "%d", r->idx);
        if (i > 0) {
            if (buf && len + 1 < cap) buf[len] = ' ';
            ++len;
        }
        for (int c = 0; c < n; ++c) {
            if (buf && len + 1 < cap) buf[len] = tmp[c];
            ++len;
        }
    }
    if (buf && cap > 0) buf[len < cap ? len : cap - 1] = 0;
    return len;
}

static int mt_state_parse(orc_mt* r, const char* s) {
    char* end = NULL;
    for (int i = 0; i < MT_N; ++i) {
        r->mt[i] = strtoull(s, &end, 10);
        if (end == s) return -1;
        s = end;
    }
    r->idx = (int)strtol(s, &end, 10);
    if (end == s) return -1;
    return 0;
}

ORC_EXPORT void orc_rng_draws(uint64_t seed, int64_t n, uint64_t* out) {
    orc_mt r;
    mt_seed(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = mt_next(&r);
}
ORC_EXPORT void orc_rng_uniform(uint64_t seed, int64_t n, double* out) {
    orc_mt r;
    mt_seed(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_uniform01(&r);
}
ORC_EXPORT void orc_rng_normal(uint64_t seed, int64_t n, double* out) {
    orc_mt r;
    mt_seed(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_normal(&r);
}
ORC_EXPORT void orc_rng_index(uint64_t seed, int64_t n, uint64_t range, uint64_t* out) {
    orc_mt r;
    mt_seed(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_index(&r, range);
}
ORC_EXPORT int64_t orc_rng_state(uint64_t seed, int64_t skip, char* buf, int64_t cap) {
    orc_mt r;
    mt_seed(&r, seed);
    for (int64_t i = 0; i < skip; ++i) mt_next(&r);
    return mt_state_text(&r, buf, cap);
}
ORC_EXPORT void orc_rng_draws_from_state(const char* state, int64_t n, uint64_t* out) {
    orc_mt r;
    mt_state_parse(&r, state);
    for (int64_t i = 0; i < n; ++i) out[i] = mt_next(&r);
}

/* ---------------------------------------------------------------- genome.hpp */
#define KTWOPI 6.283185307179586476925286766559 /* genome.hpp:16 */
#define NMAT 5

typedef struct {
    int m;
    int nh;
    int widths[16];
} orc_arch;

static int64_t arch_param_count(const orc_arch* a) {
    int64_t n = 0;
    int in = 2 * a->m;
    for (int l = 0; l < a->nh; ++l) {
        n += (int64_t)in * a->widths[l] + a->widths[l];
        in = a->widths[l];
    }
    n += (int64_t)in * NMAT + NMAT;
    n += (int64_t)in + 1;
    return n;
}

ORC_EXPORT int64_t orc_param_count(int m, int nh, const int* widths) {
    orc_arch a = {m, nh, {0}};
    for (int i = 0; i < nh; ++i) a.widths[i] = widths[i];
    return arch_param_count(&a);
}

/* detail::init_layer (genome.hpp:106-115): W row-major uniform, b = 0 */
static double* init_layer(double* p, int in, int out, orc_mt* r) {
    const double limit = sqrt(6.0 / (double)(in + out));
    for (int64_t i = 0; i < (int64_t)in * out; ++i) p[i] = (2.0 * rng_uniform01(r) - 1.0) * limit;
    p += (int64_t)in * out;
    for (int i = 0; i < out; ++i) p[i] = 0.0;
    return p + out;
}

/* sample_genome (genome.hpp:146-166) */
ORC_EXPORT void orc_sample_genome(int m, double sigma, int nh, const int* widths, uint64_t seed, double* params,
                                  double* bmat) {
    orc_mt r;
    mt_seed(&r, seed);
    for (int i = 0; i < 3 * m; ++i) bmat[i] = sigma * rng_normal(&r);
    int in = 2 * m;
    double* p = params;
    for (int l = 0; l < nh; ++l) {
        p = init_layer(p, in, widths[l], &r);
        in = widths[l];
    }
    p = init_layer(p, in, NMAT, &r);
    init_layer(p, in, 1, &r);
}

/* gaussian_encode (genome.hpp:169-179) */
static void encode(const double* v, const double* b, int m, double* out) {
    for (int r = 0; r < m; ++r) {
        const double* row = b + 3 * r;
        const double phase = KTWOPI * (row[0] * v[0] + row[1] * v[1] + row[2] * v[2]);
        out[r] = cos(phase);
        out[m + r] = sin(phase);
    }
}
ORC_EXPORT void orc_gaussian_encode(const double* v, const double* bmat, int m, double* out) {
    encode(v, bmat, m, out);
}

/* detail::affine (genome.hpp:118-126): acc = b_r; acc += w*x, c ascending */
static const double* affine(const double* p, int in, int out, const double* x, double* y) {
    const double* w = p;
    const double* b = p + (int64_t)in * out;
    for (int r = 0; r < out; ++r) {
        const double* wr = w + (int64_t)r * in;
        double acc = b[r];
        for (int c = 0; c < in; ++c) acc += wr[c] * x[c];
        y[r] = acc;
    }
    return b + out;
}

/* detail::stable_sigmoid (genome.hpp:128-138) */
static double stable_sigmoid(double z) {
    double s;
    if (z >= 0.0) {
        s = 1.0 / (1.0 + exp(-z));
    } else {
        const double e = exp(z);
        s = e / (1.0 + e);
    }
    if (s < 1e-12) s = 1e-12; /* std::clamp(s, 1e-12, 1 - 1e-12) */
    if (s > 1.0 - 1e-12) s = 1.0 - 1e-12;
    return s;
}

/* forward (genome.hpp:187-211) */
static void forward(const orc_arch* a, const double* params, const double* bmat, const double* v, double* probs,
                    double* weight) {
    double bufx[1024], bufy[1024];
    double* x = bufx;
    double* y = bufy;
    encode(v, bmat, a->m, x);
    int in = 2 * a->m;
    const double* p = params;
    for (int l = 0; l < a->nh; ++l) {
        p = affine(p, in, a->widths[l], x, y);
        for (int i = 0; i < a->widths[l]; ++i) y[i] = tanh(y[i]);
        double* t = x;
        x = y;
        y = t;
        in = a->widths[l];
    }
    double logits[NMAT];
    p = affine(p, in, NMAT, x, logits);
    double mx = logits[0]; /* std::max_element: first maximal */
    for (int i = 1; i < NMAT; ++i)
        if (mx < logits[i]) mx = logits[i];
    double sum = 0.0;
    for (int i = 0; i < NMAT; ++i) {
        probs[i] = exp(logits[i] - mx);
        sum += probs[i];
    }
    for (int i = 0; i < NMAT; ++i) probs[i] /= sum;
    double wl;
    affine(p, in, 1, x, &wl);
    *weight = stable_sigmoid(wl);
}

static orc_arch mk_arch(int m, int nh, const int* widths) {
    orc_arch a;
    memset(&a, 0, sizeof a);
    a.m = m;
    a.nh = nh;
    for (int i = 0; i < nh; ++i) a.widths[i] = widths[i];
    return a;
}

ORC_EXPORT void orc_forward(int m, int nh, const int* widths, const double* params, const double* bmat,
                            const double* v, double* probs, double* weight) {
    orc_arch a = mk_arch(m, nh, widths);
    forward(&a, params, bmat, v, probs, weight);
}

/* ------------------------------------------------------------ morphology.hpp */
/* decode (morphology.hpp:141-157) */
static void decode(const orc_arch* a, const double* params, const double* bmat, int w, int h, int d, uint8_t* mat,
                   double* wt) {
    for (int z = 0; z < d; ++z)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                const double v[3] = {(x + 0.5) / w, (y + 0.5) / h, (z + 0.5) / d};
                double probs[NMAT], weight;
                forward(a, params, bmat, v, probs, &weight);
                int best = 0;
                for (int i = 1; i < NMAT; ++i)
                    if (probs[i] > probs[best]) best = i;
                const int idx = x + w * (y + h * z);
                mat[idx] = (uint8_t)best;
                wt[idx] = weight < 0.1 ? 0.1 : (weight > 1.0 ? 1.0 : weight); /* clamp(q.weight, kMin, 1) */
            }
}
ORC_EXPORT void orc_decode(int m, int nh, const int* widths, const double* params, const double* bmat, int w, int h,
                           int d, uint8_t* mat, double* wt) {
    orc_arch a = mk_arch(m, nh, widths);
    decode(&a, params, bmat, w, h, d, mat, wt);
}

/* largest_component (morphology.hpp:162-208): DFS from ascending seeds,
 * strict > keeps the lowest-seed component on ties. */
static void largest_component(int w, int h, int d, const uint8_t* in, uint8_t* out) {
    const int n = w * h * d;
    int* label = (int*)malloc(sizeof(int) * (size_t)n);
    int* stack = (int*)malloc(sizeof(int) * (size_t)n);
    for (int i = 0; i < n; ++i) label[i] = -1;
    int best_label = -1, best_count = 0, next_label = 0;
    static const int dx[6] = {1, -1, 0, 0, 0, 0}, dy[6] = {0, 0, 1, -1, 0, 0}, dz[6] = {0, 0, 0, 0, 1, -1};
    for (int seed = 0; seed < n; ++seed) {
        if (label[seed] >= 0 || in[seed] == 0) continue;
        int count = 0, sp = 0;
        stack[sp++] = seed;
        label[seed] = next_label;
        while (sp > 0) {
            const int idx = stack[--sp];
            ++count;
            const int x = idx % w, y = (idx / w) % h, z = idx / (w * h);
            for (int k = 0; k < 6; ++k) {
                const int nx = x + dx[k], ny = y + dy[k], nz = z + dz[k];
                if (nx < 0 || nx >= w || ny < 0 || ny >= h || nz < 0 || nz >= d) continue;
                const int ni = nx + w * (ny + h * nz);
                if (label[ni] >= 0 || in[ni] == 0) continue;
                label[ni] = next_label;
                stack[sp++] = ni;
            }
        }
        if (count > best_count) {
            best_count = count;
            best_label = next_label;
        }
        ++next_label;
    }
    for (int i = 0; i < n; ++i) out[i] = (in[i] != 0 && label[i] != best_label) ? 0 : in[i];
    free(label);
    free(stack);
}
ORC_EXPORT void orc_largest_component(int w, int h, int d, const uint8_t* in, uint8_t* out) {
    largest_component(w, h, d, in, out);
}

/* bench_robot (bench.hpp:35-44) */
ORC_EXPORT void orc_bench_robot(int n, uint8_t* mat, double* wt) {
    static const uint8_t cyc[4] = {1, 3, 2, 4};
    for (int z = 0; z < n; ++z)
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < n; ++x) {
                const int i = x + n * (y + n * z);
                mat[i] = cyc[(x + 2 * y + 3 * z) % 4];
                wt[i] = 1.0;
            }
}

/* system: plain SoA owned by the handle */
typedef struct {
    int nm, ns;
    double *pos, *vel, *mass; /* 3*nm, 3*nm, nm */
    int *si, *sj;
    double *k, *rest0, *zeta, *sign, *amp, *phase;
    uint8_t* has_act;
    double plane[4];
    /* SimWorkspace (physics.hpp:127-186), built lazily */
    int ws_ready;
    double *f, *damp, *amp_rest, *sin_ph, *cos_ph, *gdamp, *inc_sign;
    int *inc_off, *inc_spring;
    double max_speed_sq;
    uint64_t spring_updates;
    int any_act;
} orc_sys;

static orc_sys* sys_alloc(int nm, int ns) {
    orc_sys* s = (orc_sys*)calloc(1, sizeof(orc_sys));
    s->nm = nm;
    s->ns = ns;
    s->pos = (double*)calloc((size_t)3 * nm + 1, sizeof(double));
    s->vel = (double*)calloc((size_t)3 * nm + 1, sizeof(double));
    s->mass = (double*)calloc((size_t)nm + 1, sizeof(double));
    s->si = (int*)calloc((size_t)ns + 1, sizeof(int));
    s->sj = (int*)calloc((size_t)ns + 1, sizeof(int));
    s->k = (double*)calloc((size_t)ns + 1, sizeof(double));
    s->rest0 = (double*)calloc((size_t)ns + 1, sizeof(double));
    s->zeta = (double*)calloc((size_t)ns + 1, sizeof(double));
    s->sign = (double*)calloc((size_t)ns + 1, sizeof(double));
    s->amp = (double*)calloc((size_t)ns + 1, sizeof(double));
    s->phase = (double*)calloc((size_t)ns + 1, sizeof(double));
    s->has_act = (uint8_t*)calloc((size_t)ns + 1, 1);
    s->plane[0] = 1e5;
    s->plane[1] = 0.1;
    s->plane[2] = 0.6;
    s->plane[3] = 1.0;
    return s;
}

static void ws_free(orc_sys* s) {
    if (!s->ws_ready) return;
    free(s->f);
    free(s->damp);
    free(s->amp_rest);
    free(s->sin_ph);
    free(s->cos_ph);
    free(s->gdamp);
    free(s->inc_sign);
    free(s->inc_off);
    free(s->inc_spring);
    s->ws_ready = 0;
}

ORC_EXPORT void orc_sys_free(void* h) {
    orc_sys* s = (orc_sys*)h;
    if (!s) return;
    ws_free(s);
    free(s->pos);
    free(s->vel);
    free(s->mass);
    free(s->si);
    free(s->sj);
    free(s->k);
    free(s->rest0);
    free(s->zeta);
    free(s->sign);
    free(s->amp);
    free(s->phase);
    free(s->has_act);
    free(s);
}

typedef struct {
    int64_t key; /* i * nm + j */
    int seq;     /* contribution order = voxel scan order */
    double k_contrib;
    int vox_mat;
    double vox_w;
} contrib_t;

static int contrib_cmp(const void* a, const void* b) {
    const contrib_t* x = (const contrib_t*)a;
    const contrib_t* y = (const contrib_t*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

static int int_cmp(const void* a, const void* b) {
    const int x = *(const int*)a, y = *(const int*)b;
    return x < y ? -1 : (x > y);
}

static double base_stiffness(const double* t, int m) {
    switch (m) {
        case 1:
        case 2: return t[0];
        case 3: return t[1];
        case 4: return t[2];
    }
    return 0.0;
}

static const double kDefaultTable[8] = {2e3, 1e3, 1e4, 0.1, 0.25, M_PI, 0.1, 0.1};

/* build_mass_spring (morphology.hpp:217-299).  std::map<pair> iteration ==
 * lexicographic (i,j) == sort by key; per-key contributions accumulate in
 * voxel scan order (stable on seq). */
ORC_EXPORT void* orc_build(int w, int h, int d, const uint8_t* mat, const double* wt, const double* table8,
                           const double* plane4) {
    const double* t = table8 ? table8 : kDefaultTable;
    const int vw = w + 1, vh = h + 1;
    int nvox = 0;
    for (int i = 0; i < w * h * d; ++i)
        if (mat[i]) ++nvox;
    if (nvox == 0) return NULL; /* empty_robot, morphology.hpp:230 */
    int* keys = (int*)malloc(sizeof(int) * 8 * (size_t)nvox);
    int nk = 0;
    for (int z = 0; z < d; ++z)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                if (!mat[x + w * (y + h * z)]) continue;
                for (int c = 0; c < 8; ++c)
                    keys[nk++] = (x + (c & 1)) + vw * ((y + ((c >> 1) & 1)) + vh * (z + ((c >> 2) & 1)));
            }
    qsort(keys, (size_t)nk, sizeof(int), int_cmp);
    int nm = 0;
    for (int i = 0; i < nk; ++i)
        if (i == 0 || keys[i] != keys[i - 1]) keys[nm++] = keys[i];
    /* key -> mass index via dense table over the vertex lattice */
    const int nvert = vw * vh * (d + 1);
    int* key_to_mass = (int*)malloc(sizeof(int) * (size_t)nvert);
    for (int i = 0; i < nm; ++i) key_to_mass[keys[i]] = i;

    contrib_t* cs = (contrib_t*)malloc(sizeof(contrib_t) * 28 * (size_t)nvox);
    int nc = 0;
    for (int z = 0; z < d; ++z)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                const int ci = x + w * (y + h * z);
                if (!mat[ci]) continue;
                int corner[8];
                for (int c = 0; c < 8; ++c)
                    corner[c] = key_to_mass[(x + (c & 1)) + vw * ((y + ((c >> 1) & 1)) + vh * (z + ((c >> 2) & 1)))];
                const double k_contrib = wt[ci] * base_stiffness(t, mat[ci]);
                for (int p = 0; p < 8; ++p)
                    for (int q = p + 1; q < 8; ++q) {
                        const int a = corner[p] < corner[q] ? corner[p] : corner[q];
                        const int b = corner[p] < corner[q] ? corner[q] : corner[p];
                        cs[nc].key = (int64_t)a * nm + b;
                        cs[nc].seq = nc;
                        cs[nc].k_contrib = k_contrib;
                        cs[nc].vox_mat = mat[ci];
                        cs[nc].vox_w = wt[ci];
                        ++nc;
                    }
            }
    qsort(cs, (size_t)nc, sizeof(contrib_t), contrib_cmp);
    int ns = 0;
    for (int i = 0; i < nc; ++i)
        if (i == 0 || cs[i].key != cs[i - 1].key) ++ns;

    orc_sys* s = sys_alloc(nm, ns);
    if (plane4) memcpy(s->plane, plane4, sizeof s->plane);
    for (int i = 0; i < nm; ++i) {
        const int key = keys[i];
        const int x = key % vw, y = (key / vw) % vh, z = key / (vw * vh);
        s->pos[3 * i] = x * t[6];
        s->pos[3 * i + 1] = y * t[6];
        s->pos[3 * i + 2] = z * t[6];
        s->mass[i] = t[7];
    }
    double min_z = s->pos[2];
    for (int i = 0; i < nm; ++i)
        if (s->pos[3 * i + 2] < min_z) min_z = s->pos[3 * i + 2];
    for (int i = 0; i < nm; ++i) s->pos[3 * i + 2] -= min_z;

    int q = -1;
    double k_sum = 0.0;
    int count = 0;
    for (int e = 0; e <= nc; ++e) {
        if (e == nc || e == 0 || cs[e].key != cs[e - 1].key) {
            if (q >= 0) {
                s->k[q] = k_sum / count;
                const double* A = s->pos + 3 * s->si[q];
                const double* B = s->pos + 3 * s->sj[q];
                s->rest0[q] = sqrt((B[0] - A[0]) * (B[0] - A[0]) + (B[1] - A[1]) * (B[1] - A[1]) +
                                   (B[2] - A[2]) * (B[2] - A[2]));
                s->zeta[q] = t[3];
            }
            if (e == nc) break;
            ++q;
            s->si[q] = (int)(cs[e].key / nm);
            s->sj[q] = (int)(cs[e].key % nm);
            k_sum = 0.0;
            count = 0;
        }
        k_sum += cs[e].k_contrib;
        count += 1;
        const int m = cs[e].vox_mat;
        if ((m == 1 || m == 2) && !s->has_act[q]) {
            s->has_act[q] = 1;
            s->sign[q] = m == 1 ? 1.0 : -1.0;
            s->amp[q] = cs[e].vox_w * t[4];
            s->phase[q] = cs[e].vox_w * t[5];
        }
    }
    free(cs);
    free(keys);
    free(key_to_mass);
    return s;
}

ORC_EXPORT void* orc_sys_make(int nm, int ns, const double* pos, const double* vel, const double* mass,
                              const int* si, const int* sj, const double* k, const double* rest0, const double* zeta,
                              const uint8_t* has_act, const double* sign, const double* amp, const double* phase,
                              const double* plane4) {
    orc_sys* s = sys_alloc(nm, ns);
    memcpy(s->pos, pos, sizeof(double) * 3 * (size_t)nm);
    memcpy(s->vel, vel, sizeof(double) * 3 * (size_t)nm);
    memcpy(s->mass, mass, sizeof(double) * (size_t)nm);
    for (int q = 0; q < ns; ++q) {
        s->si[q] = si[q];
        s->sj[q] = sj[q];
        s->k[q] = k[q];
        s->rest0[q] = rest0[q];
        s->zeta[q] = zeta[q];
        s->has_act[q] = has_act ? has_act[q] : 0;
        s->sign[q] = s->has_act[q] ? sign[q] : 0.0;
        s->amp[q] = s->has_act[q] ? amp[q] : 0.0;
        s->phase[q] = s->has_act[q] ? phase[q] : 0.0;
    }
    if (plane4) memcpy(s->plane, plane4, sizeof s->plane);
    return s;
}

ORC_EXPORT void orc_sys_sizes(void* h, int* nm, int* ns) {
    const orc_sys* s = (const orc_sys*)h;
    *nm = s->nm;
    *ns = s->ns;
}

ORC_EXPORT void orc_sys_export(void* h, double* pos, double* vel, double* mass, int* si, int* sj, double* k,
                               double* rest0, double* zeta, uint8_t* has_act, double* sign, double* amp,
                               double* phase) {
    const orc_sys* s = (const orc_sys*)h;
    const size_t nm = (size_t)s->nm, ns = (size_t)s->ns;
    if (pos) memcpy(pos, s->pos, sizeof(double) * 3 * nm);
    if (vel) memcpy(vel, s->vel, sizeof(double) * 3 * nm);
    if (mass) memcpy(mass, s->mass, sizeof(double) * nm);
    if (si) memcpy(si, s->si, sizeof(int) * ns);
    if (sj) memcpy(sj, s->sj, sizeof(int) * ns);
    if (k) memcpy(k, s->k, sizeof(double) * ns);
    if (rest0) memcpy(rest0, s->rest0, sizeof(double) * ns);
    if (zeta) memcpy(zeta, s->zeta, sizeof(double) * ns);
    if (has_act) memcpy(has_act, s->has_act, ns);
    if (sign) memcpy(sign, s->sign, sizeof(double) * ns);
    if (amp) memcpy(amp, s->amp, sizeof(double) * ns);
    if (phase) memcpy(phase, s->phase, sizeof(double) * ns);
}

/* ---------------------------------------------------------------- physics.hpp */
/* SimWorkspace ctor (physics.hpp:140-185) */
static void ws_build(orc_sys* s) {
    if (s->ws_ready) return;
    const int nm = s->nm, ns = s->ns;
    s->f = (double*)calloc((size_t)3 * ns + 1, sizeof(double));
    s->damp = (double*)calloc((size_t)ns + 1, sizeof(double));
    s->amp_rest = (double*)calloc((size_t)ns + 1, sizeof(double));
    s->sin_ph = (double*)calloc((size_t)ns + 1, sizeof(double));
    s->cos_ph = (double*)calloc((size_t)ns + 1, sizeof(double));
    s->gdamp = (double*)calloc((size_t)nm + 1, sizeof(double));
    s->inc_off = (int*)calloc((size_t)nm + 1, sizeof(int));
    s->inc_spring = (int*)calloc((size_t)2 * ns + 1, sizeof(int));
    s->inc_sign = (double*)calloc((size_t)2 * ns + 1, sizeof(double));
    s->any_act = 0;
    for (int q = 0; q < ns; ++q) {
        /* detail::damping_coefficient (physics.hpp:66-71) */
        const double mi = s->mass[s->si[q]], mj = s->mass[s->sj[q]];
        const double mu = mi * mj / (mi + mj);
        s->damp[q] = s->zeta[q] * 2.0 * sqrt(s->k[q] * mu);
        if (s->has_act[q]) {
            s->any_act = 1;
            s->amp_rest[q] = s->sign[q] * s->amp[q] * s->rest0[q];
            s->sin_ph[q] = sin(s->phase[q]);
            s->cos_ph[q] = cos(s->phase[q]);
        } else {
            s->amp_rest[q] = 0.0;
            s->sin_ph[q] = 0.0;
            s->cos_ph[q] = 1.0;
        }
    }
    for (int a = 0; a < nm; ++a) s->gdamp[a] = s->plane[1] * 2.0 * sqrt(s->plane[0] * s->mass[a]);
    for (int q = 0; q < ns; ++q) {
        s->inc_off[s->si[q] + 1]++;
        s->inc_off[s->sj[q] + 1]++;
    }
    for (int a = 0; a < nm; ++a) s->inc_off[a + 1] += s->inc_off[a];
    int* cur = (int*)malloc(sizeof(int) * ((size_t)nm + 1));
    memcpy(cur, s->inc_off, sizeof(int) * (size_t)nm);
    for (int q = 0; q < ns; ++q) {
        s->inc_spring[cur[s->si[q]]] = q;
        s->inc_sign[cur[s->si[q]]++] = 1.0;
        s->inc_spring[cur[s->sj[q]]] = q;
        s->inc_sign[cur[s->sj[q]]++] = -1.0;
    }
    free(cur);
    s->max_speed_sq = 0.0;
    s->spring_updates = 0;
    s->ws_ready = 1;
}

ORC_EXPORT void orc_sys_workspace(void* h, double* damp_coef, double* amp_rest, double* sin_ph, double* cos_ph,
                                  double* ground_damp, int* inc_off, int* inc_spring, double* inc_sign) {
    orc_sys* s = (orc_sys*)h;
    ws_build(s);
    const size_t nm = (size_t)s->nm, ns = (size_t)s->ns;
    if (damp_coef) memcpy(damp_coef, s->damp, sizeof(double) * ns);
    if (amp_rest) memcpy(amp_rest, s->amp_rest, sizeof(double) * ns);
    if (sin_ph) memcpy(sin_ph, s->sin_ph, sizeof(double) * ns);
    if (cos_ph) memcpy(cos_ph, s->cos_ph, sizeof(double) * ns);
    if (ground_damp) memcpy(ground_damp, s->gdamp, sizeof(double) * nm);
    if (inc_off) memcpy(inc_off, s->inc_off, sizeof(int) * (nm + 1));
    if (inc_spring) memcpy(inc_spring, s->inc_spring, sizeof(int) * 2 * ns);
    if (inc_sign) memcpy(inc_sign, s->inc_sign, sizeof(double) * 2 * ns);
}

typedef struct {
    double gravity, dt, duration, freq;
    int en_grav, en_contact;
} orc_simcfg;

static orc_simcfg sim_from(const double* s6) {
    orc_simcfg c = {9.81, 1e-5, 2.0, 2.0, 1, 1};
    if (s6) {
        c.gravity = s6[0];
        c.dt = s6[1];
        c.duration = s6[2];
        c.freq = s6[3];
        c.en_grav = s6[4] != 0.0;
        c.en_contact = s6[5] != 0.0;
    }
    return c;
}

/* step (physics.hpp:191-264); returns 1 when ok, 0 when diverged */
static int step(orc_sys* s, double t, const orc_simcfg* cfg) {
    const int ns = s->ns, nm = s->nm;
    double sin_wt = 0.0, cos_wt = 1.0;
    if (s->any_act) {
        const double wt = KTWOPI * cfg->freq * t;
        sin_wt = sin(wt);
        cos_wt = cos(wt);
    }
    for (int q = 0; q < ns; ++q) {
        const double* xi = s->pos + 3 * s->si[q];
        const double* xj = s->pos + 3 * s->sj[q];
        const double dx = xj[0] - xi[0], dy = xj[1] - xi[1], dz = xj[2] - xi[2];
        const double len = sqrt(dx * dx + dy * dy + dz * dz);
        if (len < 1e-9) return 0; /* kZeroLengthEps */
        const double rest = s->rest0[q] + s->amp_rest[q] * (sin_wt * s->cos_ph[q] + cos_wt * s->sin_ph[q]);
        /* detail::spring_force_on_i (physics.hpp:55-64) */
        const double* vi = s->vel + 3 * s->si[q];
        const double* vj = s->vel + 3 * s->sj[q];
        const double inv_len = 1.0 / len;
        const double nx = (xj[0] - xi[0]) * inv_len;
        const double ny = (xj[1] - xi[1]) * inv_len;
        const double nz = (xj[2] - xi[2]) * inv_len;
        const double rel = (vj[0] - vi[0]) * nx + (vj[1] - vi[1]) * ny + (vj[2] - vi[2]) * nz;
        const double mag = s->k[q] * (len - rest) + s->damp[q] * rel;
        s->f[3 * q] = mag * nx;
        s->f[3 * q + 1] = mag * ny;
        s->f[3 * q + 2] = mag * nz;
    }
    s->spring_updates += (uint64_t)ns;
    const double dt = cfg->dt;
    int ok = 1;
    for (int a = 0; a < nm; ++a) {
        double* p = s->pos + 3 * a;
        double* v = s->vel + 3 * a;
        double fx = 0.0, fy = 0.0, fz = 0.0;
        for (int e = s->inc_off[a]; e < s->inc_off[a + 1]; ++e) {
            const double* f = s->f + 3 * s->inc_spring[e];
            const double sgn = s->inc_sign[e];
            fx += sgn * f[0];
            fy += sgn * f[1];
            fz += sgn * f[2];
        }
        if (cfg->en_grav) fz -= s->mass[a] * cfg->gravity;
        if (cfg->en_contact && p[2] < 0.0) {
            const double penetration = -p[2];
            double normal = s->plane[0] * penetration - s->gdamp[a] * v[2];
            if (normal < 0.0) normal = 0.0;
            const double ft = sqrt(fx * fx + fy * fy);
            const double vt = sqrt(v[0] * v[0] + v[1] * v[1]);
            if (vt < 1e-4 && ft <= s->plane[2] * normal) { /* kStickVelocity */
                fx = 0.0;
                fy = 0.0;
            } else if (vt > 0.0) {
                const double scale = s->plane[3] * normal / vt;
                fx -= scale * v[0];
                fy -= scale * v[1];
            } else if (ft > 0.0) {
                const double scale = s->plane[3] * normal / ft;
                fx -= scale * fx;
                fy -= scale * fy;
            }
            fz += normal;
        }
        const double inv_m_dt = dt / s->mass[a];
        v[0] += fx * inv_m_dt;
        v[1] += fy * inv_m_dt;
        v[2] += fz * inv_m_dt;
        p[0] += v[0] * dt;
        p[1] += v[1] * dt;
        p[2] += v[2] * dt;
        const double sp = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
        if (sp > s->max_speed_sq) s->max_speed_sq = sp;
        for (int c = 0; c < 3; ++c)
            if (!(fabs(p[c]) <= 1e6)) ok = 0; /* kDivergenceBound, catches NaN */
    }
    return ok;
}

ORC_EXPORT int64_t orc_sys_step(void* h, const double* sim6, int64_t k0, int64_t nsteps, int64_t* steps_called,
                                uint64_t* spring_updates, double* max_speed_sq) {
    orc_sys* s = (orc_sys*)h;
    ws_build(s);
    const orc_simcfg cfg = sim_from(sim6);
    int64_t ok = 0, called = 0;
    for (int64_t k = k0; k < k0 + nsteps; ++k) {
        ++called;
        if (!step(s, (double)k * cfg.dt, &cfg)) break;
        ++ok;
    }
    if (steps_called) *steps_called = called;
    if (spring_updates) *spring_updates = s->spring_updates;
    if (max_speed_sq) *max_speed_sq = s->max_speed_sq;
    return ok;
}

/* center_of_mass (physics.hpp:266-278) */
static void com_of(const double* pos, const double* mass, int nm, double* com) {
    com[0] = com[1] = com[2] = 0.0;
    double total = 0.0;
    for (int a = 0; a < nm; ++a) {
        com[0] += mass[a] * pos[3 * a];
        com[1] += mass[a] * pos[3 * a + 1];
        com[2] += mass[a] * pos[3 * a + 2];
        total += mass[a];
    }
    if (total > 0.0)
        for (int c = 0; c < 3; ++c) com[c] /= total;
}
ORC_EXPORT void orc_center_of_mass(void* h, double* com) {
    const orc_sys* s = (const orc_sys*)h;
    com_of(s->pos, s->mass, s->nm, com);
}

/* simulate (physics.hpp:287-311) on a private copy of the state */
static void simulate(const orc_sys* s0, const orc_simcfg* cfg, double* summary) {
    orc_sys* s = (orc_sys*)orc_sys_make(s0->nm, s0->ns, s0->pos, s0->vel, s0->mass, s0->si, s0->sj, s0->k, s0->rest0,
                                        s0->zeta, s0->has_act, s0->sign, s0->amp, s0->phase, s0->plane);
    memset(summary, 0, sizeof(double) * 9);
    if (s->nm > 0) {
        ws_build(s);
        com_of(s->pos, s->mass, s->nm, summary);
        const long long n_steps = llround(cfg->duration / cfg->dt);
        for (long long k = 0; k < n_steps; ++k) {
            if (!step(s, (double)k * cfg->dt, cfg)) {
                summary[8] = 1.0;
                break;
            }
        }
        com_of(s->pos, s->mass, s->nm, summary + 3);
        const double dx = summary[3] - summary[0], dy = summary[4] - summary[1];
        summary[6] = sqrt(dx * dx + dy * dy);
        summary[7] = sqrt(s->max_speed_sq);
    }
    orc_sys_free(s);
}

ORC_EXPORT void orc_simulate(void* h, const double* sim6, double* summary) {
    const orc_simcfg cfg = sim_from(sim6);
    simulate((const orc_sys*)h, &cfg, summary);
}

/* -------------------------------------------------------------- evolution.hpp */
/* evaluate_fitness (evolution.hpp:110-119) */
static double evaluate_fitness(int w, int h, int d, const uint8_t* raw, const double* wt, const double* table8,
                               const double* plane4, const orc_simcfg* cfg) {
    const int n = w * h * d;
    uint8_t* body = (uint8_t*)malloc((size_t)n);
    largest_component(w, h, d, raw, body);
    int nonempty = 0, muscle = 0;
    for (int i = 0; i < n; ++i) {
        nonempty += body[i] != 0;
        muscle += body[i] == 1 || body[i] == 2;
    }
    double fit = 0.0;
    if (nonempty && muscle) {
        orc_sys* s = (orc_sys*)orc_build(w, h, d, body, wt, table8, plane4);
        double sum[9];
        simulate(s, cfg, sum);
        fit = sum[8] != 0.0 ? 0.0 : sum[6];
        orc_sys_free(s);
    }
    free(body);
    return fit;
}

ORC_EXPORT double orc_evaluate_fitness(int w, int h, int d, const uint8_t* mat, const double* wt,
                                       const double* table8, const double* plane4, const double* sim6) {
    const orc_simcfg cfg = sim_from(sim6);
    return evaluate_fitness(w, h, d, mat, wt, table8, plane4, &cfg);
}

/* population_diversity (evolution.hpp:89-105) */
ORC_EXPORT double orc_population_diversity(int P, int cells, const uint8_t* mats) {
    if (P < 2 || cells == 0) return 0.0;
    double sum = 0.0;
    size_t pairs = 0;
    for (int a = 0; a + 1 < P; ++a)
        for (int b = a + 1; b < P; ++b) {
            size_t differ = 0;
            const uint8_t* A = mats + (size_t)a * cells;
            const uint8_t* B = mats + (size_t)b * cells;
            for (int c = 0; c < cells; ++c) differ += A[c] != B[c];
            sum += (double)differ / (double)cells;
            ++pairs;
        }
    return sum / (double)pairs;
}

/* detail::elite_count (evolution.hpp:131-136) */
ORC_EXPORT int orc_elite_count(double ef, int population) {
    int n = (int)ceil(ef * population - 1e-9);
    if (n < 1) n = 1;
    if (n > population) n = population;
    return n;
}

/* HyperParams::clamp (evolution.hpp:29-35) */
static double clampd(double x, double lo, double hi) { return x < lo ? lo : (hi < x ? hi : x); }
ORC_EXPORT void orc_hyper_clamp(double* h) {
    h[0] = clampd(h[0], 0.001, 1.0);
    h[1] = clampd(h[1], 0.001, 1.0);
    h[2] = clampd(h[2], 0.0, 1.0);
    h[3] = clampd(h[3], 0.05, 0.9);
    for (int i = 4; i < 7; ++i) h[i] = clampd(h[i], 0.1, 10.0);
}

/* Evolution state (evolution.hpp:177-188) */
typedef struct {
    int P, gens, gw, gh, gd, tsize, cells;
    orc_arch arch;
    double sigma;
    int64_t np;
    double hyper[7];
    double table[8], plane[4];
    orc_simcfg sim;
    double *params, *bmat, *fitness;
    uint8_t* evaluated;
    uint8_t* grids; /* P x cells; has_grid marks decoded */
    double* gw_;
    uint8_t* has_grid;
    int generation;
    double best_fitness;
    int has_best;
    double* best_params;
    orc_mt rng;
} orc_evo;

ORC_EXPORT void* orc_evo_init(int population, int generations, int gw, int gh, int gd, int nh, const int* widths,
                              int m, double sigma, int tournament, int threads, uint64_t seed, const double* hyper7,
                              const double* table8, const double* plane4, const double* sim6) {
    (void)threads; /* thread count never changes results (parallel.hpp:13-16) */
    orc_evo* e = (orc_evo*)calloc(1, sizeof(orc_evo));
    e->P = population;
    e->gens = generations;
    e->gw = gw;
    e->gh = gh;
    e->gd = gd;
    e->cells = gw * gh * gd;
    e->tsize = tournament;
    e->arch = mk_arch(m, nh, widths);
    e->sigma = sigma;
    e->np = arch_param_count(&e->arch);
    const double defh[7] = {0.1, 0.1, 0.4, 0.3, 1.0, 1.0, 1.0};
    memcpy(e->hyper, hyper7 ? hyper7 : defh, sizeof e->hyper);
    orc_hyper_clamp(e->hyper);
    memcpy(e->table, table8 ? table8 : kDefaultTable, sizeof e->table);
    const double defp[4] = {1e5, 0.1, 0.6, 1.0};
    memcpy(e->plane, plane4 ? plane4 : defp, sizeof e->plane);
    e->sim = sim_from(sim6);
    const size_t P = (size_t)population;
    e->params = (double*)malloc(sizeof(double) * P * (size_t)e->np);
    e->bmat = (double*)malloc(sizeof(double) * P * 3 * (size_t)m);
    e->fitness = (double*)calloc(P, sizeof(double));
    e->evaluated = (uint8_t*)calloc(P, 1);
    e->grids = (uint8_t*)calloc(P * (size_t)e->cells, 1);
    e->gw_ = (double*)calloc(P * (size_t)e->cells, sizeof(double));
    e->has_grid = (uint8_t*)calloc(P, 1);
    e->best_params = (double*)malloc(sizeof(double) * (size_t)e->np);
    mt_seed(&e->rng, seed);
    for (size_t a = 0; a < P; ++a)
        orc_sample_genome(m, sigma, nh, widths, mt_next(&e->rng), e->params + a * (size_t)e->np,
                          e->bmat + a * 3 * (size_t)m);
    return e;
}

ORC_EXPORT void orc_evo_free(void* h) {
    orc_evo* e = (orc_evo*)h;
    free(e->params);
    free(e->bmat);
    free(e->fitness);
    free(e->evaluated);
    free(e->grids);
    free(e->gw_);
    free(e->has_grid);
    free(e->best_params);
    free(e);
}

/* evolve_generation (evolution.hpp:217-293), advisor off */
ORC_EXPORT void orc_evo_generation(void* h, double* rep) {
    orc_evo* e = (orc_evo*)h;
    const int P = e->P, cells = e->cells;
    const size_t np = (size_t)e->np, nb = 3 * (size_t)e->arch.m;
    double table[8];
    memcpy(table, e->table, sizeof table);
    table[0] *= e->hyper[4]; /* detail::scaled_materials (evolution.hpp:123-129) */
    table[1] *= e->hyper[5];
    table[2] *= e->hyper[6];
    int evaluations = 0;
    for (int a = 0; a < P; ++a) {
        if (!e->has_grid[a]) {
            decode(&e->arch, e->params + a * np, e->bmat + a * nb, e->gw, e->gh, e->gd, e->grids + (size_t)a * cells,
                   e->gw_ + (size_t)a * cells);
            e->has_grid[a] = 1;
        }
    }
    for (int a = 0; a < P; ++a) {
        if (e->evaluated[a]) continue;
        e->fitness[a] = evaluate_fitness(e->gw, e->gh, e->gd, e->grids + (size_t)a * cells,
                                         e->gw_ + (size_t)a * cells, table, e->plane, &e->sim);
        e->evaluated[a] = 1;
        ++evaluations;
    }
    /* std::stable_sort by fitness descending (evolution.hpp:243-244):
     * insertion sort is stable */
    int* order = (int*)malloc(sizeof(int) * (size_t)P);
    for (int a = 0; a < P; ++a) order[a] = a;
    for (int a = 1; a < P; ++a) {
        const int cur = order[a];
        int b = a - 1;
        while (b >= 0 && e->fitness[cur] > e->fitness[order[b]]) {
            order[b + 1] = order[b];
            --b;
        }
        order[b + 1] = cur;
    }
    /* permute population into sorted order */
    double* params = (double*)malloc(sizeof(double) * (size_t)P * np);
    double* bmat = (double*)malloc(sizeof(double) * (size_t)P * nb);
    double* fit = (double*)malloc(sizeof(double) * (size_t)P);
    uint8_t* ev = (uint8_t*)malloc((size_t)P);
    uint8_t* grids = (uint8_t*)malloc((size_t)P * cells);
    double* gw = (double*)malloc(sizeof(double) * (size_t)P * cells);
    uint8_t* hg = (uint8_t*)malloc((size_t)P);
    for (int a = 0; a < P; ++a) {
        const int o = order[a];
        memcpy(params + a * np, e->params + o * np, sizeof(double) * np);
        memcpy(bmat + a * nb, e->bmat + o * nb, sizeof(double) * nb);
        fit[a] = e->fitness[o];
        ev[a] = e->evaluated[o];
        memcpy(grids + (size_t)a * cells, e->grids + (size_t)o * cells, (size_t)cells);
        memcpy(gw + (size_t)a * cells, e->gw_ + (size_t)o * cells, sizeof(double) * cells);
        hg[a] = e->has_grid[o];
    }
    if (!e->has_best || fit[0] > e->best_fitness) {
        e->best_fitness = fit[0];
        memcpy(e->best_params, params, sizeof(double) * np);
        e->has_best = 1;
    }
    double sum = 0.0;
    for (int a = 0; a < P; ++a) sum += fit[a];
    const double mean = sum / (double)P;
    double var = 0.0;
    for (int a = 0; a < P; ++a) {
        const double dd = fit[a] - mean;
        var += dd * dd;
    }
    rep[0] = e->generation;
    rep[1] = fit[0];
    rep[2] = mean;
    rep[3] = sqrt(var / (double)P);
    rep[4] = orc_population_diversity(P, cells, grids);
    rep[5] = evaluations;
    rep[6] = 0.0;
    memcpy(rep + 7, e->hyper, sizeof(double) * 7);

    /* breed (evolution.hpp:267-289) into e->*, reading the sorted copy */
    const int n_elite = orc_elite_count(e->hyper[3], P);
    for (int a = 0; a < n_elite; ++a) {
        memcpy(e->params + a * np, params + a * np, sizeof(double) * np);
        memcpy(e->bmat + a * nb, bmat + a * nb, sizeof(double) * nb);
        e->fitness[a] = fit[a];
        e->evaluated[a] = ev[a];
        memcpy(e->grids + (size_t)a * cells, grids + (size_t)a * cells, (size_t)cells);
        memcpy(e->gw_ + (size_t)a * cells, gw + (size_t)a * cells, sizeof(double) * cells);
        e->has_grid[a] = hg[a];
    }
    for (int c = n_elite; c < P; ++c) {
        /* tournament_select (evolution.hpp:169-173) */
        uint64_t pa = rng_index(&e->rng, (uint64_t)P);
        for (int k = 1; k < e->tsize; ++k) {
            const uint64_t x = rng_index(&e->rng, (uint64_t)P);
            if (x < pa) pa = x;
        }
        double* child = e->params + (size_t)c * np;
        memcpy(child, params + pa * np, sizeof(double) * np);
        memcpy(e->bmat + (size_t)c * nb, bmat + pa * nb, sizeof(double) * nb);
        if (rng_uniform01(&e->rng) < e->hyper[2]) {
            uint64_t pb = rng_index(&e->rng, (uint64_t)P);
            for (int k = 1; k < e->tsize; ++k) {
                const uint64_t x = rng_index(&e->rng, (uint64_t)P);
                if (x < pb) pb = x;
            }
            /* crossover (evolution.hpp:143-155) */
            const double* src = params + pb * np;
            for (size_t i = 0; i < np; ++i)
                if (rng_uniform01(&e->rng) < 0.5) child[i] = src[i];
        }
        /* mutate (evolution.hpp:160-165) */
        for (size_t i = 0; i < np; ++i)
            if (rng_uniform01(&e->rng) < e->hyper[0]) child[i] += rng_normal(&e->rng) * e->hyper[1];
        e->fitness[c] = 0.0;
        e->evaluated[c] = 0;
        e->has_grid[c] = 0;
    }
    ++e->generation;
    free(order);
    free(params);
    free(bmat);
    free(fit);
    free(ev);
    free(grids);
    free(gw);
    free(hg);
}

ORC_EXPORT void orc_evo_get_population(void* h, double* params, double* bmat, double* fitness, uint8_t* evaluated,
                                       uint8_t* grids, double* grid_w) {
    const orc_evo* e = (const orc_evo*)h;
    const size_t P = (size_t)e->P, np = (size_t)e->np, nb = 3 * (size_t)e->arch.m, cells = (size_t)e->cells;
    if (params) memcpy(params, e->params, sizeof(double) * P * np);
    if (bmat) memcpy(bmat, e->bmat, sizeof(double) * P * nb);
    if (fitness) memcpy(fitness, e->fitness, sizeof(double) * P);
    if (evaluated) memcpy(evaluated, e->evaluated, P);
    for (size_t a = 0; a < P; ++a)
        for (size_t c = 0; c < cells; ++c) {
            if (grids) grids[a * cells + c] = e->has_grid[a] ? e->grids[a * cells + c] : 255;
            if (grid_w) grid_w[a * cells + c] = e->has_grid[a] ? e->gw_[a * cells + c] : 0.0;
        }
}

ORC_EXPORT void orc_evo_set_population(void* h, const double* params, const double* bmat, const double* fitness,
                                       const uint8_t* evaluated, const uint8_t* grids, const double* grid_w) {
    orc_evo* e = (orc_evo*)h;
    const size_t P = (size_t)e->P, np = (size_t)e->np, nb = 3 * (size_t)e->arch.m, cells = (size_t)e->cells;
    memcpy(e->params, params, sizeof(double) * P * np);
    memcpy(e->bmat, bmat, sizeof(double) * P * nb);
    for (size_t a = 0; a < P; ++a) {
        e->fitness[a] = fitness ? fitness[a] : 0.0;
        e->evaluated[a] = evaluated ? evaluated[a] : 0;
        e->has_grid[a] = grids != NULL;
        for (size_t c = 0; c < cells; ++c) {
            e->grids[a * cells + c] = grids ? grids[a * cells + c] : 0;
            e->gw_[a * cells + c] = grids ? (grid_w ? grid_w[a * cells + c] : 1.0) : 0.0;
        }
    }
}

ORC_EXPORT int64_t orc_evo_rng_state(void* h, char* buf, int64_t cap) {
    return mt_state_text(&((orc_evo*)h)->rng, buf, cap);
}
ORC_EXPORT void orc_evo_set_rng_state(void* h, const char* s) { mt_state_parse(&((orc_evo*)h)->rng, s); }
ORC_EXPORT void orc_evo_get_params(void* h, double* hyper7) { memcpy(hyper7, ((orc_evo*)h)->hyper, 7 * sizeof(double)); }
ORC_EXPORT void orc_evo_set_params(void* h, const double* hyper7) {
    memcpy(((orc_evo*)h)->hyper, hyper7, 7 * sizeof(double));
}
ORC_EXPORT int orc_evo_best(void* h, double* best_fitness, double* best_params) {
    const orc_evo* e = (const orc_evo*)h;
    *best_fitness = e->best_fitness;
    if (!e->has_best) return 0;
    if (best_params) memcpy(best_params, e->best_params, sizeof(double) * (size_t)e->np);
    return 1;
}

/* CPU-baseline helper mirroring ref_evaluate_batch (single thread). */
ORC_EXPORT double orc_evaluate_batch_1t(int n, int w, int h, int d, const uint8_t* mats, const double* wts,
                                        const double* table8, const double* plane4, const double* sim6,
                                        double* fitness) {
    const orc_simcfg cfg = sim_from(sim6);
    const size_t cells = (size_t)w * h * d;
    for (int a = 0; a < n; ++a)
        fitness[a] = evaluate_fitness(w, h, d, mats + a * cells, wts + a * cells, table8, plane4, &cfg);
    return 0.0;
}
