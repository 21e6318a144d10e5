/*
 * gnnsim_oracle.c — plain-C restatement of the reference's chunk-pipelined
 * training path (arXiv 2308.10087 / gnnsim). TEST INFRASTRUCTURE ONLY: it is the
 * checker for tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg;
 * the product never links or calls it.
 *
 * Pinned against the reference itself (oracle/_ref/ref_driver, built from
 * /root/reference/proj/src) and the golden fixtures in tests/golden/ by
 * tests/test_oracle.py. Compiled with -ffp-contract=off and no -march, so float
 * arithmetic is the same x86-64 SSE scalar mul-then-add as the reference; it
 * uses the same glibc expf/logf/log1p/sqrt, hence it is bit-exact with it.
 *
 * Third-party algorithm restated: libstdc++ (GCC 13.3) <random> —
 *   std::mt19937_64, uniform_int_distribution<uint64_t> (Lemire's method via
 *   unsigned __int128, bits/uniform_int_dist.h _S_nd), uniform_real_distribution
 *   <double> (generate_canonical<double,53>, bits/random.tcc:3349-3381).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng.hpp:9-38 */
static uint64_t mix1(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
static uint64_t mix2(uint64_t a, uint64_t b) { return mix1(mix1(a) ^ b); }
static uint64_t mix3(uint64_t a, uint64_t b, uint64_t c) { return mix1(mix2(a, b) ^ c); }
static double hash_unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

/* mt19937_64 (ISO C++ [rand.eng.mers], parameters of std::mt19937_64) */
typedef struct {
    uint64_t mt[312];
    int i;
} mt64;
static void mt_seed(mt64* m, uint64_t s) {
    m->mt[0] = s;
    for (int i = 1; i < 312; ++i) m->mt[i] = 6364136223846793005ull * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
    m->i = 312;
}
static uint64_t mt_next(mt64* m) {
    if (m->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            uint64_t y = (m->mt[k] & 0xFFFFFFFF80000000ull) | (m->mt[(k + 1) % 312] & 0x7FFFFFFFull);
            uint64_t v = m->mt[(k + 156) % 312] ^ (y >> 1);
            if (y & 1) v ^= 0xB5026F5AA96619E9ull;
            m->mt[k] = v;
        }
        m->i = 0;
    }
    uint64_t x = m->mt[m->i++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}
/* make_engine(seed, stream) = mt19937_64(mix64(seed, stream)) (rng.hpp:36-38) */
static void make_engine(mt64* m, uint64_t seed, uint64_t stream) { mt_seed(m, mix2(seed, stream)); }

/* uniform_int_distribution<uint64_t>(0, hi)(mt19937_64): downscaling with the
 * 128-bit Lemire method (_S_nd), range = hi + 1 < 2^64. */
static uint64_t uniform_u64(mt64* m, uint64_t hi) {
    if (hi == UINT64_MAX) return mt_next(m);
    const uint64_t range = hi + 1;
    unsigned __int128 prod = (unsigned __int128)mt_next(m) * range;
    uint64_t low = (uint64_t)prod;
    if (low < range) {
        const uint64_t thr = (uint64_t)(-range) % range;
        while (low < thr) {
            prod = (unsigned __int128)mt_next(m) * range;
            low = (uint64_t)prod;
        }
    }
    return (uint64_t)(prod >> 64);
}
/* uniform_real_distribution<double>(a, b): a + (b-a) * generate_canonical<double,53>,
 * one 64-bit draw: ret = double(x) / 2^64, clamped below 1 with nextafter. */
static double uniform_real(mt64* m, double a, double b) {
    double ret = (double)mt_next(m) / 18446744073709551616.0;
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return ret * (b - a) + a;
}

/* ---------------------------------------------------------------- graph.cpp:33-66 */
typedef struct {
    uint32_t n;
    uint64_t m;            /* undirected edges */
    uint64_t* off;         /* n+1 */
    uint32_t* nb;          /* 2m */
    uint32_t* deg;
} ograph;

static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* edges as packed (u<<32|v); canonicalise, sort, unique, drop loops, CSR with sorted rows */
static void build_graph(ograph* g, uint32_t n, uint64_t* keys, uint64_t cnt) {
    for (uint64_t i = 0; i < cnt; ++i) {
        uint32_t u = (uint32_t)(keys[i] >> 32), v = (uint32_t)keys[i];
        if (u > v) {
            uint32_t t = u;
            u = v;
            v = t;
        }
        keys[i] = ((uint64_t)u << 32) | v;
    }
    qsort(keys, cnt, 8, cmp_u64);
    uint64_t w = 0;
    for (uint64_t i = 0; i < cnt; ++i) {
        if (i > 0 && keys[i] == keys[i - 1]) continue;
        if ((uint32_t)(keys[i] >> 32) == (uint32_t)keys[i]) continue;
        keys[w++] = keys[i];
    }
    g->n = n;
    g->m = w;
    g->deg = (uint32_t*)calloc(n ? n : 1, 4);
    g->off = (uint64_t*)calloc((size_t)n + 1, 8);
    g->nb = (uint32_t*)malloc((2 * w + 1) * 4);
    for (uint64_t i = 0; i < w; ++i) {
        ++g->deg[keys[i] >> 32];
        ++g->deg[(uint32_t)keys[i]];
    }
    for (uint32_t v = 0; v < n; ++v) g->off[v + 1] = g->off[v] + g->deg[v];
    uint64_t* cur = (uint64_t*)malloc(((size_t)n + 1) * 8);
    memcpy(cur, g->off, (size_t)n * 8);
    /* sorted (u,v) order puts a vertex's lower neighbours before its upper ones */
    for (uint64_t i = 0; i < w; ++i) {
        const uint32_t u = (uint32_t)(keys[i] >> 32), v = (uint32_t)keys[i];
        g->nb[cur[u]++] = v;
        g->nb[cur[v]++] = u;
    }
    free(cur);
}

static void free_graph(ograph* g) {
    free(g->off);
    free(g->nb);
    free(g->deg);
}

/* graph.cpp:119-156 — Batagelj-Brandes geometric skipping */
static void generate_er(ograph* g, uint32_t n, double p, uint64_t seed) {
    uint64_t cap = 1024, cnt = 0;
    uint64_t* keys = (uint64_t*)malloc(cap * 8);
    if (p > 0.0) {
        const uint64_t total = (uint64_t)n * (n - 1) / 2;
        uint32_t u = 0;
        uint64_t row0 = 0, rowlen = (uint64_t)n - 1;
        mt64 eng;
        make_engine(&eng, seed, 0x45527ull);
        const double lq = log1p(-p);
        double idx = -1;
        for (uint64_t it = 0;; ++it) {
            uint64_t pi;
            if (p >= 1.0) {
                if (it >= total) break;
                pi = it;
            } else {
                const double r = uniform_real(&eng, 0.0, 1.0);
                idx += 1.0 + floor(log1p(-r) / lq);
                if (idx >= (double)total) break;
                pi = (uint64_t)idx;
            }
            while (pi >= row0 + rowlen) {
                row0 += rowlen;
                --rowlen;
                ++u;
            }
            if (cnt == cap) keys = (uint64_t*)realloc(keys, (cap *= 2) * 8);
            keys[cnt++] = ((uint64_t)u << 32) | (uint32_t)(u + 1 + (pi - row0));
        }
    }
    build_graph(g, n, keys, cnt);
    free(keys);
}

/* graph.cpp:68-98 — normalised adjacency with self-loops at the sorted position */
typedef struct {
    uint64_t* off;
    uint32_t* col;
    float* val;
} ocsr;

static void normalize(const ograph* g, ocsr* a, int loops) {
    const uint32_t n = g->n;
    a->off = (uint64_t*)calloc((size_t)n + 1, 8);
    for (uint32_t v = 0; v < n; ++v) a->off[v + 1] = a->off[v] + g->deg[v] + (loops ? 1 : 0);
    a->col = (uint32_t*)malloc((a->off[n] + 1) * 4);
    a->val = (float*)malloc((a->off[n] + 1) * 4);
    const double ex = loops ? 1.0 : 0.0;
    for (uint32_t v = 0; v < n; ++v) {
        const double dv = (double)g->deg[v] + ex;
        uint64_t w = a->off[v];
        int pending = loops;
        for (uint64_t i = g->off[v]; i <= g->off[v + 1]; ++i) {
            const int at_end = i == g->off[v + 1];
            const uint32_t u = at_end ? 0 : g->nb[i];
            if (pending && (at_end || u > v)) {
                a->col[w] = v;
                a->val[w++] = (float)(1.0 / sqrt(dv * dv));
                pending = 0;
            }
            if (at_end) break;
            const double du = (double)g->deg[u] + ex;
            a->col[w] = u;
            a->val[w++] = (float)(1.0 / sqrt(dv * du));
        }
    }
}

/* ------------------------------------------------------- partition.cpp:57-198 */
#define NONE 0xffffffffu

static void bfs(const ograph* g, const uint32_t* src, uint32_t ns, uint32_t* dist, uint32_t* q) {
    for (uint32_t v = 0; v < g->n; ++v) dist[v] = NONE;
    uint64_t h = 0, t = 0;
    for (uint32_t i = 0; i < ns; ++i) {
        dist[src[i]] = 0;
        q[t++] = src[i];
    }
    while (h < t) {
        const uint32_t v = q[h++];
        for (uint64_t i = g->off[v]; i < g->off[v + 1]; ++i) {
            const uint32_t u = g->nb[i];
            if (dist[u] == NONE) {
                dist[u] = dist[v] + 1;
                q[t++] = u;
            }
        }
    }
}

/* FIFO of vertex ids (duplicates allowed, like the reference's std::deque) */
typedef struct {
    uint32_t* b;
    uint64_t h, t, cap;
} fifo;
static void fpush(fifo* f, uint32_t v) {
    if (f->t == f->cap) {
        f->cap = f->cap ? 2 * f->cap : 64;
        f->b = (uint32_t*)realloc(f->b, f->cap * 4);
    }
    f->b[f->t++] = v;
}

static int partition(const ograph* g, uint32_t parts, uint64_t seed, uint32_t* part) {
    const uint32_t n = g->n;
    if (parts == 0 || parts > n) return 1;
    const uint64_t ceil_avg = ((uint64_t)n + parts - 1) / parts;
    const uint64_t slack = (uint64_t)floor(1.05 * (double)n / (double)parts);
    const uint64_t cap = ceil_avg > slack ? ceil_avg : slack;
    /* seeds (partition.cpp:76-108) */
    uint32_t* seeds = (uint32_t*)malloc(parts * 4);
    uint32_t* dist = (uint32_t*)malloc(((size_t)n + 1) * 4);
    uint32_t* q = (uint32_t*)malloc(((size_t)n + 1) * 4);
    uint8_t* taken = (uint8_t*)calloc(n, 1);
    mt64 eng;
    make_engine(&eng, seed, 0x504152ull);
    seeds[0] = (uint32_t)uniform_u64(&eng, n - 1);
    taken[seeds[0]] = 1;
    for (uint32_t s = 1; s < parts; ++s) {
        bfs(g, seeds, s, dist, q);
        uint32_t pick = NONE, far = 0;
        for (uint32_t v = 0; v < n; ++v) {
            if (taken[v]) continue;
            if (dist[v] == NONE) {
                pick = v;
                break;
            }
            if (dist[v] > far) {
                far = dist[v];
                pick = v;
            }
        }
        if (pick == NONE)
            for (uint32_t v = 0; v < n; ++v)
                if (!taken[v]) {
                    pick = v;
                    break;
                }
        seeds[s] = pick;
        taken[pick] = 1;
    }
    /* round-robin growth (:110-155) */
    for (uint32_t v = 0; v < n; ++v) part[v] = NONE;
    fifo* fr = (fifo*)calloc(parts, sizeof(fifo));
    uint64_t* size = (uint64_t*)calloc(parts, 8);
    uint32_t assigned = 0, fresh = 0;
    for (uint32_t i = 0; i < parts; ++i) {
        if (part[seeds[i]] != NONE) continue;
        part[seeds[i]] = i;
        ++size[i];
        ++assigned;
        for (uint64_t e = g->off[seeds[i]]; e < g->off[seeds[i] + 1]; ++e) fpush(&fr[i], g->nb[e]);
    }
    while (assigned < n) {
        int moved = 0;
        for (uint32_t i = 0; i < parts && assigned < n; ++i) {
            if (size[i] >= cap) continue;
            uint32_t claim = NONE;
            while (fr[i].h < fr[i].t) {
                const uint32_t v = fr[i].b[fr[i].h++];
                if (part[v] == NONE) {
                    claim = v;
                    break;
                }
            }
            if (claim == NONE) {
                while (fresh < n && part[fresh] != NONE) ++fresh;
                if (fresh < n) claim = fresh;
            }
            if (claim == NONE) continue;
            part[claim] = i;
            ++size[i];
            ++assigned;
            moved = 1;
            for (uint64_t e = g->off[claim]; e < g->off[claim + 1]; ++e)
                if (part[g->nb[e]] == NONE) fpush(&fr[i], g->nb[e]);
        }
        if (!moved) break;
    }
    /* one refinement sweep (:159-181) */
    for (uint32_t i = 0; i < parts; ++i) size[i] = 0;
    for (uint32_t v = 0; v < n; ++v) ++size[part[v]];
    uint32_t* votes = (uint32_t*)calloc(parts, 4);
    for (uint32_t v = 0; v < n; ++v) {
        const uint32_t home = part[v];
        if (size[home] <= 1) continue;
        for (uint64_t e = g->off[v]; e < g->off[v + 1]; ++e) ++votes[part[g->nb[e]]];
        uint32_t best = home;
        for (uint64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
            const uint32_t c = part[g->nb[e]];
            if (c == home || size[c] + 1 > cap) continue;
            if (votes[c] > votes[best] || (votes[c] == votes[best] && c < best)) best = c;
        }
        if (best != home && votes[best] > votes[home]) {
            part[v] = best;
            --size[home];
            ++size[best];
        }
        for (uint64_t e = g->off[v]; e < g->off[v + 1]; ++e) votes[part[g->nb[e]]] = 0;
        votes[home] = 0;
    }
    for (uint32_t i = 0; i < parts; ++i) free(fr[i].b);
    free(fr);
    free(size);
    free(votes);
    free(seeds);
    free(dist);
    free(q);
    free(taken);
    return 0;
}

/* partition.cpp:239-248 */
static void shuffle_order(uint32_t K, uint64_t epoch, uint64_t seed, uint32_t* order) {
    for (uint32_t k = 0; k < K; ++k) order[k] = k;
    mt64 eng;
    make_engine(&eng, seed, mix2(0x5348ull, epoch));
    for (uint32_t i = K; i > 1; --i) {
        const uint32_t j = (uint32_t)uniform_u64(&eng, i - 1);
        const uint32_t t = order[i - 1];
        order[i - 1] = order[j];
        order[j] = t;
    }
}

/* ------------------------------------------------------------------- model */
enum { DENSE = 0, GCNCONV = 1, GCN2CONV = 3 };
typedef struct {
    int kind;
    uint32_t in, out;
    int relu;
    double alpha, beta;
} ospec;

/* nn.cpp:28-64 (kind: 0 GCN, 2 GCNII) */
static uint32_t build_specs(int model, uint32_t layers, uint32_t hidden, double alpha, double lambda, uint32_t F,
                            uint32_t C, ospec* s) {
    if (model == 2) {
        s[0] = (ospec){DENSE, F, hidden, 1, 0, 0};
        for (uint32_t j = 1; j + 2 <= layers; ++j) s[j] = (ospec){GCN2CONV, hidden, hidden, 1, alpha, log(lambda / (double)j + 1.0)};
        s[layers - 1] = (ospec){DENSE, hidden, C, 0, 0, 0};
    } else {
        for (uint32_t l = 0; l < layers; ++l)
            s[l] = (ospec){GCNCONV, l == 0 ? F : hidden, l + 1 == layers ? C : hidden, l + 1 < layers, 0, 0};
    }
    return layers;
}

/* matrix.hpp:53-59 + nn.hpp:60-72 */
static void glorot(float* w, uint32_t rows, uint32_t cols, uint64_t seed, uint32_t l) {
    const double a = sqrt(6.0 / (double)(rows + cols));
    mt64 eng;
    make_engine(&eng, seed, mix2(0x57454947ull, l));
    for (uint64_t i = 0; i < (uint64_t)rows * cols; ++i) w[i] = (float)uniform_real(&eng, -a, a);
}

/* DropMask (nn.hpp:103-138) */
typedef struct {
    int on;
    float scale;
    uint32_t cols;
    uint64_t* bits;
} omask;
static void mask_make(omask* m, double rate, uint64_t seed, uint64_t epoch, uint32_t layer, uint32_t n, uint32_t cols) {
    m->on = rate > 0.0;
    m->bits = NULL;
    m->cols = cols;
    m->scale = 1.f;
    if (!m->on) return;
    const double keep = 1.0 - rate;
    m->scale = (float)(1.0 / keep);
    const uint64_t total = (uint64_t)n * cols;
    m->bits = (uint64_t*)calloc((total + 63) / 64 + 1, 8);
    const uint64_t key = mix3(seed, epoch, layer);
    for (uint64_t i = 0; i < total; ++i)
        if (hash_unit(mix2(key, i)) < keep) m->bits[i >> 6] |= 1ull << (i & 63);
}
static float mask_apply(const omask* m, float x, uint32_t v, uint32_t j) {
    if (!m->on) return x;
    const uint64_t i = (uint64_t)v * m->cols + j;
    return ((m->bits[i >> 6] >> (i & 63)) & 1) ? x * m->scale : 0.f;
}

/* dense_rows (matrix.hpp:63-74) */
static void dense_rows(const float* x, uint32_t in, const float* W, const float* b, float* y, uint32_t out) {
    for (uint32_t j = 0; j < out; ++j) y[j] = b ? b[j] : 0.f;
    for (uint32_t i = 0; i < in; ++i) {
        const float xi = x[i];
        if (xi == 0.f) continue;
        for (uint32_t j = 0; j < out; ++j) y[j] += xi * W[(size_t)i * out + j];
    }
}
/* dense_rows_wt (matrix.hpp:77-86) */
static void dense_rows_wt(const float* x, uint32_t out, const float* W, float* y, uint32_t in) {
    for (uint32_t i = 0; i < in; ++i) {
        float acc = 0.f;
        for (uint32_t j = 0; j < out; ++j) acc += x[j] * W[(size_t)i * out + j];
        y[i] = acc;
    }
}

/* ------------------------------------------------------------- trainer state */
typedef struct {
    float *h, *hs, *pre, *dz, *dagg, *daggs, *dh;
} olayer;

typedef struct {
    /* inputs */
    uint32_t n, F, C, K, S, L;
    const ocsr* A;
    const float* x0;
    const uint32_t* lab;
    const uint8_t* split;
    const uint32_t* chunk_of;
    const ospec* sp;
    float** W;
    float** b;
    double dropout;
    uint64_t seed;
    int sync, hist, shuffle, sgd;
    uint32_t fix_alpha, hidden;
    double lr, b1, b2, eps;
    uint64_t n_train, cnt[3];
} orun;

typedef struct {
    uint32_t lb, le, len;
    float *in_cur, *in_snap, *dh_in, *h0_cur, *dh0;
    olayer* ly;
    float **mW, **vW, **mb, **vb;
    uint64_t step;
    omask* masks;
} ostage;

static float* zf(uint64_t c) { return (float*)calloc(c ? c : 1, 4); }

/* ----------------------------------------------------- kernels (nn.hpp:143-293) */
typedef struct {
    const float* cur;
    const float* snap;
    const uint8_t* done; /* NULL: always cur */
    const uint32_t* chunk_of;
    uint32_t w;
} osrc;
static const float* src_row(const osrc* s, uint32_t u) {
    if (!s->done || s->done[s->chunk_of[u]]) return s->cur + (size_t)u * s->w;
    return s->snap ? s->snap + (size_t)u * s->w : NULL;
}

static void forward_row(const orun* R, const ospec* sp, uint32_t l, uint32_t v, const osrc* src, const omask* m,
                        const float* h0row, float* pre, float* out) {
    const uint32_t in = sp->in, o = sp->out;
    if (sp->kind == DENSE) {
        const float* x = src_row(src, v);
        for (uint32_t j = 0; j < in; ++j) pre[j] = mask_apply(m, x[j], v, j);
        dense_rows(pre, in, R->W[l], R->b[l], out, o);
    } else {
        for (uint32_t j = 0; j < in; ++j) pre[j] = 0.f;
        for (uint64_t i = R->A->off[v]; i < R->A->off[v + 1]; ++i) {
            const uint32_t u = R->A->col[i];
            const float w = R->A->val[i];
            const float* r = src_row(src, u);
            if (!r) continue;
            for (uint32_t j = 0; j < in; ++j) pre[j] += w * mask_apply(m, r[j], u, j);
        }
        if (sp->kind == GCN2CONV) {
            const float a = (float)sp->alpha, be = (float)sp->beta;
            for (uint32_t j = 0; j < in; ++j) pre[j] = (1.f - a) * pre[j] + a * h0row[j];
            dense_rows(pre, in, R->W[l], NULL, out, o);
            for (uint32_t j = 0; j < o; ++j) out[j] = (1.f - be) * pre[j] + be * out[j];
        } else {
            dense_rows(pre, in, R->W[l], R->b[l], out, o);
        }
    }
    if (sp->relu)
        for (uint32_t j = 0; j < o; ++j)
            if (out[j] < 0.f) out[j] = 0.f;
}

static void backward_out_row(const orun* R, const ospec* sp, uint32_t l, const float* dout, const float* outr, float* dz,
                             float* dagg, float* dh0) {
    const uint32_t o = sp->out, k = sp->in;
    for (uint32_t j = 0; j < o; ++j) dz[j] = sp->relu ? (outr[j] > 0.f ? dout[j] : 0.f) : dout[j];
    dense_rows_wt(dz, o, R->W[l], dagg, k);
    if (sp->kind == GCN2CONV) {
        const float a = (float)sp->alpha, be = (float)sp->beta;
        for (uint32_t j = 0; j < k; ++j) dagg[j] = (1.f - be) * dz[j] + be * dagg[j];
        for (uint32_t j = 0; j < k; ++j) dh0[j] += a * dagg[j];
    }
}

static void backward_prev_row(const orun* R, const ospec* sp, uint32_t u, const osrc* dg, const float* own, const omask* m,
                              float* dprev) {
    const uint32_t in = sp->in;
    if (sp->kind == DENSE) {
        for (uint32_t j = 0; j < in; ++j) dprev[j] = own[j];
    } else {
        const float oma = 1.f - (float)sp->alpha;
        for (uint32_t j = 0; j < in; ++j) dprev[j] = 0.f;
        for (uint64_t i = R->A->off[u]; i < R->A->off[u + 1]; ++i) {
            const float w = R->A->val[i];
            const float* d = src_row(dg, R->A->col[i]);
            if (!d) continue;
            if (sp->kind == GCN2CONV)
                for (uint32_t j = 0; j < in; ++j) dprev[j] += w * (oma * d[j]);
            else
                for (uint32_t j = 0; j < in; ++j) dprev[j] += w * d[j];
        }
    }
    for (uint32_t j = 0; j < in; ++j) dprev[j] = mask_apply(m, dprev[j], u, j);
}

/* softmax-xent pieces (nn.hpp:373-403) */
static double xent_loss(const float* l, uint32_t C, uint32_t label) {
    float mx = l[0];
    for (uint32_t j = 1; j < C; ++j) mx = l[j] > mx ? l[j] : mx;
    float s = 0.f;
    for (uint32_t j = 0; j < C; ++j) s += expf(l[j] - mx);
    return (double)logf(s) - (double)(l[label] - mx);
}
static void xent_grad(const float* l, uint32_t C, uint32_t label, float inv, float* g) {
    float mx = l[0];
    for (uint32_t j = 1; j < C; ++j) mx = l[j] > mx ? l[j] : mx;
    float s = 0.f;
    for (uint32_t j = 0; j < C; ++j) {
        g[j] = expf(l[j] - mx);
        s += g[j];
    }
    for (uint32_t j = 0; j < C; ++j) {
        g[j] = g[j] / s * inv;
        if (j == label) g[j] -= inv;
    }
}
static uint32_t argmax(const float* l, uint32_t C) {
    uint32_t b = 0;
    for (uint32_t j = 1; j < C; ++j)
        if (l[j] > l[b]) b = j;
    return b;
}

/* Adam / SGD (nn.hpp:474-490) */
static void optim_update(const orun* R, uint64_t step, float* p, const float* g, uint64_t n, float* m, float* v) {
    const float lr = (float)R->lr;
    if (R->sgd) {
        for (uint64_t i = 0; i < n; ++i) p[i] -= lr * g[i];
        return;
    }
    const float b1 = (float)R->b1, b2 = (float)R->b2, eps = (float)R->eps;
    const float c1 = (float)(1.0 - pow(R->b1, (double)step));
    const float c2 = (float)(1.0 - pow(R->b2, (double)step));
    for (uint64_t i = 0; i < n; ++i) {
        m[i] = b1 * m[i] + (1.f - b1) * g[i];
        v[i] = b2 * v[i] + (1.f - b2) * g[i] * g[i];
        const float mh = m[i] / c1, vh = v[i] / c2;
        p[i] -= lr * mh / (sqrtf(vh) + eps);
    }
}

/* ------------------------------------------------------------ the trainer
 * train_hybrid with G = 1 (engines_impl.hpp:515-909), stages simulated in
 * order: a stage's results depend only on its own state and on the message
 * sequence from its neighbour, so running stage 0..S-1 forward, then S-1..0
 * backward, is exactly the reference's concurrent schedule. */
typedef struct {
    uint32_t lo, len;          /* chunk row list: rows[lo..lo+len) */
} ochunk;

int or_train(uint32_t n, const uint64_t* off, const uint32_t* col, const float* val, const float* x0, uint32_t F,
             const uint32_t* lab, const uint8_t* split, uint32_t C, const uint32_t* chunk_of, uint32_t K, uint32_t S,
             int model, uint32_t layers, uint32_t hidden, double dropout, double alpha, double lambda, uint64_t seed,
             uint32_t epochs, int shuffle, uint32_t fix_alpha, int hist, int sync, int sgd, double lr,
             double* metrics /* epochs x 5 */, uint64_t* comm /* epochs */, float* params_out,
             float* h_out /* optional: final-epoch h of every layer, concatenated N x out */) {
    ocsr A = {(uint64_t*)off, (uint32_t*)col, (float*)val};
    ospec* sp = (ospec*)calloc(layers, sizeof(ospec));
    const uint32_t L = build_specs(model, layers, hidden, alpha, lambda, F, C, sp);
    orun R = {0};
    R.n = n, R.F = F, R.C = C, R.K = K, R.S = S, R.L = L, R.A = &A, R.x0 = x0, R.lab = lab, R.split = split;
    R.chunk_of = chunk_of, R.sp = sp, R.dropout = dropout, R.seed = seed, R.sync = sync, R.hist = hist && !sync;
    R.shuffle = shuffle, R.sgd = sgd, R.fix_alpha = fix_alpha ? fix_alpha : 1, R.hidden = hidden, R.lr = lr;
    R.b1 = 0.9, R.b2 = 0.999, R.eps = 1e-8;
    for (uint32_t v = 0; v < n; ++v)
        if (split[v] >= 1 && split[v] <= 3) ++R.cnt[split[v] - 1];
    if (R.cnt[0] == 0) return 1;
    const float inv_train = (float)(1.0 / (double)R.cnt[0]);
    int needs_h0 = 0;
    for (uint32_t l = 0; l < L; ++l) needs_h0 |= sp[l].kind == GCN2CONV;
    R.W = (float**)calloc(L, sizeof(float*));
    R.b = (float**)calloc(L, sizeof(float*));
    for (uint32_t l = 0; l < L; ++l) {
        R.W[l] = zf((uint64_t)sp[l].in * sp[l].out);
        glorot(R.W[l], sp[l].in, sp[l].out, seed, l);
        R.b[l] = sp[l].kind == GCN2CONV ? NULL : zf(sp[l].out);
    }
    /* chunk rows, ascending per chunk */
    uint32_t* rows = (uint32_t*)malloc(((size_t)n + 1) * 4);
    ochunk* ch = (ochunk*)calloc(K, sizeof(ochunk));
    {
        uint32_t at = 0;
        for (uint32_t k = 0; k < K; ++k) {
            ch[k].lo = at;
            for (uint32_t v = 0; v < n; ++v)
                if (chunk_of[v] == k) rows[at++] = v;
            ch[k].len = at - ch[k].lo;
        }
    }
    /* stages (engines.cpp:8-21) */
    ostage* st = (ostage*)calloc(S, sizeof(ostage));
    for (uint32_t s = 0, at = 0; s < S; ++s) {
        const uint32_t take = L / S + (s < L % S ? 1u : 0u);
        st[s].lb = at, st[s].le = at + take, st[s].len = take;
        at += take;
    }
    for (uint32_t s = 0; s < S; ++s) {
        ostage* g = &st[s];
        const uint32_t in0 = sp[g->lb].in;
        g->in_cur = s == 0 ? (float*)x0 : zf((uint64_t)n * in0);
        g->in_snap = (!sync && sp[g->lb].kind != DENSE) ? (s == 0 ? (float*)x0 : zf((uint64_t)n * in0)) : NULL;
        g->dh_in = s > 0 ? zf((uint64_t)n * in0) : NULL;
        g->h0_cur = (needs_h0 && s > 0) ? zf((uint64_t)n * hidden) : NULL;
        g->dh0 = needs_h0 ? zf((uint64_t)n * hidden) : NULL;
        g->ly = (olayer*)calloc(g->len, sizeof(olayer));
        g->mW = (float**)calloc(g->len, sizeof(float*));
        g->vW = (float**)calloc(g->len, sizeof(float*));
        g->mb = (float**)calloc(g->len, sizeof(float*));
        g->vb = (float**)calloc(g->len, sizeof(float*));
        g->masks = (omask*)calloc(g->len, sizeof(omask));
        for (uint32_t i = 0; i < g->len; ++i) {
            const ospec* q = &sp[g->lb + i];
            olayer* y = &g->ly[i];
            y->h = zf((uint64_t)n * q->out);
            y->pre = zf((uint64_t)n * q->in);
            y->dz = zf((uint64_t)n * q->out);
            y->dagg = zf((uint64_t)n * q->in);
            y->dh = zf((uint64_t)n * q->out);
            if (!sync && i + 1 < g->len && sp[g->lb + i + 1].kind != DENSE) y->hs = zf((uint64_t)n * q->out);
            if (R.hist && q->kind != DENSE) y->daggs = zf((uint64_t)n * q->in);
            g->mW[i] = zf((uint64_t)q->in * q->out);
            g->vW[i] = zf((uint64_t)q->in * q->out);
            g->mb[i] = zf(q->out);
            g->vb[i] = zf(q->out);
        }
    }
    uint32_t* order = (uint32_t*)malloc(K * 4);
    uint8_t* fdone = (uint8_t*)calloc(K, 1);
    uint8_t* bdone = (uint8_t*)calloc(K, 1);
    uint8_t* all = (uint8_t*)malloc(K);
    memset(all, 1, K);

    for (uint32_t t = 1; t <= epochs; ++t) {
        uint64_t bytes = 0;
        if (shuffle)
            shuffle_order(K, t, seed, order);
        else
            for (uint32_t k = 0; k < K; ++k) order[k] = k;
        /* snapshot + masks, every stage (:671-683) */
        for (uint32_t s = 0; s < S; ++s) {
            ostage* g = &st[s];
            if (!sync && (t - 1) % R.fix_alpha == 0) {
                if (g->in_snap && s > 0) memcpy(g->in_snap, g->in_cur, (size_t)n * sp[g->lb].in * 4);
                for (uint32_t i = 0; i < g->len; ++i) {
                    if (g->ly[i].hs) memcpy(g->ly[i].hs, g->ly[i].h, (size_t)n * sp[g->lb + i].out * 4);
                    if (g->ly[i].daggs) memcpy(g->ly[i].daggs, g->ly[i].dagg, (size_t)n * sp[g->lb + i].in * 4);
                }
            }
            for (uint32_t i = 0; i < g->len; ++i) {
                free(g->masks[i].bits);
                mask_make(&g->masks[i], dropout, seed, t, g->lb + i, n, sp[g->lb + i].in);
            }
        }
        /* ---- forward, stage by stage ---- */
        for (uint32_t s = 0; s < S; ++s) {
            ostage* g = &st[s];
            const float* h0m = needs_h0 ? (s == 0 ? g->ly[0].h : g->h0_cur) : NULL;
            const uint32_t in0 = sp[g->lb].in;
            memset(fdone, 0, K);
            const uint32_t passes = sync ? 1 : K;
            for (uint32_t kk = 0; kk < passes; ++kk) {
                /* rows processed in this pass */
                uint32_t r_lo, r_len;
                const uint32_t* rl;
                uint32_t* allrows = NULL;
                if (sync) {
                    allrows = (uint32_t*)malloc(((size_t)n + 1) * 4);
                    for (uint32_t v = 0; v < n; ++v) allrows[v] = v;
                    rl = allrows, r_lo = 0, r_len = n;
                    for (uint32_t q = 0; q < K; ++q) fdone[order[q]] = 1;
                } else {
                    const uint32_t k = order[kk];
                    fdone[k] = 1;
                    rl = rows, r_lo = ch[k].lo, r_len = ch[k].len;
                }
                /* recv: rows of the chunk(s) from the previous stage's stash (messages) */
                if (s > 0) {
                    const ostage* up = &st[s - 1];
                    const uint32_t wl = sp[up->le - 1].out;
                    const float* hsrc = needs_h0 ? (s - 1 == 0 ? up->ly[0].h : up->h0_cur) : NULL;
                    for (uint32_t r = 0; r < r_len; ++r) {
                        const uint32_t v = rl[r_lo + r];
                        memcpy(g->in_cur + (size_t)v * in0, up->ly[up->len - 1].h + (size_t)v * wl, wl * 4);
                        if (needs_h0) memcpy(g->h0_cur + (size_t)v * hidden, hsrc + (size_t)v * hidden, hidden * 4);
                    }
                    bytes += (uint64_t)r_len * (wl + (needs_h0 ? hidden : 0)) * 4;
                }
                for (uint32_t i = 0; i < g->len; ++i) {
                    const ospec* q = &sp[g->lb + i];
                    osrc src;
                    src.cur = i == 0 ? g->in_cur : g->ly[i - 1].h;
                    src.snap = i == 0 ? g->in_snap : g->ly[i - 1].hs;
                    src.done = sync ? NULL : fdone;
                    src.chunk_of = chunk_of;
                    src.w = q->in;
                    for (uint32_t r = 0; r < r_len; ++r) {
                        const uint32_t v = rl[r_lo + r];
                        forward_row(&R, q, g->lb + i, v, &src, &g->masks[i],
                                    (h0m && g->lb + i > 0) ? h0m + (size_t)v * hidden : NULL,
                                    g->ly[i].pre + (size_t)v * q->in, g->ly[i].h + (size_t)v * q->out);
                    }
                }
                free(allrows);
            }
        }
        /* ---- metrics at the last stage (:816-825) ---- */
        {
            ostage* g = &st[S - 1];
            const float* lg = g->ly[g->len - 1].h;
            double loss = 0;
            uint64_t cor[3] = {0, 0, 0};
            for (uint32_t v = 0; v < n; ++v) {
                const uint8_t sv = split[v];
                if (sv == 0) continue;
                const int ok = argmax(lg + (size_t)v * C, C) == lab[v];
                if (sv == 1) loss += xent_loss(lg + (size_t)v * C, C, lab[v]);
                cor[sv - 1] += ok;
            }
            double* mrow = metrics + (size_t)(t - 1) * 5;
            mrow[0] = t;
            mrow[1] = loss / (double)R.cnt[0];
            mrow[2] = (double)cor[0] / (double)R.cnt[0];
            mrow[3] = R.cnt[1] ? (double)cor[1] / (double)R.cnt[1] : 0.0;
            mrow[4] = R.cnt[2] ? (double)cor[2] / (double)R.cnt[2] : 0.0;
            if (needs_h0) memset(g->dh0, 0, (size_t)n * hidden * 4);
        }
        /* ---- backward, last stage first ---- */
        for (uint32_t si = S; si-- > 0;) {
            ostage* g = &st[si];
            const uint32_t in0 = sp[g->lb].in;
            memset(bdone, 0, K);
            const uint32_t passes = sync ? 1 : K;
            for (uint32_t pk = 0; pk < passes; ++pk) {
                uint32_t r_lo, r_len;
                const uint32_t* rl;
                uint32_t* allrows = NULL;
                if (sync) {
                    allrows = (uint32_t*)malloc(((size_t)n + 1) * 4);
                    for (uint32_t v = 0; v < n; ++v) allrows[v] = v;
                    rl = allrows, r_lo = 0, r_len = n;
                    for (uint32_t q = 0; q < K; ++q) bdone[q] = 1;
                } else {
                    const uint32_t k = order[K - 1 - pk];
                    bdone[k] = 1;
                    rl = rows, r_lo = ch[k].lo, r_len = ch[k].len;
                }
                olayer* top = &g->ly[g->len - 1];
                const uint32_t wl = sp[g->le - 1].out;
                if (si == S - 1) {
                    for (uint32_t r = 0; r < r_len; ++r) {
                        const uint32_t v = rl[r_lo + r];
                        float* d = top->dh + (size_t)v * wl;
                        if (split[v] == 1)
                            xent_grad(top->h + (size_t)v * wl, C, lab[v], inv_train, d);
                        else
                            memset(d, 0, wl * 4);
                    }
                } else {
                    const ostage* dn = &st[si + 1];
                    for (uint32_t r = 0; r < r_len; ++r) {
                        const uint32_t v = rl[r_lo + r];
                        memcpy(top->dh + (size_t)v * wl, dn->dh_in + (size_t)v * wl, wl * 4);
                        if (needs_h0) memcpy(g->dh0 + (size_t)v * hidden, dn->dh0 + (size_t)v * hidden, hidden * 4);
                    }
                }
                for (uint32_t i = g->len; i-- > 0;) {
                    const uint32_t l = g->lb + i;
                    const ospec* q = &sp[l];
                    olayer* y = &g->ly[i];
                    for (uint32_t r = 0; r < r_len; ++r) {
                        const uint32_t v = rl[r_lo + r];
                        if (l == 0 && needs_h0) {
                            float* d = y->dh + (size_t)v * q->out;
                            const float* a = g->dh0 + (size_t)v * hidden;
                            for (uint32_t j = 0; j < hidden; ++j) d[j] += a[j];
                        }
                        backward_out_row(&R, q, l, y->dh + (size_t)v * q->out, y->h + (size_t)v * q->out,
                                         y->dz + (size_t)v * q->out, y->dagg + (size_t)v * q->in,
                                         (needs_h0 && q->kind == GCN2CONV) ? g->dh0 + (size_t)v * hidden : NULL);
                    }
                    if (l > 0) {
                        float* target = i > 0 ? g->ly[i - 1].dh : g->dh_in;
                        osrc dg;
                        dg.cur = y->dagg;
                        dg.snap = R.hist ? y->daggs : NULL;
                        dg.done = sync ? NULL : bdone;
                        dg.chunk_of = chunk_of;
                        dg.w = q->in;
                        for (uint32_t r = 0; r < r_len; ++r) {
                            const uint32_t u = rl[r_lo + r];
                            backward_prev_row(&R, q, u, &dg, y->dagg + (size_t)u * q->in, &g->masks[i],
                                              target + (size_t)u * q->in);
                        }
                    }
                }
                if (si > 0) bytes += (uint64_t)r_len * (in0 + (needs_h0 ? hidden : 0)) * 4;
                free(allrows);
            }
            /* param grads + optimizer step (:872-878) */
            ++g->step;
            for (uint32_t i = 0; i < g->len; ++i) {
                const uint32_t l = g->lb + i;
                const ospec* q = &sp[l];
                float* gW = zf((uint64_t)q->in * q->out);
                float* gb = zf(q->out);
                for (uint32_t v = 0; v < n; ++v) {
                    const float* x = g->ly[i].pre + (size_t)v * q->in;
                    const float* d = g->ly[i].dz + (size_t)v * q->out;
                    for (uint32_t a = 0; a < q->in; ++a) {
                        const float xa = x[a];
                        if (xa == 0.f) continue;
                        for (uint32_t j = 0; j < q->out; ++j) gW[(size_t)a * q->out + j] += xa * d[j];
                    }
                    if (q->kind != GCN2CONV)
                        for (uint32_t j = 0; j < q->out; ++j) gb[j] += d[j];
                }
                if (q->kind == GCN2CONV) {
                    const float be = (float)q->beta;
                    for (uint64_t e = 0; e < (uint64_t)q->in * q->out; ++e) gW[e] *= be;
                }
                optim_update(&R, g->step, R.W[l], gW, (uint64_t)q->in * q->out, g->mW[i], g->vW[i]);
                if (R.b[l]) optim_update(&R, g->step, R.b[l], gb, q->out, g->mb[i], g->vb[i]);
                free(gW);
                free(gb);
            }
        }
        if (comm) comm[t - 1] = bytes;
    }
    /* outputs */
    {
        uint64_t at = 0;
        for (uint32_t l = 0; l < L; ++l) {
            memcpy(params_out + at, R.W[l], (size_t)sp[l].in * sp[l].out * 4);
            at += (uint64_t)sp[l].in * sp[l].out;
            if (R.b[l]) {
                memcpy(params_out + at, R.b[l], sp[l].out * 4);
                at += sp[l].out;
            }
        }
        if (h_out) {
            uint64_t ho = 0;
            for (uint32_t s = 0; s < S; ++s)
                for (uint32_t i = 0; i < st[s].len; ++i) {
                    const uint32_t w = sp[st[s].lb + i].out;
                    memcpy(h_out + ho, st[s].ly[i].h, (size_t)n * w * 4);
                    ho += (uint64_t)n * w;
                }
        }
    }
    for (uint32_t s = 0; s < S; ++s) {
        ostage* g = &st[s];
        if (s > 0) free(g->in_cur);
        if (s > 0) free(g->in_snap);
        free(g->dh_in);
        free(g->h0_cur);
        free(g->dh0);
        for (uint32_t i = 0; i < g->len; ++i) {
            olayer* y = &g->ly[i];
            free(y->h), free(y->hs), free(y->pre), free(y->dz), free(y->dagg), free(y->daggs), free(y->dh);
            free(g->mW[i]), free(g->vW[i]), free(g->mb[i]), free(g->vb[i]);
            free(g->masks[i].bits);
        }
        free(g->ly), free(g->mW), free(g->vW), free(g->mb), free(g->vb), free(g->masks);
    }
    for (uint32_t l = 0; l < L; ++l) free(R.W[l]), free(R.b[l]);
    free(R.W), free(R.b), free(st), free(rows), free(ch), free(order), free(fdone), free(bdone), free(all), free(sp);
    return 0;
}

/* ------------------------------------------------------------ exported API */
typedef struct {
    ograph g;
    float* x;
    uint32_t* lab;
    uint8_t* split;
    uint32_t F, C;
} odata;

/* synthetic dataset: generate_er + hashed features */
void* or_synthetic_er(uint32_t n, double p, uint64_t gseed, uint32_t F, uint32_t C, uint64_t fseed) {
    odata* d = (odata*)calloc(1, sizeof(odata));
    generate_er(&d->g, n, p, gseed);
    d->F = F, d->C = C;
    d->x = zf((uint64_t)n * F);
    d->lab = (uint32_t*)calloc(n ? n : 1, 4);
    d->split = (uint8_t*)calloc(n ? n : 1, 1);
    for (uint64_t v = 0; v < n; ++v) {
        for (uint64_t j = 0; j < F; ++j) d->x[v * F + j] = (float)(hash_unit(mix2(fseed, v * F + j)) * 2.0 - 1.0);
        d->lab[v] = (uint32_t)(mix3(fseed, 0x4C42ull, v) % C);
        const uint64_t r = mix3(fseed, 0x5350ull, v) % 10;
        d->split[v] = r < 6 ? 1 : (r < 8 ? 2 : 3);
    }
    return d;
}
/* arbitrary edge list (pairs) + node data */
void* or_from_edges(uint32_t n, const uint32_t* uv, uint64_t m, const float* x, uint32_t F, const uint32_t* lab,
                    uint32_t C, const uint8_t* split) {
    odata* d = (odata*)calloc(1, sizeof(odata));
    uint64_t* keys = (uint64_t*)malloc((m + 1) * 8);
    for (uint64_t i = 0; i < m; ++i) keys[i] = ((uint64_t)uv[2 * i] << 32) | uv[2 * i + 1];
    build_graph(&d->g, n, keys, m);
    free(keys);
    d->F = F, d->C = C;
    d->x = zf((uint64_t)n * F);
    memcpy(d->x, x, (size_t)n * F * 4);
    d->lab = (uint32_t*)malloc((size_t)n * 4 + 4);
    memcpy(d->lab, lab, (size_t)n * 4);
    d->split = (uint8_t*)malloc((size_t)n + 1);
    memcpy(d->split, split, n);
    return d;
}
void or_free(void* h) {
    odata* d = (odata*)h;
    if (!d) return;
    free_graph(&d->g);
    free(d->x), free(d->lab), free(d->split), free(d);
}
void or_shape(const void* h, uint32_t* n, uint64_t* m) {
    const odata* d = (const odata*)h;
    *n = d->g.n, *m = d->g.m;
}
void or_graph(const void* h, uint64_t* off, uint32_t* nb, uint32_t* deg) {
    const odata* d = (const odata*)h;
    memcpy(off, d->g.off, ((size_t)d->g.n + 1) * 8);
    memcpy(nb, d->g.nb, d->g.m * 2 * 4);
    memcpy(deg, d->g.deg, (size_t)d->g.n * 4);
}
void or_arrays(const void* h, float* x, uint32_t* lab, uint8_t* split) {
    const odata* d = (const odata*)h;
    memcpy(x, d->x, (size_t)d->g.n * d->F * 4);
    memcpy(lab, d->lab, (size_t)d->g.n * 4);
    memcpy(split, d->split, d->g.n);
}
void or_normalize(const void* h, int loops, uint64_t* off, uint32_t* col, float* val) {
    const odata* d = (const odata*)h;
    ocsr a;
    normalize(&d->g, &a, loops);
    memcpy(off, a.off, ((size_t)d->g.n + 1) * 8);
    memcpy(col, a.col, a.off[d->g.n] * 4);
    memcpy(val, a.val, a.off[d->g.n] * 4);
    free(a.off), free(a.col), free(a.val);
}
int or_partition(const void* h, uint32_t parts, uint64_t seed, uint32_t* part) {
    return partition(&((const odata*)h)->g, parts, seed, part);
}
void or_shuffle(uint32_t K, uint64_t epoch, uint64_t seed, uint32_t* order) { shuffle_order(K, epoch, seed, order); }
void or_stage_ranges(uint32_t L, uint32_t S, uint32_t* ranges) {
    for (uint32_t s = 0, at = 0; s < S; ++s) {
        const uint32_t take = L / S + (s < L % S ? 1u : 0u);
        ranges[2 * s] = at, ranges[2 * s + 1] = at + take;
        at += take;
    }
}
void or_init_params(int model, uint32_t layers, uint32_t hidden, uint32_t F, uint32_t C, uint64_t seed, float* flat) {
    ospec sp[512];
    const uint32_t L = build_specs(model, layers, hidden, 0.1, 0.5, F, C, sp);
    uint64_t at = 0;
    for (uint32_t l = 0; l < L; ++l) {
        glorot(flat + at, sp[l].in, sp[l].out, seed, l);
        at += (uint64_t)sp[l].in * sp[l].out;
        if (sp[l].kind != GCN2CONV) {
            memset(flat + at, 0, sp[l].out * 4);
            at += sp[l].out;
        }
    }
}
uint64_t or_dropmask_bits(double rate, uint64_t seed, uint64_t epoch, uint32_t layer, uint32_t n, uint32_t cols,
                          uint64_t* out_words) {
    omask m;
    mask_make(&m, rate, seed, epoch, layer, n, cols);
    const uint64_t words = ((uint64_t)n * cols + 63) / 64;
    if (m.on && out_words) memcpy(out_words, m.bits, words * 8);
    free(m.bits);
    return words;
}
/* train on a dataset handle: normalised adjacency built here */
int or_train_data(const void* h, const uint32_t* chunk_of, uint32_t K, uint32_t S, int model, uint32_t layers,
                  uint32_t hidden, double dropout, uint64_t seed, uint32_t epochs, int shuffle, uint32_t fix_alpha,
                  int hist, int sync, int sgd, double lr, double* metrics, uint64_t* comm, float* params,
                  float* h_out) {
    const odata* d = (const odata*)h;
    ocsr a;
    normalize(&d->g, &a, 1);
    const int rc = or_train(d->g.n, a.off, a.col, a.val, d->x, d->F, d->lab, d->split, d->C, chunk_of, K, S, model,
                            layers, hidden, dropout, 0.1, 0.5, seed, epochs, shuffle, fix_alpha, hist, sync, sgd, lr,
                            metrics, comm, params, h_out);
    free(a.off), free(a.col), free(a.val);
    return rc;
}
