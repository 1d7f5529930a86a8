/*
 * gee_gen.c -- TEST INFRASTRUCTURE ONLY: the CPU restatement of the
 * counter-based synthetic generators of paper_2406_03726_b200/csrc/k_gen.cu
 * (spec: include/gee.h, "On-device synthetic generators").  It produces the
 * inputs of the reference arm (bench.py --impl reference, cpu_baseline) and
 * of the full-size parity tests on the host, identical bit for bit to what
 * the device generators write, so both arms time the same graph.
 *
 * The reference generates its SBM with numpy's PCG64 stream (sbm.py:52-155);
 * these generators stand in for the BASELINE.json configurations 2-4 (and
 * 0/1) whose generators the reference does not ship.
 * The element loops are split over pthreads: every output element is a pure
 * function of its index, so the thread count never changes a bit.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

typedef void (*range_fn)(void *ctx, int64_t lo, int64_t hi);
struct job {
    range_fn fn;
    void *ctx;
    int64_t lo, hi;
};
static void *job_run(void *p) {
    struct job *j = p;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}
/* fn over [0, n) in up to 64 contiguous chunks, one thread each */
static void parallel_for(range_fn fn, void *ctx, int64_t n) {
    long t = sysconf(_SC_NPROCESSORS_ONLN);
    if (t < 1) t = 1;
    if (t > 64) t = 64;
    if (n < 65536) t = 1;
    struct job jobs[64];
    pthread_t th[64];
    for (long i = 0; i < t; ++i) {
        jobs[i].fn = fn;
        jobs[i].ctx = ctx;
        jobs[i].lo = n * i / t;
        jobs[i].hi = n * (i + 1) / t;
    }
    long started = 0;
    for (long i = 1; i < t; ++i, ++started)
        if (pthread_create(&th[i], NULL, job_run, &jobs[i]) != 0) break;
    job_run(&jobs[0]);
    for (long i = 1; i <= started; ++i) pthread_join(th[i], NULL);
    for (long i = started + 1; i < t; ++i) job_run(&jobs[i]); /* threads that failed to start */
}

#define GOLDEN 0x9e3779b97f4a7c15ull

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static inline uint64_t draw(uint64_t key, uint64_t t) { return mix64(key + (t + 1) * GOLDEN); }

uint64_t ggen_key(uint64_t seed, uint64_t stream) { return mix64(seed ^ (stream * GOLDEN)); }

struct rmat_ctx {
    uint64_t key, wkey;
    int scale;
    uint32_t t1, t2, t3;
    int64_t *rows, *cols;
    float *w;
};
static void rmat_range(void *p, int64_t lo, int64_t hi) {
    const struct rmat_ctx *c_ = p;
    const uint64_t key = c_->key, wkey = c_->wkey;
    const int scale = c_->scale;
    const uint32_t t1 = c_->t1, t2 = c_->t2, t3 = c_->t3;
    int64_t *rows = c_->rows, *cols = c_->cols;
    float *w = c_->w;
    const int words = (scale + 1) / 2;
    for (int64_t i = lo; i < hi; ++i) {
        int64_t r = 0, c = 0;
        for (int h = 0; h < words; ++h) {
            const uint64_t x = draw(key, (uint64_t)i * 16 + (uint64_t)h);
            for (int half = 0; half < 2; ++half) {
                if (2 * h + half >= scale) break;
                const uint32_t u = half ? (uint32_t)(x >> 32) : (uint32_t)x;
                const int rb = u >= t2;
                const int cb = (u >= t1 && u < t2) || u >= t3;
                r = 2 * r + rb;
                c = 2 * c + cb;
            }
        }
        rows[i] = r;
        cols[i] = c;
        if (w) {
            const uint32_t u24 = (uint32_t)(draw(wkey, (uint64_t)i) >> 40);
            w[i] = 1.0f - (float)u24 * 0x1p-24f;
        }
    }
}

void ggen_rmat(uint64_t key, uint64_t wkey, int scale, int64_t e, uint32_t t1, uint32_t t2, uint32_t t3,
               int64_t *rows, int64_t *cols, float *w) {
    struct rmat_ctx c = {key, wkey, scale, t1, t2, t3, rows, cols, w};
    parallel_for(rmat_range, &c, e);
}

static inline int64_t cdf_pick(const double *cdf, int64_t n, double u) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (cdf[mid] <= u)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo < n ? lo : n - 1;
}

struct cl_ctx {
    uint64_t rkey, ckey, wkey;
    const double *cdf;
    int64_t n;
    int64_t *rows, *cols;
    double *w;
};
static void cl_range(void *p, int64_t lo, int64_t hi) {
    const struct cl_ctx *c_ = p;
    const uint64_t rkey = c_->rkey, ckey = c_->ckey, wkey = c_->wkey;
    const double *cdf = c_->cdf;
    const int64_t n = c_->n;
    int64_t *rows = c_->rows, *cols = c_->cols;
    double *w = c_->w;
    for (int64_t i = lo; i < hi; ++i) {
        const double ur = (double)(draw(rkey, (uint64_t)i) >> 11) * 0x1p-53;
        const double uc = (double)(draw(ckey, (uint64_t)i) >> 11) * 0x1p-53;
        rows[i] = cdf_pick(cdf, n, ur);
        cols[i] = cdf_pick(cdf, n, uc);
        if (w) w[i] = 1.0 - (double)(draw(wkey, (uint64_t)i) >> 11) * 0x1p-53;
    }
}

void ggen_chunglu(uint64_t rkey, uint64_t ckey, uint64_t wkey, const double *cdf, int64_t n, int64_t e,
                  int64_t *rows, int64_t *cols, double *w) {
    struct cl_ctx c = {rkey, ckey, wkey, cdf, n, rows, cols, w};
    parallel_for(cl_range, &c, e);
}

struct pair_ctx {
    uint64_t key;
    int64_t t0, n;
    int64_t *keys;
};
static void pair_range(void *p, int64_t lo, int64_t hi) {
    const struct pair_ctx *c_ = p;
    const uint64_t key = c_->key;
    const int64_t t0 = c_->t0, n = c_->n;
    int64_t *keys = c_->keys;
    for (int64_t i = lo; i < hi; ++i) {
        const uint64_t x = draw(key, (uint64_t)(t0 + i));
        const uint32_t a = (uint32_t)(((uint64_t)(uint32_t)x * (uint64_t)n) >> 32);
        const uint32_t b = (uint32_t)(((x >> 32) * (uint64_t)n) >> 32);
        keys[i] = a == b ? -1 : (a < b ? (int64_t)a * n + b : (int64_t)b * n + a);
    }
}

void ggen_pairs(uint64_t key, int64_t t0, int64_t count, int64_t n, int64_t *keys) {
    struct pair_ctx c = {key, t0, n, keys};
    parallel_for(pair_range, &c, count);
}

/* G(n,m): the first m distinct candidate pairs in candidate order (a
 * candidate repeating an earlier one, or a self pair, is skipped).  Returns
 * the number of candidates consumed, or -1 if `limit` candidates were not
 * enough.  Stable LSD radix sort of (key, t) by key, 16-bit digits. */
int64_t ggen_gnm(uint64_t key, int64_t n, int64_t m, int64_t limit, int64_t *rows, int64_t *cols) {
    int64_t *keys = malloc(sizeof(int64_t) * (size_t)limit);
    uint64_t *a = malloc(sizeof(uint64_t) * (size_t)limit), *b = malloc(sizeof(uint64_t) * (size_t)limit);
    uint32_t *ta = malloc(sizeof(uint32_t) * (size_t)limit), *tb = malloc(sizeof(uint32_t) * (size_t)limit);
    unsigned char *keep = calloc((size_t)limit, 1);
    int64_t used = -1;
    if (!keys || !a || !b || !ta || !tb || !keep) goto done;
    ggen_pairs(key, 0, limit, n, keys);
    int64_t cnt = 0;
    for (int64_t i = 0; i < limit; ++i)
        if (keys[i] >= 0) {
            a[cnt] = (uint64_t)keys[i];
            ta[cnt] = (uint32_t)i;
            ++cnt;
        }
    uint64_t maxk = (uint64_t)n * (uint64_t)n;
    int bits = 0;
    while (bits < 64 && (maxk >> bits)) bits += 16;
    static int64_t hist[65536];
    for (int sh = 0; sh < bits; sh += 16) {
        memset(hist, 0, sizeof(hist));
        for (int64_t i = 0; i < cnt; ++i) ++hist[(a[i] >> sh) & 0xffff];
        int64_t s = 0;
        for (int d = 0; d < 65536; ++d) {
            int64_t h = hist[d];
            hist[d] = s;
            s += h;
        }
        for (int64_t i = 0; i < cnt; ++i) {
            int64_t p = hist[(a[i] >> sh) & 0xffff]++;
            b[p] = a[i];
            tb[p] = ta[i];
        }
        uint64_t *tk = a; a = b; b = tk;
        uint32_t *tt = ta; ta = tb; tb = tt;
    }
    for (int64_t i = 0; i < cnt; ++i)
        if (i == 0 || a[i] != a[i - 1]) keep[ta[i]] = 1;
    int64_t got = 0;
    for (int64_t t = 0; t < limit && got < m; ++t)
        if (keep[t]) {
            rows[got] = keys[t] / n;
            cols[got] = keys[t] % n;
            ++got;
            used = t + 1;
        }
    if (got < m) used = -1;
done:
    free(keys); free(a); free(b); free(ta); free(tb); free(keep);
    return used;
}

/* SBM pair sweep; rows/cols NULL -> count only.  Returns the edge count. */
int64_t ggen_sbm(uint64_t key, int64_t n, const int64_t *lab, uint32_t thr_in, uint32_t thr_out, int64_t *rows,
                 int64_t *cols) {
    int64_t e = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j) {
            const uint32_t u = (uint32_t)(draw(key, (uint64_t)(i * n + j)) >> 32);
            if (u < (lab[i] == lab[j] ? thr_in : thr_out)) {
                if (rows) {
                    rows[e] = i;
                    cols[e] = j;
                }
                ++e;
            }
        }
    return e;
}
