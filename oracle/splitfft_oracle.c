/*
 * splitfft_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain-C restatement of the reference CPU algorithm (the `splitfft`
 * package under /root/reference/pkg/src/splitfft) used only as the parity
 * checker by tests/, by __graft_entry__.smoke() and by bench.py's
 * cpu_baseline leg.  Nothing in paper_2504_07264_b200/ links or calls it.
 *
 * Parity status: PINNED.  tests/test_oracle_golden.py checks every function
 * here bit-for-bit against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference in the build
 * container and writes the .npz files under tests/golden).
 *
 * Restated pieces (reference file:line):
 *   oracle_twiddle_table   twiddle.py:46-57 (_snapped_cos_sin) and
 *                          transform.py:80-84 (stage factor  cos - 1j*sin)
 *   oracle_bitrev          layout.py:122-133 (bit_reverse_indices)
 *   oracle_fft_dit         transform.py:208-238 (fft_dit; per element the
 *                          executor equals the stage composition
 *                          twiddle_stage/butterfly_stage, transform.py:88-120,
 *                          pinned bitwise by test_transform.py:145-167)
 *   oracle_fft_dif         transform.py:241-270 (fft_dif)
 *   oracle_ifft            transform.py:280-298 (ifft via channel swap)
 *
 * Complex multiply.  The reference multiplies complex128 arrays with
 * numpy.multiply (transform.py:137,150).  On x86-64 with FMA numpy rounds
 *     re = fma(ar, br, -(ai*bi)),   im = fma(ar, bi, ai*br)
 * (measured here: bitwise on 2^16 random products).
 * cmul() below restates exactly that, which is what makes this oracle
 * bit-identical to the reference rather than merely close.  Build with
 * -ffp-contract=off so the compiler adds no further contractions.
 *
 * The stage factor is w = cos - 1j*sin computed by numpy
 * (transform.py:82); its imaginary part is 0.0 - sin, i.e. -sin except
 * that sin == 0 yields +0.0.  We store (wr, wi) exactly like that.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_MAX_M 30

/* twiddle.py:46-57 for stage i, index q, then transform.py:82. */
static void stage_factor(int i, int64_t q, double *wr, double *wi)
{
    double angle = 2.0 * M_PI * (double)q / (double)(1LL << i);
    double c = cos(angle);
    double s = sin(angle);
    if (((4 * q) % (1LL << i)) == 0) {       /* exact multiples of pi/2 */
        c = nearbyint(c);                      /* np.round: half-to-even */
        s = nearbyint(s);
    }
    c += 0.0;                                  /* clear -0.0 */
    s += 0.0;
    *wr = c - 0.0;      /* (cos + 0j) - (1j*sin): real part cos - (0*sin - 1*0) */
    *wi = 0.0 - s;      /* imag part 0 - sin (+0.0 when sin == 0) */
    /* cos - (+-0) == cos for every finite cos, including cos == +0 */
    if (*wr == 0.0) *wr = 0.0;
}

/* Top-stage factor table: w[q] for stage m, q in [0, 2^(m-1)).  Stage i's
 * table is w[q << (m - i)] bit-for-bit (the angle 2*pi*q*2^k / 2^m rounds
 * identically to 2*pi*q / 2^i since scaling by 2^k commutes with rounding). */
int oracle_twiddle_table(int m, double *wr, double *wi)
{
    if (m < 1 || m > ORACLE_MAX_M) return 1;
    int64_t h = 1LL << (m - 1);
    for (int64_t q = 0; q < h; ++q) stage_factor(m, q, &wr[q], &wi[q]);
    return 0;
}

/* Raw snapped (cos, sin) of stage i, twiddle.py:109-120. */
int oracle_cos_sin(int i, double *c_out, double *s_out)
{
    if (i < 1 || i > ORACLE_MAX_M) return 1;
    int64_t h = 1LL << (i - 1);
    for (int64_t q = 0; q < h; ++q) {
        double angle = 2.0 * M_PI * (double)q / (double)(1LL << i);
        double c = cos(angle), s = sin(angle);
        if (((4 * q) % (1LL << i)) == 0) { c = nearbyint(c); s = nearbyint(s); }
        c_out[q] = c + 0.0;
        s_out[q] = s + 0.0;
    }
    return 0;
}

/* layout.py:122-133 */
void oracle_bitrev(int m, int64_t *idx)
{
    int64_t n = 1LL << m;
    for (int64_t k = 0; k < n; ++k) {
        int64_t r = 0, v = k;
        for (int b = 0; b < m; ++b) { r = (r << 1) | (v & 1); v >>= 1; }
        idx[k] = r;
    }
}

static inline void cmul(double ar, double ai, double br, double bi,
                        double *cr, double *ci)
{
    *cr = fma(ar, br, -(ai * bi));
    *ci = fma(ar, bi, ai * br);
}

typedef struct {
    int m;
    int algo;             /* 0 = dit, 1 = dif */
    int inverse;
    const double *wr, *wi;
    const int64_t *rev;
    const double *x_re, *x_im;
    double *y_re, *y_im;
    int64_t row0, row1;
    int64_t in_stride, out_stride;
} job_t;

/* One forward transform of an interleaved (re, im) signal z, in place,
 * using the scratch s.  Stage order/arithmetic per transform.py:208-270. */
static void one_signal(const job_t *j, double *z, double *s)
{
    const int m = j->m;
    const int64_t n = 1LL << m;
    if (m == 0) return;
    if (j->algo == 0) {
        /* gather (transform.py:217) */
        for (int64_t k = 0; k < n; ++k) {
            s[2 * k] = z[2 * j->rev[k]];
            s[2 * k + 1] = z[2 * j->rev[k] + 1];
        }
        /* stage 1 (transform.py:218, _butterfly_all :123-128) */
        for (int64_t k = 0; k < n; k += 2) {
            z[2 * k] = s[2 * k] + s[2 * k + 2];
            z[2 * k + 1] = s[2 * k + 1] + s[2 * k + 3];
            z[2 * k + 2] = s[2 * k] - s[2 * k + 2];
            z[2 * k + 3] = s[2 * k + 1] - s[2 * k + 3];
        }
        /* stages 2..m: t = b*w; b = a - t; a = a + t (_dit_stage :131-139) */
        for (int i = 2; i <= m; ++i) {
            int64_t h = 1LL << (i - 1);
            int sh = m - i;
            for (int64_t b0 = 0; b0 < n; b0 += 2 * h) {
                for (int64_t q = 0; q < h; ++q) {
                    double *a = z + 2 * (b0 + q), *b = z + 2 * (b0 + q + h);
                    double tr, ti;
                    cmul(b[0], b[1], j->wr[q << sh], j->wi[q << sh], &tr, &ti);
                    b[0] = a[0] - tr; b[1] = a[1] - ti;
                    a[0] = a[0] + tr; a[1] = a[1] + ti;
                }
            }
        }
    } else {
        /* stages m..2: t = a - b; a = a + b; b = t*w (_dif_stage :142-150) */
        for (int i = m; i >= 2; --i) {
            int64_t h = 1LL << (i - 1);
            int sh = m - i;
            for (int64_t b0 = 0; b0 < n; b0 += 2 * h) {
                for (int64_t q = 0; q < h; ++q) {
                    double *a = z + 2 * (b0 + q), *b = z + 2 * (b0 + q + h);
                    double tr = a[0] - b[0], ti = a[1] - b[1];
                    a[0] = a[0] + b[0]; a[1] = a[1] + b[1];
                    cmul(tr, ti, j->wr[q << sh], j->wi[q << sh], &b[0], &b[1]);
                }
            }
        }
        /* stage 1 into scratch (transform.py:268) */
        for (int64_t k = 0; k < n; k += 2) {
            s[2 * k] = z[2 * k] + z[2 * k + 2];
            s[2 * k + 1] = z[2 * k + 1] + z[2 * k + 3];
            s[2 * k + 2] = z[2 * k] - z[2 * k + 2];
            s[2 * k + 3] = z[2 * k + 1] - z[2 * k + 3];
        }
        /* gather (transform.py:269) */
        for (int64_t k = 0; k < n; ++k) {
            z[2 * k] = s[2 * j->rev[k]];
            z[2 * k + 1] = s[2 * j->rev[k] + 1];
        }
    }
}

static void *run_rows(void *arg)
{
    const job_t *j = (const job_t *)arg;
    const int64_t n = 1LL << j->m;
    double *z = (double *)malloc(sizeof(double) * 4 * (size_t)n);
    double *s = z + 2 * n;
    const double scale = 1.0 / (double)n;
    for (int64_t r = j->row0; r < j->row1; ++r) {
        const double *xr = j->x_re + r * j->in_stride;
        const double *xi = j->x_im + r * j->in_stride;
        /* interleave (layout.py:89-101); ifft swaps channels first (:280-283) */
        for (int64_t k = 0; k < n; ++k) {
            z[2 * k] = j->inverse ? xi[k] : xr[k];
            z[2 * k + 1] = j->inverse ? xr[k] : xi[k];
        }
        one_signal(j, z, s);
        double *yr = j->y_re + r * j->out_stride;
        double *yi = j->y_im + r * j->out_stride;
        for (int64_t k = 0; k < n; ++k) {
            if (j->inverse) {           /* swap back, then data *= 1/N (:296-297) */
                yr[k] = z[2 * k + 1] * scale;
                yi[k] = z[2 * k] * scale;
            } else {
                yr[k] = z[2 * k];
                yi[k] = z[2 * k + 1];
            }
        }
    }
    free(z);
    return NULL;
}

/* ---- one long signal over many threads ------------------------------------
 * For batches smaller than the thread count (config 5: one 2^28-point
 * signal) the threads split the work INSIDE each stage instead of across
 * rows: every stage's n/2 butterflies are independent (transform.py:131-150
 * updates disjoint (a, b) pairs), so thread t takes a contiguous range of
 * butterfly indices, and a barrier separates the stages -- the same
 * operations on the same values in the same stage order, hence bit-identical
 * to one_signal().  The gather, stage 1 and the (de)interleave split by
 * element ranges the same way. */
typedef struct {
    const job_t *j;
    int tid, nth;
    double *z, *s;
    int64_t row;
    pthread_barrier_t *bar;
} wide_t;

static void range_of(int64_t total, int tid, int nth, int64_t *lo, int64_t *hi)
{
    int64_t per = (total + nth - 1) / nth;
    *lo = (int64_t)tid * per < total ? (int64_t)tid * per : total;
    *hi = *lo + per < total ? *lo + per : total;
}

static void *wide_worker(void *arg)
{
    wide_t *w = (wide_t *)arg;
    const job_t *j = w->j;
    const int m = j->m;
    const int64_t n = 1LL << m;
    double *z = w->z, *s = w->s;
    int64_t lo, hi;
    const int64_t r = w->row;
    const double scale = 1.0 / (double)n;
    /* interleave (layout.py:89-101; ifft swaps channels first, :280-283) */
    range_of(n, w->tid, w->nth, &lo, &hi);
    const double *xr = j->x_re + r * j->in_stride, *xi = j->x_im + r * j->in_stride;
    for (int64_t k = lo; k < hi; ++k) {
        z[2 * k] = j->inverse ? xi[k] : xr[k];
        z[2 * k + 1] = j->inverse ? xr[k] : xi[k];
    }
    pthread_barrier_wait(w->bar);
    if (j->algo == 0) {
        for (int64_t k = lo; k < hi; ++k) {                  /* gather (:217) */
            s[2 * k] = z[2 * j->rev[k]];
            s[2 * k + 1] = z[2 * j->rev[k] + 1];
        }
        pthread_barrier_wait(w->bar);
        range_of(n / 2, w->tid, w->nth, &lo, &hi);          /* stage 1 (:218) */
        for (int64_t b = lo; b < hi; ++b) {
            const int64_t k = 2 * b;
            z[2 * k] = s[2 * k] + s[2 * k + 2];
            z[2 * k + 1] = s[2 * k + 1] + s[2 * k + 3];
            z[2 * k + 2] = s[2 * k] - s[2 * k + 2];
            z[2 * k + 3] = s[2 * k + 1] - s[2 * k + 3];
        }
        for (int i = 2; i <= m; ++i) {                        /* stages 2..m (:131-139) */
            pthread_barrier_wait(w->bar);
            const int64_t h = 1LL << (i - 1);
            const int sh = m - i;
            for (int64_t b = lo; b < hi; ++b) {
                const int64_t q = b & (h - 1), b0 = (b >> (i - 1)) << i;
                double *a = z + 2 * (b0 + q), *bb = z + 2 * (b0 + q + h);
                double tr, ti;
                cmul(bb[0], bb[1], j->wr[q << sh], j->wi[q << sh], &tr, &ti);
                bb[0] = a[0] - tr; bb[1] = a[1] - ti;
                a[0] = a[0] + tr; a[1] = a[1] + ti;
            }
        }
        pthread_barrier_wait(w->bar);
    } else {
        range_of(n / 2, w->tid, w->nth, &lo, &hi);
        for (int i = m; i >= 2; --i) {                        /* stages m..2 (:142-150) */
            const int64_t h = 1LL << (i - 1);
            const int sh = m - i;
            for (int64_t b = lo; b < hi; ++b) {
                const int64_t q = b & (h - 1), b0 = (b >> (i - 1)) << i;
                double *a = z + 2 * (b0 + q), *bb = z + 2 * (b0 + q + h);
                double tr = a[0] - bb[0], ti = a[1] - bb[1];
                a[0] = a[0] + bb[0]; a[1] = a[1] + bb[1];
                cmul(tr, ti, j->wr[q << sh], j->wi[q << sh], &bb[0], &bb[1]);
            }
            pthread_barrier_wait(w->bar);
        }
        for (int64_t b = lo; b < hi; ++b) {                   /* stage 1 into scratch (:268) */
            const int64_t k = 2 * b;
            s[2 * k] = z[2 * k] + z[2 * k + 2];
            s[2 * k + 1] = z[2 * k + 1] + z[2 * k + 3];
            s[2 * k + 2] = z[2 * k] - z[2 * k + 2];
            s[2 * k + 3] = z[2 * k + 1] - z[2 * k + 3];
        }
        pthread_barrier_wait(w->bar);
        range_of(n, w->tid, w->nth, &lo, &hi);
        for (int64_t k = lo; k < hi; ++k) {                   /* gather (:269) */
            z[2 * k] = s[2 * j->rev[k]];
            z[2 * k + 1] = s[2 * j->rev[k] + 1];
        }
        pthread_barrier_wait(w->bar);
    }
    range_of(n, w->tid, w->nth, &lo, &hi);
    double *yr = j->y_re + r * j->out_stride, *yi = j->y_im + r * j->out_stride;
    for (int64_t k = lo; k < hi; ++k) {
        if (j->inverse) {               /* swap back, then data *= 1/N (:296-297) */
            yr[k] = z[2 * k + 1] * scale;
            yi[k] = z[2 * k] * scale;
        } else {
            yr[k] = z[2 * k];
            yi[k] = z[2 * k + 1];
        }
    }
    return NULL;
}

typedef struct {
    int m, tid, nth;
    double *wr, *wi;
    int64_t *rev;
} tab_t;

static void *table_worker(void *arg)
{
    tab_t *t = (tab_t *)arg;
    const int64_t n = 1LL << t->m, h = n / 2;
    int64_t lo, hi;
    range_of(h, t->tid, t->nth, &lo, &hi);
    for (int64_t q = lo; q < hi; ++q) stage_factor(t->m, q, &t->wr[q], &t->wi[q]);
    range_of(n, t->tid, t->nth, &lo, &hi);
    for (int64_t k = lo; k < hi; ++k) {
        int64_t r = 0, v = k;
        for (int b = 0; b < t->m; ++b) { r = (r << 1) | (v & 1); v >>= 1; }
        t->rev[k] = r;
    }
    return NULL;
}

static int run_wide(job_t *j, int64_t batch, int threads)
{
    const int64_t n = 1LL << j->m;
    double *z = (double *)malloc(sizeof(double) * 4 * (size_t)n);
    if (!z) return 2;
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)threads);
    pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    wide_t *ws = (wide_t *)calloc((size_t)threads, sizeof(wide_t));
    for (int64_t r = 0; r < batch; ++r) {
        for (int t = 0; t < threads; ++t) {
            ws[t].j = j; ws[t].tid = t; ws[t].nth = threads;
            ws[t].z = z; ws[t].s = z + 2 * n; ws[t].row = r; ws[t].bar = &bar;
            pthread_create(&tids[t], NULL, wide_worker, &ws[t]);
        }
        for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    }
    pthread_barrier_destroy(&bar);
    free(ws); free(tids); free(z);
    return 0;
}

/* Batched split -> split transform of `batch` rows, fp64, over `threads`
 * POSIX threads (the reference has no internal parallelism; threads split
 * independent rows, or -- fewer rows than threads and m >= 16 -- the
 * butterflies of each stage of one row, run_wide).  algo: 0 = dit,
 * 1 = dif.  Returns 0 on success. */
int oracle_fft_split(int m, int algo, int inverse,
                     const double *x_re, const double *x_im,
                     double *y_re, double *y_im,
                     int64_t batch, int64_t in_stride, int64_t out_stride,
                     int threads)
{
    if (m < 0 || m > ORACLE_MAX_M || batch < 0) return 1;
    if (threads < 1) threads = 1;
    const int wide = batch < threads && m >= 16;
    if (!wide && threads > batch) threads = batch > 0 ? (int)batch : 1;
    int64_t n = 1LL << m;
    int64_t h = m >= 1 ? n / 2 : 1;
    double *wr = (double *)malloc(sizeof(double) * 2 * (size_t)h);
    double *wi = wr + h;
    int64_t *rev = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    if (!wr || !rev) { free(wr); free(rev); return 2; }
    if (wide) {
        /* tables of a long plan in parallel (same values: stage_factor per q) */
        pthread_t *tt = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
        tab_t *ta = (tab_t *)calloc((size_t)threads, sizeof(tab_t));
        for (int t = 0; t < threads; ++t) {
            ta[t].m = m; ta[t].tid = t; ta[t].nth = threads; ta[t].wr = wr; ta[t].wi = wi; ta[t].rev = rev;
            pthread_create(&tt[t], NULL, table_worker, &ta[t]);
        }
        for (int t = 0; t < threads; ++t) pthread_join(tt[t], NULL);
        free(ta); free(tt);
        job_t j;
        memset(&j, 0, sizeof j);
        j.m = m; j.algo = algo; j.inverse = inverse;
        j.wr = wr; j.wi = wi; j.rev = rev;
        j.x_re = x_re; j.x_im = x_im; j.y_re = y_re; j.y_im = y_im;
        j.in_stride = in_stride; j.out_stride = out_stride;
        int rc = run_wide(&j, batch, threads);
        free(rev); free(wr);
        return rc;
    }
    if (m >= 1) oracle_twiddle_table(m, wr, wi);
    oracle_bitrev(m, rev);
    job_t *jobs = (job_t *)calloc((size_t)threads, sizeof(job_t));
    pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    int64_t per = (batch + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        job_t *j = &jobs[t];
        j->m = m; j->algo = algo; j->inverse = inverse;
        j->wr = wr; j->wi = wi; j->rev = rev;
        j->x_re = x_re; j->x_im = x_im; j->y_re = y_re; j->y_im = y_im;
        j->row0 = t * per < batch ? t * per : batch;
        j->row1 = (t + 1) * per < batch ? (t + 1) * per : batch;
        j->in_stride = in_stride; j->out_stride = out_stride;
    }
    if (threads == 1) {
        run_rows(&jobs[0]);
    } else {
        for (int t = 0; t < threads; ++t) pthread_create(&tids[t], NULL, run_rows, &jobs[t]);
        for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    }
    free(tids); free(jobs); free(rev); free(wr);
    return 0;
}
