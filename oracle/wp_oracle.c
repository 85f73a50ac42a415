/*
 * CPU ORACLE - TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's float64 filter kernels, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker and the CPU baseline ("port"). Nothing in the product package links
 * or calls this file.
 *
 * Each function follows the reference loop for loop, float op for float op,
 * so that its outputs are bit-identical to the reference's numba kernels
 * (compile with -ffp-contract=off: no FMA contraction, IEEE order kept, like
 * numba with fastmath off, _kernels_jit.py:1-7):
 *
 *   wpo_iir_cascade  <- _iir_channel + iir_cascade_parallel  (_kernels_jit.py:14-48)
 *   wpo_fir_direct   <- _fir_channel + fir_direct_parallel   (_kernels_jit.py:51-78)
 *   wpo_transversal  <- oracle_transversal                   (_kernels_jit.py:81-100)
 *
 * Channel parallelism mirrors numba's prange over channels with a pthread
 * fan-out; every channel is computed by exactly one thread into its own row,
 * so results do not depend on the thread count (engine.py:1-8).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int kind; /* 0 = iir, 1 = fir */
    const double *coef; /* sos [S][5] or taps [T] */
    int64_t ncoef;
    const double *x;
    double *y;
    int64_t channels, frames;
    int64_t next; /* shared channel cursor */
    pthread_mutex_t lock;
} job_t;

/* _iir_channel: copy x -> out, then section-major DF2T in place with zeroed
 * state per section (_kernels_jit.py:14-32). */
static void iir_channel(const double *sos, int64_t S, const double *x, double *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = x[i];
    for (int64_t s = 0; s < S; ++s) {
        const double b0 = sos[5 * s + 0], b1 = sos[5 * s + 1], b2 = sos[5 * s + 2];
        const double a1 = sos[5 * s + 3], a2 = sos[5 * s + 4];
        double w1 = 0.0, w2 = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            const double xi = out[i];
            const double yi = b0 * xi + w1;
            w1 = b1 * xi - a1 * yi + w2;
            w2 = b2 * xi - a2 * yi;
            out[i] = yi;
        }
    }
}

/* _fir_channel: scalar accumulation over k = 0..min(i+1,T)-1 in order
 * (_kernels_jit.py:51-62). */
static void fir_channel(const double *taps, int64_t t, const double *x, double *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        int64_t kmax = i + 1;
        if (kmax > t) kmax = t;
        double acc = 0.0;
        for (int64_t k = 0; k < kmax; ++k) acc += taps[k] * x[i - k];
        out[i] = acc;
    }
}

static void *worker(void *arg) {
    job_t *job = (job_t *)arg;
    for (;;) {
        pthread_mutex_lock(&job->lock);
        const int64_t c = job->next++;
        pthread_mutex_unlock(&job->lock);
        if (c >= job->channels) break;
        const double *xr = job->x + c * job->frames;
        double *yr = job->y + c * job->frames;
        if (job->kind == 0)
            iir_channel(job->coef, job->ncoef, xr, yr, job->frames);
        else
            fir_channel(job->coef, job->ncoef, xr, yr, job->frames);
    }
    return NULL;
}

static void run(job_t *job, int threads) {
    if (threads < 1) threads = 1;
    if (threads > job->channels) threads = (int)job->channels;
    pthread_mutex_init(&job->lock, NULL);
    job->next = 0;
    if (threads <= 1) {
        worker(job);
    } else {
        pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
        for (int i = 0; i < threads; ++i) pthread_create(&tid[i], NULL, worker, job);
        for (int i = 0; i < threads; ++i) pthread_join(tid[i], NULL);
        free(tid);
    }
    pthread_mutex_destroy(&job->lock);
}

/* iir_cascade_parallel(sos, x): sos [S][5] with the cascade gain already folded
 * into section 0 (engine.py:133-139); x, y planar [C][N] float64. */
void wpo_iir_cascade(const double *sos, int64_t S, const double *x, double *y,
                     int64_t channels, int64_t frames, int threads) {
    job_t job;
    memset(&job, 0, sizeof(job));
    job.kind = 0;
    job.coef = sos;
    job.ncoef = S;
    job.x = x;
    job.y = y;
    job.channels = channels;
    job.frames = frames;
    run(&job, threads);
}

/* fir_direct_parallel(taps, x) */
void wpo_fir_direct(const double *taps, int64_t T, const double *x, double *y,
                    int64_t channels, int64_t frames, int threads) {
    job_t job;
    memset(&job, 0, sizeof(job));
    job.kind = 1;
    job.coef = taps;
    job.ncoef = T;
    job.x = x;
    job.y = y;
    job.channels = channels;
    job.frames = frames;
    run(&job, threads);
}

/* oracle_transversal(b, a, x): literal y[n] = sum b[k] x[n-k] - sum_{k>=1} a[k] y[n-k]
 * with a[0] == 1 checked by the caller (engine.py:181-198). */
void wpo_transversal(const double *b, int64_t nb, const double *a, int64_t na,
                     const double *x, double *y, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        int64_t kb = i + 1 < nb ? i + 1 : nb;
        for (int64_t k = 0; k < kb; ++k) acc += b[k] * x[i - k];
        int64_t ka = i + 1 < na ? i + 1 : na;
        for (int64_t k = 1; k < ka; ++k) acc -= a[k] * y[i - k];
        y[i] = acc;
    }
}

int wpo_abi_version(void) { return 1; }
