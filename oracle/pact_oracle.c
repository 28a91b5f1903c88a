/*
 * pact_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker and the CPU
 * baseline leg of bench.py).  Nothing in the product path may link or call it.
 *
 * Matrix-free fp64 restatement of the reference's time-domain operator and its
 * two dense products, so that configs whose dense K does not fit in RAM (2.2 TB
 * at 512^2 x 512 x 2048) can still be checked and timed on the CPU.
 *
 * Operator (reference pkg/src/pactkit/forward.py):
 *   d      = hypot(px - sx, py - sy)                      forward.py:157-160
 *   u      = d / (c*dt);  s0 = floor(u);  f = u - s0        forward.py:180-182
 *   w      = 1 / (2*pi*c)                                  forward.py:183
 *   K[m*Q + s0-1, p] = (1-f)*w   if 1 <= s0 <= Q           forward.py:189,191,193
 *   K[m*Q + s0,   p] =  f   *w   if 0 <= s0 <= Q-1         forward.py:190,192,194
 * Products (reference pkg/src/pactkit/kernels.py):
 *   forward  out[i] = sum_j A[i,j]*x[j], ascending j         kernels.py:185-202
 *   adjoint  out[j] += A[i,j]*y[i],      ascending i         kernels.py:205-225
 * Skipping the structural zeros of K is exact: acc + (+-0) == acc for finite
 * acc, so the sums below reproduce the dense loops bit for bit (the survey
 * measured 2e-16 with a numpy restatement; this one keeps the summation order).
 *
 * Threads: a small pthread parallel-for (libgomp is absent from this image);
 * each output element has exactly one writer.
 *
 * Build with -ffp-contract=off: numba does not contract a*b+c into FMA, so
 * neither may we.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define OR_PI 3.141592653589793 /* np.pi */

/* geometry of one pair, exactly as build_time_matrix evaluates it */
static inline void pair_delay(double px, double py, double sx, double sy, double cdt,
                              int64_t* s0, double* frac)
{
    double d = hypot(px - sx, py - sy);  /* np.hypot == libm hypot */
    double u = d / cdt;
    double fl = floor(u);
    *s0 = (int64_t)fl;
    *frac = u - (double)(*s0);
}

/* ---- a minimal parallel-for over [0, n) (libgomp is not in this image) ---- */
typedef void (*or_body)(int64_t lo, int64_t hi, void* ctx);
typedef struct {
    or_body body; void* ctx; int64_t n, chunk; int64_t next; pthread_mutex_t mu;
} or_pool;

static void* or_worker(void* arg)
{
    or_pool* pl = (or_pool*)arg;
    for (;;) {
        pthread_mutex_lock(&pl->mu);
        int64_t lo = pl->next;
        pl->next += pl->chunk;
        pthread_mutex_unlock(&pl->mu);
        if (lo >= pl->n) break;
        int64_t hi = lo + pl->chunk < pl->n ? lo + pl->chunk : pl->n;
        pl->body(lo, hi, pl->ctx);
    }
    return NULL;
}

int or_max_threads(void)
{
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

/* chunks are handed out dynamically; every output element is owned by one
 * chunk, so the result does not depend on the thread count */
static void parallel_for(int64_t n, int64_t chunk, int threads, or_body body, void* ctx)
{
    if (threads <= 0) threads = or_max_threads();
    if (threads > 256) threads = 256;
    if (chunk < 1) chunk = 1;
    or_pool pl = {body, ctx, n, chunk, 0, PTHREAD_MUTEX_INITIALIZER};
    if (threads == 1 || n <= chunk) { body(0, n, ctx); return; }
    pthread_t tid[256];
    int started = 0;
    for (int t = 0; t < threads; ++t)
        if (pthread_create(&tid[t], NULL, or_worker, &pl) == 0) ++started;
    if (started == 0) or_worker(&pl);
    for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
}

typedef struct {
    int nx, ny, M, Q; const double *xx, *yy, *pos; double cdt, w;
    const double* in; double* out; int64_t* s0_out; double* frac_out;
} or_args;

double or_weight(double c) { return 1.0 / (2.0 * OR_PI * c); } /* forward.py:183 */

static void index_body(int64_t lo, int64_t hi, void* ctx)
{
    const or_args* a = (const or_args*)ctx;
    const int64_t P = (int64_t)a->nx * a->ny;
    for (int64_t m = lo; m < hi; ++m) {
        const double sx = a->pos[2 * m], sy = a->pos[2 * m + 1];
        for (int j = 0; j < a->ny; ++j)
            for (int i = 0; i < a->nx; ++i) {
                int64_t p = (int64_t)j * a->nx + i;
                int64_t s0; double f;
                pair_delay(a->xx[i], a->yy[j], sx, sy, a->cdt, &s0, &f);
                a->s0_out[m * P + p] = s0;
                if (a->frac_out) a->frac_out[m * P + p] = f;
            }
    }
}

/* s0 / frac dump for sensors [0, M): layout [m][p], p = j*nx + i (geometry.py:59-68) */
void or_index(int nx, int ny, const double* xx, const double* yy, int M, const double* pos,
              double cdt, int64_t* s0_out, double* frac_out, int threads)
{
    or_args a = {nx, ny, M, 0, xx, yy, pos, cdt, 0.0, NULL, NULL, s0_out, frac_out};
    parallel_for(M, 1, threads, index_body, &a);
}

/* number of truncated pairs, the count build_time_matrix warns about (forward.py:196-205) */
int64_t or_truncated(int nx, int ny, const double* xx, const double* yy, int M,
                     const double* pos, double cdt, int Q)
{
    int64_t n = 0;
    for (int m = 0; m < M; ++m)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                int64_t s0; double f;
                pair_delay(xx[i], yy[j], pos[2 * m], pos[2 * m + 1], cdt, &s0, &f);
                int in0 = s0 >= 1 && s0 <= Q;
                int in1 = s0 + 1 >= 1 && s0 + 1 <= Q;
                if (!in0 || (!in1 && f > 0.0)) ++n;
            }
    return n;
}

static void forward_body(int64_t lo, int64_t hi, void* ctx)
{
    const or_args* a = (const or_args*)ctx;
    const int Q = a->Q;
    const double w = a->w;
    for (int64_t m = lo; m < hi; ++m) {
        double* tr = a->out + m * Q;
        memset(tr, 0, sizeof(double) * (size_t)Q);
        const double sx = a->pos[2 * m], sy = a->pos[2 * m + 1];
        for (int j = 0; j < a->ny; ++j)
            for (int i = 0; i < a->nx; ++i) {
                const double xv = a->in[(int64_t)j * a->nx + i];
                int64_t s0; double f;
                pair_delay(a->xx[i], a->yy[j], sx, sy, a->cdt, &s0, &f);
                if (s0 >= 1 && s0 <= Q) tr[s0 - 1] += ((1.0 - f) * w) * xv;
                if (s0 >= 0 && s0 <= Q - 1) tr[s0] += (f * w) * xv;
            }
    }
}

/*
 * y = K x for sensors [0, M) of pos (pass pos + 2*m0 for a shard).
 * One sensor's trace per task; pixels visited in ascending p, which is the
 * ascending-j order of every output row of the dense product.
 */
void or_forward(int nx, int ny, const double* xx, const double* yy, int M, const double* pos,
                double cdt, double w, int Q, const double* x, double* out, int threads)
{
    or_args a = {nx, ny, M, Q, xx, yy, pos, cdt, w, x, out, NULL, NULL};
    parallel_for(M, 1, threads, forward_body, &a);
}

static void adjoint_body(int64_t lo, int64_t hi, void* ctx)
{
    const or_args* a = (const or_args*)ctx;
    const int Q = a->Q;
    const double w = a->w;
    for (int64_t p = lo; p < hi; ++p) {
        const int i = (int)(p % a->nx), j = (int)(p / a->nx);
        const double px = a->xx[i], py = a->yy[j];
        double acc = 0.0;
        for (int m = 0; m < a->M; ++m) {
            int64_t s0; double f;
            pair_delay(px, py, a->pos[2 * m], a->pos[2 * m + 1], a->cdt, &s0, &f);
            const double* tr = a->in + (int64_t)m * Q;
            if (s0 >= 1 && s0 <= Q) acc += ((1.0 - f) * w) * tr[s0 - 1];
            if (s0 >= 0 && s0 <= Q - 1) acc += (f * w) * tr[s0];
        }
        a->out[p] = acc;
    }
}

/*
 * out = K^T r: every pixel sums its sensors in ascending m, and inside one
 * sensor row s0-1 before row s0 -- the ascending-i order of the dense adjoint.
 */
void or_adjoint(int nx, int ny, const double* xx, const double* yy, int M, const double* pos,
                double cdt, double w, int Q, const double* r, double* out, int threads)
{
    or_args a = {nx, ny, M, Q, xx, yy, pos, cdt, w, r, out, NULL, NULL};
    parallel_for((int64_t)nx * ny, 256, threads, adjoint_body, &a);
}
