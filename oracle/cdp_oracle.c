/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, fp64, scalar) of the reference's per-micro-batch
 * value+gradient kernels.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the CPU baseline; the product path never does.
 *
 * Follows, loop for loop and in the same accumulation order:
 *   mlp_value_grad   pkg/src/cyclicdp/training/_kernels.pyx:25-132
 *                    (twin: _kernels_py.py:24-114)
 *     forward         _kernels.pyx:40-62
 *     MSE loss/dz     _kernels.pyx:72-79
 *     softmax-xent    _kernels.pyx:80-100
 *     backward        _kernels.pyx:102-130
 *   quad_value_grad  pkg/src/cyclicdp/training/_kernels.pyx:135-172
 *
 * Built with -O2 -ffp-contract=off (no FMA contraction, like the reference's
 * gcc -O3 build for generic x86-64), so results are bit-identical to the
 * reference; tests/test_oracle.py pins that against the committed golden
 * vectors (tests/golden/) generated from the reference itself.
 *
 * Parameter layout (ref models.py:63-68): stage j is W_j row-major
 * [din][dout] (index k*dout+o) followed by b_j [dout], stages concatenated.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

static void stage_offsets(int n_stages, const int64_t *dims, int64_t *off) {
    off[0] = 0;
    for (int j = 0; j < n_stages; ++j) off[j + 1] = off[j] + dims[j] * dims[j + 1] + dims[j + 1];
}

/* Returns the loss; grad[] (length = total params) is fully overwritten. */
double oracle_mlp_value_grad(int n_dims, const int64_t *dims, const double *theta, int batch,
                             const double *x, const double *y, const int64_t *labels, int loss_kind,
                             double *grad) {
    int n_stages = n_dims - 1;
    int64_t *off = (int64_t *)malloc(sizeof(int64_t) * (n_stages + 1));
    stage_offsets(n_stages, dims, off);
    memset(grad, 0, sizeof(double) * off[n_stages]);

    /* hs[j] = input of stage j (hs[0] = x); z = output of the last stage */
    double **hs = (double **)calloc(n_stages, sizeof(double *));
    hs[0] = (double *)x;
    double *z = NULL;
    for (int j = 0; j < n_stages; ++j) {
        int64_t din = dims[j], dout = dims[j + 1], base = off[j], bias = base + din * dout;
        const double *hin = hs[j];
        double *out = (double *)malloc(sizeof(double) * batch * dout);
        for (int s = 0; s < batch; ++s)
            for (int64_t o = 0; o < dout; ++o) {
                double acc = theta[bias + o];
                for (int64_t k = 0; k < din; ++k) acc += hin[s * din + k] * theta[base + k * dout + o];
                out[s * dout + o] = acc;
            }
        if (j < n_stages - 1) {
            for (int64_t q = 0; q < (int64_t)batch * dout; ++q) out[q] = tanh(out[q]);
            hs[j + 1] = out;
        } else {
            z = out;
        }
    }

    int64_t dlast = dims[n_stages];
    double *dz = (double *)calloc((size_t)batch * dlast, sizeof(double));
    double loss = 0.0;
    if (loss_kind == 0) {
        for (int s = 0; s < batch; ++s)
            for (int64_t o = 0; o < dlast; ++o) {
                double d = z[s * dlast + o] - y[s * dlast + o];
                loss += d * d;
                dz[s * dlast + o] = d / batch;
            }
        loss = loss / (2.0 * batch);
    } else {
        double *p = (double *)malloc(sizeof(double) * dlast);
        for (int s = 0; s < batch; ++s) {
            const double *zr = z + s * dlast;
            int64_t lab = labels[s];
            double m = zr[0];
            for (int64_t o = 1; o < dlast; ++o)
                if (zr[o] > m) m = zr[o];
            double se = 0.0;
            for (int64_t o = 0; o < dlast; ++o) {
                double e = exp(zr[o] - m);
                p[o] = e;
                se += e;
            }
            for (int64_t o = 0; o < dlast; ++o) p[o] = p[o] / se;
            loss += -log(p[lab]);
            for (int64_t o = 0; o < dlast; ++o) dz[s * dlast + o] = (p[o] - (o == lab ? 1.0 : 0.0)) / batch;
        }
        loss = loss / batch;
        free(p);
    }

    for (int j = n_stages - 1; j >= 0; --j) {
        int64_t din = dims[j], dout = dims[j + 1], base = off[j], bias = base + din * dout;
        const double *hin = hs[j];
        for (int64_t k = 0; k < din; ++k)
            for (int64_t o = 0; o < dout; ++o) {
                double acc = 0.0;
                for (int s = 0; s < batch; ++s) acc += hin[s * din + k] * dz[s * dout + o];
                grad[base + k * dout + o] = acc;
            }
        for (int64_t o = 0; o < dout; ++o) {
            double acc = 0.0;
            for (int s = 0; s < batch; ++s) acc += dz[s * dout + o];
            grad[bias + o] = acc;
        }
        if (j > 0) {
            double *prev = (double *)calloc((size_t)batch * din, sizeof(double));
            for (int s = 0; s < batch; ++s)
                for (int64_t k = 0; k < din; ++k) {
                    double acc = 0.0;
                    for (int64_t o = 0; o < dout; ++o) acc += dz[s * dout + o] * theta[base + k * dout + o];
                    double h = hin[s * din + k];
                    prev[s * din + k] = acc * (1.0 - h * h);
                }
            free(dz);
            dz = prev;
        }
    }
    free(dz);
    for (int j = 1; j < n_stages; ++j) free(hs[j]);
    free(hs);
    free(z);
    free(off);
    return loss;
}

/* Coupled quadratic fixture (ref _kernels.pyx:135-172). a is [m][p]. */
double oracle_quad_value_grad(int m, int p_dim, const double *a, const double *theta, int batch,
                              const double *targets, double *grad) {
    double *z = (double *)calloc(m, sizeof(double));
    double *rsum = (double *)calloc(m, sizeof(double));
    for (int r = 0; r < m; ++r) {
        double acc = 0.0;
        for (int p = 0; p < p_dim; ++p) acc += a[r * p_dim + p] * theta[p];
        z[r] = acc;
    }
    double loss = 0.0;
    for (int s = 0; s < batch; ++s)
        for (int r = 0; r < m; ++r) {
            double d = z[r] - targets[s * m + r];
            loss += d * d;
            rsum[r] += d;
        }
    loss = loss / (2.0 * m * batch);
    double scale = 1.0 / (m * batch);
    for (int p = 0; p < p_dim; ++p) {
        double acc = 0.0;
        for (int r = 0; r < m; ++r) acc += a[r * p_dim + p] * rsum[r];
        grad[p] = acc * scale;
    }
    free(z);
    free(rsum);
    return loss;
}

/* ---- multi-threaded driver for the CPU baseline: one thread per micro-batch ---- */
typedef struct {
    int n_dims;
    const int64_t *dims;
    const double *theta;
    int batch;
    const double *x;
    const double *y;
    const int64_t *labels;
    int loss_kind;
    double *grad;
    double loss;
} mlp_job;

static void *mlp_job_run(void *arg) {
    mlp_job *j = (mlp_job *)arg;
    j->loss = oracle_mlp_value_grad(j->n_dims, j->dims, j->theta, j->batch, j->x, j->y, j->labels,
                                    j->loss_kind, j->grad);
    return NULL;
}

/* n_jobs independent micro-batches; thetas[i], xs[i], labels[i], grads[i] per job.
 * Runs up to `threads` jobs concurrently; losses[i] receives each loss. */
void oracle_mlp_value_grad_batch(int n_jobs, int threads, int n_dims, const int64_t *dims,
                                 const double *const *thetas, int batch, const double *const *xs,
                                 const double *const *ys, const int64_t *const *labels, int loss_kind,
                                 double *const *grads, double *losses) {
    if (threads < 1) threads = 1;
    mlp_job *jobs = (mlp_job *)calloc(n_jobs, sizeof(mlp_job));
    pthread_t *tids = (pthread_t *)calloc(n_jobs, sizeof(pthread_t));
    for (int i = 0; i < n_jobs; ++i) {
        jobs[i] = (mlp_job){n_dims, dims, thetas[i], batch, xs[i], ys ? ys[i] : NULL,
                            labels ? labels[i] : NULL, loss_kind, grads[i], 0.0};
    }
    for (int lo = 0; lo < n_jobs; lo += threads) {
        int hi = lo + threads < n_jobs ? lo + threads : n_jobs;
        for (int i = lo; i < hi; ++i) pthread_create(&tids[i], NULL, mlp_job_run, &jobs[i]);
        for (int i = lo; i < hi; ++i) pthread_join(tids[i], NULL);
    }
    for (int i = 0; i < n_jobs; ++i) losses[i] = jobs[i].loss;
    free(jobs);
    free(tids);
}
