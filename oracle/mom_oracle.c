/*
 * oracle/mom_oracle.c -- the CPU ORACLE for the MOM mini-sequence prefill MLP path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2504_12526_b200/csrc); the
 * product library never links or calls it.
 *
 * What it computes (citations are /root/reference/PAPER.md line numbers, "P:<n>",
 * and SPEC.md lines, "S:<n>"):
 *   - oracle_plan            Alg. 1 P:109  M = ceil(S/C) mini-sequences, sizes (C,..,C, S-(M-1)C)
 *   - oracle_mlp_minseq      Alg. 1 P:109-113  for i = 1..M: O_i = MLP(A_i); O = concat(O_1..O_M)
 *                            MLP = SwiGLU: O = (Swish(A Wg^T) (.) A Wu^T) Wd^T,
 *                            Swish(z) = z * sigmoid(z); plus an optional residual (reading R2).
 *   - oracle_mlp_rows        the same MLP evaluated on an arbitrary list of rows (rows are
 *                            independent, so this is exact for sampled-row parity).
 *   - oracle_rmsnorm         final norm before the LM head (reading R3).
 *   - oracle_lm_head         Alg. 1 P:105  L = LM_Head(O_last): logits_v = sum_k h_k W[v,k].
 *   - oracle_argmax_f32/f64  greedy next token, ties -> lowest index.
 *
 * Arithmetic: inputs arrive as float32 arrays holding exactly the values the GPU gets
 * (bf16 widened exactly).  Every product of two float32 values is exact in float64
 * (24+24 significant bits < 53), and every sum is accumulated in float64 in ascending
 * index order with no contraction (-ffp-contract=off).  Threads split ROWS only, so each
 * output value is computed by one fixed sequence of operations: the result is bitwise
 * identical for every mini-sequence size C and every thread count.
 *
 * Parity pins (tests/test_oracle.py) tie every function to something other than itself:
 * SPEC worked values, closed forms, exact rational brute force, the paper's two facts.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ---------------------------------------------------------------------------------
 * a1. Partition plan.  Alg. 1: "Partition A into M = ceil(S/C) mini-sequences
 * {A_i}, where each A_i in R^{B x N x d} and N ~= C".  Sizes (C,...,C, S-(M-1)C).
 * Returns M; writes at most `cap` (start, length) pairs.  Returns -1 on S<0 or C<1.
 * ------------------------------------------------------------------------------- */
int64_t oracle_plan(int64_t S, int64_t C, int64_t *starts, int64_t *lens, int64_t cap)
{
    if (S < 0 || C < 1) return -1;
    int64_t M = (S + C - 1) / C;          /* ceil(S/C) */
    for (int64_t i = 0; i < M && i < cap; ++i) {
        int64_t r0 = i * C;
        int64_t r1 = r0 + C;
        if (r1 > S) r1 = S;
        starts[i] = r0;
        lens[i] = r1 - r0;
    }
    return M;
}

/* Swish with beta = 1 ("Swish(X W_gate)"; S:228 swish(z) = z * sigma(z)). */
static double swish(double z)
{
    double sigma = 1.0 / (1.0 + exp(-z));
    return z * sigma;
}

/* One row of the SwiGLU MLP:
 *   g_j = sum_k x_k Wg[j,k]      (gate projection, W_gate: d -> I)
 *   u_j = sum_k x_k Wu[j,k]      (up projection,   W_up:   d -> I)
 *   h_j = Swish(g_j) * u_j       ("multiplied element-wise")
 *   o_c = sum_j h_j Wd[c,j]      (down projection, W_down: I -> d)
 *   out_c = residual_c + o_c     (residual optional)
 * Weights are in nn.Linear layout: Wg, Wu are [I, d], Wd is [d, I], row-major. */
static void mlp_one_row(const float *x, const float *res,
                        const float *wg, const float *wu, const float *wd,
                        int64_t d, int64_t I, double *h, double *out)
{
    for (int64_t j = 0; j < I; ++j) {
        const float *wg_j = wg + j * d;
        const float *wu_j = wu + j * d;
        double g = 0.0, u = 0.0;
        for (int64_t k = 0; k < d; ++k) {
            g = g + (double)x[k] * (double)wg_j[k];
            u = u + (double)x[k] * (double)wu_j[k];
        }
        h[j] = swish(g) * u;
    }
    for (int64_t c = 0; c < d; ++c) {
        const float *wd_c = wd + c * I;
        double o = 0.0;
        for (int64_t j = 0; j < I; ++j) o = o + h[j] * (double)wd_c[j];
        out[c] = (res ? (double)res[c] : 0.0) + o;
    }
}

/* ----------------------------- row-parallel driver ------------------------------ */
typedef struct {
    const float *x, *res, *wg, *wu, *wd;
    const int64_t *rows;   /* row ids into x/res; out row t <- input row rows[t] */
    int64_t n_rows, d, I;
    double *out;           /* [n_rows, d] */
    int64_t t_begin, t_end;
    int status;
} rows_job_t;

static void *rows_worker(void *arg)
{
    rows_job_t *jb = (rows_job_t *)arg;
    double *h = (double *)malloc(sizeof(double) * (size_t)jb->I);
    if (!h) { jb->status = -1; return NULL; }
    for (int64_t t = jb->t_begin; t < jb->t_end; ++t) {
        int64_t r = jb->rows[t];
        mlp_one_row(jb->x + r * jb->d, jb->res ? jb->res + r * jb->d : NULL,
                    jb->wg, jb->wu, jb->wd, jb->d, jb->I, h, jb->out + t * jb->d);
    }
    free(h);
    jb->status = 0;
    return NULL;
}

static int run_rows(const float *x, const float *res, const float *wg, const float *wu,
                    const float *wd, const int64_t *rows, int64_t n_rows, int64_t d, int64_t I,
                    double *out, int nthreads)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads > n_rows) nthreads = (int)(n_rows > 0 ? n_rows : 1);
    rows_job_t *jobs = (rows_job_t *)calloc((size_t)nthreads, sizeof(rows_job_t));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return -1; }
    int64_t per = (n_rows + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        rows_job_t *jb = &jobs[t];
        jb->x = x; jb->res = res; jb->wg = wg; jb->wu = wu; jb->wd = wd;
        jb->rows = rows; jb->n_rows = n_rows; jb->d = d; jb->I = I; jb->out = out;
        jb->t_begin = (int64_t)t * per;
        jb->t_end = jb->t_begin + per > n_rows ? n_rows : jb->t_begin + per;
        if (jb->t_begin > n_rows) jb->t_begin = n_rows;
        jb->status = -2;
    }
    int rc = 0;
    for (int t = 1; t < nthreads; ++t)
        if (pthread_create(&th[t], NULL, rows_worker, &jobs[t]) != 0) { jobs[t].status = -3; }
    rows_worker(&jobs[0]);
    for (int t = 1; t < nthreads; ++t)
        if (jobs[t].status != -3) pthread_join(th[t], NULL);
    for (int t = 0; t < nthreads; ++t) if (jobs[t].status != 0) rc = -1;
    free(jobs); free(th);
    return rc;
}

/* The MLP on an arbitrary list of rows: out[t, :] = residual[rows[t]] + MLP(x[rows[t]]).
 * Rows are independent (position-wise op), so sampled-row parity is exact. */
int oracle_mlp_rows(const float *x, const float *residual,
                    const float *w_gate, const float *w_up, const float *w_down,
                    const int64_t *rows, int64_t n_rows, int64_t d, int64_t I,
                    double *out, int nthreads)
{
    if (!x || !w_gate || !w_up || !w_down || !out || (n_rows > 0 && !rows)) return -1;
    if (d < 1 || I < 1 || n_rows < 0) return -1;
    if (n_rows == 0) return 0;
    return run_rows(x, residual, w_gate, w_up, w_down, rows, n_rows, d, I, out, nthreads);
}

/* Alg. 1, non-final branch, step by step:
 *   Partition A into M = ceil(S/C) mini-sequences;
 *   for i = 1..M: O_i = MLP(A_i);
 *   O = concat(O_1, ..., O_M)  -- O_i written at rows [start_i, start_i+len_i)
 * out is [S, d] float64. */
int oracle_mlp_minseq(const float *x, const float *residual,
                      const float *w_gate, const float *w_up, const float *w_down,
                      int64_t S, int64_t d, int64_t I, int64_t C, double *out, int nthreads)
{
    if (S < 1 || C < 1 || d < 1 || I < 1) return -1;
    int64_t M = (S + C - 1) / C;
    int64_t *starts = (int64_t *)malloc(sizeof(int64_t) * (size_t)M);
    int64_t *lens = (int64_t *)malloc(sizeof(int64_t) * (size_t)M);
    int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * (size_t)(C < S ? C : S));
    if (!starts || !lens || !rows) { free(starts); free(lens); free(rows); return -1; }
    oracle_plan(S, C, starts, lens, M);
    int rc = 0;
    for (int64_t i = 0; i < M && rc == 0; ++i) {
        /* A_i = rows [starts[i], starts[i] + lens[i]) of A */
        for (int64_t t = 0; t < lens[i]; ++t) rows[t] = starts[i] + t;
        /* O_i = MLP(A_i), written directly into its rows of O (the concat) */
        rc = run_rows(x, residual, w_gate, w_up, w_down, rows, lens[i], d, I,
                      out + starts[i] * d, nthreads);
    }
    free(starts); free(lens); free(rows);
    return rc;
}

/* f3: the Llama pre-norm block's MLP half ("x + mlp(norm(x))"),
 *   xn = RMSNorm(x) (.) gain,  RMSNorm(x)_k = x_k / sqrt(mean(x^2) + eps)
 *   out = x + MLP(xn)
 * evaluated exactly in that order, row by row, float64. */
typedef struct {
    const float *x, *gain, *wg, *wu, *wd;
    double eps;
    const int64_t *rows;
    int64_t d, I;
    double *out;
    int64_t t_begin, t_end;
    int status;
} norm_job_t;

static void *norm_worker(void *arg)
{
    norm_job_t *jb = (norm_job_t *)arg;
    double *xn = (double *)malloc(sizeof(double) * (size_t)jb->d);
    double *h = (double *)malloc(sizeof(double) * (size_t)jb->I);
    if (!xn || !h) { free(xn); free(h); jb->status = -1; return NULL; }
    for (int64_t t = jb->t_begin; t < jb->t_end; ++t) {
        const float *x = jb->x + jb->rows[t] * jb->d;
        double ss = 0.0;
        for (int64_t k = 0; k < jb->d; ++k) ss = ss + (double)x[k] * (double)x[k];
        double inv = 1.0 / sqrt(ss / (double)jb->d + jb->eps);
        for (int64_t k = 0; k < jb->d; ++k) xn[k] = (double)x[k] * inv * (double)jb->gain[k];
        for (int64_t j = 0; j < jb->I; ++j) {
            const float *wg_j = jb->wg + j * jb->d, *wu_j = jb->wu + j * jb->d;
            double g = 0.0, u = 0.0;
            for (int64_t k = 0; k < jb->d; ++k) {
                g = g + xn[k] * (double)wg_j[k];
                u = u + xn[k] * (double)wu_j[k];
            }
            h[j] = swish(g) * u;
        }
        double *o = jb->out + t * jb->d;
        for (int64_t c = 0; c < jb->d; ++c) {
            const float *wd_c = jb->wd + c * jb->I;
            double acc = 0.0;
            for (int64_t j = 0; j < jb->I; ++j) acc = acc + h[j] * (double)wd_c[j];
            o[c] = (double)x[c] + acc;
        }
    }
    free(xn); free(h);
    jb->status = 0;
    return NULL;
}

int oracle_mlp_norm_rows(const float *x, const float *gain, double eps, const float *w_gate,
                         const float *w_up, const float *w_down, const int64_t *rows, int64_t n_rows,
                         int64_t d, int64_t I, double *out, int nthreads)
{
    if (!x || !gain || !w_gate || !w_up || !w_down || !out || (n_rows > 0 && !rows)) return -1;
    if (d < 1 || I < 1 || n_rows < 0 || eps < 0.0) return -1;
    if (n_rows == 0) return 0;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > n_rows) nthreads = (int)n_rows;
    norm_job_t *jobs = (norm_job_t *)calloc((size_t)nthreads, sizeof(norm_job_t));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    int *started = (int *)calloc((size_t)nthreads, sizeof(int));
    if (!jobs || !th || !started) { free(jobs); free(th); free(started); return -1; }
    int64_t per = (n_rows + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        norm_job_t *jb = &jobs[t];
        jb->x = x; jb->gain = gain; jb->eps = eps; jb->wg = w_gate; jb->wu = w_up; jb->wd = w_down;
        jb->rows = rows; jb->d = d; jb->I = I; jb->out = out;
        jb->t_begin = (int64_t)t * per; if (jb->t_begin > n_rows) jb->t_begin = n_rows;
        jb->t_end = jb->t_begin + per > n_rows ? n_rows : jb->t_begin + per;
        jb->status = -2;
    }
    for (int t = 1; t < nthreads; ++t) started[t] = pthread_create(&th[t], NULL, norm_worker, &jobs[t]) == 0;
    norm_worker(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) {
        if (started[t]) pthread_join(th[t], NULL); else norm_worker(&jobs[t]);
    }
    int rc = 0;
    for (int t = 0; t < nthreads; ++t) if (jobs[t].status != 0) rc = -1;
    free(jobs); free(th); free(started);
    return rc;
}

/* Final RMSNorm on one row (S:126 rmsnorm: y = x / sqrt(mean(x^2) + eps) (.) gain; applied
 * after slicing the last token).  gain may be NULL (= all ones). */
int oracle_rmsnorm(const double *y, const float *gain, double eps, int64_t d, double *out)
{
    if (!y || !out || d < 1) return -1;
    double ss = 0.0;
    for (int64_t k = 0; k < d; ++k) ss = ss + y[k] * y[k];
    double mean = ss / (double)d;
    double inv = 1.0 / sqrt(mean + eps);
    for (int64_t k = 0; k < d; ++k) out[k] = y[k] * inv * (gain ? (double)gain[k] : 1.0);
    return 0;
}

/* LM head (Alg. 1): logits[r, v] = sum_k h[r, k] W[v, k], W is [V, d] row-major.
 * n rows of h (n = 1 is the MOM last-token path; n = S is the standard path of fact F2). */
typedef struct {
    const double *h; const float *w; int64_t n, V, d; double *logits; int64_t v0, v1;
} head_job_t;

static void *head_worker(void *arg)
{
    head_job_t *jb = (head_job_t *)arg;
    for (int64_t r = 0; r < jb->n; ++r) {
        const double *hr = jb->h + r * jb->d;
        for (int64_t v = jb->v0; v < jb->v1; ++v) {
            const float *wv = jb->w + v * jb->d;
            double acc = 0.0;
            for (int64_t k = 0; k < jb->d; ++k) acc = acc + hr[k] * (double)wv[k];
            jb->logits[r * jb->V + v] = acc;
        }
    }
    return NULL;
}

int oracle_lm_head(const double *h, const float *w_head, int64_t n, int64_t V, int64_t d,
                   double *logits, int nthreads)
{
    if (!h || !w_head || !logits || n < 1 || V < 1 || d < 1) return -1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > V) nthreads = (int)V;
    head_job_t *jobs = (head_job_t *)calloc((size_t)nthreads, sizeof(head_job_t));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return -1; }
    int64_t per = (V + nthreads - 1) / nthreads;
    int *started = (int *)calloc((size_t)nthreads, sizeof(int));
    for (int t = 0; t < nthreads; ++t) {
        head_job_t *jb = &jobs[t];
        jb->h = h; jb->w = w_head; jb->n = n; jb->V = V; jb->d = d; jb->logits = logits;
        jb->v0 = (int64_t)t * per; if (jb->v0 > V) jb->v0 = V;
        jb->v1 = jb->v0 + per > V ? V : jb->v0 + per;
    }
    for (int t = 1; t < nthreads; ++t)
        started[t] = pthread_create(&th[t], NULL, head_worker, &jobs[t]) == 0;
    head_worker(&jobs[0]);
    int rc = 0;
    for (int t = 1; t < nthreads; ++t) {
        if (started[t]) pthread_join(th[t], NULL);
        else { head_worker(&jobs[t]); }
    }
    free(jobs); free(th); free(started);
    return rc;
}

/* Greedy next token: index of the maximum logit, ties -> lowest index.
 * The f32 form takes the decision in the kernel's precision (fp32 logits), the f64 form
 * in the oracle's.  NaN never wins (inputs are finite by construction). */
int64_t oracle_argmax_f32(const float *logits, int64_t V)
{
    if (!logits || V < 1) return -1;
    int64_t best = 0;
    for (int64_t v = 1; v < V; ++v) if (logits[v] > logits[best]) best = v;
    return best;
}

int64_t oracle_argmax_f64(const double *logits, int64_t V)
{
    if (!logits || V < 1) return -1;
    int64_t best = 0;
    for (int64_t v = 1; v < V; ++v) if (logits[v] > logits[best]) best = v;
    return best;
}
