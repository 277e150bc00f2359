/*
 * sos_oracle.c -- fp64 CPU ORACLE for the over-parameterised SOS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call this
 * file.  The product path (paper_2410_19844_b200/) never links it, and it
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, cited by line):
 *
 *   - PAPER.md:45-60 (sec 1.1, Eq. 1): p = m_d B m_d^T, m_d the vector of
 *     monomials; restricted to forms, m_d holds the degree-d
 *     monomials in n variables, of which there are C(n+d-1, d)
 *     (PAPER.md:58-60).  Example: n=d=2, m_d=(x1^2,x1x2,x2^2).
 *   - PAPER.md:72-76 (sec 1.1, Eq. 2): minimise ||p - m_d P P^T m_d^T||^2,
 *     "the squared norm of the difference between their coefficient vectors".
 *     Here P is called V (N x r), the k-th square is q_k = m_d . v_k.
 *   - PAPER.md:221 (sec 4): first-order optimisation ("basic ADAM approach");
 *     plain gradient descent is the other optimiser the task names.
 *
 * Reading: monomial order is colex order of the
 * sorted variable-index multiset (the order of the combinatorial number
 * system); it reproduces the paper's n=d=2 example order.  The oracle
 * realises that order by DEFINITION: enumerate every exponent vector, sort
 * with the colex comparator, look ranks up by binary search.  No binomial
 * ranking formula appears here.
 *
 * Everything is plain loops in double precision; nothing is blocked or fused.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------ */
/* Monomial basis of degree D in n variables, colex order.            */
/* ------------------------------------------------------------------ */

typedef struct {
    int n, D;
    int64_t count;
    uint8_t *ms; /* count x D : sorted variable-index multiset m_1<=...<=m_D */
    uint8_t *ex; /* count x n : exponent vector                            */
} basis_t;

static int g_cmp_D; /* qsort has no context argument; the oracle is single-threaded */

/* colex comparison of two sorted multisets: compare the LAST entries
 * first, then the previous ones (PAPER.md:53 order x1^2 < x1x2 < x2^2). */
static int colex_cmp_D(const uint8_t *a, const uint8_t *b, int D) {
    for (int k = D - 1; k >= 0; --k) {
        if (a[k] != b[k]) return a[k] < b[k] ? -1 : 1;
    }
    return 0;
}

static int colex_qsort_cmp(const void *a, const void *b) {
    return colex_cmp_D((const uint8_t *)a, (const uint8_t *)b, g_cmp_D);
}

/* Count exponent vectors of degree D in n variables by plain recursion. */
static int64_t count_rec(int n, int D) {
    if (n == 1) return 1;
    int64_t c = 0;
    for (int e = 0; e <= D; ++e) c += count_rec(n - 1, D - e);
    return c;
}

/* Emit all exponent vectors (any order) by plain recursion. */
static void emit_rec(int n, int D, int v, int left, uint8_t *cur, uint8_t *out, int64_t *pos) {
    if (v == n - 1) {
        cur[v] = (uint8_t)left;
        memcpy(out + (*pos) * n, cur, (size_t)n);
        (*pos)++;
        return;
    }
    for (int e = 0; e <= left; ++e) {
        cur[v] = (uint8_t)e;
        emit_rec(n, D, v + 1, left - e, cur, out, pos);
    }
}

static void ex_to_ms(const uint8_t *ex, int n, uint8_t *ms) {
    int k = 0;
    for (int v = 0; v < n; ++v)
        for (int t = 0; t < ex[v]; ++t) ms[k++] = (uint8_t)v;
}

static void ms_to_ex(const uint8_t *ms, int D, int n, uint8_t *ex) {
    memset(ex, 0, (size_t)n);
    for (int k = 0; k < D; ++k) ex[ms[k]]++;
}

static int basis_build(basis_t *b, int n, int D) {
    b->n = n; b->D = D;
    b->count = count_rec(n, D);
    uint8_t *raw = (uint8_t *)malloc((size_t)b->count * n);
    uint8_t cur[256];
    int64_t pos = 0;
    if (!raw) return -1;
    emit_rec(n, D, 0, D, cur, raw, &pos);
    b->ms = (uint8_t *)malloc((size_t)b->count * (D > 0 ? D : 1));
    b->ex = (uint8_t *)malloc((size_t)b->count * n);
    if (!b->ms || !b->ex) return -1;
    for (int64_t i = 0; i < b->count; ++i) ex_to_ms(raw + i * n, n, b->ms + i * D);
    free(raw);
    g_cmp_D = D;
    qsort(b->ms, (size_t)b->count, (size_t)D, colex_qsort_cmp);
    for (int64_t i = 0; i < b->count; ++i) ms_to_ex(b->ms + i * D, D, n, b->ex + i * n);
    return 0;
}

/* rank of an exponent vector by binary search in the sorted basis; -1 if absent */
static int64_t basis_rank_ex(const basis_t *b, const uint8_t *ex) {
    uint8_t key[256];
    int s = 0;
    for (int v = 0; v < b->n; ++v) s += ex[v];
    if (s != b->D) return -1;
    ex_to_ms(ex, b->n, key);
    int64_t lo = 0, hi = b->count - 1;
    while (lo <= hi) {
        int64_t mid = lo + (hi - lo) / 2;
        int c = colex_cmp_D(b->ms + mid * b->D, key, b->D);
        if (c == 0) return mid;
        if (c < 0) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* ------------------------------------------------------------------ */
/* Oracle index: alpha = degree-d basis (m_d), beta = degree-2d basis. */
/* ------------------------------------------------------------------ */

typedef struct {
    int n, d;
    basis_t a; /* degree d  : N entries */
    basis_t b; /* degree 2d : M entries */
} or_index_t;

void *or_index_create(int n, int d) {
    if (n < 1 || d < 1 || n > 255 || 2 * d > 255) return NULL;
    or_index_t *h = (or_index_t *)calloc(1, sizeof(or_index_t));
    h->n = n; h->d = d;
    if (basis_build(&h->a, n, d) || basis_build(&h->b, n, 2 * d)) return NULL;
    return h;
}

void or_index_destroy(void *hv) {
    or_index_t *h = (or_index_t *)hv;
    if (!h) return;
    free(h->a.ms); free(h->a.ex); free(h->b.ms); free(h->b.ex);
    free(h);
}

int64_t or_index_N(void *hv) { return ((or_index_t *)hv)->a.count; }
int64_t or_index_M(void *hv) { return ((or_index_t *)hv)->b.count; }
int64_t or_basis_count(int n, int D) { return count_rec(n, D); }

/* exponent tables, row-major */
void or_index_alpha(void *hv, uint8_t *out) {
    or_index_t *h = (or_index_t *)hv;
    memcpy(out, h->a.ex, (size_t)h->a.count * h->n);
}
void or_index_beta(void *hv, uint8_t *out) {
    or_index_t *h = (or_index_t *)hv;
    memcpy(out, h->b.ex, (size_t)h->b.count * h->n);
}

/* rank in the degree-2d basis of given exponent vectors (count x n); -1 if not degree 2d */
void or_rank2d(void *hv, const uint8_t *ex, int64_t count, int64_t *out) {
    or_index_t *h = (or_index_t *)hv;
    for (int64_t t = 0; t < count; ++t) out[t] = basis_rank_ex(&h->b, ex + t * h->n);
}

/* rank(alpha_i + alpha_j) for i in rows[], all j: out is nrows x N */
void or_pair_ranks(void *hv, const int64_t *rows, int64_t nrows, uint32_t *out) {
    or_index_t *h = (or_index_t *)hv;
    int n = h->n;
    int64_t N = h->a.count;
    uint8_t s[256];
    for (int64_t t = 0; t < nrows; ++t) {
        const uint8_t *ai = h->a.ex + rows[t] * n;
        for (int64_t j = 0; j < N; ++j) {
            const uint8_t *aj = h->a.ex + j * n;
            for (int v = 0; v < n; ++v) s[v] = (uint8_t)(ai[v] + aj[v]);
            out[t * N + j] = (uint32_t)basis_rank_ex(&h->b, s);
        }
    }
}

/* ------------------------------------------------------------------ */
/* Forward: coef(m_d V V^T m_d^T)   (Eq. 2)           */
/* The polynomial is sum_{i,j} G_ij x^(alpha_i) x^(alpha_j), G = V V^T */
/* ------------------------------------------------------------------ */

static double dot_row(const double *V, int64_t r, int64_t i, int64_t j) {
    double s = 0.0;
    for (int64_t k = 0; k < r; ++k) s += V[i * r + k] * V[j * r + k];
    return s;
}

void or_forward(void *hv, const double *V, int64_t r, double *coef) {
    or_index_t *h = (or_index_t *)hv;
    int n = h->n;
    int64_t N = h->a.count, M = h->b.count;
    uint8_t s[256];
    for (int64_t q = 0; q < M; ++q) coef[q] = 0.0;
    for (int64_t i = 0; i < N; ++i) {
        for (int64_t j = 0; j < N; ++j) {
            for (int v = 0; v < n; ++v) s[v] = (uint8_t)(h->a.ex[i * n + v] + h->a.ex[j * n + v]);
            int64_t q = basis_rank_ex(&h->b, s);
            coef[q] += dot_row(V, r, i, j);
        }
    }
}

/* The same pair loop restricted to rows i0 <= i < i1 (all j), ADDED into coef
 * (the caller zeroes it).  Summing the partial vectors of a partition of the
 * rows gives or_forward up to the order of the additions, so independent row
 * ranges can run on separate host threads (the loop body is unchanged). */
void or_forward_rows(void *hv, const double *V, int64_t r, int64_t i0, int64_t i1, double *coef) {
    or_index_t *h = (or_index_t *)hv;
    int n = h->n;
    int64_t N = h->a.count;
    uint8_t s[256];
    for (int64_t i = i0; i < i1 && i < N; ++i) {
        for (int64_t j = 0; j < N; ++j) {
            for (int v = 0; v < n; ++v) s[v] = (uint8_t)(h->a.ex[i * n + v] + h->a.ex[j * n + v]);
            int64_t q = basis_rank_ex(&h->b, s);
            coef[q] += dot_row(V, r, i, j);
        }
    }
}

/* Selected coefficients only: coef_beta = sum over ordered pairs (i,j) with
 * alpha_i + alpha_j = beta of <v_i, v_j>  (same definition, per beta). */
void or_coef_sample(void *hv, const double *V, int64_t r, const int64_t *betas, int64_t k, double *out) {
    or_index_t *h = (or_index_t *)hv;
    int n = h->n;
    int64_t N = h->a.count;
    uint8_t rest[256];
    for (int64_t t = 0; t < k; ++t) {
        const uint8_t *bt = h->b.ex + betas[t] * n;
        double acc = 0.0;
        for (int64_t i = 0; i < N; ++i) {
            const uint8_t *ai = h->a.ex + i * n;
            int ok = 1;
            for (int v = 0; v < n; ++v) {
                if (ai[v] > bt[v]) { ok = 0; break; }
                rest[v] = (uint8_t)(bt[v] - ai[v]);
            }
            if (!ok) continue;
            int64_t j = basis_rank_ex(&h->a, rest);
            if (j < 0) continue;
            acc += dot_row(V, r, i, j);
        }
        out[t] = acc;
    }
}

/* ------------------------------------------------------------------ */
/* Loss and gradient of Eq. 2.                       */
/* L(V) = sum_beta (coef_beta(V) - p_beta)^2.                          */
/* dcoef_beta/dV[a,c] = sum_{(i,j): a_i+a_j=beta} (d_ia V[j,c] + V[i,c] d_ja) */
/* so dL/dV[a,c] = 2 sum_beta res_beta * 2 sum_{j: a_a+a_j=beta} V[j,c]      */
/*              = 4 sum_j res[rank(alpha_a + alpha_j)] V[j,c].               */
/* ------------------------------------------------------------------ */

void or_grad_rows(void *hv, const double *V, int64_t r, const double *res,
                  const int64_t *rows, int64_t nrows, double *out) {
    or_index_t *h = (or_index_t *)hv;
    int n = h->n;
    int64_t N = h->a.count;
    uint8_t s[256];
    for (int64_t t = 0; t < nrows; ++t) {
        int64_t a = rows[t];
        double *g = out + t * r;
        for (int64_t c = 0; c < r; ++c) g[c] = 0.0;
        for (int64_t j = 0; j < N; ++j) {
            for (int v = 0; v < n; ++v) s[v] = (uint8_t)(h->a.ex[a * n + v] + h->a.ex[j * n + v]);
            double w = 4.0 * res[basis_rank_ex(&h->b, s)];
            for (int64_t c = 0; c < r; ++c) g[c] += w * V[j * r + c];
        }
    }
}

/* full loss and gradient; coef_out / res_out may be NULL */
double or_loss_grad(void *hv, const double *V, int64_t r, const double *p,
                    double *grad, double *coef_out, double *res_out) {
    or_index_t *h = (or_index_t *)hv;
    int64_t N = h->a.count, M = h->b.count;
    double *coef = (double *)malloc(sizeof(double) * M);
    double *res = (double *)malloc(sizeof(double) * M);
    or_forward(hv, V, r, coef);
    double loss = 0.0;
    for (int64_t q = 0; q < M; ++q) {
        res[q] = coef[q] - p[q];
        loss += res[q] * res[q];
    }
    if (grad) {
        int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * N);
        for (int64_t i = 0; i < N; ++i) rows[i] = i;
        or_grad_rows(hv, V, r, res, rows, N, grad);
        free(rows);
    }
    if (coef_out) memcpy(coef_out, coef, sizeof(double) * M);
    if (res_out) memcpy(res_out, res, sizeof(double) * M);
    free(coef); free(res);
    return loss;
}

/* ------------------------------------------------------------------ */
/* Optimisers ("basic ADAM approach"; plain GD).         */
/* ------------------------------------------------------------------ */

/* plain gradient descent: V <- V - lr * g */
void or_gd_update(double *V, const double *g, int64_t len, double lr) {
    for (int64_t t = 0; t < len; ++t) V[t] -= lr * g[t];
}

/* Adam (Kingma & Ba), step index t >= 1:
 * m <- b1 m + (1-b1) g ; v <- b2 v + (1-b2) g^2 ;
 * V <- V - lr * (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps) */
void or_adam_update(double *V, const double *g, double *m, double *v, int64_t len,
                    double lr, double b1, double b2, double eps, int64_t t) {
    double c1 = 1.0 - pow(b1, (double)t), c2 = 1.0 - pow(b2, (double)t);
    for (int64_t k = 0; k < len; ++k) {
        m[k] = b1 * m[k] + (1.0 - b1) * g[k];
        v[k] = b2 * v[k] + (1.0 - b2) * g[k] * g[k];
        double mh = m[k] / c1, vh = v[k] / c2;
        V[k] -= lr * mh / (sqrt(vh) + eps);
    }
}

/* Descent driver: `steps` iterations of GD (kind 0) or Adam (kind 1) from V
 * (updated in place).  losses[t] = L(V_t) before update t; losses[steps] = final. */
void or_descent(void *hv, double *V, int64_t r, const double *p, int kind, int64_t steps,
                double lr, double b1, double b2, double eps, double *losses) {
    or_index_t *h = (or_index_t *)hv;
    int64_t len = h->a.count * r;
    double *g = (double *)malloc(sizeof(double) * len);
    double *m = (double *)calloc((size_t)len, sizeof(double));
    double *v = (double *)calloc((size_t)len, sizeof(double));
    for (int64_t t = 0; t < steps; ++t) {
        losses[t] = or_loss_grad(hv, V, r, p, g, NULL, NULL);
        if (kind == 0) or_gd_update(V, g, len, lr);
        else or_adam_update(V, g, m, v, len, lr, b1, b2, eps, t + 1);
    }
    losses[steps] = or_loss_grad(hv, V, r, p, NULL, NULL, NULL);
    free(g); free(m); free(v);
}
