/*
 * oracle_setup.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the two pure-Python setup loops of the reference
 * package pslr 0.1.0, used by the oracle when the instance is too large for
 * the Python restatement (bench CPU baseline, large parity cases):
 *
 *   oracle_ilut   — ilu.py:35-138  (row-wise IKJ ILUT: heap-ordered elimination,
 *                   drop |l| < droptol*||a_i||_2, diagonal never dropped, pivot
 *                   repair, optional fill cap with stable |value| ordering)
 *   oracle_bisect — partition.py:72-132 (recursive BFS level-set bisection with
 *                   smallest-index roots; ids assigned depth-first)
 *
 * Bit-identity with the reference is pinned by tests/test_oracle_golden.py.
 * Build: oracle/Makefile (-ffp-contract=off: numpy never fuses multiply-add).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

/* numpy's float64 add-reduce of a contiguous run: first + pairwise(rest). */
static double np_pairwise(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; i++) r += a[i];
        return r;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int k = 0; k < 8; k++) r[k] = a[k];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; k++) r[k] += a[i + k];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
    }
}

static double np_reduce_add(const double *a, int64_t n) {
    if (n == 0) return 0.0;
    return a[0] + np_pairwise(a + 1, n - 1);
}

/* ---- binary min-heap of int64 ---- */
typedef struct { int64_t *v; int64_t n, cap; } heap_t;
static void hpush(heap_t *h, int64_t x) {
    if (h->n == h->cap) { h->cap = h->cap ? 2 * h->cap : 64; h->v = realloc(h->v, h->cap * sizeof(int64_t)); }
    int64_t i = h->n++;
    while (i > 0) { int64_t p = (i - 1) / 2; if (h->v[p] <= x) break; h->v[i] = h->v[p]; i = p; }
    h->v[i] = x;
}
static int64_t hpop(heap_t *h) {
    int64_t top = h->v[0], x = h->v[--h->n], i = 0;
    for (;;) {
        int64_t c = 2 * i + 1;
        if (c >= h->n) break;
        if (c + 1 < h->n && h->v[c + 1] < h->v[c]) c++;
        if (x <= h->v[c]) break;
        h->v[i] = h->v[c]; i = c;
    }
    if (h->n) h->v[i] = x;
    return top;
}

typedef struct { int64_t col; double val; int64_t seq; } ent_t;
static int cmp_col(const void *a, const void *b) {
    int64_t x = ((const ent_t *)a)->col, y = ((const ent_t *)b)->col;
    return (x > y) - (x < y);
}
/* Python's sorted(key=-|v|) is stable: descending |v|, ties by original sequence */
static int cmp_mag(const void *a, const void *b) {
    const ent_t *x = a, *y = b;
    double ax = fabs(x->val), ay = fabs(y->val);
    if (ax > ay) return -1;
    if (ax < ay) return 1;
    return (x->seq > y->seq) - (x->seq < y->seq);
}

typedef struct {
    int64_t n, nl, nu;
    int64_t *Lp, *Li, *Up, *Ui;
    double *Lx, *Ux;
} ilut_out_t;

int oracle_ilut(int64_t n, const int64_t *ip, const int64_t *ix, const double *ax,
                double droptol, int64_t fill_cap, void **handle, int64_t *sizes) {
    double *norms = malloc((n ? n : 1) * sizeof(double));
    double *sq = NULL; int64_t sqcap = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t len = ip[i + 1] - ip[i];
        if (len > sqcap) { sqcap = len; sq = realloc(sq, sqcap * sizeof(double)); }
        for (int64_t k = 0; k < len; k++) { double v = ax[ip[i] + k]; sq[k] = v * v; }
        norms[i] = sqrt(np_reduce_add(sq, len));
    }
    free(sq);
    /* U rows, stored as they are produced (diag first, then sorted upper cols) */
    int64_t *urow_start = malloc((n + 1) * sizeof(int64_t));
    int64_t ucap = 1024, unn = 0;
    int64_t *ucol = malloc(ucap * sizeof(int64_t));
    double *uval = malloc(ucap * sizeof(double));
    int64_t lcap = 1024, lnn = 0;
    int64_t *lrow = malloc(lcap * sizeof(int64_t)), *lcol = malloc(lcap * sizeof(int64_t));
    double *lval = malloc(lcap * sizeof(double));
    double *udiag = malloc((n ? n : 1) * sizeof(double));
    double *w = calloc(n ? n : 1, sizeof(double));
    char *mark = calloc(n ? n : 1, 1);
    int64_t *touched = malloc((n ? n : 1) * sizeof(int64_t));
    ent_t *lk = malloc((n ? n : 1) * sizeof(ent_t)), *up = malloc((n ? n : 1) * sizeof(ent_t));
    heap_t hp = {0};
    int64_t repairs = 0;
    const double eps = DBL_EPSILON;

    for (int64_t i = 0; i < n; i++) {
        int64_t nt = 0, nlk = 0, nup = 0;
        for (int64_t k = ip[i]; k < ip[i + 1]; k++) {
            int64_t c = ix[k];
            w[c] = ax[k];
            mark[c] = 1;
            touched[nt++] = c;
        }
        double tau = droptol * norms[i];
        hp.n = 0;
        for (int64_t k = ip[i]; k < ip[i + 1]; k++) if (ix[k] < i) hpush(&hp, ix[k]);
        while (hp.n) {
            int64_t k = hpop(&hp);
            double f = w[k] / udiag[k];
            w[k] = 0.0;
            if (fabs(f) < tau) continue;
            lk[nlk].col = k; lk[nlk].val = f; lk[nlk].seq = nlk; nlk++;
            int64_t a = urow_start[k], b = urow_start[k + 1];
            for (int64_t t = a; t < b; t++) {
                int64_t c = ucol[t];
                if (!mark[c]) {
                    mark[c] = 1;
                    touched[nt++] = c;
                    if (c < i) hpush(&hp, c);
                }
            }
            for (int64_t t = a; t < b; t++) {
                double prod = f * uval[t];
                w[ucol[t]] = w[ucol[t]] - prod;
            }
        }
        double piv = w[i];
        if (piv == 0.0) {
            double base = norms[i] > 0 ? norms[i] : 1.0;
            piv = droptol * base;
            if (piv == 0.0) piv = eps * base;
            repairs++;
        }
        for (int64_t t = 0; t < nt; t++) {
            int64_t j = touched[t];
            if (j > i && fabs(w[j]) >= tau && w[j] != 0.0) {
                up[nup].col = j; up[nup].val = w[j]; up[nup].seq = nup; nup++;
            }
        }
        if (fill_cap >= 0) {
            if (nlk > fill_cap) { qsort(lk, nlk, sizeof(ent_t), cmp_mag); nlk = fill_cap; }
            if (nup > fill_cap) { qsort(up, nup, sizeof(ent_t), cmp_mag); nup = fill_cap; }
        }
        qsort(lk, nlk, sizeof(ent_t), cmp_col);
        qsort(up, nup, sizeof(ent_t), cmp_col);
        if (lnn + nlk + 1 > lcap) {
            while (lnn + nlk + 1 > lcap) lcap *= 2;
            lrow = realloc(lrow, lcap * sizeof(int64_t)); lcol = realloc(lcol, lcap * sizeof(int64_t));
            lval = realloc(lval, lcap * sizeof(double));
        }
        for (int64_t t = 0; t < nlk; t++) { lrow[lnn] = i; lcol[lnn] = lk[t].col; lval[lnn] = lk[t].val; lnn++; }
        if (unn + nup + 1 > ucap) {
            while (unn + nup + 1 > ucap) ucap *= 2;
            ucol = realloc(ucol, ucap * sizeof(int64_t)); uval = realloc(uval, ucap * sizeof(double));
        }
        urow_start[i] = unn;
        ucol[unn] = i; uval[unn] = piv; unn++;
        for (int64_t t = 0; t < nup; t++) { ucol[unn] = up[t].col; uval[unn] = up[t].val; unn++; }
        urow_start[i + 1] = unn;
        udiag[i] = piv;
        for (int64_t t = 0; t < nt; t++) { w[touched[t]] = 0.0; mark[touched[t]] = 0; }
    }
    /* assemble L in CSR: per row, kept multipliers (ascending col) then the unit diagonal */
    ilut_out_t *o = calloc(1, sizeof(ilut_out_t));
    o->n = n; o->nl = lnn + n; o->nu = unn;
    o->Lp = malloc((n + 1) * sizeof(int64_t));
    o->Li = malloc((o->nl ? o->nl : 1) * sizeof(int64_t));
    o->Lx = malloc((o->nl ? o->nl : 1) * sizeof(double));
    int64_t pos = 0, t = 0;
    for (int64_t i = 0; i < n; i++) {
        o->Lp[i] = pos;
        while (t < lnn && lrow[t] == i) { o->Li[pos] = lcol[t]; o->Lx[pos] = lval[t]; pos++; t++; }
        o->Li[pos] = i; o->Lx[pos] = 1.0; pos++;
    }
    o->Lp[n] = pos;
    o->Up = urow_start; o->Ui = ucol; o->Ux = uval;
    free(norms); free(lrow); free(lcol); free(lval); free(udiag); free(w); free(mark);
    free(touched); free(lk); free(up); free(hp.v);
    *handle = o;
    sizes[0] = o->nl; sizes[1] = o->nu; sizes[2] = repairs;
    return 0;
}

int64_t oracle_ilut_fetch(void *h, int64_t *Lp, int64_t *Li, double *Lx,
                          int64_t *Up, int64_t *Ui, double *Ux) {
    ilut_out_t *o = h;
    memcpy(Lp, o->Lp, (o->n + 1) * sizeof(int64_t));
    memcpy(Li, o->Li, o->nl * sizeof(int64_t));
    memcpy(Lx, o->Lx, o->nl * sizeof(double));
    memcpy(Up, o->Up, (o->n + 1) * sizeof(int64_t));
    memcpy(Ui, o->Ui, o->nu * sizeof(int64_t));
    memcpy(Ux, o->Ux, o->nu * sizeof(double));
    return o->nl + o->nu;
}

void oracle_ilut_free(void *h) {
    ilut_out_t *o = h;
    if (!o) return;
    free(o->Lp); free(o->Li); free(o->Lx); free(o->Up); free(o->Ui); free(o->Ux); free(o);
}

/* ---- BFS bisection ---- */
typedef struct {
    const int64_t *ip, *ix;
    char *inset, *seen;
    int64_t *queue;
    int64_t *assign;
} bis_t;

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

static int64_t bisect_rec(bis_t *B, int64_t *verts, int64_t nv, int64_t parts, int64_t nid) {
    if (parts == 1) {
        for (int64_t k = 0; k < nv; k++) B->assign[verts[k]] = nid;
        return nid + 1;
    }
    int64_t lp = (parts + 1) / 2, rp = parts - lp;
    for (int64_t k = 0; k < nv; k++) { B->inset[verts[k]] = 1; B->seen[verts[k]] = 0; }
    int64_t head = 0, tail = 0;
    for (int64_t r = 0; r < nv; r++) {
        int64_t root = verts[r];
        if (B->seen[root]) continue;
        B->seen[root] = 1;
        B->queue[tail++] = root;
        while (head < tail) {
            int64_t v = B->queue[head++];
            for (int64_t e = B->ip[v]; e < B->ip[v + 1]; e++) {
                int64_t u = B->ix[e];
                if (B->inset[u] && !B->seen[u]) { B->seen[u] = 1; B->queue[tail++] = u; }
            }
        }
    }
    for (int64_t k = 0; k < nv; k++) B->inset[verts[k]] = 0;
    /* Python: int(round(len * lp / parts)) — true division, round-half-even */
    double x = (double)(nv * lp) / (double)parts;
    int64_t cut = (int64_t)nearbyint(x);
    if (cut < lp) cut = lp;
    if (cut > nv - rp) cut = nv - rp;
    /* the BFS order now lives in queue[0..nv); copy both halves back into verts sorted */
    memcpy(verts, B->queue, nv * sizeof(int64_t));
    qsort(verts, cut, sizeof(int64_t), cmp_i64);
    qsort(verts + cut, nv - cut, sizeof(int64_t), cmp_i64);
    nid = bisect_rec(B, verts, cut, lp, nid);
    return bisect_rec(B, verts + cut, nv - cut, rp, nid);
}

int oracle_bisect(int64_t n, const int64_t *ip, const int64_t *ix, int64_t parts, int64_t *assign) {
    if (parts < 1 || parts > n) return 1;
    bis_t B;
    B.ip = ip; B.ix = ix; B.assign = assign;
    B.inset = calloc(n ? n : 1, 1);
    B.seen = calloc(n ? n : 1, 1);
    B.queue = malloc((n ? n : 1) * sizeof(int64_t));
    int64_t *verts = malloc((n ? n : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) verts[i] = i;
    bisect_rec(&B, verts, n, parts, 0);
    free(B.inset); free(B.seen); free(B.queue); free(verts);
    return 0;
}
