/*
 * mcl_oracle.c -- the CPU ORACLE for the HipMCL expansion hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2002_10083_b200/, libmclx.so) never links, loads or calls it; the two
 * share no source, header, table or constant generator.
 *
 * Plain, slow, single-threaded, fp64, no -ffast-math.  Each function cites the
 * passage of /root/reference/PAPER.md (P:line) it writes out, or the DESIGN.md
 * reading (Q#) where the paper is silent.
 *
 *   orc_spgemm         P:159 Alg.1 l.3 (B <- AA), P:173-175 (flops)
 *                      (CSC-native).  PLAIN DEFINITION: C = A*B by Gustavson with a
 *                      dense accumulator; structure = rows touched (Q13).
 *   orc_prune_inflate  P:161 Alg.1 l.4, Alg.1 l.5.
 *                      ALGORITHM step by step (readings Q1-Q9).  Recovery (Q7) and
 *                      chaos (Q9) have no paper text: PARITY UNPINNED BY THE PAPER for
 *                      R/pct and for the chaos definition -- pinned only by hand
 *                      examples and invariants (tests/test_oracle.py).
 *   orc_preprocess     P:156 Alg.1 l.1, P:184 (column stochastic), Q10 (loops).
 *   orc_clusters       P:166 Alg.1 l.6, P:191 -- union-find, Q11.
 *   orc_philox / orc_cohen   P:609-630 §V (Cohen estimator), P:1036-1037 (lambda=1),
 *                      Q14 (garbled index read as per-output-column estimate).
 *   orc_merge          P:246 ("merging the list of intermediate products"),
 *                      P:454-467 (multiway merge) -- PLAIN DEFINITION: sum of lists.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t nrows, ncols;
    int64_t *cp;   /* [ncols+1] */
    int32_t *row;  /* [nnz] */
    double *val;   /* [nnz] */
} ocsc;

void orc_free(void *p) { free(p); }

/* ---------------------------------------------------------------- growable output */
typedef struct {
    int64_t n, cap;
    int32_t *row;
    double *val;
} obuf;

static int ob_push(obuf *b, int32_t r, double v) {
    if (b->n == b->cap) {
        int64_t nc = b->cap ? 2 * b->cap : 1024;
        int32_t *nr = (int32_t *)realloc(b->row, (size_t)nc * sizeof(int32_t));
        if (!nr) return -1;
        b->row = nr;
        double *nv = (double *)realloc(b->val, (size_t)nc * sizeof(double));
        if (!nv) return -1;
        b->val = nv;
        b->cap = nc;
    }
    b->row[b->n] = r;
    b->val[b->n] = v;
    b->n++;
    return 0;
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/*
 * C[:, cb:ce) = A * B[:, cb:ce)   (A: m x p, B: p x n; CSC; values fp64)
 *
 * For every output column j (Gustavson in CSC per P:430-437):
 *   for each (k, b_kj) in B_*j in stored order:
 *     for each (i, a_ik) in A_*k in stored order:
 *       acc[i] += a_ik * b_kj ; mark row i as touched.
 * Then the touched rows are sorted ascending and emitted with acc[i].
 * flops_j = sum_{k in inds(B_*j)} nnz(A_*k), written to flops[j-cb].
 * Outputs are malloc'ed; free with orc_free.  Returns 0, or -1 on OOM / bad dims.
 */
int orc_spgemm(int64_t m, int64_t p, int64_t n,
               const int64_t *acp, const int32_t *arow, const double *aval,
               const int64_t *bcp, const int32_t *brow, const double *bval,
               int64_t cb, int64_t ce,
               int64_t **ocp, int32_t **orow, double **oval, int64_t *flops) {
    if (cb < 0 || ce > n || cb > ce) return -1;
    (void)p;
    double *acc = (double *)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
    int64_t *mark = (int64_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
    int32_t *touched = (int32_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    int64_t *cp = (int64_t *)malloc((size_t)(ce - cb + 1) * sizeof(int64_t));
    obuf out = {0, 0, NULL, NULL};
    if (!acc || !mark || !touched || !cp) return -1;
    for (int64_t i = 0; i < m; i++) mark[i] = -1;
    cp[0] = 0;
    for (int64_t j = cb; j < ce; j++) {
        int64_t nt = 0, f = 0;
        for (int64_t q = bcp[j]; q < bcp[j + 1]; q++) {
            int32_t k = brow[q];
            double bkj = bval[q];
            f += acp[k + 1] - acp[k];
            for (int64_t t = acp[k]; t < acp[k + 1]; t++) {
                int32_t i = arow[t];
                if (mark[i] != j) {
                    mark[i] = j;
                    acc[i] = 0.0;
                    touched[nt++] = i;
                }
                acc[i] += aval[t] * bkj;
            }
        }
        qsort(touched, (size_t)nt, sizeof(int32_t), cmp_i32);
        for (int64_t t = 0; t < nt; t++)
            if (ob_push(&out, touched[t], acc[touched[t]])) return -1;
        cp[j - cb + 1] = out.n;
        if (flops) flops[j - cb] = f;
    }
    free(acc);
    free(mark);
    free(touched);
    *ocp = cp;
    *orow = out.row;
    *oval = out.val;
    return 0;
}

/* ------------------------------------------------------------ prune / inflate */
typedef struct {
    double v;
    int32_t r;
} ent;

/* order: value descending, then row ascending (Q5 tie rule) */
static int cmp_desc(const void *a, const void *b) {
    const ent *x = (const ent *)a, *y = (const ent *)b;
    if (x->v > y->v) return -1;
    if (x->v < y->v) return 1;
    return (x->r > y->r) - (x->r < y->r);
}
static int cmp_row(const void *a, const void *b) {
    const ent *x = (const ent *)a, *y = (const ent *)b;
    return (x->r > y->r) - (x->r < y->r);
}

/*
 * Per column j of C (an unpruned expansion B of Alg.1 l.3), the reading of
 * SURVEY §8(c) Q3-Q9 of Alg.1 l.4-5:
 *   m_j = #{v >= theta}, s_j = sum{v : v >= theta}   (Q3, Q4: keep v >= theta)
 *   branch 1 SELECT   if m_j > S:                       keep top-S          (Q5)
 *   branch 2 RECOVER  elif R>0 and m_j<R and s_j<pct and nnz_j>m_j:
 *                                                       keep top-min(R,nnz) (Q7)
 *   branch 0 THRESH   elif m_j > 0:                     keep {v >= theta}
 *   branch 3 ARGMAX   elif nnz_j > 0:                   keep top-1          (Q8)
 *   (empty column stays empty, branch 4)
 *   "top" = order by (value desc, row asc).
 *   w = kept / sum(kept)                          (renormalise, Q1)
 *   chaos_j = |kept| * (max w - sum w^2)          (Q9)
 *   a'_ij = w^r / sum w^r                         (P:162-164 Hadamard power, r=2 at P:770; Q1, Q2)
 * tau_j (effective cut, Q19) = theta for THRESH, the value of the last kept entry
 * otherwise.  Outputs sorted by row ascending.
 */
int orc_prune_inflate(int64_t ncols, const int64_t *ccp, const int32_t *crow, const double *cval,
                      double theta, int64_t S, int64_t R, double pct, double r,
                      int64_t **ocp, int32_t **orow, double **oval,
                      double *chaos, double *tau, int32_t *branch, int64_t *mcount, double *smass) {
    int64_t *cp = (int64_t *)malloc((size_t)(ncols + 1) * sizeof(int64_t));
    obuf out = {0, 0, NULL, NULL};
    int64_t maxlen = 1;
    for (int64_t j = 0; j < ncols; j++)
        if (ccp[j + 1] - ccp[j] > maxlen) maxlen = ccp[j + 1] - ccp[j];
    ent *e = (ent *)malloc((size_t)maxlen * sizeof(ent));
    if (!cp || !e) return -1;
    cp[0] = 0;
    for (int64_t j = 0; j < ncols; j++) {
        int64_t nz = ccp[j + 1] - ccp[j];
        int64_t m = 0;
        double s = 0.0;
        for (int64_t t = 0; t < nz; t++) {
            e[t].v = cval[ccp[j] + t];
            e[t].r = crow[ccp[j] + t];
            if (e[t].v >= theta) {
                m++;
                s += e[t].v;
            }
        }
        int64_t K;
        int32_t br;
        if (m > S) {
            K = S;
            br = 1;
        } else if (R > 0 && m < R && s < pct && nz > m) {
            K = R < nz ? R : nz;
            br = 2;
        } else if (m > 0) {
            K = m;
            br = 0;
        } else if (nz > 0) {
            K = 1;
            br = 3;
        } else {
            K = 0;
            br = 4;
        }
        qsort(e, (size_t)nz, sizeof(ent), cmp_desc);
        if (tau) tau[j] = (br == 0) ? theta : (K > 0 ? e[K - 1].v : 0.0);
        double sum = 0.0, mx = 0.0;
        for (int64_t t = 0; t < K; t++) {
            sum += e[t].v;
            if (e[t].v > mx) mx = e[t].v;
        }
        double sq = 0.0, sr = 0.0;
        for (int64_t t = 0; t < K; t++) {
            double w = e[t].v / sum;
            sq += w * w;
            double wr = (r == 2.0) ? w * w : pow(w, r);
            e[t].v = wr;
            sr += wr;
        }
        if (chaos) chaos[j] = K > 0 ? (double)K * (mx / sum - sq) : 0.0;
        if (branch) branch[j] = br;
        if (mcount) mcount[j] = m;
        if (smass) smass[j] = s;
        for (int64_t t = 0; t < K; t++) e[t].v /= sr;
        qsort(e, (size_t)K, sizeof(ent), cmp_row);
        for (int64_t t = 0; t < K; t++)
            if (ob_push(&out, e[t].r, e[t].v)) return -1;
        cp[j + 1] = out.n;
    }
    free(e);
    *ocp = cp;
    *orow = out.row;
    *oval = out.val;
    return 0;
}

/*
 * Alg.1 l.1: column-stochastic version of the weighted adjacency
 * matrix.  Reading Q10: a self-loop of weight 1.0 is added to every vertex
 * (summed onto an existing diagonal entry) before normalising each column to 1.
 */
int orc_preprocess(int64_t n, const int64_t *gcp, const int32_t *grow, const float *gw,
                   int add_loops, int64_t **ocp, int32_t **orow, double **oval) {
    int64_t *cp = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
    obuf out = {0, 0, NULL, NULL};
    if (!cp) return -1;
    cp[0] = 0;
    for (int64_t j = 0; j < n; j++) {
        int64_t start = out.n;
        int placed = !add_loops;
        for (int64_t t = gcp[j]; t < gcp[j + 1]; t++) {
            int32_t i = grow[t];
            double w = (double)gw[t];
            if (!placed && i > j) {
                if (ob_push(&out, (int32_t)j, 1.0)) return -1;
                placed = 1;
            }
            if (!placed && i == j) {
                w += 1.0;
                placed = 1;
            }
            if (ob_push(&out, i, w)) return -1;
        }
        if (!placed)
            if (ob_push(&out, (int32_t)j, 1.0)) return -1;
        double s = 0.0;
        for (int64_t t = start; t < out.n; t++) s += out.val[t];
        for (int64_t t = start; t < out.n; t++) out.val[t] /= s;
        cp[j + 1] = out.n;
    }
    *ocp = cp;
    *orow = out.row;
    *oval = out.val;
    return 0;
}

/* ------------------------------------------------------------ clusters */
static int64_t uf_find(int64_t *par, int64_t x) {
    int64_t r = x;
    while (par[r] != r) r = par[r];
    while (par[x] != r) {
        int64_t nx = par[x];
        par[x] = r;
        x = nx;
    }
    return r;
}

/*
 * Alg.1 l.6: connected components of A.  Reading Q11: weak
 * components of the symmetrised pattern (edge (i,j) for every stored entry),
 * labels numbered in order of each component's smallest vertex.
 */
int orc_clusters(int64_t n, const int64_t *cp, const int32_t *row, int32_t *labels, int64_t *ncl) {
    int64_t *par = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!par) return -1;
    for (int64_t i = 0; i < n; i++) par[i] = i;
    for (int64_t j = 0; j < n; j++)
        for (int64_t t = cp[j]; t < cp[j + 1]; t++) {
            int64_t a = uf_find(par, row[t]), b = uf_find(par, j);
            if (a != b) {
                if (a < b) par[b] = a;
                else par[a] = b;
            }
        }
    int64_t next = 0;
    int64_t *lab = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!lab) return -1;
    for (int64_t i = 0; i < n; i++) lab[i] = -1;
    for (int64_t i = 0; i < n; i++) {
        int64_t rt = uf_find(par, i);
        if (lab[rt] < 0) lab[rt] = next++;
        labels[i] = (int32_t)lab[rt];
    }
    *ncl = next;
    free(par);
    free(lab);
    return 0;
}

/* ------------------------------------------------------------ Cohen estimator */
/*
 * Philox-4x32-10 (Salmon et al., SC'11), written out from its definition:
 * 10 rounds; round: (hi0,lo0) = M0*x0, (hi1,lo1) = M1*x2;
 * x = (hi1 ^ x1 ^ k0, lo1, hi0 ^ x3 ^ k1, lo0); key bumped by W0, W1 between rounds.
 */
void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int rnd = 0; rnd < 10; rnd++) {
        uint64_t p0 = (uint64_t)M0 * x0, p1 = (uint64_t)M1 * x2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t y0 = hi1 ^ x1 ^ k0, y1 = lo1, y2 = hi0 ^ x3 ^ k1, y3 = lo0;
        x0 = y0; x1 = y1; x2 = y2; x3 = y3;
        k0 += W0;
        k1 += W1;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* Key s of first-layer vertex i (Q14): u = Philox(ctr=(i_lo,i_hi,s,0), key=(seed_lo,seed_hi))[0];
 * X = (float)(-log((u + 0.5) * 2^-32)) -- an Exp(lambda=1) variate. */
float orc_cohen_key(uint64_t seed, int64_t s, int64_t i) {
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)((uint64_t)i >> 32), (uint32_t)s, 0u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    orc_philox(ctr, key, o);
    return (float)(-log(((double)o[0] + 0.5) * (1.0 / 4294967296.0)));
}

/*
 * Cohen's size estimate for C = A*B (§V, Fig. layered-graph):
 *   layer 1 (rows of A, m vertices): r keys X[s][i] ~ Exp(1);
 *   layer 2 (cols of A = rows of B):  M[s][k] = min_{i in inds(A_*k)} X[s][i];
 *   layer 3 (cols of B):              c[s][j] = min_{k in inds(B_*j)} M[s][k];
 *   est_j = (r-1) / sum_s c[s][j], 0 if column j reaches no first-layer vertex.
 * keys_out (optional, [r*m], plane-major) receives X for the bit-exact key check.
 */
int orc_cohen(int64_t m, int64_t p, int64_t n,
              const int64_t *acp, const int32_t *arow,
              const int64_t *bcp, const int32_t *brow,
              int32_t r, uint64_t seed, float *keys_out, float *mid_out, double *est) {
    if (r < 2) return -1;
    float *X = (float *)malloc((size_t)(r * (m > 0 ? m : 1)) * sizeof(float));
    float *M = (float *)malloc((size_t)(r * (p > 0 ? p : 1)) * sizeof(float));
    if (!X || !M) return -1;
    for (int32_t s = 0; s < r; s++)
        for (int64_t i = 0; i < m; i++) X[(int64_t)s * m + i] = orc_cohen_key(seed, s, i);
    for (int32_t s = 0; s < r; s++)
        for (int64_t k = 0; k < p; k++) {
            float mn = INFINITY;
            for (int64_t t = acp[k]; t < acp[k + 1]; t++) {
                float x = X[(int64_t)s * m + arow[t]];
                if (x < mn) mn = x;
            }
            M[(int64_t)s * p + k] = mn;
        }
    for (int64_t j = 0; j < n; j++) {
        double sum = 0.0;
        int reach = 1;
        for (int32_t s = 0; s < r; s++) {
            float mn = INFINITY;
            for (int64_t t = bcp[j]; t < bcp[j + 1]; t++) {
                float x = M[(int64_t)s * p + brow[t]];
                if (x < mn) mn = x;
            }
            if (isinf(mn)) reach = 0;
            sum += (double)mn;
        }
        est[j] = reach ? (double)(r - 1) / sum : 0.0;
    }
    if (keys_out) memcpy(keys_out, X, (size_t)(r * m) * sizeof(float));
    if (mid_out) memcpy(mid_out, M, (size_t)(r * p) * sizeof(float));
    free(X);
    free(M);
    return 0;
}

/* ------------------------------------------------------------ merge of stage lists */
/*
 * Merge L lists (CSC blocks of identical shape) into one: per column, the union
 * of rows with values summed ("summation is implemented via merging the
 * list of intermediate products"; multiway merge P:454-467).  Duplicates are
 * summed in list order.  Plain definition: the sum of the L matrices.
 */
int orc_merge(int32_t L, int64_t nrows, int64_t ncols, const int64_t **cps, const int32_t **rows,
              const double **vals, int64_t **ocp, int32_t **orow, double **oval) {
    double *acc = (double *)calloc((size_t)(nrows > 0 ? nrows : 1), sizeof(double));
    int64_t *mark = (int64_t *)malloc((size_t)(nrows > 0 ? nrows : 1) * sizeof(int64_t));
    int32_t *touched = (int32_t *)malloc((size_t)(nrows > 0 ? nrows : 1) * sizeof(int32_t));
    int64_t *cp = (int64_t *)malloc((size_t)(ncols + 1) * sizeof(int64_t));
    obuf out = {0, 0, NULL, NULL};
    if (!acc || !mark || !touched || !cp) return -1;
    for (int64_t i = 0; i < nrows; i++) mark[i] = -1;
    cp[0] = 0;
    for (int64_t j = 0; j < ncols; j++) {
        int64_t nt = 0;
        for (int32_t l = 0; l < L; l++)
            for (int64_t t = cps[l][j]; t < cps[l][j + 1]; t++) {
                int32_t i = rows[l][t];
                if (mark[i] != j) {
                    mark[i] = j;
                    acc[i] = 0.0;
                    touched[nt++] = i;
                }
                acc[i] += vals[l][t];
            }
        qsort(touched, (size_t)nt, sizeof(int32_t), cmp_i32);
        for (int64_t t = 0; t < nt; t++)
            if (ob_push(&out, touched[t], acc[touched[t]])) return -1;
        cp[j + 1] = out.n;
    }
    free(acc);
    free(mark);
    free(touched);
    *ocp = cp;
    *orow = out.row;
    *oval = out.val;
    return 0;
}
