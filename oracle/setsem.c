/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU evaluator of ALCQI(D) instance
 * semantics under the closed-world and unique-name assumptions
 * (§III-A "closed world assumption (CWA) and unique world
 * assumption (UWA)").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this file's library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_2412_00802_b200/csrc); the only common thing is the input format
 * produced by synth/ (the hedl_kb_desc arrays and the node records).
 *
 * Representation (deliberately the paper's, not the GPU's): every
 * intermediate concept extension is one byte per individual, 0 or 1 --
 * the "results matrix" row of PAPER.md:65 §III-A.  Roles are sets of
 * (subject, object) pairs (duplicates collapse); an inverse
 * role swaps subject and object (§III-B2).  Every operator
 * scans assertions one by one exactly like the per-assertion loops of
 * Algs. 3-10 without their skip-ahead optimisation;
 * there is no CSE, no bytecode and no blocking: the hypothesis tree is
 * evaluated recursively, a fresh row per node.
 *
 * Readings of silent/ambiguous points are SURVEY.md 8(c) Q1..Q19, restated
 * in DESIGN.md "Readings".  Parity is pinned (see tests/test_oracle_*.py):
 * against brute force over all of Delta x Delta, SPEC.md hand examples,
 * DL identities and closed forms.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* node opcodes of the input format (synth/format.py) */
enum { O_TOP, O_BOTTOM, O_ATOM, O_NOT, O_AND, O_OR, O_EXISTS, O_FORALL,
       O_MIN, O_MAX, O_EXACT, O_DRANGE, O_SEQUAL, O_SCONTAIN };
#define F_INV 1u
#define CF_COMPAT_PAPER_MAX 4u

enum { R_OK = 0, R_INVALID = 1, R_RANGE = 2, R_CONFLICT = 3, R_BADEXPR = 4, R_OOM = 7 };

typedef struct {
    uint8_t op, flags;
    uint16_t pad;
    uint32_t arg, n;
    float lo, hi;
    uint32_t child_begin, child_count;
} onode;

typedef struct {
    uint32_t N, W, C, R, D;
    const uint32_t *concept_bits;      /* borrowed: [C][W] input words */
    uint64_t **pairs;                  /* per role: sorted unique (s<<32|o) */
    uint64_t *npairs;
    uint32_t **dsubj;                  /* per data property: assertion subjects */
    float **dval;                      /* ... and their float32 values */
    uint64_t *ndata;
    uint8_t *pos, *neg;                /* ExMat (Alg. 15 input) */
    uint64_t npos, nneg;
    uint32_t S;                        /* string concrete roles (Algs. 11-14) */
    const uint64_t *str_off;           /* borrowed: role s = assertions [str_off[s], str_off[s+1]) */
    const uint32_t *str_subj;
    const uint64_t *str_val_off;       /* assertion k's value = str_bytes[str_val_off[k] .. k+1) */
    const uint8_t *str_bytes;
} okb;

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : x > y;
}

void oracle_kb_free(okb *kb);

int oracle_kb_new(uint32_t N, uint32_t C, const uint32_t *concept_bits,
                  uint32_t R, const uint64_t *role_off, const uint32_t *esubj, const uint32_t *eobj,
                  uint32_t D, const uint64_t *data_off, const uint32_t *dsubj, const float *dval,
                  uint32_t npos, const uint32_t *pos, uint32_t nneg, const uint32_t *neg,
                  uint32_t S, const uint64_t *str_off, const uint32_t *str_subj, const uint64_t *str_val_off,
                  const uint8_t *str_bytes, okb **out) {
    okb *kb = (okb *)calloc(1, sizeof(okb));
    if (!kb) return R_OOM;
    kb->N = N; kb->W = (N + 31) / 32; kb->C = C; kb->R = R; kb->D = D;
    kb->concept_bits = concept_bits;
    kb->pairs = (uint64_t **)calloc(R ? R : 1, sizeof(uint64_t *));
    kb->npairs = (uint64_t *)calloc(R ? R : 1, sizeof(uint64_t));
    kb->dsubj = (uint32_t **)calloc(D ? D : 1, sizeof(uint32_t *));
    kb->dval = (float **)calloc(D ? D : 1, sizeof(float *));
    kb->ndata = (uint64_t *)calloc(D ? D : 1, sizeof(uint64_t));
    kb->pos = (uint8_t *)calloc(N ? N : 1, 1);
    kb->neg = (uint8_t *)calloc(N ? N : 1, 1);
    int rc = R_OK;
    /* role extensions: the set of asserted pairs */
    for (uint32_t r = 0; r < R && rc == R_OK; r++) {
        uint64_t a = role_off[r], b = role_off[r + 1], m = b - a, k = 0;
        uint64_t *p = (uint64_t *)malloc((m ? m : 1) * sizeof(uint64_t));
        for (uint64_t i = 0; i < m; i++) {
            if (esubj[a + i] >= N || eobj[a + i] >= N) { rc = R_RANGE; break; }
            p[i] = ((uint64_t)esubj[a + i] << 32) | eobj[a + i];
        }
        qsort(p, m, sizeof(uint64_t), cmp_u64);
        for (uint64_t i = 0; i < m; i++)
            if (k == 0 || p[k - 1] != p[i]) p[k++] = p[i];
        kb->pairs[r] = p; kb->npairs[r] = k;
    }
    /* numeric concrete roles: the multiset of asserted (subject, value) */
    for (uint32_t d = 0; d < D && rc == R_OK; d++) {
        uint64_t a = data_off[d], b = data_off[d + 1], m = b - a;
        kb->dsubj[d] = (uint32_t *)malloc((m ? m : 1) * sizeof(uint32_t));
        kb->dval[d] = (float *)malloc((m ? m : 1) * sizeof(float));
        for (uint64_t i = 0; i < m; i++) {
            if (dsubj[a + i] >= N) { rc = R_RANGE; break; }
            kb->dsubj[d][i] = dsubj[a + i];
            kb->dval[d][i] = dval[a + i];
        }
        kb->ndata[d] = m;
    }
    for (uint32_t i = 0; i < npos && rc == R_OK; i++) {
        if (pos[i] >= N) { rc = R_RANGE; break; }
        kb->pos[pos[i]] = 1;
    }
    for (uint32_t i = 0; i < nneg && rc == R_OK; i++) {
        if (neg[i] >= N) { rc = R_RANGE; break; }
        if (kb->pos[neg[i]]) { rc = R_CONFLICT; break; }
        kb->neg[neg[i]] = 1;
    }
    for (uint32_t i = 0; i < N; i++) { kb->npos += kb->pos[i]; kb->nneg += kb->neg[i]; }
    kb->S = S; kb->str_off = str_off; kb->str_subj = str_subj;
    kb->str_val_off = str_val_off; kb->str_bytes = str_bytes;
    for (uint32_t r = 0; r < S && rc == R_OK; r++)
        for (uint64_t k = str_off[r]; k < str_off[r + 1]; k++)
            if (str_subj[k] >= N) { rc = R_RANGE; break; }
    if (rc != R_OK) { oracle_kb_free(kb); return rc; }
    *out = kb;
    return R_OK;
}

void oracle_kb_free(okb *kb) {
    if (!kb) return;
    for (uint32_t r = 0; r < kb->R; r++) free(kb->pairs[r]);
    for (uint32_t d = 0; d < kb->D; d++) { free(kb->dsubj[d]); free(kb->dval[d]); }
    free(kb->pairs); free(kb->npairs); free(kb->dsubj); free(kb->dval); free(kb->ndata);
    free(kb->pos); free(kb->neg); free(kb);
}

typedef struct {
    const okb *kb;
    const onode *nodes;
    uint32_t n_nodes;
    const uint32_t *kids;
    uint64_t n_kids;
    uint32_t flags;
    uint32_t n_pat;                    /* string patterns of SEQUAL / SCONTAIN (node.n) */
    const uint64_t *pat_off;
    const uint8_t *pat_bytes;
} octx;

/* does the byte string h[0..hn) contain p[0..pn) as a contiguous substring? */
static int contains(const uint8_t *h, uint64_t hn, const uint8_t *p, uint64_t pn) {
    if (pn > hn) return 0;
    for (uint64_t i = 0; i + pn <= hn; i++)
        if (memcmp(h + i, p, pn) == 0) return 1;
    return 0;
}

/* eval(node) -> fresh row of N bytes in {0,1}; NULL on error (*rc set). */
static uint8_t *eval(const octx *x, uint32_t id, int depth, int *rc) {
    const okb *kb = x->kb;
    const uint32_t N = kb->N;
    if (id >= x->n_nodes) { *rc = R_RANGE; return NULL; }
    if (depth > 4096) { *rc = R_BADEXPR; return NULL; }          /* cycle guard */
    const onode *nd = &x->nodes[id];
    if ((uint64_t)nd->child_begin + nd->child_count > x->n_kids) { *rc = R_RANGE; return NULL; }
    const uint32_t *ch = x->kids + nd->child_begin;
    uint8_t *res = (uint8_t *)malloc(N ? N : 1);
    if (!res) { *rc = R_OOM; return NULL; }
    switch (nd->op) {
    case O_TOP:                      /* Delta = {0..N-1} */
    case O_BOTTOM:
        if (nd->child_count) goto bad;
        memset(res, nd->op == O_TOP, N);
        return res;
    case O_ATOM: {                   /* A^I = asserted members */
        if (nd->child_count) goto bad;
        if (nd->arg >= kb->C) { *rc = R_RANGE; free(res); return NULL; }
        const uint32_t *row = kb->concept_bits + (uint64_t)nd->arg * kb->W;
        for (uint32_t i = 0; i < N; i++) res[i] = (row[i >> 5] >> (i & 31)) & 1u;
        return res;
    }
    case O_NOT: {                    /* Delta \ C: XOR with 1 (Alg. 1) */
        if (nd->child_count != 1) goto bad;
        uint8_t *c = eval(x, ch[0], depth + 1, rc);
        if (!c) { free(res); return NULL; }
        for (uint32_t i = 0; i < N; i++) res[i] = c[i] ^ 1u;
        free(c);
        return res;
    }
    case O_AND:                      /* r=1; r &= concept (Alg. 2) */
    case O_OR: {                     /* r=0; r |= concept                           */
        memset(res, nd->op == O_AND, N);
        for (uint32_t j = 0; j < nd->child_count; j++) {
            uint8_t *c = eval(x, ch[j], depth + 1, rc);
            if (!c) { free(res); return NULL; }
            for (uint32_t i = 0; i < N; i++)
                res[i] = nd->op == O_AND ? (res[i] & c[i]) : (res[i] | c[i]);
            free(c);
        }
        return res;
    }
    case O_EXISTS: case O_FORALL: case O_MIN: case O_MAX: case O_EXACT: {
        if (nd->child_count != 1) goto bad;
        if (nd->arg >= kb->R) { *rc = R_RANGE; free(res); return NULL; }
        uint8_t *c = eval(x, ch[0], depth + 1, rc);
        if (!c) { free(res); return NULL; }
        const uint64_t *p = kb->pairs[nd->arg];
        const uint64_t m = kb->npairs[nd->arg];
        const int inv = (nd->flags & F_INV) != 0;   /* swap subj/obj */
        if (nd->op == O_EXISTS) {
            /* cleared row; an assertion whose object is in C sets its subject
               (Alg. 4) */
            memset(res, 0, N);
            for (uint64_t k = 0; k < m; k++) {
                uint32_t s = (uint32_t)(p[k] >> 32), o = (uint32_t)p[k];
                uint32_t xx = inv ? o : s, yy = inv ? s : o;
                if (c[yy]) res[xx] = 1;
            }
        } else if (nd->op == O_FORALL) {
            /* row set to 1; an assertion whose object is not in C clears its
               subject; assertion-less individuals stay 1 (Alg. 6) */
            memset(res, 1, N);
            for (uint64_t k = 0; k < m; k++) {
                uint32_t s = (uint32_t)(p[k] >> 32), o = (uint32_t)p[k];
                uint32_t xx = inv ? o : s, yy = inv ? s : o;
                if (!c[yy]) res[xx] = 0;
            }
        } else {
            /* count matching assertions per subject, then filter
               (Alg. 7) */
            uint64_t *cnt = (uint64_t *)calloc(N ? N : 1, sizeof(uint64_t));
            if (!cnt) { free(c); free(res); *rc = R_OOM; return NULL; }
            for (uint64_t k = 0; k < m; k++) {
                uint32_t s = (uint32_t)(p[k] >> 32), o = (uint32_t)p[k];
                uint32_t xx = inv ? o : s, yy = inv ? s : o;
                cnt[xx] += c[yy];
            }
            const uint64_t n = nd->n;
            for (uint32_t i = 0; i < N; i++) {
                if (nd->op == O_MIN) res[i] = cnt[i] >= n;            /* MIN: cVal>=rVal */
                else if (nd->op == O_EXACT) res[i] = cnt[i] == n;     /* EXACTLY: cVal==rVal */
                else if (x->flags & CF_COMPAT_PAPER_MAX)
                    res[i] = cnt[i] > 0 && cnt[i] <= n;               /* paper MAX */
                else res[i] = cnt[i] <= n;                            /* standard <=n (Q2) */
            }
            free(cnt);
        }
        free(c);
        return res;
    }
    case O_DRANGE: {
        /* exists d.[lo,hi]: some asserted value v with lo <= v <= hi in float32;
           the paper's >=, ==, <= comparators (Alg. 9) are the
           intervals [v,+inf], [v,v], [-inf,v]; NaN never matches */
        if (nd->child_count) goto bad;
        if (nd->flags & F_INV) goto bad;                 /* Q12 */
        if (isnan(nd->lo) || isnan(nd->hi)) goto bad;    /* Q10 */
        if (nd->arg >= kb->D) { *rc = R_RANGE; free(res); return NULL; }
        memset(res, 0, N);
        const uint32_t *s = kb->dsubj[nd->arg];
        const float *v = kb->dval[nd->arg];
        for (uint64_t k = 0; k < kb->ndata[nd->arg]; k++)
            if (nd->lo <= v[k] && v[k] <= nd->hi) res[s[k]] = 1;
        return res;
    }
    case O_SEQUAL:
    case O_SCONTAIN: {
        /* EQUAL: some assertion's value equals the pattern (Alg. 11);
           CONTAIN: some value contains the pattern as a substring (Alg. 13, PAPER.md:459-488,
           SPEC.md:229 byte-wise, case-sensitive); an empty CONTAIN pattern is rejected (Q20) */
        if (nd->child_count || (nd->flags & F_INV)) goto bad;
        if (nd->arg >= kb->S || nd->n >= x->n_pat) { *rc = R_RANGE; free(res); return NULL; }
        const uint8_t *pat = x->pat_bytes + x->pat_off[nd->n];
        const uint64_t pn = x->pat_off[nd->n + 1] - x->pat_off[nd->n];
        if (nd->op == O_SCONTAIN && pn == 0) goto bad;
        memset(res, 0, N);
        for (uint64_t k = kb->str_off[nd->arg]; k < kb->str_off[nd->arg + 1]; k++) {
            const uint8_t *v = kb->str_bytes + kb->str_val_off[k];
            const uint64_t vn = kb->str_val_off[k + 1] - kb->str_val_off[k];
            const int hit = nd->op == O_SEQUAL ? (vn == pn && memcmp(v, pat, pn) == 0) : contains(v, vn, pat, pn);
            if (hit) res[kb->str_subj[k]] = 1;
        }
        return res;
    }
    default:
        goto bad;
    }
bad:
    free(res);
    *rc = R_BADEXPR;
    return NULL;
}

typedef struct {
    const octx *x;
    const uint32_t *roots;
    uint32_t n_roots, tid, nthreads;
    uint32_t *out_bits;
    uint64_t *out_counts;
    int rc;
    uint32_t bad_root;
} ojob;

static void *run_job(void *arg) {
    ojob *j = (ojob *)arg;
    const okb *kb = j->x->kb;
    for (uint32_t r = j->tid; r < j->n_roots; r += j->nthreads) {
        int rc = R_OK;
        uint8_t *row = eval(j->x, j->roots[r], 0, &rc);
        if (!row) { if (j->rc == R_OK) { j->rc = rc; j->bad_root = r; } continue; }
        /* Alg. 15: covered positives / negatives */
        uint64_t tp = 0, fp = 0;
        for (uint32_t i = 0; i < kb->N; i++) { tp += row[i] & kb->pos[i]; fp += row[i] & kb->neg[i]; }
        uint64_t *cn = j->out_counts + 4ull * r;
        cn[0] = tp; cn[1] = fp; cn[2] = kb->npos - tp; cn[3] = kb->nneg - fp;
        if (j->out_bits) {
            uint32_t *w = j->out_bits + (uint64_t)r * kb->W;
            memset(w, 0, (size_t)kb->W * 4);
            for (uint32_t i = 0; i < kb->N; i++) w[i >> 5] |= (uint32_t)row[i] << (i & 31);
        }
        free(row);
    }
    return NULL;
}

/* Evaluate roots[0..n_roots) ; out_bits [n_roots][W] (nullable), out_counts
   [n_roots][4] = tp, fp, fn, tn.  Hypotheses are independent, so n_threads
   plain evaluators run side by side (the paper's 'Scalar' column shape,
   PAPER.md:616); each hypothesis is single-threaded. */
int oracle_eval(const okb *kb, const onode *nodes, uint32_t n_nodes,
                const uint32_t *kids, uint64_t n_kids,
                const uint32_t *roots, uint32_t n_roots, uint32_t flags,
                uint32_t n_pat, const uint64_t *pat_off, const uint8_t *pat_bytes,
                uint32_t *out_bits, uint64_t *out_counts, int n_threads, uint32_t *bad_root) {
    octx x = {kb, nodes, n_nodes, kids, n_kids, flags, n_pat, pat_off, pat_bytes};
    if (n_threads < 1) n_threads = 1;
    if ((uint32_t)n_threads > n_roots) n_threads = n_roots ? (int)n_roots : 1;
    ojob *jobs = (ojob *)calloc((size_t)n_threads, sizeof(ojob));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    for (int t = 0; t < n_threads; t++) {
        jobs[t] = (ojob){&x, roots, n_roots, (uint32_t)t, (uint32_t)n_threads, out_bits, out_counts, R_OK, 0};
        if (n_threads == 1) run_job(&jobs[t]);
        else pthread_create(&th[t], NULL, run_job, &jobs[t]);
    }
    int rc = R_OK;
    uint32_t br = 0;
    for (int t = 0; t < n_threads; t++) {
        if (n_threads > 1) pthread_join(th[t], NULL);
        if (jobs[t].rc != R_OK && (rc == R_OK || jobs[t].bad_root < br)) { rc = jobs[t].rc; br = jobs[t].bad_root; }
    }
    free(jobs); free(th);
    if (bad_root) *bad_root = br;
    return rc;
}
