/*
 * am_oracle.c -- CPU restatement of the reference analytic-marching path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file; it is loaded by tests/ (the parity checker), by
 * __graft_entry__.smoke() (checker) and by bench.py's cpu_baseline /
 * --impl reference leg.  It restates, in plain C over float64, the algorithm
 * of the reference package exactmesh (pure Python + numpy; nothing to
 * compile), function by function:
 *
 *   forward / state_at ............ reference network.py:320-392
 *   affine maps + canonical bits .. reference network.py:398-489
 *   build_cell .................... reference cells.py:127-185
 *   solve pairs (3x3 LU) .......... reference cells.py:213-249
 *   dedup / assemble polygon ...... reference cells.py:257-334
 *   naive enumeration ............. reference cells.py:337-362
 *   pivot walk (Algorithm 2) ...... reference cells.py:381-462
 *   transitions / probes / march .. reference marching.py:152-377
 *
 * Pinned against golden vectors produced by running the reference itself
 * (tests/golden/make_golden.py, tests/test_oracle_golden.py).
 *
 * State keys: bit i of the activation pattern is bit (63 - i%64) of word
 * i/64 (MSB-first, so word-wise lexicographic order equals the reference's
 * np.packbits byte order); ensembles append one word holding the branch.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TOL_DET 1e-12
#define DEGEN 1e-12

enum { K_NEURON = 0, K_BRANCH = 1, K_BBOX = 2 };
enum { F_SAVE_INPUT = 1, F_SC_IDENT = 2, F_SC_LINEAR = 4, F_FIRST = 8, F_SC_FROM_INPUT = 16 };
#define STEP_FIELDS 12
#define SUB_FIELDS 6

typedef struct {
    const double *p;
    const int64_t *steps;
    int n_steps;
    const int64_t *subs;
    int n_subs;
    int n_bits;
    int ensemble;
    int kw;         /* key words */
    int bw;         /* bit words */
    int max_width;
} om_net;

typedef struct { double tol_cell, tol_weld, tol_onplane, probe_delta; double lo[3], hi[3]; } om_cfg;

/* ------------------------------------------------------------------ keys */
static inline int key_bit(const uint64_t *k, int i) { return (int)((k[i >> 6] >> (63 - (i & 63))) & 1u); }
static inline void key_set(uint64_t *k, int i, int v) {
    uint64_t m = 1ull << (63 - (i & 63));
    if (v) k[i >> 6] |= m; else k[i >> 6] &= ~m;
}
static inline void key_flip(uint64_t *k, int i) { k[i >> 6] ^= 1ull << (63 - (i & 63)); }

static uint64_t key_hash(const uint64_t *k, int kw) {
    uint64_t h = 0x9E3779B97F4A7C15ull ^ (uint64_t)kw;
    for (int i = 0; i < kw; i++) {
        uint64_t x = k[i] + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1);
        x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
        h = (h ^ x) * 0x100000001B3ull;
        h ^= h >> 29;
    }
    return h;
}

/* ------------------------------------------------------------ hash set */
typedef struct { uint64_t *keys; uint8_t *used; size_t cap, n; int kw; } kset;

static void kset_init(kset *s, int kw, size_t cap) {
    s->kw = kw; s->cap = cap; s->n = 0;
    s->keys = (uint64_t *)malloc(cap * kw * sizeof(uint64_t));
    s->used = (uint8_t *)calloc(cap, 1);
}
static void kset_free(kset *s) { free(s->keys); free(s->used); }
static int kset_find_slot(const kset *s, const uint64_t *k, size_t *slot) {
    size_t m = s->cap - 1, i = key_hash(k, s->kw) & m;
    while (s->used[i]) {
        if (!memcmp(s->keys + i * s->kw, k, s->kw * 8)) { *slot = i; return 1; }
        i = (i + 1) & m;
    }
    *slot = i;
    return 0;
}
static void kset_grow(kset *s);
static int kset_add(kset *s, const uint64_t *k) { /* 1 if newly added */
    size_t slot;
    if (kset_find_slot(s, k, &slot)) return 0;
    memcpy(s->keys + slot * s->kw, k, s->kw * 8);
    s->used[slot] = 1;
    if (++s->n * 2 > s->cap) kset_grow(s);
    return 1;
}
static int kset_has(const kset *s, const uint64_t *k) { size_t slot; return kset_find_slot(s, k, &slot); }
static void kset_grow(kset *s) {
    kset t;
    kset_init(&t, s->kw, s->cap * 2);
    for (size_t i = 0; i < s->cap; i++) if (s->used[i]) kset_add(&t, s->keys + i * s->kw);
    kset_free(s);
    *s = t;
}

/* ------------------------------------------------------- network access */
#define ST(i, f) (net->steps[(i) * STEP_FIELDS + (f)])
#define SB(j, f) (net->subs[(j) * SUB_FIELDS + (f)])

/* forward through one subnetwork; writes pre-activation signs into key, returns F_sub(x).
 * reference network.py:320-349 (_forward_hidden) */
static double sub_forward(const om_net *net, int j, const double x[3], uint64_t *key, double *buf) {
    int W = net->max_width;
    double *h = buf, *pre = buf + W, *hin = buf + 2 * W, *tmp = buf + 3 * W;
    int first = (int)SB(j, 0), ns = (int)SB(j, 1);
    int width = 3;
    memcpy(h, x, 3 * sizeof(double));
    for (int s = first; s < first + ns; s++) {
        int n_in = (int)ST(s, 0), n_out = (int)ST(s, 1), flags = (int)ST(s, 4);
        const double *Wm = net->p + ST(s, 2), *b = net->p + ST(s, 3);
        int row = (int)ST(s, 7);
        if (flags & F_SAVE_INPUT) { memcpy(hin, h, (size_t)width * sizeof(double)); }
        for (int r = 0; r < n_out; r++) {
            double acc = 0.0;
            const double *wr = Wm + (size_t)r * n_in;
            for (int k = 0; k < n_in; k++) acc += h[k] * wr[k];
            pre[r] = acc;
        }
        if (flags & (F_SC_IDENT | F_SC_LINEAR)) {
            int n_sin = (int)ST(s, 10);
            if (flags & F_SC_IDENT) {
                for (int r = 0; r < n_out; r++) tmp[r] = hin[r];
            } else {
                const double *V = net->p + ST(s, 5);
                for (int r = 0; r < n_out; r++) {
                    double acc = 0.0;
                    for (int k = 0; k < n_sin; k++) acc += hin[k] * V[(size_t)r * n_sin + k];
                    tmp[r] = acc;
                }
                if (ST(s, 6) >= 0) { const double *vb = net->p + ST(s, 6); for (int r = 0; r < n_out; r++) tmp[r] += vb[r]; }
            }
            /* pre = shortcut(h_in) + h @ W.T + b */
            for (int r = 0; r < n_out; r++) pre[r] = (tmp[r] + pre[r]) + b[r];
        } else {
            for (int r = 0; r < n_out; r++) pre[r] += b[r];
        }
        for (int r = 0; r < n_out; r++) {
            int bit = pre[r] > 0.0;
            if (key) key_set(key, row + r, bit);
            h[r] = bit ? pre[r] : 0.0;
        }
        width = n_out;
    }
    const double *hw = net->p + SB(j, 2);
    double f = 0.0;
    for (int k = 0; k < width; k++) f += h[k] * hw[k];
    return f + net->p[SB(j, 3)];
}

/* state_at + forward (reference network.py:352-392); returns F(x), key may be NULL */
double om_forward_state(const om_net *net, const double x[3], uint64_t *key, double *buf) {
    double best = -INFINITY;
    int arg = 0;
    if (key) memset(key, 0, (size_t)net->kw * 8);
    for (int j = 0; j < net->n_subs; j++) {
        double f = sub_forward(net, j, x, key, buf);
        if (j == 0 || f > best) { best = f; arg = j; }   /* argmax: lowest index on ties */
    }
    if (key && net->ensemble) key[net->kw - 1] = (uint64_t)arg;
    return best;
}

/* ----------------------------------------------------------- affine maps */
typedef struct {
    uint64_t *key;     /* canonical */
    double *nn;        /* n_bits x 3 raw neuron normals */
    double *no;        /* n_bits */
    double face[4];    /* raw face functional (of the branch for ensembles) */
    double *sface;     /* n_subs x 4 per-subnetwork face functionals */
} om_maps;

static void maps_alloc(const om_net *net, om_maps *m) {
    m->key = (uint64_t *)calloc(net->kw, 8);
    m->nn = (double *)malloc((size_t)net->n_bits * 3 * sizeof(double));
    m->no = (double *)malloc((size_t)net->n_bits * sizeof(double));
    m->sface = (double *)malloc((size_t)net->n_subs * 4 * sizeof(double));
}
static void maps_free(om_maps *m) { free(m->key); free(m->nn); free(m->no); free(m->sface); }

/* reference network.py:398-443 (_region_maps_sub) + 446-489 (affine_maps) */
static void affine_maps(const om_net *net, const uint64_t *key_in, om_maps *m, double *buf) {
    int W = net->max_width;
    double *A = buf, *c = buf + 3 * W, *Ain = buf + 4 * W, *cin = buf + 7 * W;
    double *pA = buf + 8 * W, *pc = buf + 11 * W;
    memcpy(m->key, key_in, (size_t)net->kw * 8);
    for (int j = 0; j < net->n_subs; j++) {
        int first = (int)SB(j, 0), ns = (int)SB(j, 1);
        int width = 3;
        /* A = eye(3), c = zeros(3) */
        for (int i = 0; i < 9; i++) A[i] = (i % 4 == 0) ? 1.0 : 0.0;
        c[0] = c[1] = c[2] = 0.0;
        for (int s = first; s < first + ns; s++) {
            int n_in = (int)ST(s, 0), n_out = (int)ST(s, 1), flags = (int)ST(s, 4);
            const double *Wm = net->p + ST(s, 2), *b = net->p + ST(s, 3);
            int row = (int)ST(s, 7);
            (void)n_in;
            if (flags & F_SAVE_INPUT) {
                memcpy(Ain, A, (size_t)width * 3 * sizeof(double));
                memcpy(cin, c, (size_t)width * sizeof(double));
            }
            for (int r = 0; r < n_out; r++) {
                const double *wr = Wm + (size_t)r * width;
                double a0 = 0, a1 = 0, a2 = 0, cc = 0;
                for (int k = 0; k < width; k++) {
                    a0 += wr[k] * A[k * 3 + 0];
                    a1 += wr[k] * A[k * 3 + 1];
                    a2 += wr[k] * A[k * 3 + 2];
                    cc += wr[k] * c[k];
                }
                pA[r * 3 + 0] = a0; pA[r * 3 + 1] = a1; pA[r * 3 + 2] = a2;
                pc[r] = cc;
            }
            if (flags & (F_SC_IDENT | F_SC_LINEAR)) {
                int n_sin = (int)ST(s, 10);
                for (int r = 0; r < n_out; r++) {
                    double s0, s1, s2, sc;
                    if (flags & F_SC_IDENT) {
                        s0 = Ain[r * 3]; s1 = Ain[r * 3 + 1]; s2 = Ain[r * 3 + 2]; sc = cin[r];
                    } else {
                        const double *vr = net->p + ST(s, 5) + (size_t)r * n_sin;
                        s0 = s1 = s2 = sc = 0.0;
                        for (int k = 0; k < n_sin; k++) {
                            s0 += vr[k] * Ain[k * 3]; s1 += vr[k] * Ain[k * 3 + 1];
                            s2 += vr[k] * Ain[k * 3 + 2]; sc += vr[k] * cin[k];
                        }
                        if (ST(s, 6) >= 0) sc = sc + net->p[ST(s, 6) + r];
                    }
                    pA[r * 3] = s0 + pA[r * 3]; pA[r * 3 + 1] = s1 + pA[r * 3 + 1]; pA[r * 3 + 2] = s2 + pA[r * 3 + 2];
                    pc[r] = (sc + pc[r]) + b[r];
                }
            } else {
                for (int r = 0; r < n_out; r++) pc[r] = pc[r] + b[r];
            }
            /* step(): record planes, canonicalize constant neurons, mask */
            for (int r = 0; r < n_out; r++) {
                double *nr = m->nn + (size_t)(row + r) * 3;
                nr[0] = pA[r * 3]; nr[1] = pA[r * 3 + 1]; nr[2] = pA[r * 3 + 2];
                m->no[row + r] = pc[r];
                double nrm = sqrt((nr[0] * nr[0] + nr[1] * nr[1]) + nr[2] * nr[2]);
                int bit = key_bit(m->key, row + r);
                if (nrm <= DEGEN) { bit = pc[r] > 0.0; key_set(m->key, row + r, bit); }
                double mk = bit ? 1.0 : 0.0;
                A[r * 3] = pA[r * 3] * mk; A[r * 3 + 1] = pA[r * 3 + 1] * mk; A[r * 3 + 2] = pA[r * 3 + 2] * mk;
                c[r] = pc[r] * mk;
            }
            width = n_out;
        }
        const double *hw = net->p + SB(j, 2);
        double f0 = 0, f1 = 0, f2 = 0, fc = 0;
        for (int k = 0; k < width; k++) {
            f0 += hw[k] * A[k * 3]; f1 += hw[k] * A[k * 3 + 1]; f2 += hw[k] * A[k * 3 + 2];
            fc += hw[k] * c[k];
        }
        m->sface[j * 4] = f0; m->sface[j * 4 + 1] = f1; m->sface[j * 4 + 2] = f2;
        m->sface[j * 4 + 3] = fc + net->p[SB(j, 3)];
    }
    int br = net->ensemble ? (int)key_in[net->kw - 1] : 0;
    memcpy(m->face, m->sface + br * 4, 4 * sizeof(double));
}

/* ------------------------------------------------------------------ cell */
typedef struct { int kind, index; } ref_t;
typedef struct {
    int K;
    double *n, *o;
    ref_t *refs;
    int *row_of;        /* per neuron bit: row or -1; then per branch target: row or -1 */
    double fu[3], fo;
    int face_ok;
} om_cell;

static void cell_alloc(const om_net *net, om_cell *cl) {
    int kmax = net->n_bits + net->n_subs + 6;
    cl->n = (double *)malloc((size_t)kmax * 3 * sizeof(double));
    cl->o = (double *)malloc((size_t)kmax * sizeof(double));
    cl->refs = (ref_t *)malloc((size_t)kmax * sizeof(ref_t));
    cl->row_of = (int *)malloc((size_t)(net->n_bits + net->n_subs) * sizeof(int));
}
static void cell_free(om_cell *cl) { free(cl->n); free(cl->o); free(cl->refs); free(cl->row_of); }

/* reference cells.py:127-185 */
static void build_cell(const om_net *net, const om_maps *m, const om_cfg *cfg, om_cell *cl) {
    int K = 0;
    for (int i = 0; i < net->n_bits; i++) {
        const double *nr = m->nn + (size_t)i * 3;
        double nrm = sqrt((nr[0] * nr[0] + nr[1] * nr[1]) + nr[2] * nr[2]);
        cl->row_of[i] = -1;
        if (!(nrm > DEGEN)) continue;
        double orient = key_bit(m->key, i) ? -1.0 : 1.0;
        cl->n[K * 3] = (nr[0] * orient) / nrm; cl->n[K * 3 + 1] = (nr[1] * orient) / nrm;
        cl->n[K * 3 + 2] = (nr[2] * orient) / nrm;
        cl->o[K] = (m->no[i] * orient) / nrm;
        cl->refs[K].kind = K_NEURON; cl->refs[K].index = i;
        cl->row_of[i] = K++;
    }
    for (int t = 0; t < net->n_subs; t++) cl->row_of[net->n_bits + t] = -1;
    if (net->ensemble) {
        int br = (int)m->key[net->kw - 1];
        for (int t = 0; t < net->n_subs; t++) {
            if (t == br) continue;
            double d0 = m->sface[t * 4] - m->face[0], d1 = m->sface[t * 4 + 1] - m->face[1];
            double d2 = m->sface[t * 4 + 2] - m->face[2], dc = m->sface[t * 4 + 3] - m->face[3];
            double nrm = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
            if (!(nrm > DEGEN)) continue;
            cl->n[K * 3] = d0 / nrm; cl->n[K * 3 + 1] = d1 / nrm; cl->n[K * 3 + 2] = d2 / nrm;
            cl->o[K] = dc / nrm;
            cl->refs[K].kind = K_BRANCH; cl->refs[K].index = t;
            cl->row_of[net->n_bits + t] = K++;
        }
    }
    for (int k = 0; k < 3; k++) {
        cl->n[K * 3] = cl->n[K * 3 + 1] = cl->n[K * 3 + 2] = 0.0;
        cl->n[K * 3 + k] = 1.0; cl->o[K] = -cfg->hi[k];
        cl->refs[K].kind = K_BBOX; cl->refs[K].index = 2 * k; K++;
        cl->n[K * 3] = cl->n[K * 3 + 1] = cl->n[K * 3 + 2] = 0.0;
        cl->n[K * 3 + k] = -1.0; cl->o[K] = cfg->lo[k];
        cl->refs[K].kind = K_BBOX; cl->refs[K].index = 2 * k + 1; K++;
    }
    cl->K = K;
    double fn = sqrt((m->face[0] * m->face[0] + m->face[1] * m->face[1]) + m->face[2] * m->face[2]);
    if (fn > DEGEN) {
        cl->fu[0] = m->face[0] / fn; cl->fu[1] = m->face[1] / fn; cl->fu[2] = m->face[2] / fn;
        cl->fo = m->face[3] / fn;
        double fun = sqrt((cl->fu[0] * cl->fu[0] + cl->fu[1] * cl->fu[1]) + cl->fu[2] * cl->fu[2]);
        cl->face_ok = fun > DEGEN;     /* _face_rows */
    } else {
        cl->fu[0] = cl->fu[1] = cl->fu[2] = 0.0; cl->fo = 0.0; cl->face_ok = 0;
    }
}

static inline double row_val(const om_cell *cl, int r, const double x[3]) {
    const double *n = cl->n + r * 3;
    return ((n[0] * x[0] + n[1] * x[1]) + n[2] * x[2]) + cl->o[r];
}

/* 3x3 solve by LU with partial pivoting (LAPACK getf2/getrs order); returns |det| */
static double solve3(const double M_in[9], const double rhs_in[3], double x[3]) {
    double a[9], b[3];
    memcpy(a, M_in, sizeof a); memcpy(b, rhs_in, sizeof b);
    double sign = 1.0;
    for (int k = 0; k < 3; k++) {
        int p = k;
        double best = fabs(a[k * 3 + k]);
        for (int i = k + 1; i < 3; i++) if (fabs(a[i * 3 + k]) > best) { best = fabs(a[i * 3 + k]); p = i; }
        if (p != k) {
            for (int j = 0; j < 3; j++) { double t = a[k * 3 + j]; a[k * 3 + j] = a[p * 3 + j]; a[p * 3 + j] = t; }
            double t = b[k]; b[k] = b[p]; b[p] = t;
            sign = -sign;
        }
        double piv = a[k * 3 + k];
        if (piv == 0.0) return 0.0;
        double rp = 1.0 / piv;
        for (int i = k + 1; i < 3; i++) {
            double l = a[i * 3 + k] * rp;
            a[i * 3 + k] = l;
            for (int j = k + 1; j < 3; j++) a[i * 3 + j] -= l * a[k * 3 + j];
            b[i] -= l * b[k];
        }
    }
    double det = fabs(sign * a[0] * a[4] * a[8]);
    x[2] = b[2] / a[8];
    x[1] = (b[1] - a[5] * x[2]) / a[4];
    x[0] = ((b[0] - a[1] * x[1]) - a[2] * x[2]) / a[0];
    return det;
}

/* unit-row determinant (reference cells.py:213-228 scales rows before det) is the
 * same as the det of the stored rows: cell rows and fu are already unit */
static int solve_pair(const om_cell *cl, int i, int j, double x[3]) {
    if (i > j) { int t = i; i = j; j = t; }           /* canonical pair order */
    double M[9] = {cl->n[i * 3], cl->n[i * 3 + 1], cl->n[i * 3 + 2],
                   cl->n[j * 3], cl->n[j * 3 + 1], cl->n[j * 3 + 2],
                   cl->fu[0], cl->fu[1], cl->fu[2]};
    double r[3] = {-cl->o[i], -cl->o[j], -cl->fo};
    double det = solve3(M, r, x);
    return det >= TOL_DET;
}

static int inside(const om_cell *cl, const double x[3], double tol) {
    for (int r = 0; r < cl->K; r++) if (!(row_val(cl, r, x) <= tol)) return 0;
    return 1;
}

/* ------------------------------------------------------ small int sets */
typedef struct { int *v; int n, cap; } iset;
static void iset_add(iset *s, int x) {
    for (int i = 0; i < s->n; i++) if (s->v[i] == x) return;
    if (s->n == s->cap) { s->cap = s->cap ? s->cap * 2 : 8; s->v = (int *)realloc(s->v, s->cap * sizeof(int)); }
    s->v[s->n++] = x;
}
static int iset_has(const iset *s, int x) { for (int i = 0; i < s->n; i++) if (s->v[i] == x) return 1; return 0; }
static void iset_free(iset *s) { free(s->v); s->v = NULL; s->n = s->cap = 0; }

/* ------------------------------------------------------------ polygons */
typedef struct {
    int nv;
    double *v;          /* nv x 3 */
    int *enr;           /* refs per edge */
    ref_t *erefs;       /* concatenated */
    int ne_refs;
} om_poly;

static void poly_free(om_poly *p) { if (!p) return; free(p->v); free(p->enr); free(p->erefs); free(p); }

typedef struct { double *v; iset *sets; int n, cap; } vlist;
static void vlist_push(vlist *L, const double x[3], iset s) {
    if (L->n == L->cap) {
        L->cap = L->cap ? L->cap * 2 : 16;
        L->v = (double *)realloc(L->v, (size_t)L->cap * 3 * sizeof(double));
        L->sets = (iset *)realloc(L->sets, (size_t)L->cap * sizeof(iset));
    }
    memcpy(L->v + L->n * 3, x, 3 * sizeof(double));
    L->sets[L->n++] = s;
}
static void vlist_free(vlist *L) {
    for (int i = 0; i < L->n; i++) iset_free(&L->sets[i]);
    free(L->v); free(L->sets); L->v = NULL; L->sets = NULL; L->n = L->cap = 0;
}

static void incident(const om_cell *cl, const double x[3], double tol, iset *s) {
    for (int r = 0; r < cl->K; r++) if (fabs(row_val(cl, r, x)) <= tol) iset_add(s, r);
}

static int lex_less(const double *a, const double *b) {
    if (a[0] != b[0]) return a[0] < b[0];
    if (a[1] != b[1]) return a[1] < b[1];
    return a[2] < b[2];
}

static int cmp_ref(const void *a, const void *b) {
    const ref_t *x = (const ref_t *)a, *y = (const ref_t *)b;
    if (x->kind != y->kind) return x->kind - y->kind;
    return x->index - y->index;
}

/* _dedup_vertices + _assemble_polygon (reference cells.py:257-334); consumes L */
static om_poly *assemble(const om_cell *cl, vlist *L, const om_cfg *cfg) {
    int n = L->n;
    double *rep = (double *)malloc((size_t)(n ? n : 1) * 3 * sizeof(double));
    double *first = (double *)malloc((size_t)(n ? n : 1) * 3 * sizeof(double));
    iset *sets = (iset *)calloc(n ? n : 1, sizeof(iset));
    int nc = 0;
    for (int i = 0; i < n; i++) {
        const double *x = L->v + i * 3;
        int hit = -1;
        for (int k = 0; k < nc; k++) {
            double d0 = first[k * 3] - x[0], d1 = first[k * 3 + 1] - x[1], d2 = first[k * 3 + 2] - x[2];
            if (sqrt((d0 * d0 + d1 * d1) + d2 * d2) <= cfg->tol_weld) { hit = k; break; }
        }
        if (hit < 0) {
            hit = nc++;
            memcpy(first + hit * 3, x, 3 * sizeof(double));
            memcpy(rep + hit * 3, x, 3 * sizeof(double));
        } else if (lex_less(x, rep + hit * 3)) {
            memcpy(rep + hit * 3, x, 3 * sizeof(double));
        }
        for (int q = 0; q < L->sets[i].n; q++) iset_add(&sets[hit], L->sets[i].v[q]);
    }
    free(first);
    vlist_free(L);
    if (nc < 3) {
        for (int k = 0; k < nc; k++) iset_free(&sets[k]);
        free(sets); free(rep);
        return NULL;
    }
    /* _orient_loop */
    const double *fn = cl->fu;
    double a[3] = {1.0, 0.0, 0.0};
    if (!(fabs(fn[0]) < 0.9)) { a[0] = 0.0; a[1] = 1.0; }
    double u[3] = {fn[1] * a[2] - fn[2] * a[1], fn[2] * a[0] - fn[0] * a[2], fn[0] * a[1] - fn[1] * a[0]};
    double un = sqrt((u[0] * u[0] + u[1] * u[1]) + u[2] * u[2]);
    u[0] /= un; u[1] /= un; u[2] /= un;
    double v[3] = {fn[1] * u[2] - fn[2] * u[1], fn[2] * u[0] - fn[0] * u[2], fn[0] * u[1] - fn[1] * u[0]};
    double cen[3] = {0, 0, 0};
    for (int k = 0; k < nc; k++) { cen[0] += rep[k * 3]; cen[1] += rep[k * 3 + 1]; cen[2] += rep[k * 3 + 2]; }
    cen[0] /= nc; cen[1] /= nc; cen[2] /= nc;
    double *ang = (double *)malloc(nc * sizeof(double));
    int *ord = (int *)malloc(nc * sizeof(int));
    for (int k = 0; k < nc; k++) {
        double r0 = rep[k * 3] - cen[0], r1 = rep[k * 3 + 1] - cen[1], r2 = rep[k * 3 + 2] - cen[2];
        ang[k] = atan2((r0 * v[0] + r1 * v[1]) + r2 * v[2], (r0 * u[0] + r1 * u[1]) + r2 * u[2]);
        ord[k] = k;
    }
    for (int i = 1; i < nc; i++) {   /* stable insertion sort by angle */
        int t = ord[i], j = i - 1;
        while (j >= 0 && ang[ord[j]] > ang[t]) { ord[j + 1] = ord[j]; j--; }
        ord[j + 1] = t;
    }
    double *pv = (double *)malloc((size_t)nc * 3 * sizeof(double));
    iset *ps = (iset *)malloc(nc * sizeof(iset));
    for (int k = 0; k < nc; k++) { memcpy(pv + k * 3, rep + ord[k] * 3, 3 * sizeof(double)); ps[k] = sets[ord[k]]; }
    free(sets); free(rep); free(ang); free(ord);
    /* _loop_area */
    double tot[3] = {0, 0, 0};
    for (int i = 0; i < nc; i++) {
        const double *p = pv + i * 3, *q = pv + ((i + 1) % nc) * 3;
        tot[0] += p[1] * q[2] - p[2] * q[1];
        tot[1] += p[2] * q[0] - p[0] * q[2];
        tot[2] += p[0] * q[1] - p[1] * q[0];
    }
    double area = 0.5 * ((tot[0] * fn[0] + tot[1] * fn[1]) + tot[2] * fn[2]);
    if (area < 0.0) {
        for (int i = 0, j = nc - 1; i < j; i++, j--) {
            double t[3]; memcpy(t, pv + i * 3, sizeof t); memcpy(pv + i * 3, pv + j * 3, sizeof t); memcpy(pv + j * 3, t, sizeof t);
            iset ts = ps[i]; ps[i] = ps[j]; ps[j] = ts;
        }
    }
    int start = 0;
    for (int k = 1; k < nc; k++) if (lex_less(pv + k * 3, pv + start * 3)) start = k;
    om_poly *P = (om_poly *)calloc(1, sizeof(om_poly));
    P->nv = nc;
    P->v = (double *)malloc((size_t)nc * 3 * sizeof(double));
    iset *rs = (iset *)malloc(nc * sizeof(iset));
    for (int k = 0; k < nc; k++) { memcpy(P->v + k * 3, pv + ((k + start) % nc) * 3, 3 * sizeof(double)); rs[k] = ps[(k + start) % nc]; }
    free(pv); free(ps);
    P->enr = (int *)malloc(nc * sizeof(int));
    int cap = 4 * nc;
    P->erefs = (ref_t *)malloc(cap * sizeof(ref_t));
    P->ne_refs = 0;
    for (int i = 0; i < nc; i++) {
        const double *p = P->v + i * 3, *q = P->v + ((i + 1) % nc) * 3;
        double mid[3] = {0.5 * (p[0] + q[0]), 0.5 * (p[1] + q[1]), 0.5 * (p[2] + q[2])};
        iset on_mid = {0}, shared = {0}, rows = {0};
        int amin = 0;
        double vmin = INFINITY;
        for (int r = 0; r < cl->K; r++) {
            double val = fabs(row_val(cl, r, mid));
            if (val <= cfg->tol_onplane) iset_add(&on_mid, r);
            if (val < vmin) { vmin = val; amin = r; }
        }
        for (int q2 = 0; q2 < rs[i].n; q2++) if (iset_has(&rs[(i + 1) % nc], rs[i].v[q2])) iset_add(&shared, rs[i].v[q2]);
        for (int q2 = 0; q2 < shared.n; q2++) if (iset_has(&on_mid, shared.v[q2])) iset_add(&rows, shared.v[q2]);
        if (!rows.n) {
            const iset *src = shared.n ? &shared : &on_mid;
            for (int q2 = 0; q2 < src->n; q2++) iset_add(&rows, src->v[q2]);
        }
        if (!rows.n) iset_add(&rows, amin);
        if (P->ne_refs + rows.n > cap) { cap = 2 * (P->ne_refs + rows.n); P->erefs = (ref_t *)realloc(P->erefs, cap * sizeof(ref_t)); }
        for (int q2 = 0; q2 < rows.n; q2++) P->erefs[P->ne_refs + q2] = cl->refs[rows.v[q2]];
        qsort(P->erefs + P->ne_refs, rows.n, sizeof(ref_t), cmp_ref);
        P->enr[i] = rows.n;
        P->ne_refs += rows.n;
        iset_free(&on_mid); iset_free(&shared); iset_free(&rows);
    }
    for (int k = 0; k < nc; k++) iset_free(&rs[k]);
    free(rs);
    return P;
}

/* reference cells.py:337-362 */
static om_poly *extract_naive(const om_cell *cl, const om_cfg *cfg) {
    if (!cl->face_ok || cl->K < 2) return NULL;
    vlist L = {0};
    for (int i = 0; i < cl->K; i++) {
        for (int j = i + 1; j < cl->K; j++) {
            double x[3];
            if (!solve_pair(cl, i, j, x)) continue;
            if (!inside(cl, x, cfg->tol_cell)) continue;
            iset s = {0};
            iset_add(&s, i); iset_add(&s, j);
            incident(cl, x, cfg->tol_onplane, &s);
            vlist_push(&L, x, s);
        }
    }
    if (L.n < 3) { vlist_free(&L); return NULL; }
    return assemble(cl, &L, cfg);
}

typedef struct { double d; int i; } dsort;
static int cmp_dsort(const void *a, const void *b) {
    const dsort *x = (const dsort *)a, *y = (const dsort *)b;
    if (x->d < y->d) return -1;
    if (x->d > y->d) return 1;
    return x->i - y->i;    /* stable */
}

/* reference cells.py:381-462 (extract_face_pivot_checked); *fell_back set on fallback */
static om_poly *extract_pivot(const om_cell *cl, int start_row, const double x0[3], const om_cfg *cfg,
                              int *fell_back) {
    *fell_back = 0;
    if (!cl->face_ok) return NULL;
    if (start_row < 0) { *fell_back = 1; return extract_naive(cl, cfg); }
    int K = cl->K;
    dsort *ds = (dsort *)malloc(K * sizeof(dsort));
    for (int r = 0; r < K; r++) { ds[r].d = fabs(row_val(cl, r, x0)); ds[r].i = r; }
    qsort(ds, K, sizeof(dsort), cmp_dsort);
    uint8_t *consumed = (uint8_t *)calloc(K, 1);
    double *verts = (double *)malloc((size_t)(2 * K + 12) * 3 * sizeof(double));
    int *pa = (int *)malloc((2 * K + 12) * sizeof(int)), *pb = (int *)malloc((2 * K + 12) * sizeof(int));
    int nv = 0;
    om_poly *result = NULL;
    int ok = 0;

    /* walk_step: first candidate in distance order giving a valid vertex */
#define WALK_STEP(CUR, ALLOW, PREV, OUT_ROW, OUT_X, FOUND)                                        \
    do {                                                                                          \
        FOUND = 0;                                                                                \
        for (int q = 0; q < K && !FOUND; q++) {                                                   \
            int cand = ds[q].i;                                                                   \
            if (!(cand == (ALLOW) || (cand != (CUR) && !consumed[cand]))) continue;              \
            double xx[3];                                                                         \
            if (!solve_pair(cl, (CUR), cand, xx)) continue;                                       \
            if (!inside(cl, xx, cfg->tol_cell)) continue;                                         \
            if ((PREV) != NULL) {                                                                 \
                const double *pv_ = (PREV);                                                       \
                double d0 = xx[0] - pv_[0], d1 = xx[1] - pv_[1], d2 = xx[2] - pv_[2];             \
                if (sqrt((d0 * d0 + d1 * d1) + d2 * d2) <= cfg->tol_weld) continue;               \
            }                                                                                     \
            OUT_ROW = cand; memcpy(OUT_X, xx, sizeof xx); FOUND = 1;                              \
        }                                                                                         \
    } while (0)

    consumed[start_row] = 1;
    int cur, found;
    double x[3];
    WALK_STEP(start_row, -1, (const double *)NULL, cur, x, found);
    if (found) {
        memcpy(verts, x, sizeof x); pa[0] = start_row; pb[0] = cur; nv = 1;
        consumed[cur] = 1;
        int max_steps = 2 * K + 8;
        int st;
        for (st = 0; st < max_steps; st++) {
            int allow = nv >= 2 ? start_row : -1;
            int nxt;
            WALK_STEP(cur, allow, verts + (nv - 1) * 3, nxt, x, found);
            if (!found) break;
            memcpy(verts + nv * 3, x, sizeof x); pa[nv] = cur; pb[nv] = nxt; nv++;
            double d0 = x[0] - verts[0], d1 = x[1] - verts[1], d2 = x[2] - verts[2];
            int closed = nv > 3 && sqrt((d0 * d0 + d1 * d1) + d2 * d2) <= cfg->tol_weld;
            if (nxt == start_row || closed) { ok = 1; break; }
            consumed[nxt] = 1;
            cur = nxt;
        }
    }
#undef WALK_STEP
    if (ok) {
        vlist L = {0};
        for (int i = 0; i < nv; i++) {
            iset s = {0};
            iset_add(&s, pa[i]); iset_add(&s, pb[i]);
            incident(cl, verts + i * 3, cfg->tol_onplane, &s);
            vlist_push(&L, verts + i * 3, s);
        }
        result = assemble(cl, &L, cfg);
        if (!result) ok = 0;
    }
    free(ds); free(consumed); free(verts); free(pa); free(pb);
    if (!ok) { *fell_back = 1; return extract_naive(cl, cfg); }
    return result;
}

/* ---------------------------------------------------------------- march */
typedef struct qitem {
    uint64_t *key;
    om_maps maps;
    int has_hint;
    ref_t href;
    double hpt[3];
    struct qitem *next;
} qitem;

typedef struct {
    uint64_t *key;
    om_poly *poly;
} om_visit;

typedef struct {
    const om_net *net;
    om_cfg cfg;
    long max_cells;
    kset seen;
    qitem *qhead, *qtail;
    long outstanding;
    int capped;
    long fallbacks;
    om_visit *res;
    long nres, capres;
    pthread_mutex_t lock;
    pthread_cond_t cond;
    int threaded;
} om_marcher;

static void lock(om_marcher *M) { if (M->threaded) pthread_mutex_lock(&M->lock); }
static void unlock(om_marcher *M) { if (M->threaded) pthread_mutex_unlock(&M->lock); }

/* reference marching.py:235-245; takes ownership of maps */
static void enqueue(om_marcher *M, om_maps *maps, int has_hint, ref_t href, const double hpt[3]) {
    lock(M);
    int added = 0;
    if (!kset_has(&M->seen, maps->key)) {
        if ((long)M->seen.n >= M->max_cells) {
            M->capped = 1;
        } else {
            kset_add(&M->seen, maps->key);
            qitem *q = (qitem *)calloc(1, sizeof(qitem));
            q->key = maps->key;
            q->maps = *maps;
            q->has_hint = has_hint;
            q->href = href;
            if (hpt) memcpy(q->hpt, hpt, sizeof q->hpt);
            if (M->qtail) M->qtail->next = q; else M->qhead = q;
            M->qtail = q;
            M->outstanding++;
            added = 1;
            if (M->threaded) pthread_cond_signal(&M->cond);
        }
    }
    unlock(M);
    if (!added) maps_free(maps);
}

static void record(om_marcher *M, uint64_t *key, om_poly *P) {
    lock(M);
    if (M->nres == M->capres) {
        M->capres = M->capres ? M->capres * 2 : 1024;
        M->res = (om_visit *)realloc(M->res, M->capres * sizeof(om_visit));
    }
    M->res[M->nres].key = key;
    M->res[M->nres].poly = P;
    M->nres++;
    unlock(M);
}

/* reference marching.py:247-288 (_Marcher._process) */
static void process(om_marcher *M, qitem *q, double *buf) {
    const om_net *net = M->net;
    om_cell cl;
    cell_alloc(net, &cl);
    build_cell(net, &q->maps, &M->cfg, &cl);
    om_poly *P;
    if (q->has_hint) {
        int row = -1;
        if (q->href.kind == K_NEURON) row = cl.row_of[q->href.index];
        else if (q->href.kind == K_BRANCH) row = cl.row_of[net->n_bits + q->href.index];
        int fb = 0;
        P = extract_pivot(&cl, row, q->hpt, &M->cfg, &fb);
        if (fb) { lock(M); M->fallbacks++; unlock(M); }
    } else {
        P = extract_naive(&cl, &M->cfg);
    }
    uint64_t *state = q->key;
    free(q->maps.nn); free(q->maps.no); free(q->maps.sface);
    record(M, state, P);
    if (P) {
        int kw = net->kw;
        uint64_t *cand = (uint64_t *)malloc((size_t)kw * 8);
        int off = 0;
        for (int e = 0; e < P->nv; e++) {
            const ref_t *er = P->erefs + off;
            int ne = P->enr[e];
            off += ne;
            ref_t cross[64];
            int nc = 0;
            for (int i = 0; i < ne && nc < 64; i++) if (er[i].kind != K_BBOX) cross[nc++] = er[i];
            if (!nc) continue;
            const double *p0 = P->v + e * 3, *p1 = P->v + ((e + 1) % P->nv) * 3;
            double mid[3] = {0.5 * (p0[0] + p1[0]), 0.5 * (p0[1] + p1[1]), 0.5 * (p0[2] + p1[2])};
            int nbits = 0, nbr = 0, bits[64], brs[64];
            for (int i = 0; i < nc; i++) {
                if (cross[i].kind == K_NEURON) bits[nbits++] = cross[i].index;
                else brs[nbr++] = cross[i].index;
            }
            /* _transition_states: subsets (combinations order) x targets */
            int nsub = 0;
            int *subs_m = NULL;  /* list of bitmasks over bits[] ; >3 handled as explicit lists */
            int big = nbits > 3;
            if (big) {
                nsub = nbits + 2;
                subs_m = (int *)malloc(nsub * sizeof(int));   /* encode: -1-i single i, -100 full, -200 empty */
                for (int i = 0; i < nbits; i++) subs_m[i] = -1 - i;
                subs_m[nbits] = -100; subs_m[nbits + 1] = -200;
            } else {
                /* itertools.combinations for k = 0..n in lexicographic order */
                subs_m = (int *)malloc(16 * sizeof(int));
                for (int k = 0; k <= nbits; k++) {
                    /* enumerate k-combinations of [0, nbits) lexicographically */
                    int idx[4];
                    for (int i = 0; i < k; i++) idx[i] = i;
                    for (;;) {
                        int mask = 0;
                        for (int i = 0; i < k; i++) mask |= 1 << idx[i];
                        subs_m[nsub++] = mask;
                        int i = k - 1;
                        while (i >= 0 && idx[i] == nbits - k + i) i--;
                        if (i < 0) break;
                        idx[i]++;
                        for (int t = i + 1; t < k; t++) idx[t] = idx[t - 1] + 1;
                    }
                }
            }
            int ncand_max = nsub * (1 + nbr) + 1;
            uint64_t *cands = (uint64_t *)malloc((size_t)ncand_max * kw * 8);
            int ncand = 0;
            for (int si = 0; si < nsub; si++) {
                for (int ti = -1; ti < nbr; ti++) {
                    int empty_subset;
                    if (big) empty_subset = subs_m[si] == -200;
                    else empty_subset = subs_m[si] == 0;
                    if (empty_subset && ti < 0) continue;
                    uint64_t *t = cands + (size_t)ncand * kw;
                    memcpy(t, state, (size_t)kw * 8);
                    if (big) {
                        if (subs_m[si] == -100) { for (int i = 0; i < nbits; i++) key_flip(t, bits[i]); }
                        else if (subs_m[si] != -200) key_flip(t, bits[-1 - subs_m[si]]);
                    } else {
                        for (int i = 0; i < nbits; i++) if (subs_m[si] & (1 << i)) key_flip(t, bits[i]);
                    }
                    if (ti >= 0) t[kw - 1] = (uint64_t)brs[ti];
                    ncand++;
                }
            }
            free(subs_m);
            /* geometric probe across crossable[0] */
            int prow = cross[0].kind == K_NEURON ? cl.row_of[cross[0].index] : cl.row_of[net->n_bits + cross[0].index];
            if (prow >= 0) {
                double pp[3] = {mid[0] + M->cfg.probe_delta * cl.n[prow * 3], mid[1] + M->cfg.probe_delta * cl.n[prow * 3 + 1],
                                mid[2] + M->cfg.probe_delta * cl.n[prow * 3 + 2]};
                om_forward_state(net, pp, cands + (size_t)ncand * kw, buf);
                ncand++;
            }
            for (int ci = 0; ci < ncand; ci++) {
                uint64_t *nb = cands + (size_t)ci * kw;
                lock(M);
                int have = kset_has(&M->seen, nb);
                unlock(M);
                if (have) continue;
                om_maps nm;
                maps_alloc(net, &nm);
                affine_maps(net, nb, &nm, buf);
                if (!memcmp(nm.key, state, (size_t)kw * 8)) { maps_free(&nm); continue; }
                /* _hint_ref_for_neighbor */
                int hh = 0;
                ref_t hr = {0, 0};
                for (int i = 0; i < nc; i++) if (cross[i].kind == K_NEURON) { hr = cross[i]; hh = 1; break; }
                if (!hh) {
                    int nbbr = (int)nm.key[kw - 1];
                    for (int i = 0; i < nc; i++)
                        if (cross[i].kind == K_BRANCH && nbbr == cross[i].index) {
                            hr.kind = K_BRANCH; hr.index = (int)state[kw - 1]; hh = 1; break;
                        }
                }
                enqueue(M, &nm, hh, hr, mid);
            }
            free(cands);
        }
        free(cand);
    }
    cell_free(&cl);
    free(q);
}

static double *alloc_buf(const om_net *net) {
    return (double *)malloc((size_t)(16 * net->max_width + 64) * sizeof(double));
}

static void *worker(void *arg) {
    om_marcher *M = (om_marcher *)arg;
    double *buf = alloc_buf(M->net);
    for (;;) {
        pthread_mutex_lock(&M->lock);
        while (!M->qhead && M->outstanding > 0) pthread_cond_wait(&M->cond, &M->lock);
        if (!M->qhead && M->outstanding == 0) { pthread_mutex_unlock(&M->lock); break; }
        qitem *q = M->qhead;
        M->qhead = q->next;
        if (!M->qhead) M->qtail = NULL;
        pthread_mutex_unlock(&M->lock);
        process(M, q, buf);
        pthread_mutex_lock(&M->lock);
        M->outstanding--;
        if (M->outstanding == 0) pthread_cond_broadcast(&M->cond);
        else if (M->qhead) pthread_cond_signal(&M->cond);
        pthread_mutex_unlock(&M->lock);
    }
    free(buf);
    return NULL;
}

/* reference marching.py:201-213 (_refine_seed_state) */
static void refine_seed(const om_net *net, const double x_in[3], om_maps *out, double *buf) {
    int kw = net->kw;
    uint64_t *s = (uint64_t *)calloc(kw, 8), *s_new = (uint64_t *)calloc(kw, 8);
    double x[3] = {x_in[0], x_in[1], x_in[2]};
    om_forward_state(net, x, s, buf);
    for (int it = 0; it < 3; it++) {
        affine_maps(net, s, out, buf);
        const double *n = out->face;
        double nn = (n[0] * n[0] + n[1] * n[1]) + n[2] * n[2];
        if (nn <= 0.0) goto done;
        double t = (((n[0] * x[0] + n[1] * x[1]) + n[2] * x[2]) + n[3]) / nn;
        double xp[3] = {x[0] - t * n[0], x[1] - t * n[1], x[2] - t * n[2]};
        om_forward_state(net, xp, s_new, buf);
        if (!memcmp(s_new, out->key, (size_t)kw * 8)) goto done;
        memcpy(x, xp, sizeof x);
        memcpy(s, s_new, (size_t)kw * 8);
    }
    affine_maps(net, s, out, buf);
done:
    free(s); free(s_new);
}

/* --------------------------------------------------------------- public */
typedef struct {
    long n_cells, n_faces, n_empty, n_verts, n_erefs, open_edges, fallbacks;
    int capped;
    int kw;
    uint64_t *keys;      /* sorted */
    int32_t *nverts;
    double *verts;
    int32_t *enr;
    int32_t *erefs;      /* pairs (kind, index) */
} om_result;

static const om_net *g_sort_net;
static int cmp_visit(const void *a, const void *b) {
    const om_visit *x = (const om_visit *)a, *y = (const om_visit *)b;
    for (int i = 0; i < g_sort_net->kw; i++) {
        if (x->key[i] != y->key[i]) return x->key[i] < y->key[i] ? -1 : 1;
    }
    return 0;
}

om_net *om_net_create(const double *params, const int64_t *steps, int n_steps, const int64_t *subs,
                      int n_subs, int n_bits, int ensemble, int max_width) {
    om_net *net = (om_net *)calloc(1, sizeof(om_net));
    net->p = params; net->steps = steps; net->n_steps = n_steps; net->subs = subs; net->n_subs = n_subs;
    net->n_bits = n_bits; net->ensemble = ensemble; net->max_width = max_width;
    net->bw = (n_bits + 63) / 64;
    net->kw = net->bw + (ensemble ? 1 : 0);
    return net;
}
void om_net_free(om_net *net) { free(net); }

/* forward + state for many points: vals (n), keys (n x kw) may be NULL */
void om_forward_many(const om_net *net, const double *pts, long n, double *vals, uint64_t *keys) {
    double *buf = alloc_buf(net);
    for (long i = 0; i < n; i++) {
        double f = om_forward_state(net, pts + i * 3, keys ? keys + i * net->kw : NULL, buf);
        if (vals) vals[i] = f;
    }
    free(buf);
}

/* affine maps of one state: canonical key out, raw neuron planes (n_bits x 4), face (4) */
void om_affine_maps(const om_net *net, const uint64_t *key, uint64_t *canon, double *planes, double *face) {
    double *buf = alloc_buf(net);
    om_maps m;
    maps_alloc(net, &m);
    affine_maps(net, key, &m, buf);
    memcpy(canon, m.key, (size_t)net->kw * 8);
    for (int i = 0; i < net->n_bits; i++) {
        planes[i * 4] = m.nn[i * 3]; planes[i * 4 + 1] = m.nn[i * 3 + 1]; planes[i * 4 + 2] = m.nn[i * 3 + 2];
        planes[i * 4 + 3] = m.no[i];
    }
    memcpy(face, m.face, 4 * sizeof(double));
    maps_free(&m);
    free(buf);
}

/* reference marching.py:304-362 (march), seeds given explicitly */
om_result *om_march(const om_net *net, const double *seeds, int n_seeds, const double *bbox6, long max_cells,
                    int n_threads, double tol_cell, double tol_weld, double tol_onplane, double probe_delta) {
    om_marcher *M = (om_marcher *)calloc(1, sizeof(om_marcher));
    M->net = net;
    M->cfg.tol_cell = tol_cell; M->cfg.tol_weld = tol_weld; M->cfg.tol_onplane = tol_onplane;
    M->cfg.probe_delta = probe_delta;
    for (int k = 0; k < 3; k++) { M->cfg.lo[k] = bbox6[k]; M->cfg.hi[k] = bbox6[3 + k]; }
    M->max_cells = max_cells;
    kset_init(&M->seen, net->kw, 1024);
    M->threaded = n_threads > 1;
    pthread_mutex_init(&M->lock, NULL);
    pthread_cond_init(&M->cond, NULL);
    double *buf = alloc_buf(net);
    for (int i = 0; i < n_seeds; i++) {
        om_maps m;
        maps_alloc(net, &m);
        refine_seed(net, seeds + i * 3, &m, buf);
        ref_t none = {0, 0};
        enqueue(M, &m, 0, none, NULL);
    }
    if (!M->threaded) {
        while (M->qhead) {
            qitem *q = M->qhead;
            M->qhead = q->next;
            if (!M->qhead) M->qtail = NULL;
            M->outstanding--;
            process(M, q, buf);
        }
    } else {
        pthread_t *th = (pthread_t *)malloc(n_threads * sizeof(pthread_t));
        for (int t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, worker, M);
        for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
        free(th);
    }
    free(buf);
    g_sort_net = net;
    qsort(M->res, M->nres, sizeof(om_visit), cmp_visit);
    om_result *R = (om_result *)calloc(1, sizeof(om_result));
    R->kw = net->kw;
    R->n_cells = M->nres;
    R->capped = M->capped;
    R->fallbacks = M->fallbacks;
    for (long i = 0; i < M->nres; i++) {
        om_poly *P = M->res[i].poly;
        if (!P) { R->n_empty++; continue; }
        R->n_faces++;
        R->n_verts += P->nv;
        R->n_erefs += P->ne_refs;
        int off = 0;
        for (int e = 0; e < P->nv; e++) {
            int hit = 0;
            for (int q = 0; q < P->enr[e]; q++) if (P->erefs[off + q].kind == K_BBOX) hit = 1;
            R->open_edges += hit;
            off += P->enr[e];
        }
    }
    R->keys = (uint64_t *)malloc((size_t)(R->n_cells ? R->n_cells : 1) * net->kw * 8);
    R->nverts = (int32_t *)malloc((size_t)(R->n_cells ? R->n_cells : 1) * 4);
    R->verts = (double *)malloc((size_t)(R->n_verts ? R->n_verts : 1) * 3 * sizeof(double));
    R->enr = (int32_t *)malloc((size_t)(R->n_verts ? R->n_verts : 1) * 4);
    R->erefs = (int32_t *)malloc((size_t)(R->n_erefs ? R->n_erefs : 1) * 2 * 4);
    long vo = 0, eo = 0;
    for (long i = 0; i < M->nres; i++) {
        memcpy(R->keys + i * net->kw, M->res[i].key, (size_t)net->kw * 8);
        om_poly *P = M->res[i].poly;
        R->nverts[i] = P ? P->nv : 0;
        if (P) {
            memcpy(R->verts + vo * 3, P->v, (size_t)P->nv * 3 * sizeof(double));
            for (int e = 0; e < P->nv; e++) R->enr[vo + e] = P->enr[e];
            for (int q = 0; q < P->ne_refs; q++) { R->erefs[(eo + q) * 2] = P->erefs[q].kind; R->erefs[(eo + q) * 2 + 1] = P->erefs[q].index; }
            vo += P->nv;
            eo += P->ne_refs;
        }
        free(M->res[i].key);
        poly_free(P);
    }
    free(M->res);
    kset_free(&M->seen);
    pthread_mutex_destroy(&M->lock);
    pthread_cond_destroy(&M->cond);
    free(M);
    return R;
}

void om_result_counts(const om_result *R, long *out8) {
    out8[0] = R->n_cells; out8[1] = R->n_faces; out8[2] = R->n_empty; out8[3] = R->n_verts;
    out8[4] = R->n_erefs; out8[5] = R->open_edges; out8[6] = R->fallbacks; out8[7] = R->capped;
}
void om_result_copy(const om_result *R, uint64_t *keys, int32_t *nverts, double *verts, int32_t *enr, int32_t *erefs) {
    memcpy(keys, R->keys, (size_t)R->n_cells * R->kw * 8);
    memcpy(nverts, R->nverts, (size_t)R->n_cells * 4);
    memcpy(verts, R->verts, (size_t)R->n_verts * 3 * sizeof(double));
    memcpy(enr, R->enr, (size_t)R->n_verts * 4);
    memcpy(erefs, R->erefs, (size_t)R->n_erefs * 2 * 4);
}
void om_result_free(om_result *R) {
    if (!R) return;
    free(R->keys); free(R->nverts); free(R->verts); free(R->enr); free(R->erefs); free(R);
}

/* ------------------------------------------------ sharding / per-cell API */
/* owner rank of a state: identical arithmetic to csrc/am_internal.h key_owner (GPU) */
static uint64_t g_mix64(uint64_t x) {
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27; x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}
static uint64_t gpu_key_hash(const uint64_t *k, int kw) {
    uint64_t h = 0x9E3779B97F4A7C15ull ^ (uint64_t)kw;
    for (int i = 0; i < kw; i++) {
        uint64_t x = g_mix64(k[i] + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1));
        h = (h ^ x) * 0x100000001B3ull;
        h ^= h >> 29;
    }
    return g_mix64(h);
}
void om_key_owner(const uint64_t *keys, long n, int kw, int world, int32_t *out) {
    for (long i = 0; i < n; i++)
        out[i] = world <= 1 ? 0 : (int32_t)((gpu_key_hash(keys + i * kw, kw) >> 7) % (uint64_t)world);
}

/* canonical key of a raw state (reference network.py:446-489) */
void om_canonical(const om_net *net, const uint64_t *key, uint64_t *canon) {
    double *buf = alloc_buf(net);
    om_maps m;
    maps_alloc(net, &m);
    affine_maps(net, key, &m, buf);
    memcpy(canon, m.key, (size_t)net->kw * 8);
    maps_free(&m);
    free(buf);
}

/* face of one canonical state (naive enumeration, reference cells.py:337-362) and its
 * neighbour candidates (transition states + probe states, reference marching.py:152-288).
 * Returns the number of candidates written (<= max_out), -1 if the face is empty. */
long om_cell_expand(const om_net *net, const uint64_t *key, const double *bbox6, uint64_t *out, long max_out) {
    om_cfg cfg;
    cfg.tol_cell = 1e-9; cfg.tol_weld = 1e-7; cfg.tol_onplane = 1e-9; cfg.probe_delta = 1e-7;
    for (int k = 0; k < 3; k++) { cfg.lo[k] = bbox6[k]; cfg.hi[k] = bbox6[3 + k]; }
    double *buf = alloc_buf(net);
    om_maps m;
    maps_alloc(net, &m);
    affine_maps(net, key, &m, buf);
    om_cell cl;
    cell_alloc(net, &cl);
    build_cell(net, &m, &cfg, &cl);
    om_poly *P = extract_naive(&cl, &cfg);
    long nout = -1;
    if (P) {
        nout = 0;
        int kw = net->kw, off = 0;
        for (int e = 0; e < P->nv; e++) {
            const ref_t *er = P->erefs + off;
            int ne = P->enr[e];
            off += ne;
            int bits[64], brs[64], nb = 0, nbr = 0;
            ref_t first = {-1, -1};
            for (int i = 0; i < ne; i++) {
                if (er[i].kind == K_BBOX) continue;
                if (first.kind < 0) first = er[i];
                if (er[i].kind == K_NEURON && nb < 64) bits[nb++] = er[i].index;
                else if (er[i].kind == K_BRANCH && nbr < 64) brs[nbr++] = er[i].index;
            }
            if (first.kind < 0) continue;
            /* subsets exactly as process(): combinations (nb <= 3) or singles + full + () */
            int big = nb > 3, nsub = 0, masks[16];
            if (!big) {
                for (int k = 0; k <= nb; k++) {
                    int idx[4];
                    for (int i = 0; i < k; i++) idx[i] = i;
                    for (;;) {
                        int mk = 0;
                        for (int i = 0; i < k; i++) mk |= 1 << idx[i];
                        masks[nsub++] = mk;
                        int i = k - 1;
                        while (i >= 0 && idx[i] == nb - k + i) i--;
                        if (i < 0) break;
                        idx[i]++;
                        for (int t = i + 1; t < k; t++) idx[t] = idx[t - 1] + 1;
                    }
                }
            } else {
                nsub = nb + 2;
            }
            for (int si = 0; si < nsub; si++) {
                for (int ti = -1; ti < nbr; ti++) {
                    int empty = big ? si == nb + 1 : masks[si] == 0;
                    if (empty && ti < 0) continue;
                    if (nout >= max_out) continue;
                    uint64_t *t = out + nout * kw;
                    memcpy(t, m.key, (size_t)kw * 8);
                    if (big) {
                        if (si < nb) key_flip(t, bits[si]);
                        else if (si == nb) for (int i = 0; i < nb; i++) key_flip(t, bits[i]);
                    } else {
                        for (int i = 0; i < nb; i++) if (masks[si] & (1 << i)) key_flip(t, bits[i]);
                    }
                    if (ti >= 0) t[kw - 1] = (uint64_t)brs[ti];
                    nout++;
                }
            }
            int prow = first.kind == K_NEURON ? cl.row_of[first.index] : cl.row_of[net->n_bits + first.index];
            if (prow >= 0 && nout < max_out) {
                const double *p0 = P->v + e * 3, *p1 = P->v + ((e + 1) % P->nv) * 3;
                double pp[3];
                for (int d = 0; d < 3; d++) pp[d] = 0.5 * (p0[d] + p1[d]) + cfg.probe_delta * cl.n[prow * 3 + d];
                om_forward_state(net, pp, out + nout * kw, buf);
                nout++;
            }
        }
        poly_free(P);
    }
    cell_free(&cl);
    maps_free(&m);
    free(buf);
    return nout;
}

/* ------------------------------------------------------------------ mesh weld
 * reference meshes.py:89-148 weld(mesh, tol).  Greedy over the vertices in order: a vertex
 * merges into the FIRST kept vertex met while scanning the 27 grid cells of side tol (dx, dy,
 * dz each in the order 0, -1, 1; reference meshes.py:112-126) and, inside a cell, the kept
 * vertices in insertion order, at euclidean distance <= tol; otherwise it is kept and appended
 * to its own cell.  tol == 0: exact-coordinate buckets (-0.0 == 0.0), merge into the first kept
 * vertex with equal coordinates (reference meshes.py:104-110).  Loops are remapped, consecutive
 * repeats and a closing repeat removed, and loops with < 3 distinct indices dropped
 * (reference meshes.py:134-148).  Returns 0, or -1 on allocation failure.
 * Outputs: remap[n], kept[n_kept*3], face_off[n_faces+1], face_idx[...], face_src[n_faces],
 * counts3 = {n_kept, n_faces, n_dropped}. */
typedef struct { int64_t k[3]; long *items; long n, cap; int used; } wcell;

static uint64_t wkey_hash(const int64_t k[3]) {
    uint64_t h = 0x9e3779b97f4a7c15ull;
    for (int d = 0; d < 3; d++) {
        h ^= (uint64_t)k[d] + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
        h *= 0xff51afd7ed558ccdull;
    }
    return h ^ (h >> 33);
}
static wcell *wfind(wcell *tab, uint64_t mask, const int64_t k[3], int create) {
    for (uint64_t s = wkey_hash(k) & mask;; s = (s + 1) & mask) {
        wcell *c = &tab[s];
        if (!c->used) {
            if (!create) return NULL;
            c->used = 1;
            memcpy(c->k, k, sizeof c->k);
            return c;
        }
        if (c->k[0] == k[0] && c->k[1] == k[1] && c->k[2] == k[2]) return c;
    }
}
static int64_t wbits(double x) {
    int64_t b;
    if (x == 0.0) x = 0.0;  /* -0.0 and 0.0 hash and compare equal in the reference's tuple keys */
    memcpy(&b, &x, 8);
    return b;
}

int om_weld(const double *v, long n, const long *loop_off, const long *loop_idx, long n_loops, double tol,
            long *remap, double *kept, long *face_off, long *face_idx, long *face_src, long *counts3) {
    uint64_t cap = 16;
    while (cap < (uint64_t)(2 * n + 2)) cap <<= 1;
    wcell *tab = calloc(cap, sizeof(wcell));
    if (!tab) return -1;
    const double inv = tol > 0 ? 1.0 / tol : 0.0;
    static const int ord[3] = {0, -1, 1};
    long nk = 0;
    for (long i = 0; i < n; i++) {
        const double *p = v + i * 3;
        int64_t c[3];
        long hit = -1;
        if (tol > 0) {
            for (int d = 0; d < 3; d++) c[d] = (int64_t)floor(p[d] * inv);
            for (int a = 0; a < 3 && hit < 0; a++)
                for (int b = 0; b < 3 && hit < 0; b++)
                    for (int e = 0; e < 3 && hit < 0; e++) {
                        int64_t q[3] = {c[0] + ord[a], c[1] + ord[b], c[2] + ord[e]};
                        wcell *cl = wfind(tab, cap - 1, q, 0);
                        if (!cl) continue;
                        for (long m = 0; m < cl->n; m++) {
                            const double *r = kept + cl->items[m] * 3;
                            double d0 = r[0] - p[0], d1 = r[1] - p[1], d2 = r[2] - p[2];
                            if (sqrt((d0 * d0 + d1 * d1) + d2 * d2) <= tol) { hit = cl->items[m]; break; }
                        }
                    }
        } else {
            for (int d = 0; d < 3; d++) c[d] = wbits(p[d]);
            wcell *cl = wfind(tab, cap - 1, c, 0);
            if (cl)
                for (long m = 0; m < cl->n; m++) {
                    const double *r = kept + cl->items[m] * 3;
                    if (r[0] == p[0] && r[1] == p[1] && r[2] == p[2]) { hit = cl->items[m]; break; }
                }
        }
        if (hit < 0) {
            hit = nk++;
            memcpy(kept + hit * 3, p, 24);
            wcell *cl = wfind(tab, cap - 1, c, 1);
            if (cl->n == cl->cap) {
                cl->cap = cl->cap ? 2 * cl->cap : 4;
                cl->items = realloc(cl->items, (size_t)cl->cap * sizeof(long));
            }
            cl->items[cl->n++] = hit;
        }
        remap[i] = hit;
    }
    for (uint64_t s = 0; s < cap; s++) free(tab[s].items);
    free(tab);
    long nf = 0, dropped = 0, w = 0;
    face_off[0] = 0;
    for (long l = 0; l < n_loops; l++) {
        long a = loop_off[l], b = loop_off[l + 1];
        if (b <= a) { dropped++; continue; }
        long start = w;
        face_idx[w++] = remap[loop_idx[a]];
        for (long q = a + 1; q < b; q++) {
            long x = remap[loop_idx[q]];
            if (x != face_idx[w - 1]) face_idx[w++] = x;
        }
        if (w - start > 1 && face_idx[start] == face_idx[w - 1]) w--;
        long distinct = 0;
        for (long q = start; q < w; q++) {
            int seen = 0;
            for (long r = start; r < q; r++) if (face_idx[r] == face_idx[q]) { seen = 1; break; }
            distinct += !seen;
        }
        if (distinct < 3) { dropped++; w = start; continue; }
        face_src[nf] = l;
        face_off[++nf] = w;
    }
    counts3[0] = nk; counts3[1] = nf; counts3[2] = dropped;
    return 0;
}
