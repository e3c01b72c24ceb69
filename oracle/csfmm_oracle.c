/*
 * TEST INFRASTRUCTURE ONLY — a plain-C restatement of the reference's CSFMM hot path, the
 * CPU checker for the B200 engine.  It is never linked into the product; only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline leg may load it (via oracle/port.py).
 *
 * Restated from /root/reference/proj (C++20, csfs):
 *   geometry.cpp:19-52        face_project / face_point_from_plane / face_unproject
 *   interpolation.cpp:14-68   ChebyshevGrid1D, bary_basis_1d, CellInterpolant
 *   kernels.cpp:13-51,59-79   dilog + the four kernels (guarded forms summation.cpp:32-77)
 *   cluster_tree.cpp:16-283   transfer_matrix, ClusterTree ctor, upward/downward passes
 *   summation.cpp:89-306      group_by_target, well_separated, direct_sum,
 *                             dual_tree_traversal, evaluate_pp/pc, accumulate_cp_cc
 *   summation.cpp:383-421     csfmm_sum
 * Same operation order and the same libm calls as the reference, compiled without FMA
 * contraction (oracle/Makefile: -ffp-contract=off, no -march), so on this host it agrees
 * with the reference BITWISE (pinned by tests/test_oracle.py against oracle/_ref and the
 * committed golden fixtures).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define KPI 3.14159265358979323846
#define KINV4PI (1.0 / (4.0 * KPI))
#define KCOINC 1e-14
#define KNODETOL 1e-14
#define KMAXDEPTH 60
#define KMINEXT 1e-13

typedef struct {
    double x, y, z;
} vec3;

static double dot3(vec3 a, vec3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static vec3 sub3(vec3 a, vec3 b) { vec3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static double norm3(vec3 a) { return sqrt(dot3(a, a)); }

/* ---------------- geometry.cpp:19-52 ---------------- */
static void face_project(vec3 p, int* face, double* xi, double* eta) {
    const double v[6] = {p.x, p.y, -p.x, -p.y, p.z, -p.z};
    int f = 0;
    for (int k = 1; k < 6; ++k)
        if (v[k] > v[f]) f = k;
    double X = 0, Y = 0;
    switch (f) {
        case 0: X = p.y / p.x; Y = p.z / p.x; break;
        case 1: X = -p.x / p.y; Y = p.z / p.y; break;
        case 2: X = p.y / p.x; Y = -p.z / p.x; break;
        case 3: X = -p.x / p.y; Y = -p.z / p.y; break;
        case 4: X = p.y / p.z; Y = -p.x / p.z; break;
        case 5: X = -p.y / p.z; Y = -p.x / p.z; break;
    }
    *face = f;
    *xi = atan(X);
    *eta = atan(Y);
}

static vec3 face_point_from_plane(int face, double X, double Y) {
    const double s = 1.0 / sqrt(1.0 + X * X + Y * Y);
    vec3 r;
    switch (face) {
        case 0: r.x = s; r.y = s * X; r.z = s * Y; break;
        case 1: r.x = -s * X; r.y = s; r.z = s * Y; break;
        case 2: r.x = -s; r.y = -s * X; r.z = s * Y; break;
        case 3: r.x = s * X; r.y = -s; r.z = s * Y; break;
        case 4: r.x = -s * Y; r.y = s * X; r.z = s; break;
        default: r.x = s * Y; r.y = s * X; r.z = -s; break;
    }
    return r;
}

static vec3 face_unproject(int face, double xi, double eta) {
    return face_point_from_plane(face, tan(xi), tan(eta));
}

/* ---------------- interpolation.cpp:14-43 ---------------- */
typedef struct {
    int degree;
    double* nodes;
    double* weights;
} cheb_t;

static void cheb_init(cheb_t* g, int n) {
    g->degree = n;
    g->nodes = malloc(sizeof(double) * (n + 1));
    g->weights = malloc(sizeof(double) * (n + 1));
    for (int k = 0; k <= n; ++k) {
        g->nodes[k] = cos(k * KPI / n);
        g->weights[k] = (k % 2 == 0) ? 1.0 : -1.0;
    }
    g->weights[0] *= 0.5;
    g->weights[n] *= 0.5;
}

static void bary_basis_1d(const cheb_t* g, double x, double* out) {
    const int np = g->degree + 1;
    for (int k = 0; k < np; ++k) {
        if (fabs(x - g->nodes[k]) < KNODETOL) {
            for (int j = 0; j < np; ++j) out[j] = 0.0;
            out[k] = 1.0;
            return;
        }
    }
    double denom = 0.0;
    for (int k = 0; k < np; ++k) {
        const double q = g->weights[k] / (x - g->nodes[k]);
        out[k] = q;
        denom += q;
    }
    const double inv = 1.0 / denom;
    for (int k = 0; k < np; ++k) out[k] *= inv;
}

/* ---------------- kernels.cpp:13-51 ---------------- */
static double dilog_series(double s) {
    double term = s, sum = s;
    for (int k = 2; k < 80; ++k) {
        term *= s;
        const double add = term / (double)(k * k);
        sum += add;
        if (fabs(add) < 1e-17 * fabs(sum)) break;
    }
    return sum;
}

double port_dilog(double x) {
    const double pi2_6 = KPI * KPI / 6.0;
    if (x == 0.0) return 0.0;
    if (x == 1.0) return pi2_6;
    if (x < -1.0) {
        const double l = log(-x);
        return -pi2_6 - 0.5 * l * l - port_dilog(1.0 / x);
    }
    if (x < -0.5) {
        const double l = log(1.0 - x);
        return -0.5 * l * l - port_dilog(x / (x - 1.0));
    }
    if (x > 0.5) return pi2_6 - log(x) * log1p(-x) - dilog_series(1.0 - x);
    return dilog_series(x);
}

/* guarded kernel ops (summation.cpp:32-77); returns 0 when the guard skips the pair */
typedef struct {
    int kind; /* 0 laplace 1 biharmonic 2 biot_savart 3 sal */
    double pref, c1, c2;
} op_t;

static int op_dim(const op_t* op) { return op->kind == 2 ? 3 : 1; }

static int op_eval(const op_t* op, vec3 x, vec3 y, double* out) {
    switch (op->kind) {
        case 0: {
            const double omc = 1.0 - dot3(x, y);
            if (omc < KCOINC) return 0;
            out[0] = -log(omc) * KINV4PI;
            return 1;
        }
        case 1: {
            const double u = 0.5 * (1.0 + dot3(x, y));
            out[0] = port_dilog(u < 1.0 ? u : 1.0) * KINV4PI;
            return 1;
        }
        case 2: {
            const double omc = 1.0 - dot3(x, y);
            if (omc < KCOINC) return 0;
            const double s = -KINV4PI / omc;
            out[0] = s * (x.y * y.z - x.z * y.y);
            out[1] = s * (x.z * y.x - x.x * y.z);
            out[2] = s * (x.x * y.y - x.y * y.x);
            return 1;
        }
        default: {
            const double omc = 1.0 - dot3(x, y);
            if (omc < KCOINC) return 0;
            const double gamma = sqrt(2.0 * omc);
            const double s = 0.5 * gamma;
            out[0] = op->pref * (op->c1 / gamma - op->c2 * log(s * (1.0 + s)));
            return 1;
        }
    }
}

static op_t make_op(int kind, const double* sal4) {
    /* SalParams defaults kernels.hpp:18-23; SalOp ctor summation.cpp:67-68 */
    double a1 = -2.7, b0 = -6.21196, b1 = 6.1, rho = 1025.0 / 5517.0;
    if (sal4) {
        a1 = sal4[0];
        b0 = sal4[1];
        b1 = sal4[2];
        rho = sal4[3];
    }
    op_t op = {kind, 3.0 * rho * KINV4PI, 1.0 - b0, a1 - b1};
    return op;
}

/* ---------------- cluster_tree.cpp:29-147 ---------------- */
typedef struct {
    int face;
    double xi0, xi1, eta0, eta1; /* bounds */
    vec3 center;
    double radius;
    int begin, end, parent, depth, children[4], child_count;
    double xi_mid, xi_half, eta_mid, eta_half;
    double* xi_nodes;
    double* eta_nodes;
    vec3* proxy;
    double* pw;   /* proxy weights */
    double* pphi; /* proxy potentials */
} cluster_t;

typedef struct {
    int n, degree, np, n0, shrink;
    cheb_t cheb;
    int* perm;
    vec3* pts;
    double *xi, *eta;
    cluster_t* cl;
    int ncl, cap, max_depth;
} tree_t;

static void interp_init(tree_t* t, cluster_t* c) {
    /* CellInterpolant (interpolation.cpp:51-68) */
    const int np = t->np;
    c->xi_mid = 0.5 * (c->xi0 + c->xi1);
    c->xi_half = 0.5 * (c->xi1 - c->xi0);
    c->eta_mid = 0.5 * (c->eta0 + c->eta1);
    c->eta_half = 0.5 * (c->eta1 - c->eta0);
    c->xi_nodes = malloc(sizeof(double) * np);
    c->eta_nodes = malloc(sizeof(double) * np);
    for (int k = 0; k < np; ++k) {
        c->xi_nodes[k] = c->xi_mid + c->xi_half * t->cheb.nodes[k];
        c->eta_nodes[k] = c->eta_mid + c->eta_half * t->cheb.nodes[k];
    }
    c->proxy = malloc(sizeof(vec3) * np * np);
    for (int k1 = 0; k1 < np; ++k1)
        for (int k2 = 0; k2 < np; ++k2) c->proxy[k1 * np + k2] = face_unproject(c->face, c->xi_nodes[k1], c->eta_nodes[k2]);
    c->pw = NULL;
    c->pphi = NULL;
}

static double ref_coord(double v, double mid, double half) { return half > 0.0 ? (v - mid) / half : 0.0; }

static void finish_cluster(tree_t* t, cluster_t* c, double a0, double a1, double e0, double e1) {
    /* cluster_tree.cpp:52-70 */
    if (t->shrink && c->end - c->begin > 0) {
        double r0 = t->xi[c->begin], r1 = t->xi[c->begin], s0 = t->eta[c->begin], s1 = t->eta[c->begin];
        for (int i = c->begin + 1; i < c->end; ++i) { /* std::min(a,b) = b<a?b:a, std::max = a<b?b:a */
            r0 = (t->xi[i] < r0) ? t->xi[i] : r0;
            r1 = (r1 < t->xi[i]) ? t->xi[i] : r1;
            s0 = (t->eta[i] < s0) ? t->eta[i] : s0;
            s1 = (s1 < t->eta[i]) ? t->eta[i] : s1;
        }
        c->xi0 = r0; c->xi1 = r1; c->eta0 = s0; c->eta1 = s1;
    } else {
        c->xi0 = a0; c->xi1 = a1; c->eta0 = e0; c->eta1 = e1;
    }
    interp_init(t, c);
    c->center = face_unproject(c->face, c->xi_mid, c->eta_mid);
    c->radius = 0.0;
    for (int i = c->begin; i < c->end; ++i) {
        const double d = norm3(sub3(c->center, t->pts[i]));
        if (c->radius < d) c->radius = d;
    }
}

static cluster_t* push_cluster(tree_t* t) {
    if (t->ncl == t->cap) {
        t->cap = t->cap ? 2 * t->cap : 64;
        t->cl = realloc(t->cl, sizeof(cluster_t) * t->cap);
    }
    cluster_t* c = &t->cl[t->ncl++];
    memset(c, 0, sizeof(*c));
    c->parent = -1;
    for (int q = 0; q < 4; ++q) c->children[q] = -1;
    return c;
}

static tree_t* tree_build(const vec3* pos, int n, int degree, int n0, int shrink) {
    tree_t* t = calloc(1, sizeof(tree_t));
    t->n = n;
    t->degree = degree;
    t->np = degree + 1;
    t->n0 = n0;
    t->shrink = shrink;
    cheb_init(&t->cheb, degree);
    int* fface = malloc(sizeof(int) * n);
    double *fxi = malloc(sizeof(double) * n), *feta = malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) face_project(pos[i], &fface[i], &fxi[i], &feta[i]);
    t->perm = malloc(sizeof(int) * n);
    int m = 0;
    for (int f = 0; f < 6; ++f) /* stable bucketing by face, :38-41 */
        for (int i = 0; i < n; ++i)
            if (fface[i] == f) t->perm[m++] = i;
    t->pts = malloc(sizeof(vec3) * n);
    t->xi = malloc(sizeof(double) * n);
    t->eta = malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) {
        t->pts[i] = pos[t->perm[i]];
        t->xi[i] = fxi[t->perm[i]];
        t->eta[i] = feta[t->perm[i]];
    }
    int cursor = 0;
    for (int f = 0; f < 6; ++f) { /* roots, :72-85 */
        int count = 0;
        while (cursor + count < n && fface[t->perm[cursor + count]] == f) ++count;
        cluster_t* c = push_cluster(t);
        c->face = f;
        c->begin = cursor;
        c->end = cursor + count;
        c->depth = 0;
        finish_cluster(t, c, -KPI / 4.0, KPI / 4.0, -KPI / 4.0, KPI / 4.0);
        cursor += count;
    }
    free(fface);
    free(fxi);
    free(feta);

    int* stack = malloc(sizeof(int) * 64);
    int sp = 0, scap = 64;
    for (int f = 0; f < 6; ++f) stack[sp++] = f;
    int* tidx = malloc(sizeof(int) * (n > 0 ? n : 1));
    vec3* tpos = malloc(sizeof(vec3) * (n > 0 ? n : 1));
    double *txi = malloc(sizeof(double) * (n > 0 ? n : 1)), *teta = malloc(sizeof(double) * (n > 0 ? n : 1));
    while (sp > 0) { /* LIFO split loop, :87-141 */
        const int id = stack[--sp];
        const double b0 = t->cl[id].xi0, b1 = t->cl[id].xi1, e0 = t->cl[id].eta0, e1 = t->cl[id].eta1;
        const int begin = t->cl[id].begin, end = t->cl[id].end;
        const int depth = t->cl[id].depth, face = t->cl[id].face;
        if (end - begin <= n0 || depth >= KMAXDEPTH) continue;
        const double ex = b1 - b0, ey = e1 - e0;
        if ((ex < ey ? ey : ex) < KMINEXT) continue;
        const double mx = 0.5 * (b0 + b1), my = 0.5 * (e0 + e1);
        const int cnt = end - begin;
        memcpy(tidx, t->perm + begin, sizeof(int) * cnt);
        memcpy(tpos, t->pts + begin, sizeof(vec3) * cnt);
        memcpy(txi, t->xi + begin, sizeof(double) * cnt);
        memcpy(teta, t->eta + begin, sizeof(double) * cnt);
        int counts[4] = {0, 0, 0, 0};
        for (int k = 0; k < cnt; ++k) ++counts[(txi[k] >= mx ? 1 : 0) + (teta[k] >= my ? 2 : 0)];
        int offsets[4], acc = begin;
        for (int q = 0; q < 4; ++q) {
            offsets[q] = acc;
            acc += counts[q];
        }
        int wr[4] = {offsets[0], offsets[1], offsets[2], offsets[3]};
        for (int k = 0; k < cnt; ++k) {
            const int q = (txi[k] >= mx ? 1 : 0) + (teta[k] >= my ? 2 : 0);
            const int w = wr[q]++;
            t->perm[w] = tidx[k];
            t->pts[w] = tpos[k];
            t->xi[w] = txi[k];
            t->eta[w] = teta[k];
        }
        const double rx0[4] = {b0, mx, b0, mx}, rx1[4] = {mx, b1, mx, b1};
        const double ry0[4] = {e0, e0, my, my}, ry1[4] = {my, my, e1, e1};
        for (int q = 0; q < 4; ++q) {
            if (counts[q] == 0) continue;
            cluster_t* ch = push_cluster(t);
            ch->face = face;
            ch->begin = offsets[q];
            ch->end = offsets[q] + counts[q];
            ch->parent = id;
            ch->depth = depth + 1;
            finish_cluster(t, ch, rx0[q], rx1[q], ry0[q], ry1[q]);
            const int cid = t->ncl - 1;
            t->cl[id].children[t->cl[id].child_count++] = cid;
            if (sp == scap) {
                scap *= 2;
                stack = realloc(stack, sizeof(int) * scap);
            }
            stack[sp++] = cid;
        }
    }
    free(stack);
    free(tidx);
    free(tpos);
    free(txi);
    free(teta);
    t->max_depth = 0;
    for (int i = 0; i < t->ncl; ++i)
        if (t->cl[i].depth > t->max_depth) t->max_depth = t->cl[i].depth;
    return t;
}

static void tree_free(tree_t* t) {
    for (int i = 0; i < t->ncl; ++i) {
        free(t->cl[i].xi_nodes);
        free(t->cl[i].eta_nodes);
        free(t->cl[i].proxy);
        free(t->cl[i].pw);
        free(t->cl[i].pphi);
    }
    free(t->cl);
    free(t->perm);
    free(t->pts);
    free(t->xi);
    free(t->eta);
    free(t->cheb.nodes);
    free(t->cheb.weights);
    free(t);
}

/* transfer_matrix (cluster_tree.cpp:16-25): T[k*np+m] = L^parent_k(child node m) */
static void transfer_matrix(const cheb_t* g, double mid, double half, const double* child_nodes, double* T) {
    const int np = g->degree + 1;
    double col[64];
    for (int m = 0; m < np; ++m) {
        const double xhat = half > 0.0 ? (child_nodes[m] - mid) / half : 0.0;
        bary_basis_1d(g, xhat, col);
        for (int k = 0; k < np; ++k) T[k * np + m] = col[k];
    }
}

/* upward_pass (cluster_tree.cpp:163-220) */
static void upward(tree_t* t, const double* weights) {
    const int np = t->np, npp = np * np;
    double* w = malloc(sizeof(double) * (t->n > 0 ? t->n : 1));
    for (int i = 0; i < t->n; ++i) w[i] = weights[t->perm[i]];
    for (int c = 0; c < t->ncl; ++c) {
        free(t->cl[c].pw);
        t->cl[c].pw = calloc(npp, sizeof(double));
    }
    double lx[64], ly[64];
    double *axi = malloc(sizeof(double) * npp), *aeta = malloc(sizeof(double) * npp), *tmp = malloc(sizeof(double) * npp);
    for (int level = t->max_depth; level >= 0; --level) {
        for (int id = 0; id < t->ncl; ++id) { /* levels[level] holds ascending ids */
            cluster_t* c = &t->cl[id];
            if (c->depth != level) continue;
            double* pw = c->pw;
            if (c->child_count == 0) {
                for (int i = c->begin; i < c->end; ++i) {
                    bary_basis_1d(&t->cheb, ref_coord(t->xi[i], c->xi_mid, c->xi_half), lx);
                    bary_basis_1d(&t->cheb, ref_coord(t->eta[i], c->eta_mid, c->eta_half), ly);
                    const double wt = w[i];
                    for (int k1 = 0; k1 < np; ++k1) {
                        const double a = wt * lx[k1];
                        double* row = pw + k1 * np;
                        for (int k2 = 0; k2 < np; ++k2) row[k2] += a * ly[k2];
                    }
                }
            } else {
                for (int q = 0; q < c->child_count; ++q) {
                    const cluster_t* ch = &t->cl[c->children[q]];
                    transfer_matrix(&t->cheb, c->xi_mid, c->xi_half, ch->xi_nodes, axi);
                    transfer_matrix(&t->cheb, c->eta_mid, c->eta_half, ch->eta_nodes, aeta);
                    const double* cw = ch->pw;
                    for (int k1 = 0; k1 < np; ++k1)
                        for (int m2 = 0; m2 < np; ++m2) {
                            double s = 0.0;
                            for (int m1 = 0; m1 < np; ++m1) s += axi[k1 * np + m1] * cw[m1 * np + m2];
                            tmp[k1 * np + m2] = s;
                        }
                    for (int k1 = 0; k1 < np; ++k1)
                        for (int k2 = 0; k2 < np; ++k2) {
                            double s = 0.0;
                            for (int m2 = 0; m2 < np; ++m2) s += tmp[k1 * np + m2] * aeta[k2 * np + m2];
                            pw[k1 * np + k2] += s;
                        }
                }
            }
        }
    }
    free(axi);
    free(aeta);
    free(tmp);
    free(w);
}

/* ---------------- summation.cpp:123-203 ---------------- */
static int well_separated(vec3 c0, double r0, vec3 c1, double r1, double mac) {
    const double R = norm3(sub3(c0, c1));
    return R > 0.0 && r0 + r1 < mac * R;
}

typedef struct {
    int* p; /* (t, s) pairs */
    long n, cap;
} plist;

static void plist_push(plist* l, int t, int s) {
    if (l->n == l->cap) {
        l->cap = l->cap ? 2 * l->cap : 256;
        l->p = realloc(l->p, sizeof(int) * 2 * l->cap);
    }
    l->p[2 * l->n] = t;
    l->p[2 * l->n + 1] = s;
    ++l->n;
}

/* lists[0..3] = pp, pc, cp, cc in the reference's emission order */
static void traversal(const tree_t* T, const tree_t* S, double mac, int n0, plist lists[4]) {
    plist st = {0};
    for (int t = 0; t < 6; ++t)
        for (int s = 0; s < 6; ++s)
            if (T->cl[t].end > T->cl[t].begin && S->cl[s].end > S->cl[s].begin) plist_push(&st, t, s);
    while (st.n > 0) {
        --st.n;
        const int t = st.p[2 * st.n], s = st.p[2 * st.n + 1];
        const cluster_t* ct = &T->cl[t];
        const cluster_t* cs = &S->cl[s];
        const int big_t = ct->end - ct->begin > n0, big_s = cs->end - cs->begin > n0;
        const int sep = well_separated(ct->center, ct->radius, cs->center, cs->radius, mac);
        if (sep && (big_t || big_s)) {
            if (!big_t && big_s) plist_push(&lists[1], t, s);
            else if (big_t && !big_s) plist_push(&lists[2], t, s);
            else plist_push(&lists[3], t, s);
            continue;
        }
        if (!sep && (big_t || big_s)) {
            const int prefer_source = (cs->end - cs->begin) >= (ct->end - ct->begin);
            const int can_s = cs->child_count > 0, can_t = ct->child_count > 0;
            if (can_s && (prefer_source || !can_t)) {
                for (int q = 0; q < cs->child_count; ++q) plist_push(&st, t, cs->children[q]);
                continue;
            }
            if (can_t) {
                for (int q = 0; q < ct->child_count; ++q) plist_push(&st, ct->children[q], s);
                continue;
            }
        }
        plist_push(&lists[0], t, s);
    }
    free(st.p);
}

/* group_by_target (summation.cpp:91-96) as CSR: entries of target g in emission order */
static void group_by_target(const plist* l, int ncl, int** off, int** idx) {
    *off = calloc(ncl + 1, sizeof(int));
    *idx = malloc(sizeof(int) * (l->n > 0 ? l->n : 1));
    for (long e = 0; e < l->n; ++e) ++(*off)[l->p[2 * e] + 1];
    for (int g = 0; g < ncl; ++g) (*off)[g + 1] += (*off)[g];
    int* cur = malloc(sizeof(int) * ncl);
    memcpy(cur, *off, sizeof(int) * ncl);
    for (long e = 0; e < l->n; ++e) (*idx)[cur[l->p[2 * e]]++] = (int)e;
    free(cur);
}

/* evaluate_pp (:205-233), evaluate_pc (:235-264), accumulate_cp_cc (:266-306) */
static void evaluate_all(tree_t* T, const tree_t* S, const double* src_w_input, const op_t* op, plist lists[4],
                         double* out) {
    const int dim = op_dim(op), np = S->np, npp = np * np;
    double* w = malloc(sizeof(double) * (S->n > 0 ? S->n : 1));
    for (int i = 0; i < S->n; ++i) w[i] = src_w_input[S->perm[i]];
    int *off[4], *idx[4];
    for (int k = 0; k < 4; ++k) group_by_target(&lists[k], T->ncl, &off[k], &idx[k]);
    /* PP then PC, each accumulated per target and added to out (reference order) */
    for (int k = 0; k < 2; ++k) {
#pragma omp parallel for schedule(dynamic, 4)
        for (int g = 0; g < T->ncl; ++g) {
            if (off[k][g] == off[k][g + 1]) continue;
            const cluster_t* ct = &T->cl[g];
            for (int i = ct->begin; i < ct->end; ++i) {
                const vec3 xi = T->pts[i];
                double* dst = out + (long)T->perm[i] * dim;
                double acc[3] = {0, 0, 0}, v[3];
                for (int e = off[k][g]; e < off[k][g + 1]; ++e) {
                    const cluster_t* cs = &S->cl[lists[k].p[2 * idx[k][e] + 1]];
                    if (k == 0) {
                        for (int j = cs->begin; j < cs->end; ++j)
                            if (op_eval(op, xi, S->pts[j], v))
                                for (int d = 0; d < dim; ++d) acc[d] += w[j] * v[d];
                    } else {
                        for (int m = 0; m < npp; ++m)
                            if (op_eval(op, xi, cs->proxy[m], v))
                                for (int d = 0; d < dim; ++d) acc[d] += cs->pw[m] * v[d];
                    }
                }
                for (int d = 0; d < dim; ++d) dst[d] += acc[d];
            }
        }
    }
#pragma omp parallel for schedule(dynamic, 4)
    for (int g = 0; g < T->ncl; ++g) {
        if (off[2][g] == off[2][g + 1] && off[3][g] == off[3][g + 1]) continue;
        cluster_t* ct = &T->cl[g];
        double* phi = ct->pphi;
        double v[3];
        for (int m = 0; m < npp; ++m) {
            const vec3 tm = ct->proxy[m];
            double acc[3] = {0, 0, 0};
            for (int e = off[2][g]; e < off[2][g + 1]; ++e) {
                const cluster_t* cs = &S->cl[lists[2].p[2 * idx[2][e] + 1]];
                for (int j = cs->begin; j < cs->end; ++j)
                    if (op_eval(op, tm, S->pts[j], v))
                        for (int d = 0; d < dim; ++d) acc[d] += w[j] * v[d];
            }
            for (int e = off[3][g]; e < off[3][g + 1]; ++e) {
                const cluster_t* cs = &S->cl[lists[3].p[2 * idx[3][e] + 1]];
                for (int k = 0; k < npp; ++k)
                    if (op_eval(op, tm, cs->proxy[k], v))
                        for (int d = 0; d < dim; ++d) acc[d] += cs->pw[k] * v[d];
            }
            for (int d = 0; d < dim; ++d) phi[(long)m * dim + d] += acc[d];
        }
    }
    for (int k = 0; k < 4; ++k) {
        free(off[k]);
        free(idx[k]);
    }
    free(w);
}

/* downward_pass (cluster_tree.cpp:228-283) */
static void downward(tree_t* t, int dim, double* out) {
    const int np = t->np, npp = np * np;
    double lx[64], ly[64];
    double *axi = malloc(sizeof(double) * npp), *aeta = malloc(sizeof(double) * npp);
    for (int level = 0; level <= t->max_depth; ++level) {
        for (int id = 0; id < t->ncl; ++id) {
            cluster_t* c = &t->cl[id];
            if (c->depth != level || !c->pphi) continue;
            const double* pp = c->pphi;
            if (c->child_count == 0) {
                for (int i = c->begin; i < c->end; ++i) {
                    bary_basis_1d(&t->cheb, ref_coord(t->xi[i], c->xi_mid, c->xi_half), lx);
                    bary_basis_1d(&t->cheb, ref_coord(t->eta[i], c->eta_mid, c->eta_half), ly);
                    double* dst = out + (long)t->perm[i] * dim;
                    for (int k1 = 0; k1 < np; ++k1) {
                        const double a = lx[k1];
                        const double* row = pp + (long)k1 * np * dim;
                        for (int k2 = 0; k2 < np; ++k2) {
                            const double b = a * ly[k2];
                            for (int d = 0; d < dim; ++d) dst[d] += b * row[(long)k2 * dim + d];
                        }
                    }
                }
            } else {
                for (int q = 0; q < c->child_count; ++q) {
                    cluster_t* ch = &t->cl[c->children[q]];
                    transfer_matrix(&t->cheb, c->xi_mid, c->xi_half, ch->xi_nodes, axi);
                    transfer_matrix(&t->cheb, c->eta_mid, c->eta_half, ch->eta_nodes, aeta);
                    double* cp = ch->pphi;
                    for (int n1 = 0; n1 < np; ++n1)
                        for (int n2 = 0; n2 < np; ++n2) {
                            double* dst = cp + ((long)n1 * np + n2) * dim;
                            for (int m1 = 0; m1 < np; ++m1) {
                                const double a = axi[m1 * np + n1];
                                const double* row = pp + (long)m1 * np * dim;
                                for (int m2 = 0; m2 < np; ++m2) {
                                    const double b = a * aeta[m2 * np + n2];
                                    for (int d = 0; d < dim; ++d) dst[d] += b * row[(long)m2 * dim + d];
                                }
                            }
                        }
                }
            }
        }
    }
    free(axi);
    free(aeta);
}

static vec3* to_vec3(const double* xyz, long n) {
    vec3* v = malloc(sizeof(vec3) * (n > 0 ? n : 1));
    for (long i = 0; i < n; ++i) {
        v[i].x = xyz[3 * i];
        v[i].y = xyz[3 * i + 1];
        v[i].z = xyz[3 * i + 2];
    }
    return v;
}

/* =============================== exported (ctypes) =============================== */

/* csfmm_sum (summation.cpp:383-421).  Returns 1 for the reference's invalid_argument cases. */
int port_csfmm(const double* txyz, long nt, const double* sxyz, const double* sw, long ns, int kind,
               const double* sal4, double mac, int degree, int n0, int shrink, double* out, long long* counts4) {
    if (degree < 1) return 1;
    const int n0r = n0 >= 0 ? n0 : 4 * degree * degree;
    if (nt == 0 || ns == 0 || n0r < 1) return 1;
    vec3* tp = to_vec3(txyz, nt);
    vec3* spos = to_vec3(sxyz, ns);
    tree_t* T = tree_build(tp, (int)nt, degree, n0r, shrink);
    tree_t* S = tree_build(spos, (int)ns, degree, n0r, shrink);
    upward(S, sw);
    const op_t op = make_op(kind, sal4);
    const int dim = op_dim(&op);
    memset(out, 0, sizeof(double) * nt * dim);
    plist lists[4] = {{0}, {0}, {0}, {0}};
    traversal(T, S, mac, n0r, lists);
    const int npp = T->np * T->np;
    for (int c = 0; c < T->ncl; ++c) T->cl[c].pphi = calloc((size_t)npp * dim, sizeof(double));
    evaluate_all(T, S, sw, &op, lists, out);
    downward(T, dim, out);
    for (int k = 0; k < 4; ++k) {
        if (counts4) counts4[k] = lists[k].n;
        free(lists[k].p);
    }
    tree_free(T);
    tree_free(S);
    free(tp);
    free(spos);
    return 0;
}

/* direct_sum (summation.cpp:136-161) */
int port_direct(const double* txyz, long nt, const double* sxyz, const double* sw, long ns, int kind,
                const double* sal4, double* out) {
    const op_t op = make_op(kind, sal4);
    const int dim = op_dim(&op);
    vec3* tp = to_vec3(txyz, nt);
    vec3* spos = to_vec3(sxyz, ns);
#pragma omp parallel for schedule(static)
    for (long i = 0; i < nt; ++i) {
        double acc[3] = {0, 0, 0}, v[3];
        for (long j = 0; j < ns; ++j)
            if (op_eval(&op, tp[i], spos[j], v))
                for (int d = 0; d < dim; ++d) acc[d] += sw[j] * v[d];
        for (int d = 0; d < dim; ++d) out[i * dim + d] = acc[d];
    }
    free(tp);
    free(spos);
    return 0;
}

void* port_tree_new(const double* xyz, long n, int degree, int n0, int shrink) {
    if (degree < 1 || n == 0 || n0 < 1) return NULL;
    vec3* p = to_vec3(xyz, n);
    tree_t* t = tree_build(p, (int)n, degree, n0, shrink);
    free(p);
    return t;
}
void port_tree_free(void* h) { tree_free((tree_t*)h); }
int port_tree_ncl(void* h) { return ((tree_t*)h)->ncl; }
int port_tree_depth(void* h) { return ((tree_t*)h)->max_depth; }

void port_tree_export(void* h, int* perm, int* ints, double* dbls, double* proxy) {
    const tree_t* t = (const tree_t*)h;
    const int npp = t->np * t->np;
    if (perm) memcpy(perm, t->perm, sizeof(int) * t->n);
    for (int c = 0; c < t->ncl; ++c) {
        const cluster_t* k = &t->cl[c];
        if (ints) {
            int* r = ints + 10 * c;
            r[0] = k->face; r[1] = k->begin; r[2] = k->end; r[3] = k->parent; r[4] = k->depth;
            r[5] = k->child_count;
            for (int q = 0; q < 4; ++q) r[6 + q] = k->children[q];
        }
        if (dbls) {
            double* r = dbls + 8 * c;
            r[0] = k->xi0; r[1] = k->xi1; r[2] = k->eta0; r[3] = k->eta1;
            r[4] = k->center.x; r[5] = k->center.y; r[6] = k->center.z; r[7] = k->radius;
        }
        if (proxy)
            for (int m = 0; m < npp; ++m) {
                proxy[3 * ((long)c * npp + m)] = k->proxy[m].x;
                proxy[3 * ((long)c * npp + m) + 1] = k->proxy[m].y;
                proxy[3 * ((long)c * npp + m) + 2] = k->proxy[m].z;
            }
    }
}

void port_upward(void* h, const double* w, double* pw) {
    tree_t* t = (tree_t*)h;
    upward(t, w);
    const int npp = t->np * t->np;
    for (int c = 0; c < t->ncl; ++c) memcpy(pw + (long)c * npp, t->cl[c].pw, sizeof(double) * npp);
}

void port_lists(void* ht, void* hs, double mac, int n0, long long* counts, int* pp, int* pc, int* cp, int* cc) {
    plist lists[4] = {{0}, {0}, {0}, {0}};
    traversal((tree_t*)ht, (tree_t*)hs, mac, n0, lists);
    int* outs[4] = {pp, pc, cp, cc};
    for (int k = 0; k < 4; ++k) {
        counts[k] = lists[k].n;
        if (outs[k]) memcpy(outs[k], lists[k].p, sizeof(int) * 2 * lists[k].n);
        free(lists[k].p);
    }
}

int port_kernel_eval(int kind, const double* sal4, const double* x, const double* y, double* out) {
    const op_t op = make_op(kind, sal4);
    vec3 a = {x[0], x[1], x[2]}, b = {y[0], y[1], y[2]};
    return op_eval(&op, a, b, out);
}

void port_bary_basis_1d(int degree, double x, double* out) {
    cheb_t g;
    cheb_init(&g, degree);
    bary_basis_1d(&g, x, out);
    free(g.nodes);
    free(g.weights);
}
