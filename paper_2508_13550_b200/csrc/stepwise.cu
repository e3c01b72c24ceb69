// The stepwise half of the reference boundary on the device (include/csfs_b200.h,
// "stepwise API"): the pieces csfmm_sum is made of, callable one by one on trees the CALLER
// holds — the reference's ClusterTree (/root/reference/proj/include/csfs/cluster_tree.hpp:
// 52-67) marshalled into plain arrays (csfs_b200_tree_desc, reference cluster ids):
//
//   csfs_b200_tree_build       ClusterTree ctor            cluster_tree.cpp:29-147
//   csfs_b200_upward_tree      upward_pass                 cluster_tree.cpp:163-220
//   csfs_b200_downward_tree    downward_pass               cluster_tree.cpp:228-283
//   csfs_b200_traversal_tree   dual_tree_traversal         summation.cpp:163-203
//   csfs_b200_evaluate_tree    evaluate_pp / evaluate_pc / accumulate_cp_cc
//                                                          summation.cpp:205-306
//
// Every call uploads what it reads (the caller may have changed the tree in between, as the
// reference's own tests do — acceptance.cpp:251-258 overwrites proxy potentials) into the
// context's device trees in a level-major order (depth, then reference id), runs the same
// kernels as the fused path, and hands results back in reference ids and input order.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "context.hpp"

using namespace csfs_b200;
using namespace csfs_b200::capi;

namespace {

using Ctx = csfs_b200_ctx;

// The caller's tree description, checked.
void check_desc(const csfs_b200_tree_desc* d) {
    if (!d) throw InvalidArgument("tree description must not be null");
    if (d->degree < 1) throw InvalidArgument("interpolation degree must be positive");
    if (d->degree > kMaxNp - 1)
        throw InvalidArgument("interpolation degree above " + std::to_string(kMaxNp - 1) +
                              " is not supported by the B200 engine");
    if (d->n_clusters < 6 || !d->ints || !d->dbls || !d->proxy || !d->perm || (d->n && (!d->xyz || !d->xi || !d->eta)))
        throw InvalidArgument("incomplete tree description");
    if (d->n > 0x3fffffff) throw InvalidArgument("particle count exceeds 2^30");
}

// Uploads a described tree into T (internal ids: depth-major, reference ids ascending
// within a depth — the layout the pass kernels expect).  ref_of[i] = reference id of
// internal cluster i.  w_input: weights in input order (nullable).
void upload_tree(DeviceTree& T, const csfs_b200_tree_desc* d, const double* w_input, std::vector<int>& ref_of,
                 cudaStream_t s) {
    check_desc(d);
    const int ncl = d->n_clusters;
    const long long n = (long long)d->n;
    const int* I = d->ints;
    ref_of.resize(ncl);
    std::iota(ref_of.begin(), ref_of.end(), 0);
    std::stable_sort(ref_of.begin(), ref_of.end(), [&](int a, int b) { return I[10 * a + 4] < I[10 * b + 4]; });
    std::vector<int> int_of(ncl);
    for (int i = 0; i < ncl; ++i) int_of[ref_of[i]] = i;
    for (int r = 0; r < 6; ++r)
        if (int_of[r] != r) throw InvalidArgument("tree description: clusters 0..5 must be the face roots");

    T.n = n;
    T.degree = d->degree;
    T.np = d->degree + 1;
    T.npp = T.np * T.np;
    T.has_w = w_input != nullptr;
    T.ncl = 0;  // nothing to keep: reserve_clusters preserves the first ncl entries
    T.reserve_clusters(ncl, s);
    T.ncl = ncl;
    std::vector<int> face(ncl), depth(ncl), begin(ncl), end(ncl), parent(ncl), nch(ncl);
    std::vector<int4> child(ncl);
    std::vector<double> g[8];
    for (auto& v : g) v.resize(ncl);
    int maxd = 0;
    for (int i = 0; i < ncl; ++i) {
        const int* r = I + 10 * ref_of[i];
        face[i] = r[0];
        begin[i] = r[1];
        end[i] = r[2];
        parent[i] = r[3] < 0 ? -1 : int_of.at(r[3]);
        depth[i] = r[4];
        nch[i] = r[5];
        if (r[5] < 0 || r[5] > 4 || r[1] < 0 || r[2] < r[1] || r[2] > n)
            throw InvalidArgument("tree description: bad cluster " + std::to_string(ref_of[i]));
        int cs[4] = {-1, -1, -1, -1};
        for (int q = 0; q < r[5]; ++q) cs[q] = int_of.at(r[6 + q]);
        child[i] = make_int4(cs[0], cs[1], cs[2], cs[3]);
        for (int f = 0; f < 8; ++f) g[f][i] = d->dbls[8 * ref_of[i] + f];
        maxd = std::max(maxd, r[4]);
    }
    T.level_first.assign(maxd + 1, 0);
    T.level_count.assign(maxd + 1, 0);
    for (int i = 0; i < ncl; ++i) ++T.level_count[depth[i]];
    for (int L = 1; L <= maxd; ++L) T.level_first[L] = T.level_first[L - 1] + T.level_count[L - 1];
    T.root_count.assign(6, 0);
    for (int r = 0; r < 6; ++r) T.root_count[r] = end[r] - begin[r];
    auto put = [&](int* dst, const std::vector<int>& v) {
        CSFS_CK(cudaMemcpyAsync(dst, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    };
    put(T.face, face);
    put(T.depth, depth);
    put(T.begin, begin);
    put(T.end, end);
    put(T.parent, parent);
    put(T.nchild, nch);
    CSFS_CK(cudaMemcpyAsync(T.child.p, child.data(), ncl * sizeof(int4), cudaMemcpyHostToDevice, s));
    double* dg[8] = {T.xi0, T.xi1, T.eta0, T.eta1, T.cx, T.cy, T.cz, T.rad};
    for (int f = 0; f < 8; ++f)
        CSFS_CK(cudaMemcpyAsync(dg[f], g[f].data(), ncl * sizeof(double), cudaMemcpyHostToDevice, s));

    // particles (tree order): SoA positions, face coordinates, permutation, weights
    const size_t nn = size_t(std::max<long long>(n, 1));
    int off = 0;
    for (long long t = 0; t < n && !off; ++t) {
        const double* x = d->xyz + 3 * t;
        off = !(std::fabs(x[0] * x[0] + x[1] * x[1] + x[2] * x[2] - 1.0) <= 1e-12);
    }
    T.off_sphere.grow(1);
    CSFS_CK(cudaMemcpy(T.off_sphere.p, &off, sizeof(int), cudaMemcpyHostToDevice));
    for (DevBuf<double>* b : {&T.px, &T.py, &T.pz, &T.xi, &T.eta, &T.w}) b->grow(nn);
    for (DevBuf<int>* b : {&T.perm, &T.node}) b->grow(nn);
    std::vector<double> col(n);
    double* dp[3] = {T.px, T.py, T.pz};
    for (int f = 0; f < 3; ++f) {
        for (long long t = 0; t < n; ++t) col[t] = d->xyz[3 * t + f];
        CSFS_CK(cudaMemcpy(dp[f], col.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    }
    CSFS_CK(cudaMemcpyAsync(T.xi.p, d->xi, n * sizeof(double), cudaMemcpyHostToDevice, s));
    CSFS_CK(cudaMemcpyAsync(T.eta.p, d->eta, n * sizeof(double), cudaMemcpyHostToDevice, s));
    CSFS_CK(cudaMemcpyAsync(T.perm.p, d->perm, n * sizeof(int), cudaMemcpyHostToDevice, s));
    if (w_input) {  // permute_weights (summation.cpp:98-104)
        for (long long t = 0; t < n; ++t) {
            const int p = d->perm[t];
            if (p < 0 || p >= n) throw InvalidArgument("tree description: bad permutation");
            col[t] = w_input[p];
        }
        CSFS_CK(cudaMemcpy(T.w.p, col.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    }
    // proxy points (CellInterpolant::proxy_points), SoA, internal cluster order
    const size_t nq = size_t(ncl) * T.npp;
    T.qx.grow(nq);
    T.qy.grow(nq);
    T.qz.grow(nq);
    std::vector<double> q(nq);
    double* dq[3] = {T.qx, T.qy, T.qz};
    for (int f = 0; f < 3; ++f) {
        for (int i = 0; i < ncl; ++i)
            for (int k = 0; k < T.npp; ++k)
                q[size_t(i) * T.npp + k] = d->proxy[(size_t(ref_of[i]) * T.npp + k) * 3 + f];
        CSFS_CK(cudaMemcpy(dq[f], q.data(), nq * sizeof(double), cudaMemcpyHostToDevice));
    }
    tree_proxy_radii(T, s);
}

// per-cluster blocks of `w` doubles: reference order <-> internal order
void to_internal(const std::vector<int>& ref_of, const double* src, size_t w, std::vector<double>& dst) {
    dst.resize(ref_of.size() * w);
    for (size_t i = 0; i < ref_of.size(); ++i)
        std::memcpy(dst.data() + i * w, src + size_t(ref_of[i]) * w, w * sizeof(double));
}
void to_reference(const std::vector<int>& ref_of, const std::vector<double>& src, size_t w, double* dst, bool add) {
    for (size_t i = 0; i < ref_of.size(); ++i) {
        const double* a = src.data() + i * w;
        double* b = dst + size_t(ref_of[i]) * w;
        if (add)
            for (size_t k = 0; k < w; ++k) b[k] += a[k];
        else
            std::memcpy(b, a, w * sizeof(double));
    }
}

void forget_state(Ctx* c) {
    c->have_state = false;
    c->have_src_tree = false;
    c->have_tree = false;
    c->part_planned = false;
    c->ref_of[0].clear();
    c->ref_of[1].clear();
}

// (t, s) pairs in reference ids -> internal ids on the device list buffer
void upload_list(Ctx* c, int k, const int* pairs, long long n) {
    Lists& L = c->lists;
    L.n[k] = n;
    L.l[k].grow(size_t(std::max<long long>(n, 1)));
    if (n == 0) return;
    std::vector<int> it(c->ref_of[0].size()), is(c->ref_of[1].size());
    for (size_t i = 0; i < it.size(); ++i) it[c->ref_of[0][i]] = int(i);
    for (size_t i = 0; i < is.size(); ++i) is[c->ref_of[1][i]] = int(i);
    std::vector<int2> v(n);
    for (long long e = 0; e < n; ++e) {
        const int t = pairs[2 * e], s = pairs[2 * e + 1];
        if (t < 0 || t >= int(it.size()) || s < 0 || s >= int(is.size()))
            throw InvalidArgument("interaction list entry out of range");
        v[e] = make_int2(it[t], is[s]);
    }
    CSFS_CK(cudaMemcpy(L.l[k].p, v.data(), n * sizeof(int2), cudaMemcpyHostToDevice));
}

}  // namespace

extern "C" {

int csfs_b200_tree_build(csfs_b200_ctx* c, const double* xyz, size_t n, int degree, int n0, int shrink,
                         int* n_clusters, int* depth) {
    return guarded(c, [&] {
        FmmConfig f;
        f.degree = degree;
        f.n0 = n0;
        f.shrink = shrink != 0;
        // ClusterTree's checks in its order: the Chebyshev grid (member init), then the set
        if (degree < 1) throw InvalidArgument("interpolation degree must be positive");
        if (n == 0) throw InvalidArgument("cannot build a cluster tree from an empty particle set");
        if (n0 < 1) throw InvalidArgument("maximum leaf size must be at least 1");
        validate(f, n, n);
        forget_state(c);
        cudaStream_t s = c->own;
        c->cheb = make_cheb(degree);
        c->h_txyz.grow(n * 3);
        CSFS_CK(cudaMemcpyAsync(c->h_txyz.p, xyz, n * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
        build_tree(c->ttree, c->sc, c->h_txyz.p, nullptr, (long long)n, degree, n0, f.shrink, c->cheb, s);
        CSFS_CK(cudaStreamSynchronize(s));
        c->have_tree = true;
        if (n_clusters) *n_clusters = c->ttree.ncl;
        if (depth) *depth = c->ttree.depth_max();
    });
}

int csfs_b200_tree_particles(csfs_b200_ctx* c, int which, double* xyz, double* xi, double* eta) {
    return guarded(c, [&] {
        const DeviceTree* t = nullptr;
        if (which == 0 && c->have_tree) t = &c->ttree;
        else if (which == 1 && c->have_src_tree) t = &c->stree;
        else if (c->have_state) t = (which == 0 || c->shared) ? &c->ttree : &c->stree;
        if (!t || (which != 0 && which != 1)) throw InvalidArgument("no tree: build one first");
        const long long n = t->n;
        if (xyz) {
            std::vector<double> col(n);
            const double* src[3] = {t->px, t->py, t->pz};
            for (int f = 0; f < 3; ++f) {
                CSFS_CK(cudaMemcpy(col.data(), src[f], n * sizeof(double), cudaMemcpyDeviceToHost));
                for (long long i = 0; i < n; ++i) xyz[3 * i + f] = col[i];
            }
        }
        if (xi) CSFS_CK(cudaMemcpy(xi, t->xi.p, n * sizeof(double), cudaMemcpyDeviceToHost));
        if (eta) CSFS_CK(cudaMemcpy(eta, t->eta.p, n * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int csfs_b200_upward_tree(csfs_b200_ctx* c, const csfs_b200_tree_desc* t, const double* w, double* pw) {
    return guarded(c, [&] {
        if (!w || !pw) throw InvalidArgument("weights and proxy-weight output must not be null");
        forget_state(c);
        cudaStream_t s = c->own;
        DeviceTree& S = c->stree;
        upload_tree(S, t, w, c->ref_of[1], s);
        c->cheb = make_cheb(t->degree);
        upward_pass(S, c->cheb, s);
        std::vector<double> q(size_t(S.ncl) * S.npp);
        CSFS_CK(cudaMemcpyAsync(q.data(), S.qw.p, q.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaStreamSynchronize(s));
        to_reference(c->ref_of[1], q, S.npp, pw, false);
    });
}

int csfs_b200_downward_tree(csfs_b200_ctx* c, const csfs_b200_tree_desc* t, int dim, double* qphi, double* out) {
    return guarded(c, [&] {
        if (dim != 1 && dim != 3) throw InvalidArgument("out_dim must be 1 or 3");
        if (!qphi || !out) throw InvalidArgument("proxy potentials and output must not be null");
        forget_state(c);
        cudaStream_t s = c->own;
        DeviceTree& T = c->ttree;
        upload_tree(T, t, nullptr, c->ref_of[0], s);
        c->cheb = make_cheb(t->degree);
        const size_t blk = size_t(T.npp) * dim;
        std::vector<double> q;
        to_internal(c->ref_of[0], qphi, blk, q);
        T.qphi.grow(q.size());
        CSFS_CK(cudaMemcpyAsync(T.qphi.p, q.data(), q.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        // L2P adds into the caller's out: near = out in tree order, written back through perm
        const long long n = T.n;
        std::vector<double> near(size_t(n) * dim);
        for (long long i = 0; i < n; ++i)
            for (int d = 0; d < dim; ++d) near[size_t(i) * dim + d] = out[size_t(t->perm[i]) * dim + d];
        c->phi_near.grow(near.size() + 1);
        c->h_out.grow(near.size() + 1);
        CSFS_CK(cudaMemcpyAsync(c->phi_near.p, near.data(), near.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        CSFS_CK(cudaMemcpyAsync(c->h_out.p, out, near.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        downward_pass(T, c->cheb, dim, c->phi_near, c->h_out, s, Own{0, n}, true);
        CSFS_CK(cudaMemcpyAsync(out, c->h_out.p, near.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaMemcpyAsync(q.data(), T.qphi.p, q.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaStreamSynchronize(s));
        to_reference(c->ref_of[0], q, blk, qphi, false);  // children received their parents' share
    });
}

int csfs_b200_traversal_tree(csfs_b200_ctx* c, const csfs_b200_tree_desc* t, const csfs_b200_tree_desc* src,
                             double mac, int n0, long long* counts) {
    return guarded(c, [&] {
        forget_state(c);
        cudaStream_t s = c->own;
        upload_tree(c->ttree, t, nullptr, c->ref_of[0], s);
        upload_tree(c->stree, src, nullptr, c->ref_of[1], s);
        c->shared = false;
        dual_traversal(c->ttree, c->stree, mac, n0, c->lists, c->sc, s);
        CSFS_CK(cudaStreamSynchronize(s));
        c->have_state = true;  // lists_export / tree_export see the uploaded trees
        if (counts)
            for (int k = 0; k < 4; ++k) counts[k] = c->lists.n[k];
    });
}

int csfs_b200_evaluate_tree(csfs_b200_ctx* c, const csfs_b200_tree_desc* t, const csfs_b200_tree_desc* src,
                            const double* w, const double* src_pw, const csfs_b200_kernel* k, const int* pp,
                            long long n_pp, const int* pc, long long n_pc, const int* cp, long long n_cp,
                            const int* cc, long long n_cc, double* out, double* qphi) {
    return guarded(c, [&] {
        const KernelSpec ks = to_spec(k);
        if ((n_pp || n_cp) && !w) throw InvalidArgument("PP / CP evaluation needs the source weights");
        if ((n_pc || n_cc) && !src_pw) throw InvalidArgument("PC / CC evaluation needs the source proxy weights");
        if ((n_pp || n_pc) && !out) throw InvalidArgument("PP / PC evaluation needs the output field");
        if ((n_cp || n_cc) && !qphi) throw InvalidArgument("CP / CC evaluation needs the proxy potentials");
        if (t && src && t->degree != src->degree && (n_pc || n_cc || n_cp))
            throw InvalidArgument("target and source trees differ in degree");
        forget_state(c);
        cudaStream_t s = c->own;
        DeviceTree& T = c->ttree;
        DeviceTree& S = c->stree;
        upload_tree(T, t, nullptr, c->ref_of[0], s);
        upload_tree(S, src, w, c->ref_of[1], s);
        c->shared = false;
        c->kspec = ks;
        c->dim = ks.out_dim();
        const int dim = c->dim;
        S.qw.grow(size_t(S.ncl) * S.npp);
        if (src_pw) {
            std::vector<double> q;
            to_internal(c->ref_of[1], src_pw, S.npp, q);
            CSFS_CK(cudaMemcpy(S.qw.p, q.data(), q.size() * sizeof(double), cudaMemcpyHostToDevice));
        }
        upload_list(c, 0, pp, n_pp);
        upload_list(c, 1, pc, n_pc);
        upload_list(c, 2, cp, n_cp);
        upload_list(c, 3, cc, n_cc);
        build_items(T, S, c->lists, c->items, c->sc, s);
        c->items.mutual = false;
        const long long n = T.n;
        c->phi_near.grow(size_t(n) * dim + 1);
        T.qphi.grow(size_t(T.ncl) * T.npp * dim);
        CSFS_CK(cudaMemsetAsync(c->phi_near.p, 0, size_t(n) * dim * sizeof(double), s));
        CSFS_CK(cudaMemsetAsync(T.qphi.p, 0, size_t(T.ncl) * T.npp * dim * sizeof(double), s));
        c->counter.grow(4);
        interact(ks, T, S, c->items, c->phi_near, c->counter, c->log_tab, s, Own{0, n});
        if (n_pp || n_pc) {  // out.at(perm[i]) += acc (summation.cpp:224-227, 254-257)
            std::vector<double> near(size_t(n) * dim);
            CSFS_CK(cudaMemcpyAsync(near.data(), c->phi_near.p, near.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                    s));
            CSFS_CK(cudaStreamSynchronize(s));
            for (long long i = 0; i < n; ++i)
                for (int d = 0; d < dim; ++d) out[size_t(t->perm[i]) * dim + d] += near[size_t(i) * dim + d];
        }
        if (n_cp || n_cc) {  // phi[m * dim + d] += acc (summation.cpp:302)
            std::vector<double> q(size_t(T.ncl) * T.npp * dim);
            CSFS_CK(cudaMemcpyAsync(q.data(), T.qphi.p, q.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
            CSFS_CK(cudaStreamSynchronize(s));
            to_reference(c->ref_of[0], q, size_t(T.npp) * dim, qphi, true);
        }
        CSFS_CK(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
