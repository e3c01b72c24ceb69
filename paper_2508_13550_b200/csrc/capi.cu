// C-ABI of the B200 CSFMM (include/csfs_b200.h) and the orchestration that replaces
// csfs::csfmm_sum (/root/reference/proj/src/summation.cpp:383-421):
//   tree build (targets, sources) -> upward pass -> dual traversal -> PP/PC/CP/CC
//   -> downward pass, every phase a device kernel on the context's stream, phase times
//   from CUDA events (the reference's steady_clock SumStats, summation.cpp:407-419).
// There is no CPU fallback: without a usable sm_100a device every call fails.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <thread>
#include <memory>
#include <string>
#include <vector>

#include "context.hpp"

using namespace csfs_b200;

namespace csfs_b200 {
namespace capi {

namespace {
int fail(csfs_b200_ctx* c, int code, const std::string& m) {
    if (c) c->err = m;
    return code;
}
}  // namespace

int guarded_call(csfs_b200_ctx* c, void (*f)(void*), void* arg) {
    if (!c) return CSFS_B200_INVALID_ARGUMENT;
    try {
        CSFS_CK(cudaSetDevice(c->device));
        f(arg);
        c->err.clear();
        return CSFS_B200_OK;
    } catch (const InvalidArgument& e) {
        return fail(c, CSFS_B200_INVALID_ARGUMENT, e.what());
    } catch (const OutOfMemory& e) {
        return fail(c, CSFS_B200_OUT_OF_MEMORY, e.what());
    } catch (const NcclFailure& e) {
        return fail(c, CSFS_B200_NCCL_ERROR, e.what());
    } catch (const CudaFailure& e) {
        return fail(c, CSFS_B200_CUDA_ERROR, e.what());
    } catch (const std::exception& e) {
        return fail(c, CSFS_B200_CUDA_ERROR, e.what());
    }
}

void rethrow(csfs_b200_ctx* c, int rc) {
    if (rc == CSFS_B200_OK) return;
    if (rc == CSFS_B200_INVALID_ARGUMENT) throw InvalidArgument(c->err);
    if (rc == CSFS_B200_OUT_OF_MEMORY) throw OutOfMemory(c->err);
    if (rc == CSFS_B200_NCCL_ERROR) throw NcclFailure(c->err);
    throw CudaFailure(c->err);
}

KernelSpec to_spec(const csfs_b200_kernel* k) {
    if (!k) throw InvalidArgument("kernel must not be null");
    if (k->kind < 0 || k->kind > 3) throw InvalidArgument("unknown kernel kind: " + std::to_string(k->kind));
    KernelSpec s;
    s.kind = k->kind;
    s.a1 = k->a1;
    s.b0 = k->b0;
    s.b1 = k->b1;
    s.rho_ratio = k->rho_ratio;
    return s;
}

FmmConfig to_cfg(const csfs_b200_config* c) {
    if (!c) throw InvalidArgument("config must not be null");
    FmmConfig f;
    f.mac = c->mac;
    f.degree = c->degree;
    f.n0 = c->n0;
    f.shrink = c->shrink != 0;
    return f;
}

void validate(const FmmConfig& f, size_t nt, size_t ns) {
    if (f.degree < 1) throw InvalidArgument("interpolation degree must be positive");
    if (f.degree > kMaxNp - 1)
        throw InvalidArgument("interpolation degree above " + std::to_string(kMaxNp - 1) +
                              " is not supported by the B200 engine");
    if (nt == 0 || ns == 0) throw InvalidArgument("cannot build a cluster tree from an empty particle set");
    if (f.resolved_n0() < 1) throw InvalidArgument("maximum leaf size must be at least 1");
    if (nt > 0x3fffffff || ns > 0x3fffffff) throw InvalidArgument("particle count exceeds 2^30");
}

Cheb make_cheb(int degree) {
    // ChebyshevGrid1D (interpolation.cpp:14-24), same libm call on the host.
    Cheb c{};
    c.np = degree + 1;
    for (int k = 0; k <= degree; ++k) {
        c.nodes[k] = std::cos(k * kPi / degree);
        c.weights[k] = (k % 2 == 0) ? 1.0 : -1.0;
    }
    c.weights[0] *= 0.5;
    c.weights[degree] *= 0.5;
    return c;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    CSFS_CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

int count_internal(const DeviceTree& t) {
    std::vector<int> nch(t.ncl);
    CSFS_CK(cudaMemcpy(nch.data(), t.nchild.p, t.ncl * sizeof(int), cudaMemcpyDeviceToHost));
    int k = 0;
    for (int v : nch) k += v > 0;
    return k;
}

std::unique_ptr<csfs_b200_ctx> new_context(int device) {
    auto c = std::make_unique<csfs_b200_ctx>();
    c->device = device;
    int count = 0;
    CSFS_CK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw InvalidArgument("no CUDA device " + std::to_string(device));
    cudaDeviceProp prop{};
    CSFS_CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        throw CudaFailure("csfs_b200 is built for sm_100a; device " + std::to_string(device) + " is sm_" +
                          std::to_string(prop.major) + std::to_string(prop.minor));
    CSFS_CK(cudaSetDevice(device));
    CSFS_CK(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    {
        // the upward pass runs on `aux` under the list phase, which runs on `hi`: the
        // latency-bound list kernels (the critical path) get the SMs first.  (The least
        // priority is also the default one, so `aux` alone could not rank below the caller's
        // stream.)
        int lo = 0, hi = 0;
        CSFS_CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CSFS_CK(cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, lo));
        CSFS_CK(cudaStreamCreateWithPriority(&c->hi, cudaStreamNonBlocking, hi));
    }
    CSFS_CK(cudaEventCreateWithFlags(&c->w_copied, cudaEventDisableTiming));
    for (auto& e : c->ev) CSFS_CK(cudaEventCreate(&e));
    CSFS_CK(cudaMallocHost(&c->sc.host, kHostInts * sizeof(int)));
    const char* nosym = std::getenv("CSFS_B200_NO_SYMMETRIC");
    c->use_mutual = !(nosym && nosym[0] == '1');
    const char* scope = std::getenv("CSFS_B200_MUTUAL_SCOPE");
    c->mutual_unit_scope = scope && std::string(scope) == "unit";
    std::vector<double2> tab(kLogTabWords);
    make_log_table(tab.data());
    c->log_tab.grow(kLogTabWords);
    CSFS_CK(cudaMemcpy(c->log_tab.p, tab.data(), kLogTabWords * sizeof(double2), cudaMemcpyHostToDevice));
    return c;
}

void free_context(csfs_b200_ctx* c) {
    if (!c) return;
    for (auto& p : c->peers) {
        free_context(p.get());
        p.release();
    }
    cudaSetDevice(c->device);
    if (c->own) cudaStreamSynchronize(c->own);
    if (c->aux) cudaStreamSynchronize(c->aux);
    if (c->hi) cudaStreamSynchronize(c->hi);
    if (c->comm) ncclCommDestroy(c->comm);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->sc.host) cudaFreeHost(c->sc.host);
    for (int b = 0; b < 2; ++b) {
        if (c->stage_pin[b]) cudaFreeHost(c->stage_pin[b]);
        if (c->stage_ev[b]) cudaEventDestroy(c->stage_ev[b]);
    }
    if (c->own) cudaStreamDestroy(c->own);
    if (c->aux) cudaStreamDestroy(c->aux);
    if (c->hi) cudaStreamDestroy(c->hi);
    if (c->w_copied) cudaEventDestroy(c->w_copied);
    delete c;
}

namespace {

// Symmetric PP/CC pairs (k_mutual).  Scope: one GPU pairs every mirrored leaf pair
// (`global`); the partitioned multi-GPU path restricts them to pairs inside one partition
// unit, so no pair straddles two ranks and every rank count sums in the same order
// (results bitwise equal across rank counts; equal to the single-GPU result to rounding).
void prepare_mutual(csfs_b200_ctx* c, cudaStream_t s, bool global) {
    c->items.mutual = false;
    if (!c->shared || !c->use_mutual || c->kspec.out_dim() != 1) return;
    std::vector<long long> ub, ue;
    if (global && !c->mutual_unit_scope) ub.push_back(0);
    else partition_units(c->ttree, ub, ue, s);
    build_mutual(c->ttree, c->items, ub, c->sc, s);
    c->items.mutual = c->items.n_partial > 0;
}

}  // namespace

// Stats of the last run_csfmm from c->ev[0..5] (tree, upward on aux, lists, interact,
// downward); the partitioned path overwrites the phase times it measures itself.
void fill_stats(csfs_b200_ctx* c, csfs_b200_stats* st) {
    cudaEvent_t* ev = c->ev;
    const DeviceTree& T = c->ttree;
    const DeviceTree& S = c->shared ? c->ttree : c->stree;
    std::memset(st, 0, sizeof(*st));
    st->t_tree_build = ev_ms(ev[0], ev[1]) * 1e-3;
    // upward and lists overlap (both start at ev[1]); the reference's phases are
    // sequential, so here tree + upward + traversal + downward >= total
    st->t_upward = ev_ms(ev[1], ev[2]) * 1e-3;
    st->t_traversal = ev_ms(ev[1], ev[4]) * 1e-3;
    st->t_lists = ev_ms(ev[1], ev[3]) * 1e-3;
    st->t_interact = ev_ms(ev[3], ev[4]) * 1e-3;
    st->t_downward = ev_ms(ev[4], ev[5]) * 1e-3;
    st->t_total = ev_ms(ev[0], ev[5]) * 1e-3;
    st->pp = c->lists.n[0];
    st->pc = c->lists.n[1];
    st->cp = c->lists.n[2];
    st->cc = c->lists.n[3];
    st->evals_pp = c->items.pair_evals[0];
    st->evals_pc = c->items.pair_evals[1];
    st->evals_cp = c->items.pair_evals[2];
    st->evals_cc = c->items.pair_evals[3];
    st->evals_executed = c->items.pair_evals[0] + c->items.pair_evals[1] + c->items.pair_evals[2] +
                         c->items.pair_evals[3] - (c->items.mutual ? c->items.skipped_pairs : 0);
    st->symmetric_pairs = c->items.mutual ? c->items.n_mutual : 0;
    st->tgt_depth = T.depth_max();
    st->tgt_clusters = T.ncl;
    st->tgt_leaves = T.ncl - count_internal(T);
    st->src_depth = S.depth_max();
    st->src_clusters = S.ncl;
    st->src_leaves = c->shared ? st->tgt_leaves : S.ncl - count_internal(S);
    st->shared_tree = c->shared ? 1 : 0;
    st->n_ranks = 1;
    st->traversal_fallback = c->lists.fallback ? 1 : 0;
    st->symmetric_partials = c->items.mutual ? (uint64_t)c->items.n_partial : 0;
}

// w_ready: optional event the weights' producer records (the host API copies them on
// the aux stream while the tree levels are built).
void run_csfmm(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz,
               const double* sw, size_t ns, const KernelSpec& ks, const FmmConfig& f, double* out,
               csfs_b200_stats* st, cudaStream_t s, cudaEvent_t w_ready) {
    validate(f, nt, ns);
    c->have_state = false;
    c->have_src_tree = false;
    c->have_tree = false;
    c->ref_of[0].clear();
    c->ref_of[1].clear();
    c->part_planned = false;
    c->kspec = ks;
    c->cfg = f;
    c->dim = ks.out_dim();
    c->cheb = make_cheb(f.degree);
    const int n0 = f.resolved_n0();
    cudaEvent_t* ev = c->ev;

    CSFS_CK(cudaEventRecord(ev[0], s));
    c->shared = (nt == ns) && device_equal(txyz, sxyz, nt * 3 * sizeof(double), c->sc, s);
    DeviceTree& T = c->ttree;
    DeviceTree& S = c->shared ? c->ttree : c->stree;
    build_tree(T, c->sc, txyz, c->shared ? sw : nullptr, (long long)nt, f.degree, n0, f.shrink,
               c->cheb, s, w_ready);
    if (!c->shared) build_tree(S, c->sc, sxyz, sw, (long long)ns, f.degree, n0, f.shrink, c->cheb, s, w_ready);
    CSFS_CK(cudaEventRecord(ev[1], s));

    // the upward pass (weights -> proxy weights) and the dual traversal (geometry -> lists)
    // are independent: the upward pass runs on the aux stream meanwhile
    static const bool serial_up = std::getenv("CSFS_B200_TRACE_SERIAL_UPWARD") != nullptr;
    CSFS_CK(cudaStreamWaitEvent(c->aux, ev[1], 0));
    upward_pass(S, c->cheb, serial_up ? s : c->aux);
    CSFS_CK(cudaEventRecord(ev[2], serial_up ? s : c->aux));
    if (serial_up) CSFS_CK(cudaEventRecord(ev[1], s));

    static const bool trace = std::getenv("CSFS_B200_TRACE_LISTS") != nullptr;
    cudaStream_t ls = c->hi;  // the list phase, forked from s at ev[1] and joined at ev[3]
    CSFS_CK(cudaStreamWaitEvent(ls, ev[1], 0));
    dual_traversal(T, S, f.mac, n0, c->lists, c->sc, ls);
    if (trace) CSFS_CK(cudaEventRecord(ev[8], ls));
    build_items(T, S, c->lists, c->items, c->sc, ls);
    if (trace) CSFS_CK(cudaEventRecord(ev[9], ls));
    prepare_mutual(c, ls, true);
    CSFS_CK(cudaEventRecord(ev[3], ls));
    CSFS_CK(cudaStreamWaitEvent(s, ev[3], 0));
    if (trace) {
        CSFS_CK(cudaEventSynchronize(ev[3]));
        fprintf(stderr, "lists: traversal %.3f items %.3f mutual %.3f ms\n", ev_ms(ev[1], ev[8]), ev_ms(ev[8], ev[9]),
                ev_ms(ev[9], ev[3]));
    }
    CSFS_CK(cudaStreamWaitEvent(s, ev[2], 0));

    const int dim = c->dim;
    c->phi_near.grow(nt * dim);
    T.qphi.grow(size_t(T.ncl) * T.npp * dim);
    CSFS_CK(cudaMemsetAsync(c->phi_near.p, 0, nt * dim * sizeof(double), s));
    CSFS_CK(cudaMemsetAsync(T.qphi.p, 0, size_t(T.ncl) * T.npp * dim * sizeof(double), s));
    c->counter.grow(4);
    interact(ks, T, S, c->items, c->phi_near, c->counter, c->log_tab, s, Own{0, (long long)nt});
    CSFS_CK(cudaEventRecord(ev[4], s));

    downward_pass(T, c->cheb, dim, c->phi_near, out, s, Own{0, (long long)nt}, true);
    CSFS_CK(cudaEventRecord(ev[5], s));
    CSFS_CK(cudaEventSynchronize(ev[5]));
    c->have_state = true;
    if (st) fill_stats(c, st);
}

void part_plan(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz, const double* sw, size_t ns,
               const KernelSpec& ks, const FmmConfig& f, cudaStream_t s, bool early_upward) {
    validate(f, nt, ns);
    c->have_state = false;
    c->have_src_tree = false;
    c->have_tree = false;
    c->ref_of[0].clear();
    c->ref_of[1].clear();
    c->part_planned = false;
    c->part_stream = s;
    c->kspec = ks;
    c->cfg = f;
    c->dim = ks.out_dim();
    c->cheb = make_cheb(f.degree);
    const int n0 = f.resolved_n0();
    static const bool trace = std::getenv("CSFS_B200_TRACE_PLAN") != nullptr;
    std::vector<std::pair<const char*, double>> marks;
    auto mark = [&](const char* what) {
        if (!trace) return;
        CSFS_CK(cudaDeviceSynchronize());
        marks.push_back({what, std::chrono::duration<double, std::milli>(
                                   std::chrono::steady_clock::now().time_since_epoch()).count()});
    };
    mark("start");
    c->shared = (nt == ns) && device_equal(txyz, sxyz, nt * 3 * sizeof(double), c->sc, s);
    DeviceTree& T = c->ttree;
    DeviceTree& S = c->shared ? c->ttree : c->stree;
    build_tree(T, c->sc, txyz, c->shared ? sw : nullptr, (long long)nt, f.degree, n0, f.shrink, c->cheb, s);
    if (!c->shared) build_tree(S, c->sc, sxyz, sw, (long long)ns, f.degree, n0, f.shrink, c->cheb, s);
    mark("trees");
    // partition units: depth-1 subtrees plus unsplit roots, in tree order
    for (int w = 0; w < 2; ++w) {
        const DeviceTree& t = (w == 0 || c->shared) ? T : S;
        partition_units(t, c->unit_b[w], c->unit_e[w], s);
        c->unit_cost[w].assign(c->unit_b[w].size(), 0.0);
        if (w == 1)
            for (size_t i = 0; i < c->unit_b[1].size(); ++i)
                c->unit_cost[1][i] = double(c->unit_e[1][i] - c->unit_b[1][i]);
    }
    if (early_upward) {  // sources split by particle count: known now
        const int R = c->nranks;
        const auto srun = split_contiguous(c->unit_cost[1], R);
        c->s_range.assign(2 * R, 0);
        for (int r = 0; r < R; ++r)
            if (srun[r].second > srun[r].first) {
                c->s_range[2 * r] = c->unit_b[1][srun[r].first];
                c->s_range[2 * r + 1] = c->unit_e[1][srun[r].second - 1];
            }
        CSFS_CK(cudaEventRecord(c->ev[10], s));
        CSFS_CK(cudaStreamWaitEvent(c->aux, c->ev[10], 0));
        upward_pass(S, c->cheb, c->aux, 1, Own{c->s_range[2 * c->rank], c->s_range[2 * c->rank + 1]});
        CSFS_CK(cudaEventRecord(c->ev[11], c->aux));
        exchange_order(c, S, s);  // host work while the upward pass runs
    }
    mark("units+upward+order");
    // the list phase on the greatest-priority stream (as in run_csfmm)
    cudaStream_t ls = c->hi;
    CSFS_CK(cudaEventRecord(c->ev[10], s));
    CSFS_CK(cudaStreamWaitEvent(ls, c->ev[10], 0));
    dual_traversal(T, S, f.mac, n0, c->lists, c->sc, ls);
    mark("traversal");
    // target units' costs: the pair evaluations of their list entries, summed on the device
    // in exact integer arithmetic (every rank must derive the same split)
    const int nu = int(c->unit_b[0].size());
    c->ubeg.grow(std::max(nu, 1));
    c->ucost.grow(std::max(nu, 1));
    CSFS_CK(cudaMemcpyAsync(c->ubeg.p, c->unit_b[0].data(), nu * sizeof(long long), cudaMemcpyHostToDevice, ls));
    CSFS_CK(cudaMemsetAsync(c->ucost.p, 0, std::max(nu, 1) * sizeof(unsigned long long), ls));
    list_unit_costs(T, S, c->lists, c->ubeg.p, nu, c->ucost.p, ls);
    {
        std::vector<unsigned long long> uc(std::max(nu, 1));
        CSFS_CK(cudaMemcpyAsync(uc.data(), c->ucost.p, std::max(nu, 1) * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, ls));
        CSFS_CK(cudaStreamSynchronize(ls));
        for (int u = 0; u < nu; ++u) c->unit_cost[0][u] = double(uc[u]);
    }
    mark("costs");
    if (early_upward) {  // the group rank program: the target split now, and only our items
        const int R = c->nranks;
        const auto trun = split_contiguous(c->unit_cost[0], R);
        c->t_range.assign(2 * R, 0);
        for (int r = 0; r < R; ++r)
            if (trun[r].second > trun[r].first) {
                c->t_range[2 * r] = c->unit_b[0][trun[r].first];
                c->t_range[2 * r + 1] = c->unit_e[0][trun[r].second - 1];
            }
        const long long ob = c->t_range[2 * c->rank], oe = c->t_range[2 * c->rank + 1];
        const long long n = (long long)T.n;
        build_items(T, S, c->lists, c->items, c->sc, ls, oe > ob ? ob : n, oe > ob ? oe : n);
    } else {
        build_items(T, S, c->lists, c->items, c->sc, ls);
    }
    mark("items");
    prepare_mutual(c, ls, false);  // unit scope: the same pairs for every rank count
    mark("mutual");
    CSFS_CK(cudaEventRecord(c->ev[10], ls));  // the lists are ready for work on s
    CSFS_CK(cudaStreamWaitEvent(s, c->ev[10], 0));
    if (trace) {
        for (size_t i = 1; i < marks.size(); ++i)
            fprintf(stderr, "plan %s %.3f ms\n", marks[i].first, marks[i].second - marks[i - 1].second);
    }
    c->part_planned = true;
}

}  // namespace capi
}  // namespace csfs_b200

using namespace csfs_b200::capi;

namespace {

// Device-pointer entry points run on the caller's stream; NULL is CUDA's legacy default
// stream (what torch reports as cuda_stream == 0), never a private stream, so work stays
// ordered with the caller's producers and consumers.
cudaStream_t pick(csfs_b200_ctx*, void* stream) { return static_cast<cudaStream_t>(stream); }

// csfmm on a context: one device, or the partitioned evaluation over its group.
void csfmm_any(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz, const double* sw, size_t ns,
               const KernelSpec& ks, const FmmConfig& f, double* out, csfs_b200_stats* st, cudaStream_t s,
               cudaEvent_t w_ready = nullptr) {
    if (c->mode == csfs_b200_ctx::Mode::Single) run_csfmm(c, txyz, nt, sxyz, sw, ns, ks, f, out, st, s, w_ready);
    else run_csfmm_group(c, txyz, nt, sxyz, sw, ns, ks, f, out, st, s, w_ready);
}

struct HostTree {
    std::vector<int> face, depth, begin, end, parent, nchild, ref, inv;
    std::vector<int4> child;
};

HostTree fetch_topology(const DeviceTree& t, const std::vector<int>* ref_of = nullptr) {
    HostTree h;
    const int n = t.ncl;
    auto get = [&](std::vector<int>& v, const int* p) {
        v.resize(n);
        CSFS_CK(cudaMemcpy(v.data(), p, n * sizeof(int), cudaMemcpyDeviceToHost));
    };
    get(h.face, t.face);
    get(h.depth, t.depth);
    get(h.begin, t.begin);
    get(h.end, t.end);
    get(h.parent, t.parent);
    get(h.nchild, t.nchild);
    h.child.resize(n);
    CSFS_CK(cudaMemcpy(h.child.data(), t.child.p, n * sizeof(int4), cudaMemcpyDeviceToHost));
    h.ref = (ref_of && !ref_of->empty()) ? *ref_of : reference_ids(h.parent, h.depth, h.child, h.nchild);
    h.inv.assign(n, -1);
    for (int i = 0; i < n; ++i) h.inv[h.ref[i]] = i;
    return h;
}

const DeviceTree& which_tree(const csfs_b200_ctx* c, int which) {
    if (which != 0 && which != 1) throw InvalidArgument("which must be 0 (target) or 1 (source)");
    if (c->have_src_tree && which == 1) return c->stree;  // after cstc
    if (c->have_tree && which == 0) return c->ttree;      // after tree_build
    if (!c->have_state) throw InvalidArgument("no csfmm state: call csfs_b200_csfmm first");
    return (which == 0 || c->shared) ? c->ttree : c->stree;
}

}  // namespace

namespace {

// ---- pageable caller buffers ---------------------------------------------------------------
// cudaMemcpyAsync from / to pageable memory goes through the driver's staging buffer with a
// single-threaded copy (~12 GB/s here: 251 MB of C5 inputs and results cost 17 ms more than
// from pinned memory).  The host-pointer csfmm stages such buffers itself: a few host threads
// copy 32 MB pieces into / out of two pinned bounce buffers while the DMA of the previous piece
// runs.  Pinned or registered caller memory, small buffers and CSFS_B200_NO_STAGE=1 take the
// plain cudaMemcpyAsync.  (Page-locking the caller's memory per call is slower than either:
// INTEGRATION.md.)
constexpr size_t kStageBytes = size_t(32) << 20;
constexpr size_t kStageMin = size_t(48) << 20;  // smaller buffers gain nothing (measured: 9 MB slower, 38 MB even)

bool host_pageable(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

void par_memcpy(char* dst, const char* src, size_t bytes) {
    static const int nthr = [] {
        const unsigned h = std::thread::hardware_concurrency();
        return int(std::max(1u, std::min(8u, h / 2)));
    }();
    const size_t per = (bytes / size_t(nthr) + 4095) & ~size_t(4095);
    if (nthr == 1 || per == 0 || bytes < (size_t(2) << 20)) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 1; t < nthr; ++t) {
        const size_t off = size_t(t) * per;
        if (off >= bytes) break;
        const size_t n = std::min(per, bytes - off);
        th.emplace_back([=] { std::memcpy(dst + off, src + off, n); });
    }
    std::memcpy(dst, src, std::min(per, bytes));
    for (auto& t : th) t.join();
}

bool stage_ready(csfs_b200_ctx* c) {
    for (int b = 0; b < 2; ++b) {
        if (!c->stage_pin[b] && cudaHostAlloc(&c->stage_pin[b], kStageBytes, cudaHostAllocDefault) != cudaSuccess) {
            (void)cudaGetLastError();
            c->stage_pin[b] = nullptr;
            return false;
        }
        if (!c->stage_ev[b] && cudaEventCreateWithFlags(&c->stage_ev[b], cudaEventDisableTiming) != cudaSuccess) {
            (void)cudaGetLastError();
            c->stage_ev[b] = nullptr;
            return false;
        }
    }
    return true;
}

bool want_stage(csfs_b200_ctx* c, const void* host, size_t bytes) {
    static const bool off = std::getenv("CSFS_B200_NO_STAGE") != nullptr;
    return !off && bytes >= kStageMin && host_pageable(host) && stage_ready(c);
}

// host -> device on `s`; returns once the host buffer has been read (the DMA may still run)
void h2d_staged(csfs_b200_ctx* c, double* dst, const double* src, size_t bytes, cudaStream_t s) {
    if (!want_stage(c, src, bytes)) {
        CSFS_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    int b = 0;
    for (size_t done = 0; done < bytes; b ^= 1) {
        const size_t n = std::min(kStageBytes, bytes - done);
        CSFS_CK(cudaEventSynchronize(c->stage_ev[b]));  // the DMA that last used this buffer
        par_memcpy(static_cast<char*>(c->stage_pin[b]), reinterpret_cast<const char*>(src) + done, n);
        CSFS_CK(cudaMemcpyAsync(reinterpret_cast<char*>(dst) + done, c->stage_pin[b], n, cudaMemcpyHostToDevice, s));
        CSFS_CK(cudaEventRecord(c->stage_ev[b], s));
        done += n;
    }
}

// device -> host on `s`; returns with the data in `dst` when it was staged (else the caller
// synchronizes `s` as before)
void d2h_staged(csfs_b200_ctx* c, double* dst, const double* src, size_t bytes, cudaStream_t s) {
    if (!want_stage(c, dst, bytes)) {
        CSFS_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        return;
    }
    auto issue = [&](size_t off, int b) {
        const size_t n = std::min(kStageBytes, bytes - off);
        CSFS_CK(cudaEventSynchronize(c->stage_ev[b]));
        CSFS_CK(cudaMemcpyAsync(c->stage_pin[b], reinterpret_cast<const char*>(src) + off, n, cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaEventRecord(c->stage_ev[b], s));
    };
    issue(0, 0);
    int b = 0;
    for (size_t off = 0; off < bytes; off += kStageBytes, b ^= 1) {
        if (off + kStageBytes < bytes) issue(off + kStageBytes, b ^ 1);  // the next piece flies meanwhile
        CSFS_CK(cudaEventSynchronize(c->stage_ev[b]));
        par_memcpy(reinterpret_cast<char*>(dst) + off, static_cast<const char*>(c->stage_pin[b]),
                   std::min(kStageBytes, bytes - off));
    }
}

}  // namespace

extern "C" {

int csfs_b200_create(csfs_b200_ctx** out, int device) {
    if (!out) return CSFS_B200_INVALID_ARGUMENT;
    *out = nullptr;
    try {
        *out = new_context(device).release();
        return CSFS_B200_OK;
    } catch (const InvalidArgument&) {
        return CSFS_B200_INVALID_ARGUMENT;
    } catch (const OutOfMemory&) {
        return CSFS_B200_OUT_OF_MEMORY;
    } catch (const std::exception&) {
        return CSFS_B200_CUDA_ERROR;
    }
}

void csfs_b200_destroy(csfs_b200_ctx* c) { free_context(c); }

const char* csfs_b200_last_error(const csfs_b200_ctx* c) { return c ? c->err.c_str() : "null context"; }

int csfs_b200_csfmm_device(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz,
                           const double* sw, size_t ns, const csfs_b200_kernel* k,
                           const csfs_b200_config* cfg, double* out, csfs_b200_stats* st,
                           void* stream) {
    return guarded(c, [&] {
        csfmm_any(c, txyz, nt, sxyz, sw, ns, to_spec(k), to_cfg(cfg), out, st, pick(c, stream));
    });
}

int csfs_b200_csfmm(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz,
                    const double* sw, size_t ns, const csfs_b200_kernel* k,
                    const csfs_b200_config* cfg, double* out, csfs_b200_stats* st) {
    return guarded(c, [&] {
        const KernelSpec ks = to_spec(k);
        const FmmConfig f = to_cfg(cfg);
        validate(f, nt, ns);
        cudaStream_t s = c->own;
        const bool same = (txyz == sxyz && nt == ns);
        c->h_txyz.grow(nt * 3);
        h2d_staged(c, c->h_txyz.p, txyz, nt * 3 * sizeof(double), s);
        const double* dsrc = c->h_txyz.p;
        if (!same) {
            c->h_sxyz.grow(ns * 3);
            h2d_staged(c, c->h_sxyz.p, sxyz, ns * 3 * sizeof(double), s);
            dsrc = c->h_sxyz.p;
        }
        c->h_w.grow(ns);
        // the weights are first needed after the tree levels: copy them on the aux stream
        // while the positions' tree is built — after the positions, which the build needs
        // first (two concurrent host-to-device copies share the PCIe link and would delay
        // the positions by the weights' transfer time)
        CSFS_CK(cudaEventRecord(c->ev[10], s));
        CSFS_CK(cudaStreamWaitEvent(c->aux, c->ev[10], 0));
        h2d_staged(c, c->h_w.p, sw, ns * sizeof(double), c->aux);
        CSFS_CK(cudaEventRecord(c->w_copied, c->aux));
        const size_t nout = nt * size_t(ks.out_dim());
        c->h_out.grow(nout);
        csfmm_any(c, c->h_txyz.p, nt, dsrc, c->h_w.p, ns, ks, f, c->h_out.p, st, s, c->w_copied);
        d2h_staged(c, out, c->h_out.p, nout * sizeof(double), s);
        CSFS_CK(cudaStreamSynchronize(s));
    });
}

int csfs_b200_direct_device(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz,
                            const double* sw, size_t ns, const csfs_b200_kernel* k, double* out,
                            void* stream) {
    return guarded(c, [&] {
        const KernelSpec ks = to_spec(k);
        c->counter.grow(4);
        direct_allpairs(ks, txyz, (long long)nt, sxyz, sw, (long long)ns, out, c->d_soa, c->d_items,
                        c->d_segs, c->counter, c->log_tab, pick(c, stream));
    });
}

int csfs_b200_direct(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz,
                     const double* sw, size_t ns, const csfs_b200_kernel* k, double* out) {
    return guarded(c, [&] {
        const KernelSpec ks = to_spec(k);
        cudaStream_t s = c->own;
        c->h_txyz.grow(std::max<size_t>(nt * 3, 1));
        c->h_sxyz.grow(std::max<size_t>(ns * 3, 1));
        c->h_w.grow(std::max<size_t>(ns, 1));
        const size_t nout = nt * size_t(ks.out_dim());
        c->h_out.grow(std::max<size_t>(nout, 1));
        if (nt) CSFS_CK(cudaMemcpyAsync(c->h_txyz.p, txyz, nt * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
        if (ns) {
            CSFS_CK(cudaMemcpyAsync(c->h_sxyz.p, sxyz, ns * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
            CSFS_CK(cudaMemcpyAsync(c->h_w.p, sw, ns * sizeof(double), cudaMemcpyHostToDevice, s));
        }
        if (nout) CSFS_CK(cudaMemsetAsync(c->h_out.p, 0, nout * sizeof(double), s));
        c->counter.grow(4);
        direct_allpairs(ks, c->h_txyz.p, (long long)nt, c->h_sxyz.p, c->h_w.p, (long long)ns, c->h_out.p,
                        c->d_soa, c->d_items, c->d_segs, c->counter, c->log_tab, s);
        if (nout) CSFS_CK(cudaMemcpyAsync(out, c->h_out.p, nout * sizeof(double), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaStreamSynchronize(s));
    });
}

int csfs_b200_tree_info(const csfs_b200_ctx* c, int which, int* ncl, int* depth, size_t* n, int* npp) {
    if (!c) return CSFS_B200_INVALID_ARGUMENT;
    const bool src_only = c->have_src_tree && which == 1;
    const bool tree_only = c->have_tree && which == 0;
    if ((!c->have_state && !src_only && !tree_only) || (which != 0 && which != 1)) return CSFS_B200_INVALID_ARGUMENT;
    const DeviceTree& t = src_only ? c->stree : tree_only ? c->ttree : (which == 0 || c->shared) ? c->ttree : c->stree;
    if (ncl) *ncl = t.ncl;
    if (depth) *depth = t.depth_max();
    if (n) *n = size_t(t.n);
    if (npp) *npp = t.npp;
    return CSFS_B200_OK;
}

int csfs_b200_tree_export(csfs_b200_ctx* c, int which, int* perm, int* ints, double* dbls, double* proxy) {
    return guarded(c, [&] {
        const DeviceTree& t = which_tree(c, which);
        const HostTree h = fetch_topology(t, &c->ref_of[(&t == &c->stree) ? 1 : 0]);
        const int n = t.ncl;
        if (perm) CSFS_CK(cudaMemcpy(perm, t.perm.p, t.n * sizeof(int), cudaMemcpyDeviceToHost));
        if (ints) {
            for (int i = 0; i < n; ++i) {
                int* r = ints + 10 * h.ref[i];
                r[0] = h.face[i];
                r[1] = h.begin[i];
                r[2] = h.end[i];
                r[3] = h.parent[i] < 0 ? -1 : h.ref[h.parent[i]];
                r[4] = h.depth[i];
                r[5] = h.nchild[i];
                const int cs[4] = {h.child[i].x, h.child[i].y, h.child[i].z, h.child[i].w};
                for (int q = 0; q < 4; ++q) r[6 + q] = (q < h.nchild[i]) ? h.ref[cs[q]] : -1;
            }
        }
        if (dbls) {
            const double* src[8] = {t.xi0, t.xi1, t.eta0, t.eta1, t.cx, t.cy, t.cz, t.rad};
            std::vector<double> col(n);
            for (int f = 0; f < 8; ++f) {
                CSFS_CK(cudaMemcpy(col.data(), src[f], n * sizeof(double), cudaMemcpyDeviceToHost));
                for (int i = 0; i < n; ++i) dbls[8 * h.ref[i] + f] = col[i];
            }
        }
        if (proxy) {
            const size_t nq = size_t(n) * t.npp;
            std::vector<double> q[3];
            const double* src[3] = {t.qx, t.qy, t.qz};
            for (int f = 0; f < 3; ++f) {
                q[f].resize(nq);
                CSFS_CK(cudaMemcpy(q[f].data(), src[f], nq * sizeof(double), cudaMemcpyDeviceToHost));
            }
            for (int i = 0; i < n; ++i)
                for (int k = 0; k < t.npp; ++k)
                    for (int f = 0; f < 3; ++f)
                        proxy[(size_t(h.ref[i]) * t.npp + k) * 3 + f] = q[f][size_t(i) * t.npp + k];
        }
    });
}

int csfs_b200_leaf_histogram(csfs_b200_ctx* c, int which, int* hist, int cap, int* len) {
    return guarded(c, [&] {
        const DeviceTree& t = which_tree(c, which);
        std::vector<int> b(t.ncl), e(t.ncl), nch(t.ncl);
        CSFS_CK(cudaMemcpy(b.data(), t.begin.p, t.ncl * sizeof(int), cudaMemcpyDeviceToHost));
        CSFS_CK(cudaMemcpy(e.data(), t.end.p, t.ncl * sizeof(int), cudaMemcpyDeviceToHost));
        CSFS_CK(cudaMemcpy(nch.data(), t.nchild.p, t.ncl * sizeof(int), cudaMemcpyDeviceToHost));
        std::vector<int> h;
        for (int i = 0; i < t.ncl; ++i) {
            if (nch[i] > 0) continue;
            const int n = e[i] - b[i];
            if (int(h.size()) <= n) h.resize(n + 1, 0);
            ++h[n];
        }
        if (len) *len = int(h.size());
        for (int i = 0; i < std::min<int>(cap, int(h.size())); ++i) hist[i] = h[i];
    });
}

int csfs_b200_lists_export(csfs_b200_ctx* c, long long* counts, int* pp, int* pc, int* cp, int* cc) {
    return guarded(c, [&] {
        if (!c->have_state) throw InvalidArgument("no csfmm state: call csfs_b200_csfmm first");
        const HostTree ht = fetch_topology(c->ttree, &c->ref_of[0]);
        const HostTree hs = c->shared ? ht : fetch_topology(c->stree, &c->ref_of[1]);
        int* outs[4] = {pp, pc, cp, cc};
        for (int k = 0; k < 4; ++k) {
            if (counts) counts[k] = c->lists.n[k];
            if (!outs[k]) continue;
            std::vector<int2> v(c->lists.n[k]);
            if (!v.empty())
                CSFS_CK(cudaMemcpy(v.data(), c->lists.l[k].p, v.size() * sizeof(int2), cudaMemcpyDeviceToHost));
            std::vector<std::pair<int, int>> r(v.size());
            for (size_t e = 0; e < v.size(); ++e) r[e] = {ht.ref[v[e].x], hs.ref[v[e].y]};
            std::sort(r.begin(), r.end());
            for (size_t e = 0; e < r.size(); ++e) {
                outs[k][2 * e] = r[e].first;
                outs[k][2 * e + 1] = r[e].second;
            }
        }
    });
}

int csfs_b200_proxy_weights_export(csfs_b200_ctx* c, double* pw) {
    return guarded(c, [&] {
        const DeviceTree& s = which_tree(c, 1);
        const HostTree h = fetch_topology(s, &c->ref_of[(&s == &c->stree) ? 1 : 0]);
        const size_t nq = size_t(s.ncl) * s.npp;
        std::vector<double> q(nq);
        CSFS_CK(cudaMemcpy(q.data(), s.qw.p, nq * sizeof(double), cudaMemcpyDeviceToHost));
        for (int i = 0; i < s.ncl; ++i)
            std::memcpy(pw + size_t(h.ref[i]) * s.npp, q.data() + size_t(i) * s.npp, s.npp * sizeof(double));
    });
}

// --- CSTC treecode (cstc_sum, summation.cpp:308-381) ---------------------------------------

int csfs_b200_cstc_device(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz, const double* sw,
                          size_t ns, const csfs_b200_kernel* k, const csfs_b200_config* cfg, double* out,
                          csfs_b200_stats* st, void* stream) {
    return guarded(c, [&] {
        const KernelSpec ks = to_spec(k);
        const FmmConfig f = to_cfg(cfg);
        // the reference builds only the source tree (its checks: degree, empty set, n0)
        if (f.degree < 1) throw InvalidArgument("interpolation degree must be positive");
        if (f.degree > kMaxNp - 1)
            throw InvalidArgument("interpolation degree above " + std::to_string(kMaxNp - 1) +
                                  " is not supported by the B200 engine");
        if (ns == 0) throw InvalidArgument("cannot build a cluster tree from an empty particle set");
        if (f.resolved_n0() < 1) throw InvalidArgument("maximum leaf size must be at least 1");
        cudaStream_t s = pick(c, stream);
        c->have_state = false;
        c->have_src_tree = false;
        c->have_tree = false;
        c->ref_of[0].clear();
        c->ref_of[1].clear();
        c->cheb = make_cheb(f.degree);
        const int n0 = f.resolved_n0();
        cudaEvent_t* ev = c->ev;
        CSFS_CK(cudaEventRecord(ev[0], s));
        const bool same = (nt == ns) && device_equal(txyz, sxyz, nt * 3 * sizeof(double), c->sc, s);
        DeviceTree& S = c->stree;
        build_tree(S, c->sc, sxyz, sw, (long long)ns, f.degree, n0, f.shrink, c->cheb, s);
        CSFS_CK(cudaEventRecord(ev[1], s));
        upward_pass(S, c->cheb, s);
        CSFS_CK(cudaEventRecord(ev[2], s));
        c->items.pairs.grow(8);
        cstc_eval(ks, txyz, (long long)nt, same ? S.perm.p : nullptr, S, f.mac, n0, c->log_tab, out,
                  c->items.pairs.p + 6, s);
        CSFS_CK(cudaEventRecord(ev[3], s));
        unsigned long long cnt[2] = {0, 0};
        CSFS_CK(cudaMemcpyAsync(cnt, c->items.pairs.p + 6, sizeof(cnt), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaEventSynchronize(ev[3]));
        CSFS_CK(cudaStreamSynchronize(s));
        c->have_src_tree = true;
        if (st) {
            std::memset(st, 0, sizeof(*st));
            st->t_tree_build = ev_ms(ev[0], ev[1]) * 1e-3;
            st->t_upward = ev_ms(ev[1], ev[2]) * 1e-3;
            st->t_traversal = st->t_interact = ev_ms(ev[2], ev[3]) * 1e-3;
            st->t_total = ev_ms(ev[0], ev[3]) * 1e-3;
            st->pp = cnt[0];
            st->pc = cnt[1];
            st->src_depth = S.depth_max();
            st->src_clusters = S.ncl;
            st->src_leaves = S.ncl - count_internal(S);
        }
    });
}

int csfs_b200_cstc(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz, const double* sw,
                   size_t ns, const csfs_b200_kernel* k, const csfs_b200_config* cfg, double* out,
                   csfs_b200_stats* st) {
    return guarded(c, [&] {
        const KernelSpec ks = to_spec(k);
        cudaStream_t s = c->own;
        const bool same = (txyz == sxyz && nt == ns);
        c->h_txyz.grow(std::max<size_t>(nt * 3, 1));
        if (nt) CSFS_CK(cudaMemcpyAsync(c->h_txyz.p, txyz, nt * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
        const double* dsrc = c->h_txyz.p;
        if (!same) {
            c->h_sxyz.grow(std::max<size_t>(ns * 3, 1));
            if (ns) CSFS_CK(cudaMemcpyAsync(c->h_sxyz.p, sxyz, ns * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
            dsrc = c->h_sxyz.p;
        }
        c->h_w.grow(std::max<size_t>(ns, 1));
        if (ns) CSFS_CK(cudaMemcpyAsync(c->h_w.p, sw, ns * sizeof(double), cudaMemcpyHostToDevice, s));
        const size_t nout = nt * size_t(ks.out_dim());
        c->h_out.grow(std::max<size_t>(nout, 1));
        const int rc = csfs_b200_cstc_device(c, c->h_txyz.p, nt, dsrc, c->h_w.p, ns, k, cfg, c->h_out.p, st, s);
        if (rc == CSFS_B200_INVALID_ARGUMENT) throw InvalidArgument(c->err);
        rethrow(c, rc);
        if (nout) CSFS_CK(cudaMemcpyAsync(out, c->h_out.p, nout * sizeof(double), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaStreamSynchronize(s));
    });
}

// --- BVE RK4 step (applications.cpp:378-412, remesh off) ---------------------------------

int csfs_b200_bve_step_device(csfs_b200_ctx* c, double* xyz, double* zeta, const double* areas, size_t n,
                              double omega, double dt, const csfs_b200_config* cfg,
                              csfs_b200_stats* stage_stats, void* stream) {
    return guarded(c, [&] {
        if (dt <= 0.0) throw InvalidArgument("time step must be positive");
        const FmmConfig f = to_cfg(cfg);
        validate(f, n, n);
        cudaStream_t s = pick(c, stream);
        KernelSpec ks;
        ks.kind = 2;  // Biot-Savart (biot_savart_velocity, applications.cpp:181-196)
        const long long N = (long long)n;
        c->bve.grow(size_t(N) * 17);
        double* k[4];  // stage velocities, n x 3 each
        for (int q = 0; q < 4; ++q) k[q] = c->bve.p + size_t(N) * 3 * q;
        double* pos = c->bve.p + size_t(N) * 12;  // stage positions
        double* zs = pos + size_t(N) * 3;         // stage vorticity
        double* w = zs + N;                       // stage weights zeta * area
        const double* x0 = xyz;  // xyz and zeta keep the step's initial state until bve_final
        bve_weights(N, zeta, areas, w, s);
        const double hs[3] = {0.5 * dt, 0.5 * dt, dt};
        for (int q = 0; q < 4; ++q) {
            const double* P = q == 0 ? x0 : pos;
            csfmm_any(c, P, n, P, w, n, ks, f, k[q], stage_stats ? stage_stats + q : nullptr, s);
            if (q < 3) bve_advance(N, x0, zeta, k[q], hs[q], omega, areas, pos, zs, w, s);
        }
        bve_final(N, xyz, zeta, k[0], k[1], k[2], k[3], dt, omega, s);
        CSFS_CK(cudaStreamSynchronize(s));
    });
}

int csfs_b200_bve_step(csfs_b200_ctx* c, double* xyz, double* zeta, const double* areas, size_t n, double omega,
                       double dt, const csfs_b200_config* cfg, csfs_b200_stats* stage_stats) {
    return guarded(c, [&] {
        if (dt <= 0.0) throw InvalidArgument("time step must be positive");
        validate(to_cfg(cfg), n, n);
        cudaStream_t s = c->own;
        c->h_txyz.grow(n * 3);
        c->h_w.grow(n);
        c->h_out.grow(n);
        CSFS_CK(cudaMemcpyAsync(c->h_txyz.p, xyz, n * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
        CSFS_CK(cudaMemcpyAsync(c->h_w.p, zeta, n * sizeof(double), cudaMemcpyHostToDevice, s));
        CSFS_CK(cudaMemcpyAsync(c->h_out.p, areas, n * sizeof(double), cudaMemcpyHostToDevice, s));
        const int rc = csfs_b200_bve_step_device(c, c->h_txyz.p, c->h_w.p, c->h_out.p, n, omega, dt, cfg,
                                                 stage_stats, s);
        rethrow(c, rc);
        CSFS_CK(cudaMemcpyAsync(xyz, c->h_txyz.p, n * 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaMemcpyAsync(zeta, c->h_w.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaStreamSynchronize(s));
    });
}

// --- BVE remesh (applications.cpp:329-371) -----------------------------------------------

namespace {
void check_remesh(int neighbors) {
    if (neighbors > kRemeshMaxK)
        throw InvalidArgument("remesh_neighbors above " + std::to_string(kRemeshMaxK) + " is not supported");
}
}  // namespace

int csfs_b200_bve_remesh_device(csfs_b200_ctx* c, double* xyz, double* zeta, double* tracer,
                                const double* grid_xyz, size_t n, int neighbors, void* stream) {
    return guarded(c, [&] {
        check_remesh(neighbors);
        cudaStream_t s = pick(c, stream);
        bve_remesh(xyz, zeta, tracer, grid_xyz, (long long)n, neighbors, c->rm_i, c->rm_d, s);
        CSFS_CK(cudaStreamSynchronize(s));
    });
}

int csfs_b200_bve_remesh(csfs_b200_ctx* c, double* xyz, double* zeta, double* tracer, const double* grid_xyz,
                         size_t n, int neighbors) {
    return guarded(c, [&] {
        check_remesh(neighbors);
        if (n == 0) return;
        cudaStream_t s = c->own;
        c->rm_h.grow(n * (tracer ? 8 : 7));
        double* dx = c->rm_h.p;
        double* dg = dx + 3 * n;
        double* dz = dg + 3 * n;
        double* dt = tracer ? dz + n : nullptr;
        CSFS_CK(cudaMemcpyAsync(dx, xyz, n * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
        CSFS_CK(cudaMemcpyAsync(dg, grid_xyz, n * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
        CSFS_CK(cudaMemcpyAsync(dz, zeta, n * sizeof(double), cudaMemcpyHostToDevice, s));
        if (tracer) CSFS_CK(cudaMemcpyAsync(dt, tracer, n * sizeof(double), cudaMemcpyHostToDevice, s));
        bve_remesh(dx, dz, dt, dg, (long long)n, neighbors, c->rm_i, c->rm_d, s);
        CSFS_CK(cudaMemcpyAsync(xyz, dx, n * 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaMemcpyAsync(zeta, dz, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        if (tracer) CSFS_CK(cudaMemcpyAsync(tracer, dt, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaStreamSynchronize(s));
    });
}

// --- multi-GPU target partitioning ------------------------------------------------------

int csfs_b200_part_plan(csfs_b200_ctx* c, const double* txyz, size_t nt, const double* sxyz,
                        const double* sw, size_t ns, const csfs_b200_kernel* k,
                        const csfs_b200_config* cfg, void* stream) {
    return guarded(c, [&] { part_plan(c, txyz, nt, sxyz, sw, ns, to_spec(k), to_cfg(cfg), pick(c, stream)); });
}

int csfs_b200_part_units(csfs_b200_ctx* c, int which, int* n_units, long long* begin, long long* end,
                         double* cost) {
    return guarded(c, [&] {
        if (!c->part_planned) throw InvalidArgument("call csfs_b200_part_plan first");
        if (which != 0 && which != 1) throw InvalidArgument("which must be 0 (target) or 1 (source)");
        const size_t n = c->unit_b[which].size();
        if (n_units) *n_units = int(n);
        for (size_t i = 0; i < n; ++i) {
            if (begin) begin[i] = c->unit_b[which][i];
            if (end) end[i] = c->unit_e[which][i];
            if (cost) cost[i] = c->unit_cost[which][i];
        }
    });
}

int csfs_b200_part_sizes(csfs_b200_ctx* c, size_t* n_pw, size_t* n_phi) {
    return guarded(c, [&] {
        if (!c->part_planned) throw InvalidArgument("call csfs_b200_part_plan first");
        const DeviceTree& S = c->shared ? c->ttree : c->stree;
        if (n_pw) *n_pw = size_t(S.ncl) * S.npp;
        if (n_phi) *n_phi = size_t(c->ttree.n) * c->dim;
    });
}

int csfs_b200_part_upward(csfs_b200_ctx* c, long long src_b, long long src_e, double* pw) {
    return guarded(c, [&] {
        if (!c->part_planned) throw InvalidArgument("call csfs_b200_part_plan first");
        DeviceTree& S = c->shared ? c->ttree : c->stree;
        upward_pass(S, c->cheb, c->part_stream, 1, Own{src_b, src_e});
        CSFS_CK(cudaMemcpyAsync(pw, S.qw.p, size_t(S.ncl) * S.npp * sizeof(double), cudaMemcpyDeviceToDevice,
                                c->part_stream));
    });
}

int csfs_b200_part_eval(csfs_b200_ctx* c, long long tgt_b, long long tgt_e, const double* pw_reduced,
                        double* phi) {
    return guarded(c, [&] {
        if (!c->part_planned) throw InvalidArgument("call csfs_b200_part_plan first");
        cudaStream_t s = c->part_stream;
        DeviceTree& T = c->ttree;
        DeviceTree& S = c->shared ? c->ttree : c->stree;
        CSFS_CK(cudaMemcpyAsync(S.qw.p, pw_reduced, size_t(S.ncl) * S.npp * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
        upward_pass(S, c->cheb, s, 2);  // depth-0 proxy weights, from the reduced depth-1 ones
        const int dim = c->dim;
        const size_t nt = size_t(T.n);
        c->phi_near.grow(nt * dim);
        T.qphi.grow(size_t(T.ncl) * T.npp * dim);
        CSFS_CK(cudaMemsetAsync(c->phi_near.p, 0, nt * dim * sizeof(double), s));
        CSFS_CK(cudaMemsetAsync(phi, 0, nt * dim * sizeof(double), s));
        CSFS_CK(cudaMemsetAsync(T.qphi.p, 0, size_t(T.ncl) * T.npp * dim * sizeof(double), s));
        c->counter.grow(4);
        interact(c->kspec, T, S, c->items, c->phi_near, c->counter, c->log_tab, s, Own{tgt_b, tgt_e});
        downward_pass(T, c->cheb, dim, c->phi_near, phi, s, Own{tgt_b, tgt_e}, false);
    });
}

int csfs_b200_part_finish(csfs_b200_ctx* c, const double* phi_reduced, double* out) {
    return guarded(c, [&] {
        if (!c->part_planned) throw InvalidArgument("call csfs_b200_part_plan first");
        scatter_to_input(c->ttree, c->dim, phi_reduced, out, c->part_stream);
        CSFS_CK(cudaStreamSynchronize(c->part_stream));
        c->have_state = true;
    });
}

int csfs_b200_eval_pairs(csfs_b200_ctx* c, const csfs_b200_kernel* k, const double* x, const double* y,
                         size_t n, double* out) {
    return guarded(c, [&] {
        const KernelSpec ks = to_spec(k);
        DevBuf<double> d;
        d.grow(std::max<size_t>(n * 9, 1));
        cudaStream_t s = c->own;
        const size_t nout = n * ks.out_dim();
        if (n) {
            CSFS_CK(cudaMemcpyAsync(d.p, x, n * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
            CSFS_CK(cudaMemcpyAsync(d.p + 3 * n, y, n * 3 * sizeof(double), cudaMemcpyHostToDevice, s));
        }
        eval_pairs(ks, d.p, d.p + 3 * n, (long long)n, d.p + 6 * n, c->log_tab, s);
        if (n) CSFS_CK(cudaMemcpyAsync(out, d.p + 6 * n, nout * sizeof(double), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaStreamSynchronize(s));
    });
}

int csfs_b200_eval_math(csfs_b200_ctx* c, int fn, const double* x, size_t n, double* out) {
    return guarded(c, [&] {
        if (fn < 0 || fn > 3) throw InvalidArgument("fn must be 0 (log), 1 (rsqrt), 2 (rcp) or 3 (dilog)");
        DevBuf<double> d;
        d.grow(std::max<size_t>(2 * n, 1));
        cudaStream_t s = c->own;
        if (n) CSFS_CK(cudaMemcpyAsync(d.p, x, n * sizeof(double), cudaMemcpyHostToDevice, s));
        eval_math(fn, d.p, (long long)n, d.p + n, c->log_tab, s);
        if (n) CSFS_CK(cudaMemcpyAsync(out, d.p + n, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CSFS_CK(cudaStreamSynchronize(s));
    });
}

uint64_t csfs_b200_kernel_launches(void) { return launch_counter(); }

int csfs_b200_probe_fp64(csfs_b200_ctx* c, double* tflops) {
    return guarded(c, [&] { *tflops = probe_fp64_tflops(c->own); });
}

}  // extern "C"
