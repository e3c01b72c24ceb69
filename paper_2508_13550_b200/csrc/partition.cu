// Multi-GPU CSFMM: target partitioning by cubed-sphere subtree with the exchanges in
// NCCL.  The reference's parallel CSFMM gives "each MPI rank an equal
// portion of the interactions followed by a global reduction"; its
// serial library is csfmm_sum (/root/reference/proj/src/summation.cpp:383-421).  Here:
//
//   every rank   plan: full trees, lists and work items (replicated; unit-scope symmetric
//                pairs so no pair straddles two ranks), partition units = depth-1
//                subtrees (+ unsplit roots) with their evaluation cost
//                split: one contiguous run of units per rank — targets by cost, sources by
//                particle count (split_contiguous; identical on every rank)
//                upward pass of the OWNED source subtrees, packed into the rank's segment
//   exchange 1   all-gather of the packed proxy weights (grouped ncclBroadcast, one per
//                owner: NCCL's all-gather with per-rank counts), unpacked into the tree
//   every rank   depth-0 proxy weights (redundant), PP/PC/CP/CC of the OWNED targets,
//                downward pass into the tree-order potentials of the owned range
//   exchange 2   all-gather of the owned tree-order potential ranges (in place)
//   every rank   scatter to input order.
//
// Every target is evaluated by exactly one rank in the same order for every rank count,
// so results are bitwise identical across rank counts (tests/test_gpu_partition.py).
//
// Three group kinds share this code (include/csfs_b200.h):
//   Rank      one process per GPU (torchrun): this process's rank, NCCL from a unique id
//   Multi     one process drives N devices (ncclCommInitAll); one host thread per device
//             runs the rank program, rank 0 on the caller's thread
//   Emulated  N ranks on ONE device with device copies instead of NCCL, run phase by
//             phase in lockstep (parity tests of the partition / exchange layout on one
//             GPU; never ranks that wait on each other on one device)
#include <algorithm>
#include <atomic>
#include <cstring>
#include <exception>
#include <thread>

#include "context.hpp"

namespace csfs_b200 {

using capi::count_internal;
using capi::ev_ms;

std::vector<std::pair<int, int>> split_contiguous(const std::vector<double>& costs, int world) {
    const int n = int(costs.size());
    std::vector<double> pre(n + 1, 0.0);
    for (int i = 0; i < n; ++i) pre[i + 1] = pre[i] + costs[i];
    const double total = pre[n];
    std::vector<int> cuts{0};
    for (int k = 1; k < world; ++k) {
        const double goal = total * k / world;
        const int j = int(std::lower_bound(pre.begin(), pre.end(), goal) - pre.begin());
        int best = -1;
        for (int x : {j - 1, j}) {
            if (x < 0 || x > n) continue;
            if (best < 0 || std::abs(pre[x] - goal) < std::abs(pre[best] - goal)) best = x;
        }
        cuts.push_back(std::max(best, cuts.back()));
    }
    cuts.push_back(n);
    std::vector<std::pair<int, int>> runs;
    for (int r = 0; r < world; ++r) runs.push_back({cuts[r], cuts[r + 1]});
    return runs;
}

namespace {

constexpr int kTB = 256;

__global__ void k_pack(const int* __restrict__ idx, long long n, int npp, const double* __restrict__ qw,
                       double* __restrict__ xq) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n * npp) return;
    const long long i = g / npp;
    xq[g] = qw[(long long)idx[i] * npp + (g - i * npp)];
}

// unpack every segment but [skip_b, skip_e) (this rank's own, already in qw)
__global__ void k_unpack(const int* __restrict__ idx, long long n, int npp, long long skip_b, long long skip_e,
                         const double* __restrict__ xq, double* __restrict__ qw) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n * npp) return;
    const long long i = g / npp;
    if (i >= skip_b && i < skip_e) return;
    qw[(long long)idx[i] * npp + (g - i * npp)] = xq[g];
}

// Executed pairwise evaluations of the items and symmetric pairs this rank runs (items
// anchored in [own_b, own_e) or at depth 0, pairs anchored in the range): the work the
// roofline counts.  One warp per item.
__global__ void k_exec_count(const int4* __restrict__ item, int n_items, const int2* __restrict__ seg,
                             const int* __restrict__ anchor, const int4* __restrict__ mpair,
                             const int* __restrict__ manchor, int n_mutual, long long own_b, long long own_e,
                             unsigned long long* out) {
    const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int w = int(gt >> 5), lane = threadIdx.x & 31;
    unsigned long long v = 0;
    if (w < n_items) {
        const int a = anchor[w];
        if (a < 0 || (a >= own_b && a < own_e)) {
            const int4 it = item[w];
            const long long tl = it.y < 0 ? -it.y : it.y;
            long long src = 0;
            for (int e = it.z + lane; e < it.w; e += 32) src += seg_len(seg[e].y);
            v = (unsigned long long)(tl * src);
        }
    }
    if (gt < n_mutual) {
        const int a = manchor[gt];
        if (a >= own_b && a < own_e) {
            const int4 p = mpair[gt];
            v += (unsigned long long)seg_len(p.y) * (unsigned long long)seg_len(p.w);
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0 && v) atomicAdd(out, v);
}

using Ctx = csfs_b200_ctx;

struct Inputs {
    const double *txyz = nullptr, *sxyz = nullptr, *sw = nullptr;
    size_t nt = 0, ns = 0;
};

// Rank r's inputs in Multi mode: rank 0 broadcasts the caller's arrays into the peers'
// staging buffers (NVLink); Rank mode: every process already holds them; Emulated: the
// same device pointers.
Inputs share_inputs(Ctx* c, const Inputs& in0, bool same_xyz, cudaStream_t s) {
    if (c->mode != Ctx::Mode::Multi) return in0;
    Inputs in = in0;
    const size_t nt = in0.nt, ns = in0.ns;
    if (c->rank != 0) {
        c->h_txyz.grow(nt * 3);
        c->h_w.grow(ns);
        in.txyz = c->h_txyz.p;
        in.sw = c->h_w.p;
        if (same_xyz) {
            in.sxyz = in.txyz;
        } else {
            c->h_sxyz.grow(ns * 3);
            in.sxyz = c->h_sxyz.p;
        }
    }
    // the send buffer is read on the root only; the others pass their receive buffer
    CSFS_NCCL(ncclGroupStart());
    CSFS_NCCL(ncclBroadcast(in.txyz, const_cast<double*>(in.txyz), nt * 3, ncclFloat64, 0, c->comm, s));
    if (!same_xyz)
        CSFS_NCCL(ncclBroadcast(in.sxyz, const_cast<double*>(in.sxyz), ns * 3, ncclFloat64, 0, c->comm, s));
    CSFS_NCCL(ncclBroadcast(in.sw, const_cast<double*>(in.sw), ns, ncclFloat64, 0, c->comm, s));
    CSFS_NCCL(ncclGroupEnd());
    return in;
}

}  // namespace

// Exchange order of the proxy weights: the owned source clusters (depth >= 1) of rank 0,
// rank 1, ... (c->xidx on the device, c->xq_off per rank); c->s_range must be set.
void exchange_order(csfs_b200_ctx* c, const DeviceTree& S, cudaStream_t s) {
    const int R = c->nranks;
    std::vector<int> beg(S.ncl), dep(S.ncl);
    CSFS_CK(cudaMemcpyAsync(beg.data(), S.begin.p, S.ncl * sizeof(int), cudaMemcpyDeviceToHost, s));
    CSFS_CK(cudaMemcpyAsync(dep.data(), S.depth.p, S.ncl * sizeof(int), cudaMemcpyDeviceToHost, s));
    CSFS_CK(cudaStreamSynchronize(s));
    // owner of each depth >= 1 cluster (its first particle's rank range), then a counting
    // sort by owner that keeps cluster order inside each rank: O(ncl)
    std::vector<int> owner(S.ncl, -1);
    c->xq_off.assign(R + 1, 0);
    for (int i = 0; i < S.ncl; ++i) {
        if (dep[i] < 1) continue;
        for (int r = 0; r < R; ++r)
            if (beg[i] >= c->s_range[2 * r] && beg[i] < c->s_range[2 * r + 1]) {
                owner[i] = r;
                ++c->xq_off[r + 1];
                break;
            }
    }
    for (int r = 0; r < R; ++r) c->xq_off[r + 1] += c->xq_off[r];
    std::vector<int> idx(size_t(c->xq_off[R]));
    std::vector<long long> at(c->xq_off.begin(), c->xq_off.end() - 1);
    for (int i = 0; i < S.ncl; ++i)
        if (owner[i] >= 0) idx[size_t(at[owner[i]]++)] = i;
    const long long n = (long long)idx.size();
    c->xidx.grow(std::max<long long>(n, 1));
    c->xq.grow(size_t(std::max<long long>(n, 1)) * S.npp);
    if (n) CSFS_CK(cudaMemcpyAsync(c->xidx.p, idx.data(), n * sizeof(int), cudaMemcpyHostToDevice, s));
    CSFS_CK(cudaStreamSynchronize(s));  // idx's lifetime
}

namespace {


// Phase A: plan, split, owned upward pass, own segment packed into xq.
void phase_plan(Ctx* c, const Inputs& in, const KernelSpec& ks, const FmmConfig& f, cudaStream_t s) {
    cudaEvent_t* ev = c->ev;
    CSFS_CK(cudaEventRecord(ev[0], s));
    // the owned upward pass starts inside the plan, under the traversal (part_plan early_upward)
    capi::part_plan(c, in.txyz, in.nt, in.sxyz, in.sw, in.ns, ks, f, s, true);
    CSFS_CK(cudaEventRecord(ev[1], s));
    // c->t_range (the target split) is set by part_plan, which built only our items
    DeviceTree& S = c->shared ? c->ttree : c->stree;
    CSFS_CK(cudaStreamWaitEvent(s, ev[11], 0));  // the owned upward pass (aux)
    // c->xidx / c->xq_off: the exchange order, set by part_plan (exchange_order)
    const long long ob = c->xq_off[c->rank], on = c->xq_off[c->rank + 1] - ob;
    if (on) {
        k_pack<<<ceil_div(on * S.npp, kTB), kTB, 0, s>>>(c->xidx.p + ob, on, S.npp, S.qw.p, c->xq.p + ob * S.npp);
        CSFS_LAUNCH_CHECK();
    }
    CSFS_CK(cudaEventRecord(ev[2], s));
}

// Phase B: unpack the gathered proxy weights, depth-0 proxy weights, owned evaluation and
// downward pass into the tree-order potentials c->phi_tree.
void phase_eval(Ctx* c, cudaStream_t s, bool count_exec) {
    cudaEvent_t* ev = c->ev;
    CSFS_CK(cudaEventRecord(ev[3], s));
    DeviceTree& T = c->ttree;
    DeviceTree& S = c->shared ? c->ttree : c->stree;
    const long long n = c->xq_off[c->nranks];
    if (n) {
        k_unpack<<<ceil_div(n * S.npp, kTB), kTB, 0, s>>>(c->xidx.p, n, S.npp, c->xq_off[c->rank],
                                                          c->xq_off[c->rank + 1], c->xq.p, S.qw.p);
        CSFS_LAUNCH_CHECK();
    }
    upward_pass(S, c->cheb, s, 2);  // depth-0 proxy weights from the gathered depth-1 ones
    const int dim = c->dim;
    const size_t nt = size_t(T.n);
    const Own own{c->t_range[2 * c->rank], c->t_range[2 * c->rank + 1]};
    c->phi_near.grow(nt * dim);
    c->phi_tree.grow(nt * dim);
    T.qphi.grow(size_t(T.ncl) * T.npp * dim);
    CSFS_CK(cudaMemsetAsync(c->phi_near.p, 0, nt * dim * sizeof(double), s));
    CSFS_CK(cudaMemsetAsync(T.qphi.p, 0, size_t(T.ncl) * T.npp * dim * sizeof(double), s));
    if (count_exec) {
        c->xcount.grow(1);
        CSFS_CK(cudaMemsetAsync(c->xcount.p, 0, sizeof(unsigned long long), s));
        const Items& it = c->items;
        const long long nthr = std::max<long long>((long long)it.n_items * 32, it.mutual ? it.n_mutual : 0);
        if (nthr > 0) {
            k_exec_count<<<ceil_div(nthr, kTB), kTB, 0, s>>>(it.item, it.n_items, it.seg, it.anchor, it.mpair,
                                                             it.manchor, it.mutual ? it.n_mutual : 0, own.b, own.e,
                                                             c->xcount.p);
            CSFS_LAUNCH_CHECK();
        }
    }
    c->counter.grow(4);
    interact(c->kspec, T, S, c->items, c->phi_near, c->counter, c->log_tab, s, own);
    CSFS_CK(cudaEventRecord(ev[4], s));
    downward_pass(T, c->cheb, dim, c->phi_near, c->phi_tree, s, own, false);
    CSFS_CK(cudaEventRecord(ev[5], s));
}

// Exchange 2 done: out[perm[t]] = phi_tree[t].
void phase_finish(Ctx* c, double* out, cudaStream_t s) {
    CSFS_CK(cudaEventRecord(c->ev[6], s));
    if (out) scatter_to_input(c->ttree, c->dim, c->phi_tree, out, s);
    CSFS_CK(cudaEventRecord(c->ev[7], s));
}

// All-gather of per-rank segments [off[r], off[r+1]) x unit doubles of buf over NCCL:
// one in-place broadcast per owner, grouped (NCCL's all-gather with per-rank counts).
void nccl_gather_segments(Ctx* c, double* buf, const std::vector<long long>& off, long long unit, cudaStream_t s) {
    CSFS_NCCL(ncclGroupStart());
    for (int r = 0; r < c->nranks; ++r) {
        const long long cnt = (off[r + 1] - off[r]) * unit;
        if (cnt > 0) {
            double* p = buf + off[r] * unit;
            CSFS_NCCL(ncclBroadcast(p, p, size_t(cnt), ncclFloat64, r, c->comm, s));
        }
    }
    CSFS_NCCL(ncclGroupEnd());
}

// Rank r's potentials are the tree-order range [off[r], off[r+1]) (x dim): the owned
// target ranges tile [0, n) in rank order; an empty run is a zero-length segment.
std::vector<long long> phi_offsets(const Ctx* c) {
    std::vector<long long> off(c->nranks + 1, 0);
    long long at = 0;
    for (int r = 0; r < c->nranks; ++r) {
        const long long b = c->t_range[2 * r], e = c->t_range[2 * r + 1];
        off[r] = at;
        if (e > b) {
            if (b != at) throw CudaFailure("partition: owned target ranges are not contiguous");
            at = e;
        }
    }
    off[c->nranks] = at;
    if (at != c->ttree.n) throw CudaFailure("partition: owned target ranges do not cover the targets");
    return off;
}

// The whole rank program for NCCL-connected ranks (Rank / Multi mode).
void rank_program(Ctx* c, const Inputs& in0, bool same_xyz, const KernelSpec& ks, const FmmConfig& f, double* out,
                  cudaStream_t s, bool count_exec) {
    CSFS_CK(cudaSetDevice(c->device));
    const Inputs in = share_inputs(c, in0, same_xyz, s);
    phase_plan(c, in, ks, f, s);
    const int npp = (c->shared ? c->ttree : c->stree).npp;
    nccl_gather_segments(c, c->xq.p, c->xq_off, npp, s);
    phase_eval(c, s, count_exec);
    const std::vector<long long> off = phi_offsets(c);
    nccl_gather_segments(c, c->phi_tree.p, off, c->dim, s);
    phase_finish(c, out, s);
    CSFS_CK(cudaStreamSynchronize(s));
}

// The same all-gather for Emulated ranks on one device: device-to-device copies.
void emulated_gather(const std::vector<double*>& bufs, const std::vector<long long>& off, long long unit,
                     cudaStream_t s) {
    const int R = int(bufs.size());
    for (int r = 0; r < R; ++r) {
        const long long cnt = (off[r + 1] - off[r]) * unit;
        if (cnt <= 0) continue;
        for (int q = 0; q < R; ++q)
            if (q != r)
                CSFS_CK(cudaMemcpyAsync(bufs[q] + off[r] * unit, bufs[r] + off[r] * unit, size_t(cnt) * sizeof(double),
                                        cudaMemcpyDeviceToDevice, s));
    }
}

// Per-rank statistics of the last call into st (rank 0's phases; t_total = max over the
// ranks held by this process; evals summed over them).
void group_stats(Ctx* c, const std::vector<Ctx*>& ranks, const std::vector<unsigned long long>& exec,
                 csfs_b200_stats* st) {
    capi::fill_stats(c, st);  // counts, tree shapes (events 0..5 are re-read below)
    cudaEvent_t* ev = c->ev;
    st->t_tree_build = ev_ms(ev[0], ev[1]) * 1e-3;  // trees + lists + items (replicated plan)
    st->t_lists = 0.0;
    st->t_upward = ev_ms(ev[1], ev[2]) * 1e-3;
    st->t_interact = ev_ms(ev[3], ev[4]) * 1e-3;
    st->t_traversal = ev_ms(ev[3], ev[4]) * 1e-3;
    st->t_downward = ev_ms(ev[4], ev[5]) * 1e-3;
    st->t_exchange = (ev_ms(ev[2], ev[3]) + ev_ms(ev[5], ev[6])) * 1e-3;
    double tmax = 0.0;
    unsigned long long ex = 0;
    for (size_t r = 0; r < ranks.size(); ++r) {
        tmax = std::max(tmax, double(ev_ms(ranks[r]->ev[0], ranks[r]->ev[7])) * 1e-3);
        ex += exec[r];
    }
    st->t_total = tmax;
    st->evals_executed = ex;
    c->rank_phases.clear();
    for (size_t r = 0; r < ranks.size(); ++r) {
        const Ctx* q = ranks[r];
        const cudaEvent_t* e = q->ev;
        const int rk = q->rank;
        const DeviceTree& S = q->shared ? q->ttree : q->stree;
        const double bytes = 8.0 * double(q->xq_off[rk + 1] - q->xq_off[rk]) * S.npp +
                             8.0 * double(q->t_range[2 * rk + 1] - q->t_range[2 * rk]) * q->dim;
        for (double v : {double(ev_ms(e[0], e[1])), double(ev_ms(e[1], e[2])), double(ev_ms(e[3], e[4])),
                         double(ev_ms(e[4], e[5])), double(ev_ms(e[6], e[7])), bytes})
            c->rank_phases.push_back(v);
    }
    st->n_ranks = c->nranks;
    st->symmetric_pairs = c->items.mutual ? c->items.n_mutual : 0;
}

}  // namespace

void run_csfmm_group(Ctx* c, const double* txyz, size_t nt, const double* sxyz, const double* sw, size_t ns,
                     const KernelSpec& ks, const FmmConfig& f, double* out, csfs_b200_stats* st, cudaStream_t s,
                     cudaEvent_t w_ready) {
    capi::validate(f, nt, ns);
    if (w_ready) CSFS_CK(cudaStreamWaitEvent(s, w_ready, 0));
    const bool same_xyz = txyz == sxyz;
    const Inputs in0{txyz, sxyz, sw, nt, ns};
    const bool count_exec = st != nullptr;
    std::vector<Ctx*> ranks{c};
    for (auto& p : c->peers) ranks.push_back(p.get());
    std::vector<unsigned long long> exec(ranks.size(), 0);
    c->have_state = false;

    if (c->mode == Ctx::Mode::Emulated) {
        // lockstep on one device: every rank's phase, then the exchange as device copies
        const int R = int(ranks.size());
        for (Ctx* r : ranks) phase_plan(r, in0, ks, f, s);
        CSFS_CK(cudaStreamSynchronize(s));
        std::vector<double*> xq;
        for (Ctx* r : ranks) xq.push_back(r->xq.p);
        const int npp = (c->shared ? c->ttree : c->stree).npp;
        emulated_gather(xq, c->xq_off, npp, s);
        for (Ctx* r : ranks) phase_eval(r, s, count_exec);
        const std::vector<long long> off = phi_offsets(c);
        std::vector<double*> phi;
        for (Ctx* r : ranks) phi.push_back(r->phi_tree.p);
        emulated_gather(phi, off, c->dim, s);
        for (int r = 0; r < R; ++r) phase_finish(ranks[r], r == 0 ? out : nullptr, s);
        CSFS_CK(cudaStreamSynchronize(s));
    } else if (c->mode == Ctx::Mode::Rank) {
        rank_program(c, in0, same_xyz, ks, f, out, s, count_exec);
    } else {  // Multi: one host thread per device; rank 0 here on the caller's stream
        std::vector<std::exception_ptr> errs(ranks.size());
        std::vector<std::thread> th;
        std::atomic<bool> aborted{false};
        // a rank that fails would leave the others waiting inside an all-gather forever:
        // the first failure aborts every communicator, which unblocks them with an NCCL
        // error (the group is unusable afterwards; csfs_b200.h)
        auto fail_all = [&] {
            if (aborted.exchange(true)) return;
            for (Ctx* r : ranks)
                if (r->comm) ncclCommAbort(r->comm);
            for (Ctx* r : ranks) r->comm = nullptr;
        };
        for (size_t r = 1; r < ranks.size(); ++r)
            th.emplace_back([&, r] {
                try {
                    rank_program(ranks[r], in0, same_xyz, ks, f, nullptr, ranks[r]->own, count_exec);
                } catch (...) {
                    errs[r] = std::current_exception();
                    fail_all();
                }
            });
        try {
            rank_program(c, in0, same_xyz, ks, f, out, s, count_exec);
        } catch (...) {
            errs[0] = std::current_exception();
            fail_all();
        }
        for (auto& t : th) t.join();
        CSFS_CK(cudaSetDevice(c->device));
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    }
    if (count_exec)
        for (size_t r = 0; r < ranks.size(); ++r) {
            CSFS_CK(cudaSetDevice(ranks[r]->device));
            CSFS_CK(cudaMemcpy(&exec[r], ranks[r]->xcount.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        }
    CSFS_CK(cudaSetDevice(c->device));
    c->have_state = true;
    c->t_exchange = 0.0;
    if (st) {
        group_stats(c, ranks, exec, st);
        c->t_exchange = st->t_exchange;
    }
}

}  // namespace csfs_b200

using namespace csfs_b200;
using namespace csfs_b200::capi;

extern "C" {

int csfs_b200_nccl_unique_id(unsigned char* id) {
    if (!id) return CSFS_B200_INVALID_ARGUMENT;
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) return CSFS_B200_NCCL_ERROR;
    static_assert(sizeof(u.internal) == CSFS_B200_NCCL_ID_BYTES, "NCCL unique id size");
    std::memcpy(id, u.internal, CSFS_B200_NCCL_ID_BYTES);
    return CSFS_B200_OK;
}

int csfs_b200_create_rank(csfs_b200_ctx** out, int device, int nranks, int rank, const unsigned char* id) {
    if (!out) return CSFS_B200_INVALID_ARGUMENT;
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks || !id) return CSFS_B200_INVALID_ARGUMENT;
    std::unique_ptr<Ctx> c;
    try {
        c = new_context(device);
    } catch (const InvalidArgument&) {
        return CSFS_B200_INVALID_ARGUMENT;
    } catch (const std::exception&) {
        return CSFS_B200_CUDA_ERROR;
    }
    ncclUniqueId u;
    std::memcpy(u.internal, id, CSFS_B200_NCCL_ID_BYTES);
    if (cudaSetDevice(device) != cudaSuccess) return CSFS_B200_CUDA_ERROR;  // no exception across the C boundary
    if (ncclCommInitRank(&c->comm, nranks, u, rank) != ncclSuccess) return CSFS_B200_NCCL_ERROR;
    c->mode = Ctx::Mode::Rank;
    c->nranks = nranks;
    c->rank = rank;
    *out = c.release();
    return CSFS_B200_OK;
}

int csfs_b200_create_multi(csfs_b200_ctx** out, int num_gpus, const int* device_ids) {
    if (!out) return CSFS_B200_INVALID_ARGUMENT;
    *out = nullptr;
    if (num_gpus < 1) return CSFS_B200_INVALID_ARGUMENT;
    std::vector<int> dev(num_gpus);
    for (int i = 0; i < num_gpus; ++i) dev[i] = device_ids ? device_ids[i] : i;
    for (int i = 0; i < num_gpus; ++i)
        for (int j = 0; j < i; ++j)
            if (dev[i] == dev[j]) return CSFS_B200_INVALID_ARGUMENT;  // one rank per device
    std::vector<std::unique_ptr<Ctx>> cs;
    try {
        for (int d : dev) cs.push_back(new_context(d));
    } catch (const InvalidArgument&) {
        return CSFS_B200_INVALID_ARGUMENT;
    } catch (const std::exception&) {
        return CSFS_B200_CUDA_ERROR;
    }
    std::vector<ncclComm_t> comms(num_gpus);
    if (ncclCommInitAll(comms.data(), num_gpus, dev.data()) != ncclSuccess) return CSFS_B200_NCCL_ERROR;
    for (int i = 0; i < num_gpus; ++i) {
        cs[i]->mode = Ctx::Mode::Multi;
        cs[i]->nranks = num_gpus;
        cs[i]->rank = i;
        cs[i]->comm = comms[i];
    }
    std::unique_ptr<Ctx> root = std::move(cs[0]);
    for (int i = 1; i < num_gpus; ++i) root->peers.push_back(std::move(cs[i]));
    *out = root.release();
    return CSFS_B200_OK;
}

int csfs_b200_create_emulated(csfs_b200_ctx** out, int device, int nranks) {
    if (!out) return CSFS_B200_INVALID_ARGUMENT;
    *out = nullptr;
    if (nranks < 1) return CSFS_B200_INVALID_ARGUMENT;
    std::vector<std::unique_ptr<Ctx>> cs;
    try {
        for (int i = 0; i < nranks; ++i) cs.push_back(new_context(device));
    } catch (const InvalidArgument&) {
        return CSFS_B200_INVALID_ARGUMENT;
    } catch (const std::exception&) {
        return CSFS_B200_CUDA_ERROR;
    }
    for (int i = 0; i < nranks; ++i) {
        cs[i]->mode = Ctx::Mode::Emulated;
        cs[i]->nranks = nranks;
        cs[i]->rank = i;
    }
    std::unique_ptr<Ctx> root = std::move(cs[0]);
    for (int i = 1; i < nranks; ++i) root->peers.push_back(std::move(cs[i]));
    *out = root.release();
    return CSFS_B200_OK;
}

int csfs_b200_group_phases(const csfs_b200_ctx* c, double* out, int cap, int* n) {
    if (!c) return CSFS_B200_INVALID_ARGUMENT;
    if (n) *n = int(c->rank_phases.size());
    for (int i = 0; i < std::min<int>(cap, int(c->rank_phases.size())); ++i) out[i] = c->rank_phases[i];
    return CSFS_B200_OK;
}

int csfs_b200_group_info(const csfs_b200_ctx* c, int* nranks, int* rank, int* devices, long long* t_ranges,
                         long long* s_ranges) {
    if (!c) return CSFS_B200_INVALID_ARGUMENT;
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
    if (devices) {
        devices[0] = c->device;
        for (size_t i = 0; i < c->peers.size(); ++i) devices[i + 1] = c->peers[i]->device;
    }
    if (c->mode != Ctx::Mode::Single && (t_ranges || s_ranges)) {
        if (c->t_range.size() != size_t(2 * c->nranks)) return CSFS_B200_INVALID_ARGUMENT;  // no call yet
        for (int i = 0; i < 2 * c->nranks; ++i) {
            if (t_ranges) t_ranges[i] = c->t_range[i];
            if (s_ranges) s_ranges[i] = c->s_range[i];
        }
    }
    return CSFS_B200_OK;
}

}  // extern "C"
