// comm.cpp -- a2 halo exchange and a3 Gram allreduce over NCCL (NVLink/NVSwitch).
//
// contiguous row partition (z-slabs of a lexicographic grid);
// each apply sends the rows a neighbour needs and receives this rank's ghost
// rows with grouped ncclSend/ncclRecv on a comm stream, while the interior
// rows (no ghost column) are computed on the compute stream; the boundary
// rows run after the receive event.  Row-major X makes a contiguous send set
// a contiguous slice of X, so slab halos need no packing.  Gram matrices are
// summed in place with ncclAllReduce; every rank receives identical bits, so
// the replicated small-dense stage takes identical decisions on all ranks.
//
// Two transports behind the same calls: NCCL (one process per GPU, the product path) and an
// in-process LOOPBACK hub (bk_local_hub_create / bk_ctx_set_comm_local: several virtual ranks,
// one host thread each, in one process -- e.g. all on one GPU).  The hub exists so the
// multi-rank code (halo plan exchange, interior / boundary split, ghost-row kernels, Gram
// allreduce, the solvers' p > 1 path) runs under the GPU parity tests on a one-GPU box; it moves
// data with device-to-device copies between host barriers and reduces on the device in rank
// order, so no kernel ever waits on another rank's kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "bk_internal.h"

using namespace bk;

namespace bk {
// One posted point-to-point transfer of a grouped exchange.
struct P2POp {
    int peer;
    bool send;
    void* buf;
    size_t bytes;
};

// out[i] = op over ranks q = 0..P-1 (in rank order) of stage[q * n + i]; op 0 sum, 1 max
__global__ void hub_reduce_kernel(const double* __restrict__ stage, double* __restrict__ out, int P, int64_t n,
                                  int op) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double v = stage[i];
        for (int q = 1; q < P; ++q) {
            const double w = stage[(int64_t)q * n + i];
            v = op == 0 ? v + w : (w > v ? w : v);
        }
        out[i] = v;
    }
}

struct LocalHub {
    explicit LocalHub(int p) : P(p), ptr(p, nullptr), ops(p) {}
    const int P;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long gen = 0;
    std::vector<const void*> ptr;            // per rank: buffer posted to the current collective
    std::vector<std::vector<P2POp>> ops;     // per rank: posted point-to-point transfers
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const unsigned long g = gen;
        if (++arrived == P) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};
}  // namespace bk

namespace {

void* grow(bk_buf& b, size_t bytes, cudaStream_t st) {
    if (b.bytes >= bytes && b.p) return b.p;
    if (b.p) {
        cudaStreamSynchronize(st);
        cudaFree(b.p);
        b.p = nullptr;
        b.bytes = 0;
    }
    size_t want = std::max<size_t>(bytes + 256, 4096);
    if (cudaMalloc(&b.p, want) != cudaSuccess) {
        cudaGetLastError();
        throw bk_error(BK_ERR_OOM, "halo buffer allocation failed");
    }
    b.bytes = want;
    return b.p;
}

#ifndef BK_NO_NCCL
int nccl_check(bk_ctx* ctx, ncclResult_t r, const char* where) {
    if (r == ncclSuccess) return BK_OK;
    return set_error(ctx, BK_ERR_NCCL, std::string(where) + ": " + ncclGetErrorString(r));
}
#define NCCL_OK(ctx, call) \
    do { int _r = nccl_check(ctx, (call), #call); if (_r) return _r; } while (0)
#endif

}  // namespace

extern "C" int bk_get_nccl_unique_id(void* out128) {
#ifdef BK_NO_NCCL
    (void)out128;
    return BK_ERR_UNSUPPORTED;
#else
    if (!out128) return BK_ERR_ARG;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    return ncclGetUniqueId((ncclUniqueId*)out128) == ncclSuccess ? BK_OK : BK_ERR_NCCL;
#endif
}

extern "C" int bk_ctx_set_comm(bk_ctx* ctx, const void* uid128, int nranks, int rank) {
    if (!ctx) return BK_ERR_ARG;
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(ctx, BK_ERR_ARG, "bk_ctx_set_comm: bad rank");
    if (nranks == 1) {
        ctx->nranks = 1;
        ctx->rank = 0;
        return BK_OK;
    }
#ifdef BK_NO_NCCL
    return set_error(ctx, BK_ERR_UNSUPPORTED, "built without NCCL");
#else
    if (!uid128) return set_error(ctx, BK_ERR_ARG, "bk_ctx_set_comm: uid is NULL");
    cudaSetDevice(ctx->device);
    ncclUniqueId id;
    memcpy(&id, uid128, sizeof id);
    if (ctx->comm) {
        ncclCommDestroy(ctx->comm);
        ctx->comm = nullptr;
    }
    NCCL_OK(ctx, ncclCommInitRank(&ctx->comm, nranks, id, rank));
    ctx->hub = nullptr;
    ctx->nranks = nranks;
    ctx->rank = rank;
    return BK_OK;
#endif
}

extern "C" int bk_local_hub_create(void** hub, int nranks) {
    if (!hub || nranks < 1 || nranks > 1024) return BK_ERR_ARG;
    *hub = new LocalHub(nranks);
    return BK_OK;
}

extern "C" int bk_local_hub_destroy(void* hub) {
    delete static_cast<LocalHub*>(hub);
    return BK_OK;
}

extern "C" int bk_ctx_set_comm_local(bk_ctx* ctx, void* hub, int rank) {
    if (!ctx) return BK_ERR_ARG;
    LocalHub* h = static_cast<LocalHub*>(hub);
    if (!h || rank < 0 || rank >= h->P) return set_error(ctx, BK_ERR_ARG, "bk_ctx_set_comm_local: bad hub or rank");
#ifndef BK_NO_NCCL
    if (ctx->comm) {
        ncclCommDestroy(ctx->comm);
        ctx->comm = nullptr;
    }
#endif
    ctx->hub = h;
    ctx->nranks = h->P;
    ctx->rank = rank;
    return BK_OK;
}

namespace bk {

namespace {
constexpr int WS_HUB_STAGE = 120;   // workspace slot of the loopback reduction staging
int hub_cuda(bk_ctx* ctx, cudaError_t e, const char* where) { return cuda_check(ctx, e, where); }

// every rank's `send` (bytes each) -> recv[q * bytes ...] on every rank
int hub_allgather(bk_ctx* ctx, const void* send, void* recv, size_t bytes, cudaStream_t st) {
    LocalHub* h = ctx->hub;
    int r = hub_cuda(ctx, cudaStreamSynchronize(st), "hub allgather");
    h->ptr[ctx->rank] = send;
    h->barrier();
    for (int q = 0; q < h->P && !r; ++q)
        r = hub_cuda(ctx, cudaMemcpy((char*)recv + (size_t)q * bytes, h->ptr[q], bytes, cudaMemcpyDefault),
                     "hub allgather copy");
    h->barrier();
    return r;
}

// in-place reduction (0 sum, 1 max) of n doubles, rank order, on the device
int hub_allreduce(bk_ctx* ctx, double* d, int64_t n, int op) {
    LocalHub* h = ctx->hub;
    const int P = h->P;
    int r = hub_cuda(ctx, cudaStreamSynchronize(ctx->stream), "hub allreduce");
    double* stage = (double*)ws_get(ctx, WS_HUB_STAGE, sizeof(double) * (size_t)P * n);
    h->ptr[ctx->rank] = d;
    h->barrier();
    for (int q = 0; q < P && !r; ++q)
        r = hub_cuda(ctx, cudaMemcpy(stage + (int64_t)q * n, h->ptr[q], sizeof(double) * n, cudaMemcpyDefault),
                     "hub allreduce copy");
    h->barrier();   // every rank holds every contribution: d may be overwritten now
    if (!r) {
        const int blocks = (int)std::min<int64_t>((n + 255) / 256, 1024);
        BK_KERNEL(hub_reduce_kernel<<<blocks, 256, 0, ctx->stream>>>(stage, d, P, n, op));
        r = hub_cuda(ctx, cudaGetLastError(), "hub reduce");
    }
    return r;
}

// grouped point-to-point transfers; the n-th send to a peer matches that peer's n-th receive from me
int hub_p2p(bk_ctx* ctx, const std::vector<P2POp>& ops, cudaStream_t st) {
    LocalHub* h = ctx->hub;
    int r = hub_cuda(ctx, cudaStreamSynchronize(st), "hub p2p");
    h->ops[ctx->rank] = ops;
    h->barrier();
    std::vector<int> seen(h->P, 0);
    for (const P2POp& o : ops) {
        if (o.send || r) continue;
        const int nth = seen[o.peer]++;
        int c = 0;
        const P2POp* match = nullptr;
        for (const P2POp& p : h->ops[o.peer])
            if (p.send && p.peer == ctx->rank && c++ == nth) { match = &p; break; }
        if (!match || match->bytes != o.bytes) {
            r = set_error(ctx, BK_ERR_ARG, "hub p2p: unmatched receive");
            break;
        }
        r = hub_cuda(ctx, cudaMemcpy(o.buf, match->buf, o.bytes, cudaMemcpyDefault), "hub p2p copy");
    }
    h->barrier();
    return r;
}
}  // namespace

int allreduce_sum(bk_ctx* ctx, double* d, int64_t n) {
    if (ctx->nranks <= 1 || n == 0) return BK_OK;
    if (ctx->hub) return hub_allreduce(ctx, d, n, 0);
#ifdef BK_NO_NCCL
    (void)d;
    return set_error(ctx, BK_ERR_UNSUPPORTED, "built without NCCL");
#else
    NCCL_OK(ctx, ncclAllReduce(d, d, (size_t)n, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    return BK_OK;
#endif
}

int allreduce_max(bk_ctx* ctx, double* d, int64_t n) {
    if (ctx->nranks <= 1 || n == 0) return BK_OK;
    if (ctx->hub) return hub_allreduce(ctx, d, n, 1);
#ifdef BK_NO_NCCL
    (void)d;
    return set_error(ctx, BK_ERR_UNSUPPORTED, "built without NCCL");
#else
    NCCL_OK(ctx, ncclAllReduce(d, d, (size_t)n, ncclDouble, ncclMax, ctx->comm, ctx->stream));
    return BK_OK;
#endif
}

namespace {
int xport_allgather(bk_ctx* ctx, const void* send, void* recv, size_t bytes, cudaStream_t st) {
    if (ctx->hub) return hub_allgather(ctx, send, recv, bytes, st);
#ifdef BK_NO_NCCL
    (void)send; (void)recv; (void)bytes; (void)st;
    return set_error(ctx, BK_ERR_UNSUPPORTED, "built without NCCL");
#else
    return nccl_check(ctx, ncclAllGather(send, recv, bytes, ncclChar, ctx->comm, st), "allgather");
#endif
}

int xport_p2p(bk_ctx* ctx, const std::vector<P2POp>& ops, cudaStream_t st) {
    if (ctx->hub) return hub_p2p(ctx, ops, st);
#ifdef BK_NO_NCCL
    (void)ops; (void)st;
    return set_error(ctx, BK_ERR_UNSUPPORTED, "built without NCCL");
#else
    NCCL_OK(ctx, ncclGroupStart());
    for (const P2POp& o : ops) {
        if (o.send) ncclSend(o.buf, o.bytes, ncclChar, o.peer, ctx->comm, st);
        else ncclRecv(o.buf, o.bytes, ncclChar, o.peer, ctx->comm, st);
    }
    return nccl_check(ctx, ncclGroupEnd(), "grouped send/recv");
#endif
}
}  // namespace

int csr_setup_comm(bk_ctx* ctx, bk_csr* A, const std::vector<int32_t>& rp, std::vector<int32_t>& col_local,
                   const std::vector<int32_t>& colg) {
    const int P = ctx->nranks, me = ctx->rank;
    cudaStream_t st = ctx->stream;
    // 1. allgather (row_begin, n_local) -> partition bounds
    int64_t* d_pair = nullptr;
    if (cudaMalloc(&d_pair, sizeof(int64_t) * 2 * (P + 1)) != cudaSuccess) return set_error(ctx, BK_ERR_OOM, "oom");
    int64_t mine[2] = {A->row_begin, A->n_local};
    cudaMemcpy(d_pair + 2 * P, mine, sizeof mine, cudaMemcpyHostToDevice);
    int r = xport_allgather(ctx, d_pair + 2 * P, d_pair, 2 * sizeof(int64_t), st);
    std::vector<int64_t> pairs(2 * P);
    cudaStreamSynchronize(st);
    cudaMemcpy(pairs.data(), d_pair, sizeof(int64_t) * 2 * P, cudaMemcpyDeviceToHost);
    cudaFree(d_pair);
    if (r) return r;
    std::vector<int64_t> rb(P + 1);
    for (int q = 0; q < P; ++q) {
        rb[q] = pairs[2 * q];
        if (q > 0 && rb[q] != pairs[2 * (q - 1)] + pairs[2 * (q - 1) + 1])
            return set_error(ctx, BK_ERR_ARG, "bk_csr_create: ranks must own consecutive contiguous row ranges");
    }
    rb[P] = pairs[2 * (P - 1)] + pairs[2 * (P - 1) + 1];
    if (rb[0] != 0 || rb[P] != A->n_global)
        return set_error(ctx, BK_ERR_ARG, "bk_csr_create: row ranges must cover [0, n_global)");
    // 2. host halo plan
    const int64_t nnz = A->nnz, nl = A->n_local;
    std::vector<int64_t> gid(std::max<int64_t>(nnz, 1));
    std::vector<int32_t> gown(std::max<int64_t>(nnz, 1));
    std::vector<uint8_t> bnd(std::max<int64_t>(nl, 1));
    int64_t ng = 0;
    int pr = bk_plan_halo(P, me, rb.data(), nl, rp.data(), colg.data(), nnz, &ng, gid.data(), gown.data(),
                          col_local.data(), bnd.data());
    if (pr) return set_error(ctx, pr, "bk_csr_create: halo plan failed");
    A->n_ghost = ng;
    // 3. exchange request counts: need[q] = #ghost rows owned by q
    std::vector<int64_t> need(P, 0), recv_off(P, 0);
    for (int64_t g = 0; g < ng; ++g) need[gown[g]]++;
    for (int q = 1; q < P; ++q) recv_off[q] = recv_off[q - 1] + need[q - 1];
    int64_t* d_cnt = nullptr;
    cudaMalloc(&d_cnt, sizeof(int64_t) * P * (P + 1));
    cudaMemcpy(d_cnt + (int64_t)P * P, need.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice);
    r = xport_allgather(ctx, d_cnt + (int64_t)P * P, d_cnt, P * sizeof(int64_t), st);
    std::vector<int64_t> cnt((size_t)P * P);
    cudaStreamSynchronize(st);
    cudaMemcpy(cnt.data(), d_cnt, sizeof(int64_t) * P * P, cudaMemcpyDeviceToHost);
    cudaFree(d_cnt);
    if (r) return r;
    // 4. send the requested global ids to their owners, receive what others need from me
    std::vector<int64_t> give(P);
    for (int q = 0; q < P; ++q) give[q] = cnt[(size_t)q * P + me];  // rows rank q needs from me
    int64_t total_give = 0;
    for (int q = 0; q < P; ++q) total_give += give[q];
    int64_t *d_req = nullptr, *d_give = nullptr;
    cudaMalloc(&d_req, sizeof(int64_t) * std::max<int64_t>(ng, 1));
    cudaMalloc(&d_give, sizeof(int64_t) * std::max<int64_t>(total_give, 1));
    if (ng) cudaMemcpy(d_req, gid.data(), sizeof(int64_t) * ng, cudaMemcpyHostToDevice);
    std::vector<int64_t> give_off(P, 0);
    for (int q = 1; q < P; ++q) give_off[q] = give_off[q - 1] + give[q - 1];
    std::vector<P2POp> ops;
    for (int q = 0; q < P; ++q) {
        if (q == me) continue;
        if (need[q]) ops.push_back({q, true, d_req + recv_off[q], sizeof(int64_t) * (size_t)need[q]});
        if (give[q]) ops.push_back({q, false, d_give + give_off[q], sizeof(int64_t) * (size_t)give[q]});
    }
    r = xport_p2p(ctx, ops, st);
    std::vector<int64_t> give_ids(std::max<int64_t>(total_give, 1));
    cudaStreamSynchronize(st);
    if (total_give) cudaMemcpy(give_ids.data(), d_give, sizeof(int64_t) * total_give, cudaMemcpyDeviceToHost);
    cudaFree(d_req);
    cudaFree(d_give);
    if (r) return r;
    // 5. neighbours
    A->nbs.clear();
    A->n_send_total = 0;
    int64_t send_off = 0;
    for (int q = 0; q < P; ++q) {
        if (q == me || (need[q] == 0 && give[q] == 0)) continue;
        bk_neighbor nb;
        nb.rank = q;
        nb.recv_off = recv_off[q];
        nb.recv_cnt = need[q];
        nb.send_cnt = give[q];
        nb.send_off = send_off;
        if (give[q]) {
            std::vector<int32_t> rows(give[q]);
            bool contig = true;
            for (int64_t t = 0; t < give[q]; ++t) {
                const int64_t id = give_ids[give_off[q] + t];
                if (id < A->row_begin || id >= A->row_begin + nl)
                    return set_error(ctx, BK_ERR_ARG, "bk_csr_create: peer requested a row this rank does not own");
                rows[t] = (int32_t)(id - A->row_begin);
                if (t > 0 && rows[t] != rows[t - 1] + 1) contig = false;
            }
            nb.send_contig = contig ? 1 : 0;
            nb.send_begin = rows[0];
            cudaMalloc(&nb.d_send_rows, sizeof(int32_t) * give[q]);
            cudaMemcpy(nb.d_send_rows, rows.data(), sizeof(int32_t) * give[q], cudaMemcpyHostToDevice);
            send_off += give[q];
        }
        A->n_send_total += give[q];
        A->nbs.push_back(nb);
    }
    // 6. interior / boundary row lists
    std::vector<int32_t> inter, bound;
    for (int64_t i = 0; i < nl; ++i) (bnd[i] ? bound : inter).push_back((int32_t)i);
    A->n_boundary = (int64_t)bound.size();
    A->n_interior = (int64_t)inter.size();
    A->interior_contig = 1;
    for (size_t t = 1; t < inter.size(); ++t)
        if (inter[t] != inter[t - 1] + 1) A->interior_contig = 0;
    A->interior_begin = inter.empty() ? 0 : inter[0];
    if (!bound.empty()) {
        cudaMalloc(&A->d_boundary_rows, sizeof(int32_t) * bound.size());
        cudaMemcpy(A->d_boundary_rows, bound.data(), sizeof(int32_t) * bound.size(), cudaMemcpyHostToDevice);
    }
    if (!A->interior_contig) {
        cudaMalloc(&A->d_interior_rows, sizeof(int32_t) * inter.size());
        cudaMemcpy(A->d_interior_rows, inter.data(), sizeof(int32_t) * inter.size(), cudaMemcpyHostToDevice);
    }
    return cuda_check(ctx, cudaGetLastError(), "csr_setup_comm");
}

int halo_exchange(bk_ctx* ctx, const bk_csr* Ac, int k, const double* X, int64_t ldx) {
    bk_csr* A = const_cast<bk_csr*>(Ac);
    cudaStream_t cs = ctx->comm_stream;
    double* ghost = (double*)grow(A->ghost, sizeof(double) * std::max<int64_t>(A->n_ghost, 1) * k, ctx->stream);
    double* sendbuf = (double*)grow(A->sendbuf, sizeof(double) * std::max<int64_t>(A->n_send_total, 1) * k, ctx->stream);
    // X is produced on the compute stream (and the previous apply's boundary rows still read the
    // ghost buffer there): the comm stream waits for it
    cudaEventRecord(ctx->ev_a, ctx->stream);
    cudaStreamWaitEvent(cs, ctx->ev_a, 0);
    for (const auto& nb : A->nbs)
        if (nb.send_cnt && !(nb.send_contig && ldx == k))
            launch_pack_rows(nb.send_cnt, k, nb.d_send_rows, X, ldx, sendbuf + nb.send_off * k, cs);
    std::vector<P2POp> ops;
    for (const auto& nb : A->nbs) {
        if (nb.send_cnt) {
            const double* src = (nb.send_contig && ldx == k) ? X + nb.send_begin * ldx : sendbuf + nb.send_off * k;
            ops.push_back({nb.rank, true, const_cast<double*>(src), sizeof(double) * (size_t)nb.send_cnt * k});
        }
        if (nb.recv_cnt) ops.push_back({nb.rank, false, ghost + nb.recv_off * k, sizeof(double) * (size_t)nb.recv_cnt * k});
    }
    int r = xport_p2p(ctx, ops, cs);
    if (r) return r;
    cudaEventRecord(ctx->ev_b, cs);
    return cuda_check(ctx, cudaGetLastError(), "halo_exchange");
}

}  // namespace bk
