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
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "bk_internal.h"

using namespace bk;

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
    ctx->nranks = nranks;
    ctx->rank = rank;
    return BK_OK;
#endif
}

namespace bk {

int allreduce_sum(bk_ctx* ctx, double* d, int64_t n) {
#ifdef BK_NO_NCCL
    (void)d; (void)n;
    return set_error(ctx, BK_ERR_UNSUPPORTED, "built without NCCL");
#else
    if (ctx->nranks <= 1 || n == 0) return BK_OK;
    NCCL_OK(ctx, ncclAllReduce(d, d, (size_t)n, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    return BK_OK;
#endif
}

int allreduce_max(bk_ctx* ctx, double* d, int64_t n) {
#ifdef BK_NO_NCCL
    (void)d; (void)n;
    return ctx->nranks <= 1 ? BK_OK : set_error(ctx, BK_ERR_UNSUPPORTED, "built without NCCL");
#else
    if (ctx->nranks <= 1 || n == 0) return BK_OK;
    NCCL_OK(ctx, ncclAllReduce(d, d, (size_t)n, ncclDouble, ncclMax, ctx->comm, ctx->stream));
    return BK_OK;
#endif
}

int csr_setup_comm(bk_ctx* ctx, bk_csr* A, const std::vector<int32_t>& rp, std::vector<int32_t>& col_local,
                   const std::vector<int32_t>& colg) {
#ifdef BK_NO_NCCL
    (void)A; (void)rp; (void)col_local; (void)colg;
    return set_error(ctx, BK_ERR_UNSUPPORTED, "built without NCCL");
#else
    const int P = ctx->nranks, me = ctx->rank;
    cudaStream_t st = ctx->stream;
    // 1. allgather (row_begin, n_local) -> partition bounds
    int64_t* d_pair = nullptr;
    if (cudaMalloc(&d_pair, sizeof(int64_t) * 2 * (P + 1)) != cudaSuccess) return set_error(ctx, BK_ERR_OOM, "oom");
    int64_t mine[2] = {A->row_begin, A->n_local};
    cudaMemcpy(d_pair + 2 * P, mine, sizeof mine, cudaMemcpyHostToDevice);
    int r = nccl_check(ctx, ncclAllGather(d_pair + 2 * P, d_pair, 2, ncclInt64, ctx->comm, st), "allgather ranges");
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
    r = nccl_check(ctx, ncclAllGather(d_cnt + (int64_t)P * P, d_cnt, P, ncclInt64, ctx->comm, st), "allgather counts");
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
    ncclGroupStart();
    for (int q = 0; q < P; ++q) {
        if (q == me) continue;
        if (need[q]) ncclSend(d_req + recv_off[q], (size_t)need[q], ncclInt64, q, ctx->comm, st);
        if (give[q]) ncclRecv(d_give + give_off[q], (size_t)give[q], ncclInt64, q, ctx->comm, st);
    }
    r = nccl_check(ctx, ncclGroupEnd(), "exchange halo requests");
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
#endif
}

int halo_exchange(bk_ctx* ctx, const bk_csr* Ac, int k, const double* X, int64_t ldx) {
#ifdef BK_NO_NCCL
    (void)Ac; (void)k; (void)X; (void)ldx;
    return set_error(ctx, BK_ERR_UNSUPPORTED, "built without NCCL");
#else
    bk_csr* A = const_cast<bk_csr*>(Ac);
    cudaStream_t cs = ctx->comm_stream;
    double* ghost = (double*)grow(A->ghost, sizeof(double) * std::max<int64_t>(A->n_ghost, 1) * k, ctx->stream);
    double* sendbuf = (double*)grow(A->sendbuf, sizeof(double) * std::max<int64_t>(A->n_send_total, 1) * k, ctx->stream);
    // X is produced on the compute stream: the comm stream waits for it
    cudaEventRecord(ctx->ev_a, ctx->stream);
    cudaStreamWaitEvent(cs, ctx->ev_a, 0);
    for (const auto& nb : A->nbs)
        if (nb.send_cnt && !(nb.send_contig && ldx == k))
            launch_pack_rows(nb.send_cnt, k, nb.d_send_rows, X, ldx, sendbuf + nb.send_off * k, cs);
    NCCL_OK(ctx, ncclGroupStart());
    for (const auto& nb : A->nbs) {
        if (nb.send_cnt) {
            const double* src = (nb.send_contig && ldx == k) ? X + nb.send_begin * ldx : sendbuf + nb.send_off * k;
            ncclSend(src, (size_t)nb.send_cnt * k, ncclDouble, nb.rank, ctx->comm, cs);
        }
        if (nb.recv_cnt) ncclRecv(ghost + nb.recv_off * k, (size_t)nb.recv_cnt * k, ncclDouble, nb.rank, ctx->comm, cs);
    }
    NCCL_OK(ctx, ncclGroupEnd());
    cudaEventRecord(ctx->ev_b, cs);
    return cuda_check(ctx, cudaGetLastError(), "halo_exchange");
#endif
}

}  // namespace bk
