// abi.cpp -- the C ABI of include/bk.h: argument validation, host/device
// staging, contexts, matrix ingest (copy + renumbering + halo plan) and the
// three kernel entry points.  Every numeric step is a kernel launched from
// here or from solve.cpp; there is no CPU compute path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <vector>

#include "bk_internal.h"
#include "reduce.cuh"

using namespace bk;

namespace bk {

std::atomic<long long> g_launches{0};

int set_error(bk_ctx* ctx, int code, const std::string& msg) {
    if (ctx) {
        ctx->last_error = msg;
        if (code == BK_ERR_CUDA || code == BK_ERR_NCCL) ctx->sticky = code;
    }
    return code;
}

int cuda_check(bk_ctx* ctx, cudaError_t e, const char* where) {
    if (e == cudaSuccess) return BK_OK;
    char buf[512];
    snprintf(buf, sizeof buf, "%s: %s", where, cudaGetErrorString(e));
    return set_error(ctx, e == cudaErrorMemoryAllocation ? BK_ERR_OOM : BK_ERR_CUDA, buf);
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

void* ws_get(bk_ctx* ctx, int slot, size_t bytes) {
    if ((int)ctx->ws.size() <= slot) ctx->ws.resize(slot + 1);
    bk_buf& b = ctx->ws[slot];
    if (b.bytes >= bytes && b.p) return b.p;
    if (b.p) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(b.p);
        b.p = nullptr;
        b.bytes = 0;
    }
    size_t want = std::max<size_t>(bytes + 256, 4096);
    if (cudaMalloc(&b.p, want) != cudaSuccess) {
        cudaGetLastError();
        b.p = nullptr;
        throw bk_error(BK_ERR_OOM, "workspace allocation of " + std::to_string(want) + " bytes failed");
    }
    b.bytes = want;
    return b.p;
}

static void* grow(bk_buf& b, size_t bytes, cudaStream_t st) {
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
        throw bk_error(BK_ERR_OOM, "buffer allocation failed");
    }
    b.bytes = want;
    return b.p;
}

}  // namespace bk

#define BK_TRY try {
#define BK_CATCH(ctx)                                              \
    }                                                              \
    catch (const bk_error& e) { return set_error(ctx, e.code, e.msg); } \
    catch (const std::exception& e) { return set_error(ctx, BK_ERR_CUDA, e.what()); }

#define ARG_CHECK(ctx, cond, msg) \
    do { if (!(cond)) return set_error(ctx, BK_ERR_ARG, msg); } while (0)

#define CUDA_OK(ctx, call) \
    do { int _r = cuda_check(ctx, (call), #call); if (_r) return _r; } while (0)

static int enter(bk_ctx* ctx) {
    if (!ctx) return BK_ERR_ARG;
    if (ctx->sticky) return ctx->sticky;
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaSetDevice");
    ctx->last_error.clear();
    return BK_OK;
}

// After a batch of launches: surface launch errors.
static int post_launch(bk_ctx* ctx, const char* where) {
    cudaError_t e = cudaGetLastError();
    return cuda_check(ctx, e, where);
}

// Stage an N x k (ld) host multivector to device (ld preserved) or return the device pointer.
static const double* stage_in(bk_ctx* ctx, int slot, const double* p, int64_t n, int64_t ld,
                              bool* is_host) {
    *is_host = !is_device_ptr(p);
    if (!*is_host) return p;
    size_t bytes = (size_t)n * ld * sizeof(double);
    double* d = (double*)ws_get(ctx, slot, bytes);
    if (bytes) {
        cudaError_t e = cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, ctx->stream);
        if (e != cudaSuccess) throw bk_error(BK_ERR_CUDA, std::string("H2D copy: ") + cudaGetErrorString(e));
    }
    return d;
}

// ------------------------------------------------------------------ context
extern "C" int bk_version(void) { return 100; }

extern "C" int64_t bk_kernel_launch_count(void) { return (int64_t)g_launches.load(); }

extern "C" const char* bk_status_string(int s) {
    switch (s) {
        case BK_OK: return "ok";
        case BK_ERR_ARG: return "invalid argument";
        case BK_NOT_CONVERGED: return "not converged";
        case BK_BREAKDOWN: return "breakdown";
        case BK_ERR_CUDA: return "CUDA error";
        case BK_ERR_NCCL: return "NCCL error";
        case BK_ERR_OOM: return "out of memory";
        case BK_ERR_UNSUPPORTED: return "unsupported";
        default: return "unknown status";
    }
}

extern "C" const char* bk_last_error(const bk_ctx* ctx) { return ctx ? ctx->last_error.c_str() : ""; }

extern "C" int bk_ctx_create(bk_ctx** out, int device, void* cuda_stream) {
    if (!out) return BK_ERR_ARG;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return BK_ERR_CUDA;
    }
    if (device < 0 || device >= ndev) return BK_ERR_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return BK_ERR_CUDA;
    bk_ctx* c = new bk_ctx();
    c->device = device;
    c->stream = (cudaStream_t)cuda_stream;   // NULL = the legacy default stream
    c->own_stream = false;
    cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&c->ev_a, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming);
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    // last-CTA tickets: [0, 33) stream Grams, [32, 65) column dots, 96 flat Grams
    if (cudaMalloc(&c->d_tickets, 128 * sizeof(int)) != cudaSuccess ||
        cudaMemset(c->d_tickets, 0, 128 * sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return BK_ERR_CUDA;
    }
    c->h_pinned_bytes = 1 << 20;
    if (cudaMallocHost(&c->h_pinned, c->h_pinned_bytes) != cudaSuccess) {
        cudaGetLastError();
        c->h_pinned = nullptr;
        c->h_pinned_bytes = 0;
    }
    *out = c;
    return BK_OK;
}

extern "C" int bk_ctx_set_stream(bk_ctx* ctx, void* cuda_stream) {
    int r = enter(ctx);
    if (r) return r;
    if (ctx->own_stream) {
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        ctx->own_stream = false;
    }
    ctx->stream = (cudaStream_t)cuda_stream;
    return BK_OK;
}

extern "C" int bk_ctx_synchronize(bk_ctx* ctx) {
    int r = enter(ctx);
    if (r) return r;
    CUDA_OK(ctx, cudaStreamSynchronize(ctx->stream));
    return BK_OK;
}

extern "C" int bk_ctx_destroy(bk_ctx* ctx) {
    if (!ctx) return BK_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (bk_csr* A : ctx->mats) A->ctx = nullptr;   // still valid handles; destroy frees their memory
    for (cudaEvent_t e : ctx->tev) cudaEventDestroy(e);
    for (auto& b : ctx->ws)
        if (b.p) cudaFree(b.p);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
    if (ctx->d_tickets) cudaFree(ctx->d_tickets);
#ifndef BK_NO_NCCL
    if (ctx->comm) ncclCommDestroy(ctx->comm);
#endif
    if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
    if (ctx->ev_a) cudaEventDestroy(ctx->ev_a);
    if (ctx->ev_b) cudaEventDestroy(ctx->ev_b);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    cudaGetLastError();
    return BK_OK;
}

extern "C" int bk_ctx_comm_info(const bk_ctx* ctx, int* nranks, int* rank) {
    if (!ctx) return BK_ERR_ARG;
    if (nranks) *nranks = ctx->nranks;
    if (rank) *rank = ctx->rank;
    return BK_OK;
}

// ------------------------------------------------------------------ halo plan (host only)
extern "C" int bk_plan_halo(int nranks, int rank, const int64_t* rank_begin, int64_t n_local,
                            const int32_t* row_ptr, const int32_t* col_global, int64_t nnz,
                            int64_t* n_ghost, int64_t* ghost_ids, int32_t* ghost_owner, int32_t* col_local,
                            uint8_t* is_boundary) {
    if (nranks < 1 || rank < 0 || rank >= nranks || !rank_begin || !row_ptr || !n_ghost) return BK_ERR_ARG;
    if (nnz > 0 && (!col_global || !col_local)) return BK_ERR_ARG;
    for (int r = 0; r < nranks; ++r)
        if (rank_begin[r + 1] < rank_begin[r]) return BK_ERR_ARG;
    const int64_t b0 = rank_begin[rank], b1 = rank_begin[rank + 1];
    if (b1 - b0 != n_local) return BK_ERR_ARG;
    if (row_ptr[0] != 0 || row_ptr[n_local] != nnz) return BK_ERR_ARG;
    const int64_t n_global = rank_begin[nranks];
    std::vector<int64_t> ghosts;
    for (int64_t p = 0; p < nnz; ++p) {
        const int64_t c = col_global[p];
        if (c < 0 || c >= n_global) return BK_ERR_ARG;
        if (c < b0 || c >= b1) ghosts.push_back(c);
    }
    std::sort(ghosts.begin(), ghosts.end());
    ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
    *n_ghost = (int64_t)ghosts.size();
    for (size_t g = 0; g < ghosts.size(); ++g) {
        if (ghost_ids) ghost_ids[g] = ghosts[g];
        if (ghost_owner) {
            // owner: last r with rank_begin[r] <= id (skip empty ranks)
            int r = (int)(std::upper_bound(rank_begin, rank_begin + nranks + 1, ghosts[g]) - rank_begin) - 1;
            while (r > 0 && rank_begin[r] == rank_begin[r + 1]) --r;
            ghost_owner[g] = r;
        }
    }
    for (int64_t i = 0; i < n_local; ++i) {
        if (row_ptr[i + 1] < row_ptr[i]) return BK_ERR_ARG;
        uint8_t bnd = 0;
        for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            const int64_t c = col_global[p];
            if (c >= b0 && c < b1) {
                col_local[p] = (int32_t)(c - b0);
            } else {
                const int64_t g = std::lower_bound(ghosts.begin(), ghosts.end(), c) - ghosts.begin();
                col_local[p] = (int32_t)(n_local + g);
                bnd = 1;
            }
        }
        if (is_boundary) is_boundary[i] = bnd;
    }
    return BK_OK;
}

// ------------------------------------------------------------------ matrix

extern "C" int bk_csr_create(bk_ctx* ctx, bk_csr** out, int64_t n_global, int64_t row_begin, int64_t n_local,
                             const int32_t* row_ptr, const int32_t* col_global, const double* val, int64_t nnz) {
    int r = enter(ctx);
    if (r) return r;
    ARG_CHECK(ctx, out != nullptr, "bk_csr_create: out is NULL");
    ARG_CHECK(ctx, n_global >= 0 && n_local >= 0 && row_begin >= 0 && row_begin + n_local <= n_global,
              "bk_csr_create: bad row range");
    ARG_CHECK(ctx, n_global < ((int64_t)1 << 31), "bk_csr_create: n_global must be < 2^31 (int32 columns)");
    ARG_CHECK(ctx, nnz >= 0 && nnz < ((int64_t)1 << 31) - 16, "bk_csr_create: nnz must be < 2^31");
    ARG_CHECK(ctx, row_ptr != nullptr, "bk_csr_create: row_ptr is NULL");
    ARG_CHECK(ctx, nnz == 0 || (col_global && val), "bk_csr_create: col/val NULL");
    if (ctx->nranks == 1)
        ARG_CHECK(ctx, row_begin == 0 && n_local == n_global,
                  "bk_csr_create: a single-rank ctx needs the whole matrix (row_begin 0, n_local == n_global)");
    *out = nullptr;
    BK_TRY
    cudaStream_t st = ctx->stream;
    // host copies of the index structure (validation + halo plan are host work at setup)
    std::vector<int32_t> rp(n_local + 1), colg(nnz);
    const bool rp_dev = is_device_ptr(row_ptr), col_dev = is_device_ptr(col_global);
    CUDA_OK(ctx, cudaMemcpy(rp.data(), row_ptr, sizeof(int32_t) * (n_local + 1),
                            rp_dev ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
    if (nnz)
        CUDA_OK(ctx, cudaMemcpy(colg.data(), col_global, sizeof(int32_t) * nnz,
                                col_dev ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
    ARG_CHECK(ctx, rp[0] == 0 && rp[n_local] == nnz, "bk_csr_create: row_ptr[0] must be 0 and row_ptr[n] == nnz");
    for (int64_t i = 0; i < n_local; ++i) {
        ARG_CHECK(ctx, rp[i + 1] >= rp[i], "bk_csr_create: row_ptr must be non-decreasing");
        for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
            ARG_CHECK(ctx, colg[p] >= 0 && colg[p] < n_global, "bk_csr_create: column id out of range");
            ARG_CHECK(ctx, p == rp[i] || colg[p] > colg[p - 1],
                      "bk_csr_create: columns must be strictly increasing within a row");
        }
    }
    bk_csr* A = new bk_csr();
    A->ctx = ctx;
    A->n_global = n_global;
    A->row_begin = row_begin;
    A->n_local = n_local;
    A->nnz = nnz;
    // device arrays, 256-byte aligned (cudaMalloc) and padded by 8 elements so
    // the 16-byte vector loads of the apply kernel never leave the allocation
    const size_t pad = 8;
    if (cudaMalloc(&A->d_rp, sizeof(int32_t) * (n_local + 1 + pad)) != cudaSuccess ||
        cudaMalloc(&A->d_col, sizeof(int32_t) * (nnz + pad)) != cudaSuccess ||
        cudaMalloc(&A->d_val, sizeof(double) * (nnz + pad)) != cudaSuccess ||
        cudaMalloc(&A->d_dinv, sizeof(double) * (n_local + pad)) != cudaSuccess) {
        cudaGetLastError();
        bk_csr_destroy(A);
        return set_error(ctx, BK_ERR_OOM, "bk_csr_create: device allocation failed");
    }
    cudaMemsetAsync(A->d_col, 0, sizeof(int32_t) * (nnz + pad), st);
    cudaMemsetAsync(A->d_val, 0, sizeof(double) * (nnz + pad), st);
    std::vector<int32_t> col_local(colg);
    if (ctx->nranks > 1) {
        int rr = csr_setup_comm(ctx, A, rp, col_local, colg);
        if (rr) { bk_csr_destroy(A); return rr; }
    } else {
        A->n_interior = n_local;
        A->interior_contig = 1;
        A->interior_begin = 0;
    }
    cudaMemcpyAsync(A->d_rp, rp.data(), sizeof(int32_t) * (n_local + 1), cudaMemcpyHostToDevice, st);
    if (nnz) {
        cudaMemcpyAsync(A->d_col, col_local.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(A->d_val, val, sizeof(double) * nnz, cudaMemcpyDefault, st);
    }
    // band plan of the contiguous (interior) row range (window.cpp)
    if (A->interior_contig && A->n_interior > 0 && nnz > 0) {
        const int64_t ib = A->interior_begin, ni = A->n_interior;
        bk_band_plan bp;
        // rows of the range are numbered from 0 by the planner: offsets d = col - (row - ib)
        std::vector<int32_t> rp_range(rp.begin() + ib, rp.begin() + ib + ni + 1);
        std::vector<int32_t> col_shift;
        const int32_t* cols = col_local.data();
        if (ib != 0) {   // shift to range-local row numbering: d = col - row
            col_shift.resize(nnz);
            for (int64_t i = 0; i < ni; ++i)
                for (int32_t p = rp_range[i]; p < rp_range[i + 1]; ++p) col_shift[p] = col_local[p] - (int32_t)ib;
            cols = col_shift.data();
        }
        if (bk_plan_bands(ni, rp_range.data(), cols, 96, &bp) == BK_OK && bp.nbands > 0) {
            A->band.nbands = bp.nbands;
            A->band.extra = bp.extra_rows;
            A->band.max_row_nnz = bp.max_row_nnz;
            for (int g = 0; g < bp.nbands; ++g) {
                A->band.lo[g] = bp.lo[g];
                A->band.hi[g] = bp.hi[g];
                A->band.dmin[g] = bp.dmin[g];
                A->band.dmax[g] = bp.dmax[g];
            }
            A->band.row0 = ib;
            A->band.nrows = ni;
        }
    }
    // Jacobi diagonal (local numbering: diagonal column of row i is i)
    launch_extract_diag_inv(n_local, 0, A->d_rp, A->d_col, A->d_val, A->d_dinv, st);
    // Gershgorin bound of D^-1 A for the Chebyshev preconditioner (max over ranks)
    unsigned long long* d_g = nullptr;
    int rr = cuda_check(ctx, cudaMalloc(&d_g, sizeof *d_g), "bk_csr_create gershgorin");
    if (!rr) rr = cuda_check(ctx, cudaMemsetAsync(d_g, 0, sizeof *d_g, st), "bk_csr_create gershgorin");
    if (!rr) launch_gershgorin(n_local, A->d_rp, A->d_val, A->d_dinv, d_g, st);
    if (!rr) rr = post_launch(ctx, "bk_csr_create");
    if (!rr) rr = allreduce_max(ctx, reinterpret_cast<double*>(d_g), 1);
    if (!rr) rr = cuda_check(ctx, cudaMemcpyAsync(&A->gersh, d_g, sizeof(double), cudaMemcpyDeviceToHost, st),
                             "bk_csr_create gershgorin");
    if (!rr) rr = cuda_check(ctx, cudaStreamSynchronize(st), "bk_csr_create sync");
    if (d_g) cudaFree(d_g);
    if (rr) { bk_csr_destroy(A); return rr; }
    ctx->mats.push_back(A);
    *out = A;
    return BK_OK;
    BK_CATCH(ctx)
}

extern "C" int bk_csr_destroy(bk_csr* A) {
    if (!A) return BK_OK;
    if (A->ctx) {
        cudaSetDevice(A->ctx->device);
        cudaStreamSynchronize(A->ctx->stream);
        auto& v = A->ctx->mats;
        v.erase(std::remove(v.begin(), v.end(), A), v.end());
    }
    cudaFree(A->d_rp);
    cudaFree(A->d_col);
    cudaFree(A->d_val);
    cudaFree(A->d_dinv);
    cudaFree(A->d_boundary_rows);
    cudaFree(A->d_interior_rows);
    for (auto& nb : A->nbs) cudaFree(nb.d_send_rows);
    if (A->ghost.p) cudaFree(A->ghost.p);
    if (A->sendbuf.p) cudaFree(A->sendbuf.p);
    delete A;
    cudaGetLastError();
    return BK_OK;
}

extern "C" int bk_csr_get_info(const bk_csr* A, bk_csr_info* info) {
    if (!A || !info) return BK_ERR_ARG;
    info->n_global = A->n_global;
    info->row_begin = A->row_begin;
    info->n_local = A->n_local;
    info->nnz = A->nnz;
    info->n_ghost = A->n_ghost;
    info->n_boundary_rows = A->n_boundary;
    info->n_send_rows = A->n_send_total;
    info->n_neighbors = (int)A->nbs.size();
    info->interior_contiguous = A->interior_contig;
    info->n_bands = A->band.nbands;
    info->band_extra_rows = A->band.extra;
    info->jacobi_gershgorin = A->gersh;
    return BK_OK;
}

// ------------------------------------------------------------------ a1 apply
namespace bk {
// 3-D lattices: y-slab tile order for the gather kernel (sets a.sl_*; no-op otherwise)
static void slab_order(SpmmArgs& a, const BandPlan& bp_, int k) {
    // 3-D lattice whose z-neighbour planes do not stay in L2 across two planes of streaming
    // (c4 / c5: 256^2 / 512^2 planes): y-slab tile order.  S = the smallest power of two with
    // 2 (ny / S) nx (16 k + 88) B <= 28 MB.  Round 1 (56 MB, 12 <= k <= 16 only): ncu c5 k = 16
    // DRAM reads 20.3 -> 16.5 GB (14.5 algorithmic).  Round 2 (28 MB, every k):
    // c5 k = 8 / 16 / 32 0.83 / 0.64 / 0.57 -> 0.84 / 0.76 / 0.66 of HBM, c4 0.86 / 0.71 / 0.64
    // -> 0.87 / 0.75 / 0.68; ncu c5 k = 32 without it read X 1.9 times from DRAM.  BK_SLAB=0: off
    static const int slab = env_int("BK_SLAB", 1);
    const BandPlan& bp = bp_;
    const bool slab_k = slab != 0;
    if (slab_k && bp.nbands == 5 && bp.dmin[0] == bp.dmax[0] && bp.dmin[1] == bp.dmax[1] && bp.dmin[1] < 0 &&
        bp.dmin[0] < bp.dmin[1] && a.row0 == bp.row0 && a.nrows == bp.nrows) {
        const int64_t nx = -(int64_t)bp.dmin[1], plane = -(int64_t)bp.dmin[0];
        if (plane % nx == 0 && a.nrows % plane == 0) {
            const int64_t ny = plane / nx, nz = a.nrows / plane;
            const double row_bytes = 16.0 * k + 88.0;
            const double budget = 28.0 * 1024 * 1024;   // of the 126 MB L2 (two 63 MB partitions)
            int S = 1;
            while (2.0 * (double)(ny / S) * nx * row_bytes > budget && ny % (2 * S) == 0 && ny / (2 * S) >= 8)
                S *= 2;
            if (S > 1 && ny < (1 << 30) && nz < (1 << 30) && nx < (1 << 30)) {
                a.sl_S = S; a.sl_tpl = (int)nx; a.sl_ny = (int)ny; a.sl_nz = (int)nz;
            }
        }
    }
}
}  // namespace bk

namespace bk {
int spmm_dev(bk_ctx* ctx, const bk_csr* A, int k, const double* X, int64_t ldx, const double* C, int kout,
             double alpha, double beta, double* Y, int64_t ldy) {
    SpmmArgs a{};
    a.rp = A->d_rp;
    a.col = A->d_col;
    a.val = A->d_val;
    a.X = X;
    a.ldx = ldx;
    a.C = C;
    a.k = k;
    a.kout = kout;
    a.alpha = alpha;
    a.beta = beta;
    a.Y = Y;
    a.ldy = ldy;
    a.ncol_local = (int32_t)A->n_local;
    if (ctx->nranks == 1 || A->n_ghost == 0) {
        a.row0 = 0;
        a.nrows = A->n_local;
        slab_order(a, A->band, k);
        if (!launch_bspmm_win(a, A->band, ctx->stream)) launch_bspmm(a, ctx->stream);
        return post_launch(ctx, "bspmm_apply");
    }
    // p > 1: halo exchange on the comm stream overlapped with the interior rows
    int r = halo_exchange(ctx, A, k, X, ldx);   // records ctx->ev_b when the ghosts have landed
    if (r) return r;
    // the interior rows run while the halo is in flight: leave SMs for NCCL's send/recv kernels
    // (a persistent grid over every SM would only let them in once the interior is done)
    constexpr int kCommSms = 8;
    a.grid_sms = ctx->num_sms > 2 * kCommSms ? ctx->num_sms - kCommSms : 0;
    if (A->interior_contig) {
        a.row0 = A->interior_begin;
        a.nrows = A->n_interior;
        a.rows = nullptr;
    } else {
        a.rows = A->d_interior_rows;
        a.nrows = A->n_interior;
    }
    if (!a.rows) slab_order(a, A->band, k);
    if (!launch_bspmm_win(a, A->band, ctx->stream)) launch_bspmm(a, ctx->stream);
    a.sl_S = 0;
    cudaStreamWaitEvent(ctx->stream, ctx->ev_b, 0);
    a.grid_sms = 0;
    a.rows = A->d_boundary_rows;
    a.nrows = A->n_boundary;
    a.Xg = (const double*)A->ghost.p;
    a.ldg = k;
    launch_bspmm(a, ctx->stream);
    return post_launch(ctx, "bspmm_apply");
}
}  // namespace bk

extern "C" int bspmm_apply(bk_ctx* ctx, const bk_csr* A, int k, const double* X, int64_t ldx, const double* C,
                           int k_out, double alpha, double beta, double* Y, int64_t ldy) {
    int r = enter(ctx);
    if (r) return r;
    ARG_CHECK(ctx, A != nullptr && A->ctx == ctx, "bspmm_apply: matrix is NULL or from another ctx");
    ARG_CHECK(ctx, k >= 1 && k <= BK_MAX_K, "bspmm_apply: need 1 <= k <= 32");
    ARG_CHECK(ctx, k_out >= 1 && k_out <= BK_MAX_K, "bspmm_apply: need 1 <= k_out <= 32");
    ARG_CHECK(ctx, C != nullptr || k_out == k, "bspmm_apply: C == NULL requires k_out == k");
    ARG_CHECK(ctx, ldx >= k && ldy >= k_out, "bspmm_apply: leading dimension too small");
    ARG_CHECK(ctx, A->n_local == 0 || (X != nullptr && Y != nullptr), "bspmm_apply: X or Y is NULL");
    ARG_CHECK(ctx, (const void*)X != (const void*)Y, "bspmm_apply: Y must not alias X");
    if (A->n_local == 0) return BK_OK;
    BK_TRY
    bool xh, ch = false;
    const double* dX = stage_in(ctx, WS_STAGE_X, X, A->n_local, ldx, &xh);
    const double* dC = nullptr;
    if (C) dC = stage_in(ctx, WS_STAGE_C, C, k, k_out, &ch);
    const bool yh = !is_device_ptr(Y);
    double* dY = Y;
    if (yh) {
        dY = (double*)ws_get(ctx, WS_STAGE_Y, (size_t)A->n_local * ldy * sizeof(double));
        if (beta != 0.0)
            CUDA_OK(ctx, cudaMemcpyAsync(dY, Y, (size_t)A->n_local * ldy * sizeof(double), cudaMemcpyHostToDevice,
                                         ctx->stream));
    }
    r = spmm_dev(ctx, A, k, dX, ldx, dC, k_out, alpha, beta, dY, ldy);
    if (r) return r;
    if (yh) {
        CUDA_OK(ctx, cudaMemcpyAsync(Y, dY, (size_t)A->n_local * ldy * sizeof(double), cudaMemcpyDeviceToHost,
                                     ctx->stream));
    }
    if (xh || ch || yh) CUDA_OK(ctx, cudaStreamSynchronize(ctx->stream));
    return BK_OK;
    BK_CATCH(ctx)
}

namespace bk {
bool spmm_red_dev(bk_ctx* ctx, const bk_csr* A, int k, const double* X, double* Y, int red, const double* e0,
                  const double* e1, double* blk0, double* blk1, double* dot0, double* dot1, const SmallEpi* epi) {
    if (ctx->nranks > 1 || A->n_local <= 0 || !use_stream_kernels()) return false;
    SpmmArgs a{};
    a.rp = A->d_rp;
    a.col = A->d_col;
    a.val = A->d_val;
    a.X = X;
    a.ldx = k;
    a.k = k;
    a.kout = k;
    a.alpha = 1.0;
    a.beta = 0.0;
    a.Y = Y;
    a.ldy = k;
    a.ncol_local = (int32_t)A->n_local;
    a.row0 = 0;
    a.nrows = A->n_local;
    RedOut ro;
    ro.part = (double*)ws_get(ctx, WS_GRAM_PART + 32, stream_part_doubles(ctx->num_sms) * sizeof(double));
    ro.ticket = ctx->d_tickets;
    ro.blk[0][0] = blk0;
    ro.blk[0][1] = blk1;
    ro.dots[0] = dot0;
    ro.dots[1] = dot1;
    return launch_bspmm_win_red(a, A->band, ctx->stream, red, e0, e1, ro, epi);
}
}  // namespace bk

// ------------------------------------------------------------------ a3 gram
namespace bk {
int gram_dev(bk_ctx* ctx, int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y, int64_t ldy,
             double* G, bool allreduce) {
    static int use_mma = -1;
    if (use_mma < 0) {
        const char* e = getenv("BK_GRAM");
        use_mma = (e && strcmp(e, "fma") == 0) ? 0 : 1;
    }
    double* spart = nullptr;
    if (n > 0 && use_stream_kernels())
        spart = (double*)ws_get(ctx, WS_GRAM_PART + 32, stream_part_doubles(ctx->num_sms) * sizeof(double));
    const bool wide = n > 0 && ka >= 16 && (ka > 32 || ldx != ka || ldy != kb);
    if (n > 0 && launch_gram_flat(n, ka, kb, X, ldx, Y, ldy, G,
                                  (double*)ws_get(ctx, WS_GRAM_PART + 34, flat_part_doubles(ctx->num_sms) * sizeof(double)),
                                  ctx->d_tickets + 96, ctx->num_sms, ctx->stream)) {
        // k <= 4: flat grid-stride Gram (flat.cu)
    } else if (wide && launch_gram_wide(n, ka, kb, X, ldx, Y, ldy, G,
                                 (double*)ws_get(ctx, WS_GRAM_PART + 33,
                                                 gram_wide_ws_doubles(ka, kb, ctx->num_sms) * sizeof(double)),
                                 ctx->num_sms, ctx->stream)) {
        // strided / wide multi-Gram (GMRES basis): cp.async-staged DMMA
    } else if (spart && launch_gram_stream(n, ka, kb, X, ldx, Y, ldy, G, spart, ctx->d_tickets, ctx->num_sms, ctx->stream)) {
        // TMA-staged DMMA Gram
    } else if (n > 0 && use_mma && (ka >= 8 || kb >= 8)) {
        double* part = (double*)ws_get(ctx, WS_GRAM_PART, gram_mma_ws_doubles(n, ka, kb, ctx->num_sms) * sizeof(double));
        launch_gram_mma(n, ka, kb, X, ldx, Y, ldy, G, part, ctx->d_tickets, ctx->num_sms, ctx->stream);
    } else if (n > 0) {
        double* part = (double*)ws_get(ctx, WS_GRAM_PART, gram_ws_doubles(n, ka, kb, ctx->num_sms) * sizeof(double));
        launch_gram(n, ka, kb, X, ldx, Y, ldy, G, part, ctx->num_sms, ctx->stream);
    } else {
        cudaMemsetAsync(G, 0, sizeof(double) * ka * kb, ctx->stream);
    }
    int r = post_launch(ctx, "block_gram");
    if (r) return r;
    if (allreduce && ctx->nranks > 1) return allreduce_sum(ctx, G, (int64_t)ka * kb);
    return BK_OK;
}
}  // namespace bk

extern "C" int block_gram(bk_ctx* ctx, int64_t n, int ka, int kb, const double* X, int64_t ldx, const double* Y,
                          int64_t ldy, double* G, int flags) {
    int r = enter(ctx);
    if (r) return r;
    ARG_CHECK(ctx, n >= 0, "block_gram: n < 0");
    ARG_CHECK(ctx, ka >= 1 && ka <= BK_MAX_KA, "block_gram: need 1 <= ka <= 4096");
    ARG_CHECK(ctx, kb >= 1 && kb <= BK_MAX_K, "block_gram: need 1 <= kb <= 32");
    ARG_CHECK(ctx, ldx >= ka && ldy >= kb, "block_gram: leading dimension too small");
    ARG_CHECK(ctx, G != nullptr && (n == 0 || (X && Y)), "block_gram: NULL pointer");
    BK_TRY
    bool xh, yh;
    const double* dX = stage_in(ctx, WS_STAGE_X, X, n, ldx, &xh);
    const double* dY = (Y == X && ldy == ldx) ? dX : stage_in(ctx, WS_STAGE_Y, Y, n, ldy, &yh);
    const bool gh = !is_device_ptr(G);
    double* dG = gh ? (double*)ws_get(ctx, WS_STAGE_G, sizeof(double) * ka * kb) : G;
    r = gram_dev(ctx, n, ka, kb, dX, ldx, dY, ldy, dG, (flags & BK_GRAM_ALLREDUCE) != 0);
    if (r) return r;
    if (gh) {
        CUDA_OK(ctx, cudaMemcpyAsync(G, dG, sizeof(double) * ka * kb, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_OK(ctx, cudaStreamSynchronize(ctx->stream));
    } else if (xh || (dY != Y)) {
        CUDA_OK(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return BK_OK;
    BK_CATCH(ctx)
}

// ------------------------------------------------------------------ a5 update
extern "C" int block_update(bk_ctx* ctx, int64_t n, int kp, int k, double a, double* X, int64_t ldx, double s,
                            const double* P, int64_t ldp, const double* C) {
    int r = enter(ctx);
    if (r) return r;
    ARG_CHECK(ctx, n >= 0, "block_update: n < 0");
    ARG_CHECK(ctx, k >= 1 && k <= BK_MAX_K, "block_update: need 1 <= k <= 32");
    ARG_CHECK(ctx, kp >= 1 && kp <= BK_MAX_KA, "block_update: need 1 <= kp <= 4096");
    ARG_CHECK(ctx, ldx >= k && ldp >= kp, "block_update: leading dimension too small");
    ARG_CHECK(ctx, n == 0 || (X && P && C), "block_update: NULL pointer");
    const bool alias = (const void*)P == (const void*)X;
    ARG_CHECK(ctx, !alias || (ldp == ldx && kp == k), "block_update: P may alias X only with kp == k, ldp == ldx");
    if (n == 0) return BK_OK;
    BK_TRY
    bool xh = !is_device_ptr(X), ph = false, ch = false;
    double* dX = X;
    if (xh) {
        dX = (double*)ws_get(ctx, WS_STAGE_Y, (size_t)n * ldx * sizeof(double));
        CUDA_OK(ctx, cudaMemcpyAsync(dX, X, (size_t)n * ldx * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
    const double* dP = alias ? dX : stage_in(ctx, WS_STAGE_X, P, n, ldp, &ph);
    const double* dC = stage_in(ctx, WS_STAGE_C, C, kp, k, &ch);
    UpdArgs u{};
    u.n = n; u.kp = kp; u.k = k;
    u.a = a; u.Xin = dX; u.ldxin = ldx;
    u.s = s; u.P = dP; u.ldp = ldp; u.C = dC;
    u.out = dX; u.ldo = ldx;
    launch_update(u, ctx->stream);
    r = post_launch(ctx, "block_update");
    if (r) return r;
    if (xh) CUDA_OK(ctx, cudaMemcpyAsync(X, dX, (size_t)n * ldx * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (xh || ph || ch) CUDA_OK(ctx, cudaStreamSynchronize(ctx->stream));
    return BK_OK;
    BK_CATCH(ctx)
}

// ------------------------------------------------------------------ a6 solve
extern "C" void bk_solve_opts_default(bk_solve_opts* o) {
    if (!o) return;
    memset(o, 0, sizeof *o);
    o->method = BK_CG;
    o->max_iters = 1000;
    o->restart = 30;
    o->precond = BK_PRECOND_NONE;
    o->conv_mode = BK_CONV_ALL;
    o->x0_is_zero = 0;
    o->check_every = 1;
    o->use_graphs = 0;
    o->rtol = 1e-10;
    o->breakdown_tol = 1e-13;
    o->cheb_steps = 4;
}

extern "C" int block_krylov_solve(bk_ctx* ctx, const bk_csr* A, int k, const double* B, int64_t ldb, double* X,
                                  int64_t ldx, const bk_solve_opts* o, bk_solve_report* rep) {
    int r = enter(ctx);
    if (r) return r;
    ARG_CHECK(ctx, A && A->ctx == ctx, "block_krylov_solve: matrix is NULL or from another ctx");
    ARG_CHECK(ctx, o && rep, "block_krylov_solve: opts/report NULL");
    ARG_CHECK(ctx, k >= 1 && k <= BK_MAX_K, "block_krylov_solve: need 1 <= k <= 32");
    ARG_CHECK(ctx, ldb >= k && ldx >= k, "block_krylov_solve: leading dimension too small");
    ARG_CHECK(ctx, A->n_local == 0 || (B && X), "block_krylov_solve: NULL pointer");
    ARG_CHECK(ctx, (const void*)B != (const void*)X, "block_krylov_solve: X must not alias B");
    ARG_CHECK(ctx, o->method >= BK_CG && o->method <= BK_CG1, "block_krylov_solve: unknown method");
    ARG_CHECK(ctx, o->max_iters >= 0 && o->check_every >= 1, "block_krylov_solve: bad max_iters/check_every");
    ARG_CHECK(ctx, o->method != BK_GMRES || (o->restart >= 1 && (int64_t)(o->restart + 1) * k <= BK_MAX_KA),
              "block_krylov_solve: GMRES needs restart >= 1 and (restart+1)*k <= 4096");
    ARG_CHECK(ctx, o->rtol >= 0.0 && o->breakdown_tol >= 0.0, "block_krylov_solve: negative tolerance");
    ARG_CHECK(ctx, o->precond == BK_PRECOND_NONE ||
                       ((o->precond == BK_PRECOND_JACOBI || o->precond == BK_PRECOND_CHEBYSHEV) && o->method == BK_CG),
              "block_krylov_solve: JACOBI / CHEBYSHEV preconditioning is implemented for CG only");
    ARG_CHECK(ctx, o->precond != BK_PRECOND_CHEBYSHEV || cheb_opts_ok(A, o),
              "block_krylov_solve: CHEBYSHEV needs cheb_steps >= 1 and 0 < lmin < lmax (after defaults)");
    BK_TRY
    bool bh;
    const double* dB = stage_in(ctx, WS_STAGE_X, B, A->n_local, ldb, &bh);
    const bool xh = !is_device_ptr(X);
    double* dX = X;
    if (xh) {
        dX = (double*)ws_get(ctx, WS_STAGE_Y, (size_t)A->n_local * ldx * sizeof(double));
        if (!o->x0_is_zero)
            CUDA_OK(ctx, cudaMemcpyAsync(dX, X, (size_t)A->n_local * ldx * sizeof(double), cudaMemcpyHostToDevice,
                                         ctx->stream));
    }
    r = solve_impl(ctx, A, k, dB, ldb, dX, ldx, o, rep);
    if (r == BK_ERR_CUDA || r == BK_ERR_NCCL || r == BK_ERR_OOM || r == BK_ERR_ARG) return r;
    if (xh) {
        CUDA_OK(ctx, cudaMemcpyAsync(X, dX, (size_t)A->n_local * ldx * sizeof(double), cudaMemcpyDeviceToHost,
                                     ctx->stream));
    }
    CUDA_OK(ctx, cudaStreamSynchronize(ctx->stream));
    return r;
    BK_CATCH(ctx)
}

// ------------------------------------------------------------------ NEXT-4 preconditioner apply
extern "C" int bk_precond_apply(bk_ctx* ctx, const bk_csr* A, int k, const bk_solve_opts* o, const double* R,
                                int64_t ldr, double* Z, int64_t ldz) {
    int r = enter(ctx);
    if (r) return r;
    ARG_CHECK(ctx, A && A->ctx == ctx && o, "bk_precond_apply: NULL matrix/opts or matrix from another ctx");
    ARG_CHECK(ctx, k >= 1 && k <= BK_MAX_K && ldr >= k && ldz >= k, "bk_precond_apply: bad k / leading dims");
    ARG_CHECK(ctx, A->n_local == 0 || (R && Z), "bk_precond_apply: NULL pointer");
    ARG_CHECK(ctx, (const void*)R != (const void*)Z, "bk_precond_apply: Z must not alias R");
    ARG_CHECK(ctx, o->precond >= BK_PRECOND_NONE && o->precond <= BK_PRECOND_CHEBYSHEV,
              "bk_precond_apply: unknown preconditioner");
    ARG_CHECK(ctx, o->precond != BK_PRECOND_CHEBYSHEV || cheb_opts_ok(A, o),
              "bk_precond_apply: CHEBYSHEV needs cheb_steps >= 1 and 0 < lmin < lmax (after defaults)");
    BK_TRY
    bool rh;
    const double* dR = stage_in(ctx, WS_STAGE_X, R, A->n_local, ldr, &rh);
    const bool zh = !is_device_ptr(Z);
    double* dZ = zh ? (double*)ws_get(ctx, WS_STAGE_Y, (size_t)A->n_local * ldz * sizeof(double)) : Z;
    r = precond_apply_impl(ctx, A, k, o, dR, ldr, dZ, ldz);
    if (r) return r;
    if (zh)
        CUDA_OK(ctx, cudaMemcpyAsync(Z, dZ, (size_t)A->n_local * ldz * sizeof(double), cudaMemcpyDeviceToHost,
                                     ctx->stream));
    CUDA_OK(ctx, cudaStreamSynchronize(ctx->stream));
    return BK_OK;
    BK_CATCH(ctx)
}

// ------------------------------------------------------------------ NEXT-3 Algorithm 1 (alg1.cpp)
extern "C" int bk_alg1_run(bk_ctx* ctx, const bk_dr_problem* pb, int m, const double* A, int n_steps, int window,
                           double eps, int max_newton, const bk_solve_opts* inner, double* traj, int64_t ldt,
                           int* newton_its, bk_alg1_report* rep) {
    int r = enter(ctx);
    if (r) return r;
    ARG_CHECK(ctx, pb && A && inner && rep, "bk_alg1_run: NULL problem/tableau/opts/report");
    ARG_CHECK(ctx, ctx->nranks <= 1, "bk_alg1_run: single rank only");
    ARG_CHECK(ctx, pb->nx >= 1 && pb->ny >= 1 && pb->nz >= 1 && pb->nx * pb->ny * pb->nz < (1ll << 31) &&
                       pb->tau > 0.0 && pb->y0 && pb->g,
              "bk_alg1_run: bad lattice / tau / NULL y0, g");
    ARG_CHECK(ctx, m >= 1 && m <= 8 && n_steps >= 0 && window >= 1 && window <= BK_MAX_K && eps > 0.0 &&
                       max_newton >= 0,
              "bk_alg1_run: need 1 <= m <= 8, n_steps >= 0, 1 <= window <= 32, eps > 0, max_newton >= 0");
    ARG_CHECK(ctx, !is_device_ptr(A), "bk_alg1_run: A must be a host array");
    ARG_CHECK(ctx, !traj || ldt >= n_steps, "bk_alg1_run: ldt < n_steps");
    ARG_CHECK(ctx, inner->method >= BK_CG && inner->method <= BK_CG1 && inner->check_every >= 1 &&
                       inner->max_iters >= 0 && inner->rtol >= 0.0 &&
                       (inner->method != BK_GMRES || (int64_t)(inner->restart + 1) * window <= BK_MAX_KA),
              "bk_alg1_run: bad inner solver options");
    for (int i = 0; i < m; ++i)
        for (int j = i + 1; j < m; ++j)
            ARG_CHECK(ctx, A[i * m + j] == 0.0, "bk_alg1_run: A must be lower triangular (DIRK)");
    BK_TRY
    return alg1_impl(ctx, pb, m, A, n_steps, window, eps, max_newton, inner, traj, ldt, newton_its, rep);
    BK_CATCH(ctx)
}

// ------------------------------------------------------------------ NEXT-1 DIRK window (dirk.cpp)
static int dirk_entry(bk_ctx* ctx, const bk_csr* L, const bk_csr* K, double mass, double tau, int k,
                      const double* A1, const double* A2, const double* B, const double* B0, int64_t ldb,
                      double* Y, int64_t ldy, int max_outer, double outer_tol, const bk_solve_opts* inner,
                      bk_dirk_report* rep, bool correction) {
    int r = enter(ctx);
    if (r) return r;
    ARG_CHECK(ctx, L && K && L->ctx == ctx && K->ctx == ctx, "bk_dirk_solve: matrix NULL or from another ctx");
    ARG_CHECK(ctx, L->n_local == K->n_local && L->row_begin == K->row_begin && L->n_global == K->n_global,
              "bk_dirk_solve: L and K must have the same row partition");
    ARG_CHECK(ctx, k >= 1 && k <= BK_MAX_K, "bk_dirk_solve: need 1 <= k <= 32");
    ARG_CHECK(ctx, A1 && A2 && inner && rep, "bk_dirk_solve: NULL A1/A2/opts/report");
    ARG_CHECK(ctx, !is_device_ptr(A1) && !is_device_ptr(A2), "bk_dirk_solve: A1, A2 must be host arrays");
    ARG_CHECK(ctx, tau > 0.0 && mass >= 0.0 && max_outer >= 0 && outer_tol >= 0.0,
              "bk_dirk_solve: need tau > 0, mass >= 0, max_outer >= 0, outer_tol >= 0");
    ARG_CHECK(ctx, ldb >= k && ldy >= k, "bk_dirk_solve: leading dimension too small");
    ARG_CHECK(ctx, L->n_local == 0 || (B && B0 && Y), "bk_dirk_solve: NULL B/B0/Y");
    ARG_CHECK(ctx, (const void*)Y != (const void*)B && (const void*)Y != (const void*)B0,
              "bk_dirk_solve: Y must not alias B or B0");
    ARG_CHECK(ctx, inner->method >= BK_CG && inner->method <= BK_CG1 && inner->check_every >= 1 &&
                       inner->max_iters >= 0 && inner->rtol >= 0.0,
              "bk_dirk_solve: bad inner solver options");
    ARG_CHECK(ctx, inner->method != BK_GMRES || (inner->restart >= 1 && (int64_t)(inner->restart + 1) * k <= BK_MAX_KA),
              "bk_dirk_solve: GMRES needs restart >= 1 and (restart+1)*k <= 4096");
    ARG_CHECK(ctx, inner->precond == BK_PRECOND_NONE ||
                       ((inner->precond == BK_PRECOND_JACOBI || inner->precond == BK_PRECOND_CHEBYSHEV) &&
                        inner->method == BK_CG),
              "bk_dirk_solve: JACOBI / CHEBYSHEV preconditioning is implemented for CG only");
    ARG_CHECK(ctx, inner->precond != BK_PRECOND_CHEBYSHEV || cheb_opts_ok(L, inner),
              "bk_dirk_solve: CHEBYSHEV needs cheb_steps >= 1 and 0 < lmin < lmax (after defaults)");
    BK_TRY
    const int64_t n = L->n_local;
    bool bh, b0h;
    const double* dB = stage_in(ctx, WS_STAGE_X, B, n, ldb, &bh);
    const double* dB0 = stage_in(ctx, WS_STAGE_C, B0, n, ldb, &b0h);
    const bool yh = !is_device_ptr(Y);
    double* dY = Y;
    if (yh) {
        dY = (double*)ws_get(ctx, WS_STAGE_Y, (size_t)n * ldy * sizeof(double));
        CUDA_OK(ctx, cudaMemcpyAsync(dY, Y, (size_t)n * ldy * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
    r = dirk_impl(ctx, L, K, mass, tau, k, A1, A2, dB, dB0, ldb, dY, ldy, max_outer, outer_tol, inner, rep,
                  correction);
    if (r == BK_ERR_CUDA || r == BK_ERR_NCCL || r == BK_ERR_OOM || r == BK_ERR_ARG) return r;
    if (yh)
        CUDA_OK(ctx, cudaMemcpyAsync(Y, dY, (size_t)n * ldy * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_OK(ctx, cudaStreamSynchronize(ctx->stream));
    return r;
    BK_CATCH(ctx)
}

extern "C" int bk_dirk_solve(bk_ctx* ctx, const bk_csr* L, const bk_csr* K, double mass, double tau, int k,
                             const double* A1, const double* A2, const double* B, const double* B0, int64_t ldb,
                             double* Y, int64_t ldy, int max_outer, double outer_tol, const bk_solve_opts* inner,
                             bk_dirk_report* rep) {
    return dirk_entry(ctx, L, K, mass, tau, k, A1, A2, B, B0, ldb, Y, ldy, max_outer, outer_tol, inner, rep, false);
}

extern "C" int bk_dirk_b0(bk_ctx* ctx, const bk_csr* K, double mass, double tau, int m, const double* A, int s,
                          const double* yn, const double* bn, double* B0, int64_t ldb) {
    int r = enter(ctx);
    if (r) return r;
    ARG_CHECK(ctx, K && K->ctx == ctx, "bk_dirk_b0: matrix NULL or from another ctx");
    int k = 0;
    std::vector<double> A1((size_t)BK_MAX_K * BK_MAX_K), A2((size_t)BK_MAX_K * BK_MAX_K);
    ARG_CHECK(ctx, A && !is_device_ptr(A) && m >= 1 && m <= BK_MAX_K && s >= 1 && s <= BK_MAX_K,
              "bk_dirk_b0: A must be a host m x m tableau");
    ARG_CHECK(ctx, bk_dirk_window(m, A, s, tau, &k, A1.data(), A2.data(), nullptr) == BK_OK,
              "bk_dirk_b0: bad tableau / s / tau (see bk_dirk_window)");
    ARG_CHECK(ctx, mass >= 0.0 && ldb >= k, "bk_dirk_b0: need mass >= 0 and ldb >= k");
    ARG_CHECK(ctx, K->n_local == 0 || (yn && B0), "bk_dirk_b0: NULL y^n / B0");
    BK_TRY
    const int64_t n = K->n_local;
    bool yh, bh = false;
    const double* dy = stage_in(ctx, WS_STAGE_X, yn, n, 1, &yh);
    const double* db = bn ? stage_in(ctx, WS_STAGE_C, bn, n, 1, &bh) : nullptr;
    const bool oh = !is_device_ptr(B0);
    double* dB0 = oh ? (double*)ws_get(ctx, WS_STAGE_Y, (size_t)std::max<int64_t>(n, 1) * ldb * sizeof(double)) : B0;
    double* scratch = (double*)ws_get(ctx, WS_STAGE_G, (size_t)(n + 2 * BK_MAX_K) * sizeof(double));
    r = dirk_b0_impl(ctx, K, mass, tau, m, A, s, dy, db, dB0, ldb, scratch);
    if (r) return r;
    if (oh && n)
        CUDA_OK(ctx, cudaMemcpyAsync(B0, dB0, (size_t)n * ldb * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_OK(ctx, cudaStreamSynchronize(ctx->stream));
    return BK_OK;
    BK_CATCH(ctx)
}

extern "C" int bk_dirk_solve_dc(bk_ctx* ctx, const bk_csr* L, const bk_csr* K, double mass, double tau, int k,
                                const double* A1, const double* A2, const double* B, const double* B0, int64_t ldb,
                                double* Y, int64_t ldy, int max_outer, double outer_tol, const bk_solve_opts* inner,
                                bk_dirk_report* rep) {
    return dirk_entry(ctx, L, K, mass, tau, k, A1, A2, B, B0, ldb, Y, ldy, max_outer, outer_tol, inner, rep, true);
}
