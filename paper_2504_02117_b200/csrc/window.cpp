// window.cpp -- host-side band plan of the windowed apply (include/bk.h
// bk_plan_bands).  Setup work, done once in bk_csr_create
// (the paper times setup apart from the solve); pure host code, tested
// on CPU (tests/test_abi_cpu.py).
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>
#include <vector>

#include "bk.h"

namespace {
constexpr int64_t kGap = 4;        // offsets closer than this share a band
constexpr int kMaxDistinct = 256;  // more distinct offsets: not band structured
}

extern "C" int bk_plan_bands(int64_t n_rows, const int32_t* row_ptr, const int32_t* col, int max_extra,
                             bk_band_plan* out) {
    if (n_rows < 0 || !row_ptr || !out || max_extra < 0) return BK_ERR_ARG;
    std::memset(out, 0, sizeof(*out));
    for (int64_t i = 0; i < n_rows; ++i)
        if (row_ptr[i + 1] < row_ptr[i]) return BK_ERR_ARG;
    if (n_rows > 0 && row_ptr[n_rows] > row_ptr[0] && !col) return BK_ERR_ARG;
    // distinct diagonal offsets d = col - row (stencil operators have a handful)
    std::vector<int64_t> ds;
    int64_t last = INT64_MIN;
    for (int64_t i = 0; i < n_rows; ++i) {
        for (int32_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            const int64_t d = (int64_t)col[p] - i;
            if (d == last) continue;
            last = d;
            if (std::find(ds.begin(), ds.end(), d) == ds.end()) {
                ds.push_back(d);
                if ((int)ds.size() > kMaxDistinct) return BK_OK;   // not band structured
            }
        }
    }
    if (ds.empty()) return BK_OK;
    std::sort(ds.begin(), ds.end());
    std::vector<int64_t> b0, b1;   // bands [b0, b1] of offsets
    for (int64_t d : ds) {
        if (b1.empty() || d > b1.back() + kGap) {
            b0.push_back(d);
            b1.push_back(d);
        } else {
            b1.back() = d;
        }
    }
    if ((int)b0.size() > BK_BAND_MAX) return BK_OK;
    int64_t extra = 0;
    bk_band_plan pl;
    std::memset(&pl, 0, sizeof(pl));
    for (size_t g = 0; g < b0.size(); ++g) {
        if (b0[g] < INT32_MIN / 2 || b1[g] > INT32_MAX / 2) return BK_OK;
        // segment of band g for rows [r0, r0 + T): X rows [r0 + lo, r0 + T + hi),
        // lo / hi even so every segment is 16-byte aligned for any k (r0, T even)
        const int64_t lo = b0[g] - (((b0[g] % 2) + 2) % 2);
        const int64_t e = b1[g] + 1;
        const int64_t hi = e + (((e % 2) + 2) % 2);
        pl.dmin[g] = (int32_t)b0[g];
        pl.dmax[g] = (int32_t)b1[g];
        pl.lo[g] = (int32_t)lo;
        pl.hi[g] = (int32_t)hi;
        pl.width[g] = (int32_t)(b1[g] - b0[g] + 1);
        extra += hi - lo;
    }
    if (extra > max_extra) return BK_OK;
    pl.nbands = (int32_t)b0.size();
    pl.extra_rows = (int32_t)extra;
    int64_t wsum = 0;
    for (int g = 0; g < pl.nbands; ++g) wsum += pl.width[g];
    pl.max_row_nnz = (int32_t)wsum;
    *out = pl;
    return BK_OK;
}
