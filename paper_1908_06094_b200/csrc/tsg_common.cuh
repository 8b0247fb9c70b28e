// Shared definitions of libtsg: grid handle, error state, layout arithmetic,
// and the reference's exact fp64 operation helpers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tsg.h"

struct tsg_grid {
    int rows, cols, levels, flags;
    int row0, global_rows;  // strip origin inside the global patch (multi-GPU); 0 / rows otherwise
    int device, num_sms;
};

namespace tsg {

int fail(int code, const char *fmt, ...);
void clear_error();

#define TSG_CHECK_CUDA(call)                                                              \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return ::tsg::fail(TSG_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

#define TSG_CHECK_LAUNCH()                                                                 \
    do {                                                                                   \
        cudaError_t e_ = cudaGetLastError();                                               \
        if (e_ != cudaSuccess)                                                             \
            return ::tsg::fail(TSG_ECUDA, "kernel launch failed: %s", cudaGetErrorString(e_)); \
    } while (0)

inline int colors_of(int loc) { return loc == TSG_VERTICES ? 1 : (loc == TSG_CELLS ? 2 : 3); }
__host__ __device__ inline int64_t pitch_of(int inner) { return inner <= 1 ? 1 : ((inner + 1) & ~1); }
inline bool valid_loc(int loc) { return loc >= 0 && loc <= 2; }

// Index helper for one structured field: [rows+2][colors][cols+2][pitch].
struct FieldIx {
    int rows, cols, colors;
    int64_t pitch;     // innermost
    int64_t cstride;   // one storage column = pitch
    int64_t colorstr;  // (cols+2) * pitch
    int64_t rowstr;    // colors * (cols+2) * pitch
    __host__ __device__ FieldIx() {}
    __host__ __device__ FieldIx(int r, int c, int ncol, int inner)
        : rows(r), cols(c), colors(ncol), pitch(pitch_of(inner)) {
        cstride = pitch;
        colorstr = (int64_t)(c + 2) * pitch;
        rowstr = (int64_t)ncol * colorstr;
    }
    // logical (i, c, j) with -1 <= i <= rows, -1 <= j <= cols
    __host__ __device__ int64_t at(int i, int c, int j) const {
        return (int64_t)(i + 1) * rowstr + (int64_t)c * colorstr + (int64_t)(j + 1) * cstride;
    }
    __host__ __device__ int64_t elems() const { return (int64_t)(rows + 2) * rowstr; }
};

// Store `v` at interior (i, c, j, k) and at every periodic halo image of it.
__device__ __forceinline__ void store_img(double *f, const FieldIx &F, int i, int c, int j,
                                          int k, double v, int flags) {
    f[F.at(i, c, j) + k] = v;
    int ri = -2, cj = -2;
    if (flags & TSG_PERIODIC_ROWS) {
        if (i == 0) ri = F.rows;
        else if (i == F.rows - 1) ri = -1;
    }
    if (flags & TSG_PERIODIC_COLS) {
        if (j == 0) cj = F.cols;
        else if (j == F.cols - 1) cj = -1;
    }
    if (ri != -2) f[F.at(ri, c, j) + k] = v;
    if (cj != -2) f[F.at(i, c, cj) + k] = v;
    if (ri != -2 && cj != -2) f[F.at(ri, c, cj) + k] = v;
}

// numpy.maximum(a, 0.0) / numpy.minimum(a, 0.0): NaN in `a` propagates, ties return
// the second operand (+0.0) -- measured numpy 2.3 semantics, SURVEY Appendix A.
__device__ __forceinline__ double npmax0(double a) { return (a > 0.0 || a != a) ? a : 0.0; }
__device__ __forceinline__ double npmin0(double a) { return (a < 0.0 || a != a) ? a : 0.0; }

// Explicitly rounded fp64 ops: no contraction into FMA regardless of compiler flags,
// so every result is bitwise what the reference's numpy expression produces.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

// mpdata.py:189-199 / reference.py:18-35
template <int OP>
__device__ __forceinline__ double edge_flux(double p_origin, double p_other, double vn) {
    if (OP == TSG_UPWIND) return add(mul(p_origin, npmax0(vn)), mul(p_other, npmin0(vn)));
    return mul(mul(0.5, vn), add(p_origin, p_other));
}
// reference.py:52-56: max(w,0)*pd(k-1) + min(w,0)*pd(k)
__device__ __forceinline__ double fluz_interior(double w, double p_below, double p_above) {
    return add(mul(npmax0(w), p_below), mul(npmin0(w), p_above));
}

// Vertex->edge slot n of vertex (i, j): edge (i + dI[n], colour n%3 ... ) per
// connectivity.py:66 -- (0,0,0),(0,1,0),(0,2,0),(0,0,-1),(-1,1,-1),(-1,2,0).
// Edge (i,c,j) endpoints (connectivity.py:38-42): origin (i,j); other
// c0 -> (i, j+1), c1 -> (i+1, j+1), c2 -> (i+1, j).

}  // namespace tsg
