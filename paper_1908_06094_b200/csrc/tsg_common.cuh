// Shared definitions of libtsg: grid handle, error state, layout arithmetic,
// and the reference's exact fp64 operation helpers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "tsg.h"

struct tsg_grid {
    int rows, cols, levels, flags;
    int row0, global_rows;  // strip origin inside the global patch (multi-GPU); 0 / rows otherwise
    int device, num_sms;
    void *graph;  // cached two-step CUDA graph of the time loops (mpdata_fused.cu), or NULL
    void *launches;  // prepared fused launches (tensor maps, arguments, grid) keyed by their
                     // arguments (mpdata_fused.cu), or NULL
    void *dyn_ws;    // device workspace of the dynamically dealt fused launches: ticket words,
                     // tile counters of the multi-step loop (mpdata_fused.cu), or NULL
    int64_t dyn_tiles;  // tile counters in dyn_ws
};

namespace tsg {
// dyn_ws header bytes [192, 200): the dynamically dealt TMA reduce's ticket words
// (reduce_tma.cu); [0, 160) belong to the fused launches (mpdata_fused.cu)
constexpr int kDynReduceTicketOff = 192;
void destroy_graph_cache(tsg_grid *g);
void destroy_launch_cache(tsg_grid *g);
int create_dyn_workspace(tsg_grid *g);
void destroy_dyn_workspace(tsg_grid *g);
}

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
// Innermost (level) pitch: even, so level pairs are 16-byte aligned; from 64 levels up a
// multiple of 16, so every element's level run starts on a 128-byte line and a 16-level
// TMA chunk is whole lines (O1280, K = 137: 10.3 vs 10.6 ms per fused step), at <= 19 %
// padding that the tensor maps never fetch (their level extent is the logical count).
#ifndef TSG_LONG_PITCH_ALIGN  // A/B builds only (-DTSG_LONG_PITCH_ALIGN=2)
#define TSG_LONG_PITCH_ALIGN 16
#endif
__host__ __device__ inline int64_t pitch_of(int inner) {
    constexpr int kA = TSG_LONG_PITCH_ALIGN;
    return inner <= 1 ? 1 : (inner < 64 ? ((inner + 1) & ~1) : ((inner + kA - 1) / kA * kA));
}
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

// Division by a run-time invariant divisor in three instructions (Granlund & Montgomery,
// "Division by invariant integers using multiplication", 1994, fig. 4.1): valid for every
// 32-bit n.  Element/level decompositions of the streaming kernels use it instead of
// 64-bit integer division.
struct FastDiv {
    uint32_t d, m, s;
    __host__ __device__ FastDiv() : d(1), m(0), s(0) {}
    __host__ explicit FastDiv(uint32_t div) : d(div), m(0), s(0) {
        if (d <= 1) return;
        uint32_t l = 0;
        while ((1ull << l) < d) ++l;  // ceil(log2 d)
        m = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
        s = l;
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        if (d == 1) return n;
        const uint32_t t = __umulhi(n, m);
        return (t + ((n - t) >> 1)) >> (s - 1);
    }
};

// Points one launch may index with 32 bits (tsg_set_point_limit lowers it for tests).
int64_t point_limit();

// (element, level) decomposition of a flat point index t = ((i*colors + c)*cols + j)*nk + k
// over a band of rows starting at row i0 (for_point_bands splits larger fields).
struct PointDec {
    FastDiv nk, cols, colors;
    uint32_t n;   // number of points of the band (< 2^32)
    int i0;       // first row of the band
    uint32_t e0;  // canonical id of its first element
    __host__ PointDec() {}
    __host__ PointDec(int64_t rows, int ncols, int ncolors, int nlev, int row0 = 0)
        : nk(nlev), cols(ncols), colors(ncolors), n((uint32_t)(rows * ncolors * ncols * nlev)), i0(row0),
          e0((uint32_t)((int64_t)row0 * ncolors * ncols)) {}
    static bool fits(int64_t rows, int ncols, int ncolors, int nlev) {
        return rows * ncolors * ncols * nlev < point_limit();
    }
};

// Launch fn(PointDec) over row bands that each fit a 32-bit point index: one band unless
// the field has more than point_limit() points (an O1280 edge field at 137 levels has
// 2.7e9; a 180 GB GPU holds patches of up to ~22 M vertices at that depth).
template <class Fn>
inline void for_point_bands(int64_t rows, int ncols, int ncolors, int nlev, Fn fn) {
    const int64_t per_row = (int64_t)ncolors * ncols * nlev;
    const int64_t band = std::max<int64_t>(1, point_limit() / std::max<int64_t>(1, per_row));
    for (int64_t r = 0; r < rows; r += band) fn(PointDec(std::min(band, rows - r), ncols, ncolors, nlev, (int)r));
}

struct Pt {
    int i, c, j, k;
    uint32_t e;  // canonical element id
};

__device__ __forceinline__ Pt decompose(uint32_t t, const PointDec &D) {
    Pt p;
    const uint32_t e = D.nk.div(t);
    p.k = (int)(t - e * D.nk.d);
    const uint32_t rest = D.cols.div(e);
    p.j = (int)(e - rest * D.cols.d);
    const uint32_t i = D.colors.div(rest);
    p.c = (int)(rest - i * D.colors.d);
    p.i = (int)i + D.i0;
    p.e = e + D.e0;
    return p;
}

#define TSG_POINTS(t, D)                                                             \
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < (D).n;             \
         t += gridDim.x * blockDim.x)

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

// Launch geometry of the element-line kernels: one warp per element, lanes along the
// contiguous level run (coalesced 256-byte accesses), 8 elements (warps) per block along j,
// one block row per (row, colour) line.  Neighbour pointers, periodic-image offsets and
// table rows are resolved once per element and reused for every level.
constexpr int kWarps = 8;

// resident 256-thread blocks per SM of a kernel (cached occupancy query)
inline int resident_blocks(const void *kernel) {
    static std::mutex mu;
    static std::unordered_map<const void *, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(kernel);
    if (it != cache.end()) return it->second;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, 32 * kWarps, 0) != cudaSuccess || n < 1)
        n = 1;
    cache[kernel] = n;
    return n;
}

// exactly one wave of resident blocks; blocks then walk their share of the work items
inline dim3 one_wave(const void *kernel, int64_t items, int num_sms) {
    int64_t g = (int64_t)num_sms * resident_blocks(kernel);
    if (g > items) g = items;
    return dim3((unsigned)(g < 1 ? 1 : g));
}
inline dim3 line_block() { return dim3(32, kWarps); }

// grid of a grid-stride item kernel (256 threads, `per_thread` items per thread per pass).
// Small sweeps: one wave of resident blocks (no tail wave).  Long sweeps (more than 16
// passes of that wave): one pass per block instead.  Persistent blocks drift apart over
// hundreds of passes, so a neighbour row fetched by one block is evicted from L2 before the
// block that owns it arrives; blocks dispatched in index order keep one coherent wavefront.
// The unfused step at O1280 (2560x2576x137): 25.7 vs 32.7 ms, its flux kernel reading
// 36 vs 56 GB (ncu, tools/prof_unfused_o1280.py); at 279x256x80 (4 passes) the resident
// wave stays ahead (162 vs 167 us).  `persistent` keeps the resident wave whatever the
// length (kernels that prefetch their next item across passes).
inline unsigned item_grid(const void *kernel, int64_t items, int per_thread, int num_sms,
                          bool persistent = false) {
    const int64_t need = (items + 256LL * per_thread - 1) / (256LL * per_thread);
    const int64_t cap = (int64_t)num_sms * resident_blocks(kernel);
    const int64_t g = (!persistent && need > 16 * cap) ? need : std::min(need, cap);
    return (unsigned)std::max<int64_t>(1, g);
}

// launch an element-line kernel over `lines` (row, colour) lines of `cols` elements
template <typename... Params, typename... Args>
inline void launch_lines(void (*kernel)(Params...), int cols, int64_t lines, int num_sms,
                         cudaStream_t st, Args... args) {
    const int64_t items = lines * ((cols + kWarps - 1) / kWarps);
    kernel<<<one_wave((const void *)kernel, items, num_sms), line_block(), 0, st>>>(args...);
}

// launch a flat-row kernel (one warp per table row) over `rows` rows
template <typename... Params, typename... Args>
inline void launch_rows(void (*kernel)(Params...), int64_t rows, int num_sms, cudaStream_t st,
                        Args... args) {
    kernel<<<one_wave((const void *)kernel, (rows + kWarps - 1) / kWarps, num_sms), line_block(), 0,
             st>>>(args...);
}

#define TSG_LINES(F, i, c, j)                                                                  \
    for (int item_ = blockIdx.x, ngrp_ = ((F).cols + kWarps - 1) / kWarps,                       \
             nitem_ = (F).rows * (F).colors * ngrp_;                                             \
         item_ < nitem_; item_ += gridDim.x)                                                     \
        for (int line_ = item_ / ngrp_, j = (item_ - line_ * ngrp_) * kWarps + threadIdx.y,      \
                 i = line_ / (F).colors, c = line_ - i * (F).colors, once_ = 1;                  \
             once_ && j < (F).cols; once_ = 0)

// offsets of the periodic halo images of element (i, j) (0 = none)
struct Img {
    int64_t dr, dc;
};
__device__ __forceinline__ Img images(const FieldIx &F, int i, int j, int flags) {
    Img m{0, 0};
    if (flags & TSG_PERIODIC_ROWS) {
        if (i == 0) m.dr = (int64_t)F.rows * F.rowstr;
        else if (i == F.rows - 1) m.dr = -(int64_t)F.rows * F.rowstr;
    }
    if (flags & TSG_PERIODIC_COLS) {
        if (j == 0) m.dc = (int64_t)F.cols * F.cstride;
        else if (j == F.cols - 1) m.dc = -(int64_t)F.cols * F.cstride;
    }
    return m;
}
__device__ __forceinline__ void put(double *o, const Img &m, int k, double v) {
    o[k] = v;
    if (m.dr | m.dc) {
        if (m.dr) o[m.dr + k] = v;
        if (m.dc) o[m.dc + k] = v;
        if (m.dr && m.dc) o[m.dr + m.dc + k] = v;
    }
}

// 16-byte level pairs: every structured field has an even pitch, so (k, k+1) with k even
// is aligned; the partner of the last odd level is padding, which may be written.
__device__ __forceinline__ double2 ld2(const double *p) { return *reinterpret_cast<const double2 *>(p); }
__device__ __forceinline__ void st2(double *p, double2 v) { *reinterpret_cast<double2 *>(p) = v; }
__device__ __forceinline__ void put2(double *o, const Img &m, int k, double2 v) {
    st2(o + k, v);
    if (m.dr | m.dc) {
        if (m.dr) st2(o + m.dr + k, v);
        if (m.dc) st2(o + m.dc + k, v);
        if (m.dr && m.dc) st2(o + m.dr + m.dc + k, v);
    }
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
    if (OP != TSG_CENTRED) return add(mul(p_origin, npmax0(vn)), mul(p_other, npmin0(vn)));
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
