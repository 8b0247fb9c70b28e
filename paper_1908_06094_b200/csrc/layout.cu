// Field layout kernels: flat(any numbering) <-> structured reorder, periodic halo,
// on-device index maps, synthetic fills and the mass diagnostic.
//
// All of these are HBM-bound integer/byte-movement kernels: threads are mapped with the
// innermost (level) axis fastest so both sides of every copy are coalesced, and grids
// are sized as a multiple of the SM count (grid-stride loops).
#include "tsg_common.cuh"
#include "tsg_offsets.cuh"

namespace tsg {

static inline int grid_for(int64_t work, int threads, int num_sms) {
    int64_t blocks = (work + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms * 16;
    if (blocks > cap) blocks = cap;
    return (int)(blocks < 1 ? 1 : blocks);
}

// -- pack / unpack: the "Atlas -> structured" reorder (kernels.py:107-134) ------------

__global__ void pack_kernel(FieldIx F, int inner, PointDec D, const double *__restrict__ flat,
                            const int64_t *__restrict__ forward, double *__restrict__ f,
                            int flags) {
    TSG_POINTS(t, D) {
        const Pt p = decompose(t, D);
        const int i = p.i, c = p.c, j = p.j, k = p.k;
        const int64_t id = p.e;
        int64_t rank = forward ? forward[id] : id;
        store_img(f, F, i, c, j, k, flat[rank * inner + k], flags);
    }
}

__global__ void unpack_kernel(FieldIx F, int inner, PointDec D, const double *__restrict__ f,
                              const int64_t *__restrict__ forward, double *__restrict__ flat) {
    TSG_POINTS(t, D) {
        const Pt p = decompose(t, D);
        const int i = p.i, c = p.c, j = p.j, k = p.k;
        const int64_t id = p.e;
        int64_t rank = forward ? forward[id] : id;
        flat[rank * inner + k] = f[F.at(i, c, j) + k];
    }
}

// element-line variants (one warp per element, lanes along the level run) for long runs
__global__ void __launch_bounds__(256) pack_lines_kernel(FieldIx F, int inner,
                                                         const double *__restrict__ flat,
                                                         const int64_t *__restrict__ forward,
                                                         double *__restrict__ f, int flags) {
    TSG_LINES(F, i, c, j) {
        const int64_t id = ((int64_t)i * F.colors + c) * F.cols + j;
        const double *src = flat + (forward ? __ldg(forward + id) : id) * inner;
        double *o = f + F.at(i, c, j);
        const Img m = images(F, i, j, flags);
        if ((inner & 1) == 0) {  // level pairs: flat rows are 16-byte aligned too
            for (int k = 2 * threadIdx.x; k < inner; k += 64) put2(o, m, k, ld2(src + k));
        } else {
            for (int k = threadIdx.x; k < inner; k += 32) put(o, m, k, src[k]);
        }
    }
}

__global__ void __launch_bounds__(256) unpack_lines_kernel(FieldIx F, int inner,
                                                           const double *__restrict__ f,
                                                           const int64_t *__restrict__ forward,
                                                           double *__restrict__ flat) {
    TSG_LINES(F, i, c, j) {
        const int64_t id = ((int64_t)i * F.colors + c) * F.cols + j;
        double *dst = flat + (forward ? __ldg(forward + id) : id) * inner;
        const double *src = f + F.at(i, c, j);
        if ((inner & 1) == 0) {
            for (int k = 2 * threadIdx.x; k < inner; k += 64) st2(dst + k, ld2(src + k));
        } else {
            for (int k = threadIdx.x; k < inner; k += 32) dst[k] = src[k];
        }
    }
}

// level-pair item variants for even level counts: one thread per (element, level pair),
// items flattened over the field so every lane is busy whatever the level count, with
// kItemUnroll items per thread in flight (the element-line kernels leave 24 of 32 lanes
// idle in the second pass of an 80-level run and are latency-bound).
constexpr int kItemUnroll = 4;

// The gathered side of pack is a dependent load (forward[e], then the flat row), so the
// next batch's element ids and ranks are fetched while this batch's rows are in flight:
// one load latency per batch instead of two (the unpack side stores through the rank and
// does not wait on it).  One item per batch: the fewest registers, so the most resident
// threads -- 1024x1024x80 SN / UN / HN 433 / 450 / 448 us (0.93-0.96 of the copy peak)
// against 445-470 us with two items, 520-540 with three and 529-548 us for round 1's
// unpipelined four (tools/pack_variants.py, TSG_PACK_V A/B build).
constexpr int kPackUnroll = 1;
// FA = false: an odd level count (flat rows not 16-byte aligned) -- the flat side is read
// as two scalars, the field side still stored as aligned pairs (even pitch), the last
// pair's second value (the first padding slot) as 0.
template <int U, bool FA = true>
__global__ void __launch_bounds__(256) pack_pairs_kernel(FieldIx F, int inner, PointDec D,
                                                         const double *__restrict__ flat,
                                                         const int64_t *__restrict__ forward,
                                                         double *__restrict__ f, int flags) {
    constexpr int kItemUnroll = U;
    const uint32_t T = gridDim.x * blockDim.x;
    Pt p[kItemUnroll];
    int64_t rank[kItemUnroll];
    auto fetch = [&](uint32_t b) {
#pragma unroll
        for (int u = 0; u < kItemUnroll; ++u) {
            const uint32_t t = b + u * T;
            if (t < D.n) {
                p[u] = decompose(t, D);
                rank[u] = forward ? __ldg(forward + p[u].e) : p[u].e;
            }
        }
    };
    uint32_t base = blockIdx.x * blockDim.x + threadIdx.x;
    fetch(base);
    for (; base < D.n; base += kItemUnroll * T) {
        double2 v[kItemUnroll];
        Pt q[kItemUnroll];
#pragma unroll
        for (int u = 0; u < kItemUnroll; ++u) {
            if (base + u * T < D.n) {
                if constexpr (FA) {
                    v[u] = __ldg(reinterpret_cast<const double2 *>(flat + rank[u] * inner + 2 * p[u].k));
                } else {
                    const double *row = flat + rank[u] * inner + 2 * p[u].k;
                    v[u] = make_double2(__ldg(row), 2 * p[u].k + 1 < inner ? __ldg(row + 1) : 0.0);
                }
                q[u] = p[u];
            }
        }
        if (base + kItemUnroll * T < D.n) fetch(base + kItemUnroll * T);
#pragma unroll
        for (int u = 0; u < kItemUnroll; ++u) {
            if (base + u * T >= D.n) break;
            put2(f + F.at(q[u].i, q[u].c, q[u].j), images(F, q[u].i, q[u].j, flags), 2 * q[u].k, v[u]);
        }
    }
}

template <bool FA = true>
__global__ void __launch_bounds__(256) unpack_pairs_kernel(FieldIx F, int inner, PointDec D,
                                                           const double *__restrict__ f,
                                                           const int64_t *__restrict__ forward,
                                                           double *__restrict__ flat) {
    const uint32_t T = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < D.n; base += kItemUnroll * T) {
        double2 v[kItemUnroll];
        Pt p[kItemUnroll];
#pragma unroll
        for (int u = 0; u < kItemUnroll; ++u) {
            const uint32_t t = base + u * T;
            if (t < D.n) {
                p[u] = decompose(t, D);
                v[u] = __ldg(reinterpret_cast<const double2 *>(f + F.at(p[u].i, p[u].c, p[u].j) + 2 * p[u].k));
            }
        }
#pragma unroll
        for (int u = 0; u < kItemUnroll; ++u) {
            if (base + u * T >= D.n) break;
            const int64_t rank = forward ? __ldg(forward + p[u].e) : p[u].e;
            if constexpr (FA) {
                st2(flat + rank * inner + 2 * p[u].k, v[u]);
            } else {
                double *row = flat + rank * inner + 2 * p[u].k;
                row[0] = v[u].x;
                if (2 * p[u].k + 1 < inner) row[1] = v[u].y;
            }
        }
    }
}

// Grids of the level-pair reorders.  Long sweeps (more than 16 passes of one resident wave,
// item_grid's rule) take one pass per block -- O1280 edge field at 137 levels: pack 8.0 vs
// 10.2 ms, unpack 6.5 vs 9.3 ms; at 136 levels unpack 6.4 vs 7.5 ms -- against grid_for's
// 16 blocks per SM walking the field in grid-stride passes, which stays ahead on short
// sweeps (279x256x80 unpack 42.6 vs 44.8 us) and for the even pack, whose pipelined rank
// fetch wants several items per thread (tools/reorder_probe.py).
static unsigned reorder_grid(const void *kernel, int64_t n, int per, int num_sms) {
    const unsigned g = item_grid(kernel, n, per, num_sms);
    return (int64_t)g * 256 * per >= n ? g : (unsigned)grid_for((n + per - 1) / per, 256, num_sms);
}
#define TSG_ODD_GRID(K, n, per) reorder_grid((const void *)K, n, per, g->num_sms)
#define TSG_EVEN_GRID(K, n, per, persist) \
    ((persist) ? (unsigned)grid_for(((n) + (per) - 1) / (per), 256, g->num_sms) : reorder_grid((const void *)K, n, per, g->num_sms))
static bool pairs_ok(int inner, const void *flat) {
    return inner >= 16 && (inner & 1) == 0 && (reinterpret_cast<uintptr_t>(flat) % 16) == 0;
}

// -- periodic halo (executors.py:74-86): rows then columns, corners wrap both ways ----

__global__ void halo_kernel(FieldIx F, int inner, double *__restrict__ f, int flags) {
    // ring positions: top + bottom storage rows (cols+2 each), then left + right
    // storage columns of the interior rows.
    const int W = F.cols + 2;
    const int64_t nring = 2LL * W + 2LL * F.rows;
    const int64_t n = nring * F.colors * inner;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = t / inner;
        int k = (int)(t - p * inner);
        int c = (int)(p % F.colors);
        p /= F.colors;
        int si, sj;  // storage coordinates of the halo cell
        if (p < 2LL * W) {
            if (!(flags & TSG_PERIODIC_ROWS)) continue;
            si = p < W ? 0 : F.rows + 1;
            sj = (int)(p % W);
        } else {
            if (!(flags & TSG_PERIODIC_COLS)) continue;
            p -= 2LL * W;
            si = 1 + (int)(p % F.rows);
            sj = p < F.rows ? 0 : F.cols + 1;
        }
        // source: wrap logical coordinates onto the interior
        int li = si - 1, lj = sj - 1;
        if (flags & TSG_PERIODIC_ROWS) li = (li + F.rows) % F.rows;
        if (flags & TSG_PERIODIC_COLS) lj = (lj + F.cols) % F.cols;
        if (li < 0 || li >= F.rows) continue;  // strip halo row: owned by the exchange
        f[(int64_t)si * F.rowstr + (int64_t)c * F.colorstr + (int64_t)sj * F.cstride + k] =
            f[F.at(li, c, lj) + k];
    }
}

// -- synthetic counter-hash fill -------------------------------------------------------

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

__global__ void fill_hash_kernel(FieldIx F, int inner, PointDec D, int row0, uint64_t seed,
                                 double lo, double hi, double *__restrict__ f, int flags) {
    TSG_POINTS(t, D) {
        const Pt p = decompose(t, D);
        const int i = p.i, c = p.c, j = p.j, k = p.k;
        const int64_t id = p.e;
        // global canonical id of the element: decomposition-invariant
        uint64_t gid = ((uint64_t)(i + row0) * F.colors + c) * F.cols + j;
        uint64_t h = mix64(seed * 0x9e3779b97f4a7c15ULL + mix64(gid * 4099ULL + (uint64_t)k));
        double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
        store_img(f, F, i, c, j, k, lo + (hi - lo) * u, flags);
    }
}

// -- mass diagnostic (mpdata.py:496-500): deterministic two-pass sum -----------------

constexpr int kMassBlocks = 1024;

__global__ void mass_partial_kernel(FieldIx Fp, FieldIx Fd, int K, const double *__restrict__ pd,
                                    const double *__restrict__ dual, double *__restrict__ work) {
    __shared__ double red[256];
    const int64_t n = (int64_t)Fp.rows * Fp.cols * K;
    double acc = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = t / K;
        int k = (int)(t - v * K);
        int i = (int)(v / Fp.cols), j = (int)(v % Fp.cols);
        acc += pd[Fp.at(i, 0, j) + k] * dual[Fd.at(i, 0, j)];
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) work[blockIdx.x] = red[0];
}

__global__ void mass_final_kernel(const double *__restrict__ work, int n, double *out) {
    __shared__ double red[kMassBlocks];
    for (int t = threadIdx.x; t < kMassBlocks; t += blockDim.x) red[t] = t < n ? work[t] : 0.0;
    __syncthreads();
    for (int s = kMassBlocks / 2; s > 0; s >>= 1) {
        for (int t = threadIdx.x; t < s; t += blockDim.x) red[t] += red[t + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

// -- on-device index maps (connectivity.py:130-194) -----------------------------------

__global__ void table_kernel(int rows, int cols, int from_loc, int to_loc,
                             const int64_t *__restrict__ from_inverse,
                             const int64_t *__restrict__ to_forward, int64_t *__restrict__ out) {
    const int rel = from_loc * 3 + to_loc;
    const int width = c_rel_width[rel];
    const int cf = c_colors[from_loc], ct = c_colors[to_loc];
    const int64_t n = (int64_t)rows * cf * cols * width;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = t / width;
        int slot = (int)(t - r * width);
        int64_t id = from_inverse ? from_inverse[r] : r;
        int j = (int)(id % cols);
        int64_t rest = id / cols;
        int c = (int)(rest % cf);
        int i = (int)(rest / cf);
        const int8_t *o = c_offsets[rel][c][slot];
        int ni = (i + o[0] + rows) % rows, nj = (j + o[2] + cols) % cols;
        int64_t nid = ((int64_t)ni * ct + o[1]) * cols + nj;
        out[t] = to_forward ? to_forward[nid] : nid;
    }
}

__global__ void signs_kernel(int rows, int cols, double *__restrict__ out) {
    const int64_t n = (int64_t)rows * cols * 6;
    const int relVE = TSG_VERTICES * 3 + TSG_EDGES, relEV = TSG_EDGES * 3 + TSG_VERTICES;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = t / 6;
        int slot = (int)(t - v * 6);
        int i = (int)(v / cols), j = (int)(v % cols);
        const int8_t *o = c_offsets[relVE][0][slot];
        int ei = (i + o[0] + rows) % rows, ec = o[1], ej = (j + o[2] + cols) % cols;
        // the two endpoints of edge (ei, ec, ej)
        int64_t lower = INT64_MAX;
        for (int e = 0; e < 2; ++e) {
            const int8_t *q = c_offsets[relEV][ec][e];
            int64_t vid = (int64_t)((ei + q[0] + rows) % rows) * cols + (ej + q[2] + cols) % cols;
            lower = vid < lower ? vid : lower;
        }
        out[t] = (lower == v) ? 1.0 : -1.0;
    }
}


// -- host LinearLayout buffer <-> structured device field (layouts.py:55-104) --------
// `lay` = {front_pad, stride_row, stride_color, stride_column, stride_level, stride_extra}
// in elements; the host buffer carries a halo of width `h`.
struct HostLayout {
    int64_t front, s[5];
};

// rows [i0, i1) of the field (the whole field, or one band of a streamed upload)
__global__ void pack_strided_kernel(FieldIx F, int inner, int inner_is_level, HostLayout L, int h,
                                    const double *__restrict__ src, double *__restrict__ f,
                                    int flags, int i0, int i1) {
    const int64_t n = (int64_t)(i1 - i0) * F.colors * F.cols * inner;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t id = t / inner;
        int q = (int)(t - id * inner);
        int j = (int)(id % F.cols);
        int64_t rest = id / F.cols;
        int c = (int)(rest % F.colors);
        int i = i0 + (int)(rest / F.colors);
        int64_t off = L.front + (int64_t)(i + h) * L.s[0] + (int64_t)c * L.s[1] +
                      (int64_t)(j + h) * L.s[2] + (int64_t)q * L.s[inner_is_level ? 3 : 4];
        store_img(f, F, i, c, j, q, src[off], flags);
    }
}

// host storage rows [s0, s1) (halo rows included: 0 .. rows + 2h)
__global__ void unpack_strided_kernel(FieldIx F, int inner, int inner_is_level, HostLayout L,
                                      int h, const double *__restrict__ f,
                                      double *__restrict__ dst, int s0, int s1) {
    const int Cc = F.cols + 2 * h;
    const int64_t n = (int64_t)(s1 - s0) * F.colors * Cc * inner;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t id = t / inner;
        int q = (int)(t - id * inner);
        int sj = (int)(id % Cc);
        int64_t rest = id / Cc;
        int c = (int)(rest % F.colors);
        int si = s0 + (int)(rest / F.colors);
        // host halo cells are periodic images of the interior
        int i = ((si - h) % F.rows + F.rows) % F.rows, j = ((sj - h) % F.cols + F.cols) % F.cols;
        int64_t off = L.front + (int64_t)si * L.s[0] + (int64_t)c * L.s[1] + (int64_t)sj * L.s[2] +
                      (int64_t)q * L.s[inner_is_level ? 3 : 4];
        dst[off] = f[F.at(i, c, j) + q];
    }
}

// -- cell weights w[c, n] = length(e_n) / area(c) (mpdata.py:152-169) ------------------

__global__ void cell_weights_kernel(FieldIx Fl, FieldIx Fa, FieldIx Fw, const double *__restrict__ length,
                                    const double *__restrict__ area, double *__restrict__ w,
                                    int flags) {
    const int rel = TSG_CELLS * 3 + TSG_EDGES;
    const int64_t n = (int64_t)Fw.rows * 2 * Fw.cols * 3;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t id = t / 3;
        int s = (int)(t - id * 3);
        int j = (int)(id % Fw.cols);
        int64_t rest = id / Fw.cols;
        int c = (int)(rest % 2);
        int i = (int)(rest / 2);
        const int8_t *o = c_offsets[rel][c][s];
        double l = length[Fl.at(i + o[0], o[1], j + o[2])];
        store_img(w, Fw, i, c, j, s, dvd(l, area[Fa.at(i, c, j)]), flags);
    }
}

// -- numberings (layouts.py:134-279): SN identity, UN colour interleave, HN Hilbert ----

__device__ __forceinline__ void hilbert_xy(int64_t n, int64_t d, int64_t &x, int64_t &y) {
    x = 0;
    y = 0;
    int64_t t = d;
    for (int64_t s = 1; s < n; s *= 2) {
        int64_t rx = 1 & (t / 2);
        int64_t ry = 1 & (t ^ rx);
        if (ry == 0) {
            if (rx == 1) {
                x = s - 1 - x;
                y = s - 1 - y;
            }
            int64_t tmp = x;
            x = y;
            y = tmp;
        }
        x += s * rx;
        y += s * ry;
        t /= 4;
    }
}

__global__ void perm_simple_kernel(int rows, int cols, int colors, int un, int64_t *__restrict__ fwd) {
    const int64_t n = (int64_t)rows * colors * cols;
    for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < n;
         id += (int64_t)gridDim.x * blockDim.x) {
        if (!un) {
            fwd[id] = id;
            continue;
        }
        int j = (int)(id % cols);
        int64_t rest = id / cols;
        int c = (int)(rest % colors);
        int64_t i = rest / colors;
        fwd[id] = (i * cols + j) * colors + c;
    }
}

constexpr int kHilbertBlock = 1024;

__device__ __forceinline__ bool hilbert_keep(int64_t side, int64_t d, int gx, int gy, int64_t &x,
                                             int64_t &y) {
    hilbert_xy(side, d, x, y);
    return x < gx && y < gy;
}

__global__ void hilbert_count_kernel(int64_t side, int gx, int gy, int64_t *__restrict__ counts) {
    int64_t d = (int64_t)blockIdx.x * kHilbertBlock + threadIdx.x, x, y;
    bool keep = d < side * side && hilbert_keep(side, d, gx, gy, x, y);
    int c = __syncthreads_count(keep);
    if (threadIdx.x == 0) counts[blockIdx.x] = c;
}

__global__ void exclusive_scan_kernel(int64_t *__restrict__ v, int64_t n) {
    __shared__ int64_t part[1024];
    const int64_t per = (n + blockDim.x - 1) / blockDim.x;
    const int64_t b = threadIdx.x * per, e = b + per < n ? b + per : n;
    int64_t s = 0;
    for (int64_t q = b; q < e; ++q) s += v[q];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t run = 0;
        for (int q = 0; q < (int)blockDim.x; ++q) {
            int64_t tmp = part[q];
            part[q] = run;
            run += tmp;
        }
    }
    __syncthreads();
    int64_t run = part[threadIdx.x];
    for (int64_t q = b; q < e; ++q) {
        int64_t tmp = v[q];
        v[q] = run;
        run += tmp;
    }
}

__global__ void hilbert_write_kernel(int64_t side, int gx, int gy, int cols, int cells,
                                     const int64_t *__restrict__ offsets, int64_t *__restrict__ fwd) {
    __shared__ int warp_sums[kHilbertBlock / 32];
    int64_t d = (int64_t)blockIdx.x * kHilbertBlock + threadIdx.x, x = 0, y = 0;
    bool keep = d < side * side && hilbert_keep(side, d, gx, gy, x, y);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned ballot = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_sums[warp] = __popc(ballot);
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int w = 0; w < kHilbertBlock / 32; ++w) {
            int tmp = warp_sums[w];
            warp_sums[w] = run;
            run += tmp;
        }
    }
    __syncthreads();
    if (keep) {
        int64_t rank = offsets[blockIdx.x] + warp_sums[warp] + __popc(ballot & ((1u << lane) - 1));
        // vertices embed as (i, j); cells as (i, 2j + c) (layouts.py:221-232)
        int64_t id = cells ? (x * 2 + (y % 2)) * cols + y / 2 : x * cols + y;
        fwd[id] = rank;
    }
}

}  // namespace tsg

using namespace tsg;

#define CHECK_GRID(g) \
    if (!(g)) return fail(TSG_EVALUE, "grid is NULL")

extern "C" int tsg_pack(const tsg_grid *g, int loc, int inner, const double *flat,
                        const int64_t *forward, double *field, tsg_stream s) {
    CHECK_GRID(g);
    if (!valid_loc(loc) || inner < 1) return fail(TSG_EVALUE, "tsg_pack: bad location/inner");
    if (!flat || !field) return fail(TSG_EVALUE, "tsg_pack: NULL array");
    FieldIx F(g->rows, g->cols, colors_of(loc), inner);
    if (pairs_ok(inner, flat)) {
        for_point_bands(g->rows, g->cols, F.colors, inner / 2, [&](const PointDec &Dp) {
            pack_pairs_kernel<kPackUnroll><<<TSG_EVEN_GRID((pack_pairs_kernel<kPackUnroll>), Dp.n, kPackUnroll, true),
                                             256, 0, (cudaStream_t)s>>>(F, inner, Dp, flat, forward, field,
                                                                        g->flags);
        });
    } else if (inner >= 16 && (inner & 1)) {  // odd: scalar flat side, aligned field pairs
        for_point_bands(g->rows, g->cols, F.colors, (inner + 1) / 2, [&](const PointDec &Dp) {
            pack_pairs_kernel<kPackUnroll, false><<<TSG_ODD_GRID((pack_pairs_kernel<kPackUnroll, false>), Dp.n, 1), 256, 0,
                                                   (cudaStream_t)s>>>(
                F, inner, Dp, flat, forward, field, g->flags);
        });
    } else if (inner >= 16) {
        launch_lines(pack_lines_kernel, g->cols, (int64_t)g->rows * F.colors, g->num_sms,
                     (cudaStream_t)s, F, inner, flat, forward, field, g->flags);
    } else {
        for_point_bands(g->rows, g->cols, F.colors, inner, [&](const PointDec &D) {
            pack_kernel<<<grid_for(D.n, 256, g->num_sms), 256, 0, (cudaStream_t)s>>>(F, inner, D, flat,
                                                                                     forward, field, g->flags);
        });
    }
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_unpack(const tsg_grid *g, int loc, int inner, const double *field,
                          const int64_t *forward, double *flat, tsg_stream s) {
    CHECK_GRID(g);
    if (!valid_loc(loc) || inner < 1) return fail(TSG_EVALUE, "tsg_unpack: bad location/inner");
    if (!flat || !field) return fail(TSG_EVALUE, "tsg_unpack: NULL array");
    FieldIx F(g->rows, g->cols, colors_of(loc), inner);
    if (pairs_ok(inner, flat)) {
        for_point_bands(g->rows, g->cols, F.colors, inner / 2, [&](const PointDec &Dp) {
            unpack_pairs_kernel<<<TSG_EVEN_GRID((unpack_pairs_kernel<true>), Dp.n, kItemUnroll, false), 256, 0,
                                  (cudaStream_t)s>>>(F, inner, Dp, field, forward, flat);
        });
    } else if (inner >= 16 && (inner & 1)) {  // odd: aligned field pairs, scalar flat side
        for_point_bands(g->rows, g->cols, F.colors, (inner + 1) / 2, [&](const PointDec &Dp) {
            unpack_pairs_kernel<false><<<TSG_ODD_GRID((unpack_pairs_kernel<false>), Dp.n, kItemUnroll), 256, 0,
                                         (cudaStream_t)s>>>(F, inner, Dp, field, forward, flat);
        });
    } else if (inner >= 16) {
        launch_lines(unpack_lines_kernel, g->cols, (int64_t)g->rows * F.colors, g->num_sms,
                     (cudaStream_t)s, F, inner, field, forward, flat);
    } else {
        for_point_bands(g->rows, g->cols, F.colors, inner, [&](const PointDec &D) {
            unpack_kernel<<<grid_for(D.n, 256, g->num_sms), 256, 0, (cudaStream_t)s>>>(F, inner, D, field,
                                                                                       forward, flat);
        });
    }
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_halo_update(const tsg_grid *g, int loc, int inner, double *field,
                               tsg_stream s) {
    CHECK_GRID(g);
    if (!valid_loc(loc) || inner < 1) return fail(TSG_EVALUE, "tsg_halo_update: bad location/inner");
    if (!field) return fail(TSG_EVALUE, "tsg_halo_update: NULL field");
    FieldIx F(g->rows, g->cols, colors_of(loc), inner);
    int64_t n = (2LL * (g->cols + 2) + 2LL * g->rows) * F.colors * inner;
    halo_kernel<<<grid_for(n, 256, g->num_sms), 256, 0, (cudaStream_t)s>>>(F, inner, field,
                                                                           g->flags);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_fill_hash(const tsg_grid *g, int loc, int inner, uint64_t seed, double lo,
                             double hi, double *field, tsg_stream s) {
    CHECK_GRID(g);
    if (!valid_loc(loc) || inner < 1) return fail(TSG_EVALUE, "tsg_fill_hash: bad location/inner");
    if (!field) return fail(TSG_EVALUE, "tsg_fill_hash: NULL field");
    FieldIx F(g->rows, g->cols, colors_of(loc), inner);
    for_point_bands(g->rows, g->cols, F.colors, inner, [&](const PointDec &D) {
        fill_hash_kernel<<<grid_for(D.n, 256, g->num_sms), 256, 0, (cudaStream_t)s>>>(
            F, inner, D, g->row0, seed, lo, hi, field, g->flags);
    });
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_total_mass(const tsg_grid *g, const double *pd, const double *dual,
                              double *work, double *out, tsg_stream s) {
    CHECK_GRID(g);
    if (!pd || !dual || !work || !out) return fail(TSG_EVALUE, "tsg_total_mass: NULL array");
    FieldIx Fp(g->rows, g->cols, 1, g->levels), Fd(g->rows, g->cols, 1, 1);
    mass_partial_kernel<<<kMassBlocks, 256, 0, (cudaStream_t)s>>>(Fp, Fd, g->levels, pd, dual, work);
    mass_final_kernel<<<1, 256, 0, (cudaStream_t)s>>>(work, kMassBlocks, out);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_build_neighbor_table(int rows, int cols, int from_loc, int to_loc,
                                        const int64_t *from_inverse, const int64_t *to_forward,
                                        int64_t *out, tsg_stream s) {
    if (rows < 2 || cols < 2) return fail(TSG_EVALUE, "rows and cols must each be >= 2");
    if (!valid_loc(from_loc) || !valid_loc(to_loc))
        return fail(TSG_EVALUE, "no structured relation %d -> %d", from_loc, to_loc);
    if (!out) return fail(TSG_EVALUE, "tsg_build_neighbor_table: NULL output");
    int width = host_rel_width(from_loc, to_loc);
    int64_t n = (int64_t)rows * colors_of(from_loc) * cols * width;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    table_kernel<<<grid_for(n, 256, sms), 256, 0, (cudaStream_t)s>>>(rows, cols, from_loc, to_loc,
                                                                    from_inverse, to_forward, out);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_edge_signs(int rows, int cols, double *out, tsg_stream s) {
    if (rows < 2 || cols < 2) return fail(TSG_EVALUE, "rows and cols must each be >= 2");
    if (!out) return fail(TSG_EVALUE, "tsg_edge_signs: NULL output");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    signs_kernel<<<grid_for((int64_t)rows * cols * 6, 256, sms), 256, 0, (cudaStream_t)s>>>(rows, cols,
                                                                                          out);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}


static int to_layout(const int64_t *lay, HostLayout &L) {
    if (!lay) return fail(TSG_EVALUE, "host layout is NULL");
    L.front = lay[0];
    for (int q = 0; q < 5; ++q) L.s[q] = lay[1 + q];
    return TSG_OK;
}

extern "C" int tsg_pack_strided_rows(const tsg_grid *g, int loc, int inner, const double *src,
                                     const int64_t *layout6, int host_halo, int row_lo, int row_hi,
                                     double *field, tsg_stream s) {
    CHECK_GRID(g);
    if (!valid_loc(loc) || inner < 1) return fail(TSG_EVALUE, "tsg_pack_strided: bad location/inner");
    if (!src || !field) return fail(TSG_EVALUE, "tsg_pack_strided: NULL array");
    if (row_lo < 0 || row_hi > g->rows || row_lo > row_hi)
        return fail(TSG_EVALUE, "row range [%d, %d) outside [0, %d)", row_lo, row_hi, g->rows);
    HostLayout L;
    if (int rc = to_layout(layout6, L)) return rc;
    // inner runs along `level` when the level stride is set, else along `extra`
    int inner_is_level = inner == 1 ? 1 : (L.s[3] != 0);
    FieldIx F(g->rows, g->cols, colors_of(loc), inner);
    int64_t n = (int64_t)(row_hi - row_lo) * F.colors * g->cols * inner;
    if (n == 0) return TSG_OK;
    pack_strided_kernel<<<grid_for(n, 256, g->num_sms), 256, 0, (cudaStream_t)s>>>(
        F, inner, inner_is_level, L, host_halo, src, field, g->flags, row_lo, row_hi);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_pack_strided(const tsg_grid *g, int loc, int inner, const double *src,
                                const int64_t *layout6, int host_halo, double *field, tsg_stream s) {
    CHECK_GRID(g);
    return tsg_pack_strided_rows(g, loc, inner, src, layout6, host_halo, 0, g->rows, field, s);
}

extern "C" int tsg_unpack_strided_rows(const tsg_grid *g, int loc, int inner, const double *field,
                                       const int64_t *layout6, int host_halo, int srow_lo, int srow_hi,
                                       double *dst, tsg_stream s) {
    CHECK_GRID(g);
    if (!valid_loc(loc) || inner < 1) return fail(TSG_EVALUE, "tsg_unpack_strided: bad location/inner");
    if (!dst || !field) return fail(TSG_EVALUE, "tsg_unpack_strided: NULL array");
    if (host_halo < 0 || host_halo > g->rows || host_halo > g->cols)
        return fail(TSG_EVALUE, "host halo %d out of range", host_halo);
    if (srow_lo < 0 || srow_hi > g->rows + 2 * host_halo || srow_lo > srow_hi)
        return fail(TSG_EVALUE, "storage row range [%d, %d) outside [0, %d)", srow_lo, srow_hi,
                    g->rows + 2 * host_halo);
    HostLayout L;
    if (int rc = to_layout(layout6, L)) return rc;
    int inner_is_level = inner == 1 ? 1 : (L.s[3] != 0);
    FieldIx F(g->rows, g->cols, colors_of(loc), inner);
    int64_t n = (int64_t)(srow_hi - srow_lo) * F.colors * (g->cols + 2 * host_halo) * inner;
    if (n == 0) return TSG_OK;
    unpack_strided_kernel<<<grid_for(n, 256, g->num_sms), 256, 0, (cudaStream_t)s>>>(
        F, inner, inner_is_level, L, host_halo, field, dst, srow_lo, srow_hi);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_unpack_strided(const tsg_grid *g, int loc, int inner, const double *field,
                                  const int64_t *layout6, int host_halo, double *dst, tsg_stream s) {
    CHECK_GRID(g);
    return tsg_unpack_strided_rows(g, loc, inner, field, layout6, host_halo, 0, g->rows + 2 * host_halo,
                                   dst, s);
}

extern "C" int tsg_cell_weights(const tsg_grid *g, const double *length, const double *area,
                                double *weights, tsg_stream s) {
    CHECK_GRID(g);
    if (!length || !area || !weights) return fail(TSG_EVALUE, "tsg_cell_weights: NULL array");
    FieldIx Fl(g->rows, g->cols, 3, 1), Fa(g->rows, g->cols, 2, 1), Fw(g->rows, g->cols, 2, 3);
    int64_t n = (int64_t)g->rows * 2 * g->cols * 3;
    cell_weights_kernel<<<grid_for(n, 256, g->num_sms), 256, 0, (cudaStream_t)s>>>(
        Fl, Fa, Fw, length, area, weights, g->flags);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

static int64_t hilbert_side(int rows, int cols, int loc) {
    int64_t gx = rows, gy = loc == TSG_CELLS ? 2LL * cols : cols, side = 2;
    while (side < (gx > gy ? gx : gy)) side *= 2;
    return side;
}

extern "C" int64_t tsg_permutation_work_elems(int rows, int cols, int loc) {
    int64_t side = hilbert_side(rows, cols, loc);
    return (side * side + kHilbertBlock - 1) / kHilbertBlock;
}

extern "C" int tsg_make_permutation(int rows, int cols, int loc, int numbering, int64_t *forward,
                                    int64_t *work, tsg_stream s) {
    if (rows < 2 || cols < 2) return fail(TSG_EVALUE, "rows and cols must each be >= 2");
    if (!valid_loc(loc)) return fail(TSG_EVALUE, "bad location %d", loc);
    if (!forward) return fail(TSG_EVALUE, "tsg_make_permutation: NULL output");
    cudaStream_t st = (cudaStream_t)s;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int colors = colors_of(loc);
    if (numbering == 0 || numbering == 1) {
        int64_t n = (int64_t)rows * colors * cols;
        perm_simple_kernel<<<grid_for(n, 256, sms), 256, 0, st>>>(rows, cols, colors, numbering, forward);
        TSG_CHECK_LAUNCH();
        return TSG_OK;
    }
    if (numbering != 2) return fail(TSG_EVALUE, "unknown numbering %d", numbering);
    if (loc == TSG_EDGES) return fail(TSG_EVALUE, "hn numbering is not defined for edges");
    if (!work) return fail(TSG_EVALUE, "tsg_make_permutation: hn needs a work buffer");
    const int64_t side = hilbert_side(rows, cols, loc);
    const int64_t nb = (side * side + kHilbertBlock - 1) / kHilbertBlock;
    const int gx = rows, gy = loc == TSG_CELLS ? 2 * cols : cols;
    hilbert_count_kernel<<<(unsigned)nb, kHilbertBlock, 0, st>>>(side, gx, gy, work);
    exclusive_scan_kernel<<<1, 1024, 0, st>>>(work, nb);
    hilbert_write_kernel<<<(unsigned)nb, kHilbertBlock, 0, st>>>(side, gx, gy, cols,
                                                                 loc == TSG_CELLS, work, forward);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

// Strided host <-> device copy of `height` rows of `width` bytes (cudaMemcpy2DAsync): one
// band of storage rows of a level-outer host layout is one such copy (executors.py's
// streamed run_fused).  kind 1 = host to device, 2 = device to host.
extern "C" int tsg_memcpy2d(void *dst, int64_t dpitch, const void *src, int64_t spitch, int64_t width,
                            int64_t height, int kind, tsg_stream s) {
    if (!dst || !src) return fail(TSG_EVALUE, "tsg_memcpy2d: NULL pointer");
    if (kind != 1 && kind != 2) return fail(TSG_EVALUE, "tsg_memcpy2d: kind must be 1 (H2D) or 2 (D2H)");
    if (width < 0 || height < 0 || dpitch < width || spitch < width)
        return fail(TSG_EVALUE, "tsg_memcpy2d: bad extents");
    if (width == 0 || height == 0) return TSG_OK;
    TSG_CHECK_CUDA(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width, (size_t)height,
                                     kind == 1 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                                     (cudaStream_t)s));
    return TSG_OK;
}
