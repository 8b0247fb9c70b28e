// Neighbour-reduction stencils and the materialising (unfused / indirect) MPDATA steps.
//
// These kernels are HBM-bound streaming sweeps: one thread per (element, level) with the
// level axis fastest, so every neighbour read is a contiguous run of a neighbouring
// element's level column (coalesced; neighbour reuse is served by L1/L2).  Grids are a
// multiple of the SM count with grid-stride loops.
#include <algorithm>

#include "tsg_common.cuh"
#include "tsg_offsets.cuh"

namespace tsg {

int reduce_tma(const tsg_grid *g, int rel, int inner, const double *src, const double *scale,
               double *dst, cudaStream_t st);
int cell_divergence_tma(const tsg_grid *g, int weighted, const double *vn, const double *length,
                        const double *area, const double *weights, double *out, cudaStream_t st);

// -- structured reduce over any relation (stencil.py:404-408 with the sum fold) -------

template <int REL, bool SCALE>
__global__ void __launch_bounds__(256) reduce_kernel(FieldIx Fs, FieldIx Fd, FieldIx Fsc, int nk,
                                                     const double *__restrict__ src,
                                                     const double *__restrict__ scale,
                                                     double *__restrict__ dst, int flags) {
    constexpr int W = REL < 3 ? 6 : (REL < 6 ? 3 : (REL == 8 ? 4 : 2));
    TSG_LINES(Fd, i, c, j) {
        const double *nb[W];
#pragma unroll
        for (int s = 0; s < W; ++s) {
            const int8_t *o = c_offsets[REL][c][s];
            nb[s] = src + Fs.at(i + o[0], o[1], j + o[2]);
        }
        const double sc = SCALE ? scale[Fsc.at(i, c, j)] : 1.0;
        double *out = dst + Fd.at(i, c, j);
        const Img m = images(Fd, i, j, flags);
        if (nk > 1) {  // level pairs, 16-byte accesses
            for (int k = 2 * threadIdx.x; k < nk; k += 64) {
                double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                for (int s = 0; s < W; ++s) {
                    const double2 v = ld2(nb[s] + k);
                    acc.x = add(v.x, acc.x);
                    acc.y = add(v.y, acc.y);
                }
                if (SCALE) acc = make_double2(mul(acc.x, sc), mul(acc.y, sc));
                put2(out, m, k, acc);
            }
        } else if (threadIdx.x == 0) {
            double acc = 0.0;
#pragma unroll
            for (int s = 0; s < W; ++s) acc = add(nb[s][0], acc);
            if (SCALE) acc = mul(acc, sc);
            put(out, m, 0, acc);
        }
    }
}

// -- table-driven reduce over flat arrays (kernels.py:83-104, reference.py:137-157) -----

template <int W>
__global__ void __launch_bounds__(256) reduce_indirect_kernel(const int64_t *__restrict__ table,
                                                              int64_t nrows, int width, int nlev,
                                                              const double *__restrict__ src,
                                                              const double *__restrict__ scale,
                                                              double *__restrict__ dst) {
    const int wd = W > 0 ? W : width;
    for (int64_t r = (int64_t)blockIdx.x * kWarps + threadIdx.y; r < nrows;
         r += (int64_t)gridDim.x * kWarps) {
        const int64_t *row = table + r * wd;
        const double sc = scale ? scale[r] : 1.0;
        double *out = dst + r * nlev;
        if (W > 0 && (nlev & 1) == 0) {  // level pairs, 16-byte accesses
            const double *nb[W > 0 ? W : 1];
#pragma unroll
            for (int s = 0; s < W; ++s) nb[s] = src + __ldg(row + s) * nlev;
            for (int k = 2 * threadIdx.x; k < nlev; k += 64) {
                double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                for (int s = 0; s < W; ++s) {
                    const double2 v = ld2(nb[s] + k);
                    acc.x = add(v.x, acc.x);
                    acc.y = add(v.y, acc.y);
                }
                st2(out + k, scale ? make_double2(mul(acc.x, sc), mul(acc.y, sc)) : acc);
            }
        } else if (W > 0) {
            const double *nb[W > 0 ? W : 1];
#pragma unroll
            for (int s = 0; s < W; ++s) nb[s] = src + __ldg(row + s) * nlev;
            for (int k = threadIdx.x; k < nlev; k += 32) {
                double acc = 0.0;
#pragma unroll
                for (int s = 0; s < W; ++s) acc = add(nb[s][k], acc);
                out[k] = scale ? mul(acc, sc) : acc;
            }
        } else {
            for (int k = threadIdx.x; k < nlev; k += 32) {
                double acc = 0.0;
                for (int s = 0; s < wd; ++s) acc = add(src[__ldg(row + s) * nlev + k], acc);
                out[k] = scale ? mul(acc, sc) : acc;
            }
        }
    }
}

// Level-pair item kernels (the table-driven MPDATA stages below, the reorders): kUnroll
// items per thread per pass with all their loads issued before any use.  Lanes of one row
// share its table entries (broadcast loads) and read consecutive 16-byte pairs of each
// neighbour row (coalesced).
constexpr int kUnroll = 4;

// Level-pair items (one thread per (row, level pair), flattened over the field so every
// lane is busy whatever the level count), with the next batch's table row (and scale)
// fetched while this batch's W neighbour runs are in flight: the table load and the
// gather it feeds are dependent, so an unpipelined batch waits two load latencies.  One
// item per batch (32 registers, full occupancy): Table-1 k1 / k2 at 1024x1024x80
// 443-472 us (0.89-0.94 of the copy peak) against 553-566 us for round 1's four
// unpipelined items per thread and 594-1028 us for two / three pipelined ones
// (tools/indirect_variants.py, TSG_IND_V A/B build; outputs bitwise identical).
template <int W, bool SCALE, int U>
__global__ void __launch_bounds__(256) reduce_indirect_pipe_kernel(
    const int64_t *__restrict__ table, uint32_t nitems, FastDiv npairs, int nlev,
    const double *__restrict__ src, const double *__restrict__ scale, double *__restrict__ dst) {
    const uint32_t T = gridDim.x * blockDim.x;
    int64_t nb[U][W];
    uint32_t row[U], kp[U];
    double sc[U];
    auto fetch = [&](uint32_t b) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t it = b + u * T;
            if (it < nitems) {
                row[u] = npairs.div(it);
                kp[u] = 2 * (it - row[u] * npairs.d);
                sc[u] = SCALE ? __ldg(scale + row[u]) : 1.0;
#pragma unroll
                for (int s = 0; s < W; ++s) nb[u][s] = __ldg(table + (int64_t)row[u] * W + s);
            }
        }
    };
    uint32_t base = blockIdx.x * blockDim.x + threadIdx.x;
    fetch(base);
    for (; base < nitems; base += U * T) {
        double2 v[U][W];
        uint32_t r2[U], k2[U];
        double s2[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u * T < nitems) {
#pragma unroll
                for (int s = 0; s < W; ++s)
                    v[u][s] = __ldg(reinterpret_cast<const double2 *>(src + nb[u][s] * nlev + kp[u]));
                r2[u] = row[u];
                k2[u] = kp[u];
                s2[u] = sc[u];
            }
        }
        if (base + U * T < nitems) fetch(base + U * T);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u * T >= nitems) break;
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int s = 0; s < W; ++s) {
                acc.x = add(v[u][s].x, acc.x);
                acc.y = add(v[u][s].y, acc.y);
            }
            if (SCALE) acc = make_double2(mul(acc.x, s2[u]), mul(acc.y, s2[u]));
            st2(dst + (int64_t)r2[u] * nlev + k2[u], acc);
        }
    }
}

// -- cell divergence (mpdata.py:361-416, reference.py:119-134) --------------------------

template <bool WEIGHTED>
__global__ void __launch_bounds__(256) cell_div_kernel(FieldIx Fvn, FieldIx Fl, FieldIx Fa,
                                                       FieldIx Fw, FieldIx Fo, int nk,
                                                       const double *__restrict__ vn,
                                                       const double *__restrict__ length,
                                                       const double *__restrict__ area,
                                                       const double *__restrict__ weights,
                                                       double *__restrict__ out, int flags) {
    constexpr int REL = TSG_CELLS * 3 + TSG_EDGES;
    TSG_LINES(Fo, i, c, j) {
        const double *v[3];
        double w[3];
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const int8_t *o = c_offsets[REL][c][s];
            v[s] = vn + Fvn.at(i + o[0], o[1], j + o[2]);
            w[s] = WEIGHTED ? weights[Fw.at(i, c, j) + s] : length[Fl.at(i + o[0], o[1], j + o[2])];
        }
        const double a = WEIGHTED ? 1.0 : area[Fa.at(i, c, j)];
        double *o = out + Fo.at(i, c, j);
        const Img m = images(Fo, i, j, flags);
        for (int k = threadIdx.x; k < nk; k += 32) {
            double acc = 0.0;
#pragma unroll
            for (int s = 0; s < 3; ++s) acc = add(mul(v[s][k], w[s]), acc);
            if (!WEIGHTED) acc = dvd(acc, a);
            put(o, m, k, acc);
        }
    }
}

// -- unfused MPDATA (run_naive analogue, executors.py:213-245) --------------------------

// Level-pair item forms of the four unfused stages: one thread per
// (element, level pair) over the whole field, kUnroll items per thread per pass, 16-byte
// loads and stores (round 1's element-line forms, one warp per element, were latency-bound
// with a quarter of their lanes idle in the last pass of an 80-level run).  Item order: on a resident grid
// (item_grid, short sweeps) thread t's items of a pass are t, t + T, ... (T = all threads);
// on a one-pass grid (long sweeps) the stencil stages take a block's kUnroll x 256 items
// contiguously instead, so the items in flight form one wavefront rather than kUnroll
// wavefronts a quarter of the field apart, and the row a stencil reads one row ahead is
// still in L2 when its own items arrive: O1280 flux reads 31.6 vs 36.4 GB, divergence 31.4
// vs 38.7 GB, the step 25.9 vs 27.1 ms (profiles/unfused_o1280_r2.csv).  On the resident
// grid of a short sweep the strided order is faster (279x256x80: 170 vs 176 us).
// 64-bit pass arithmetic: n may approach 2^32.
#ifndef TSG_CHUNK_MASK  // A/B builds only: which stages take contiguous chunks on one pass
#define TSG_CHUNK_MASK 7
#endif
#define TSG_ITEMS(base, u, D, BIT)                                                               \
    const bool ch_ = (TSG_CHUNK_MASK & (BIT)) && (uint64_t)kUnroll * gridDim.x * blockDim.x >= (D).n; \
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * (ch_ ? kUnroll : 1) + threadIdx.x, \
                  T_ = ch_ ? blockDim.x : (uint64_t)gridDim.x * blockDim.x;                      \
         base < (D).n; base += (uint64_t)kUnroll * gridDim.x * blockDim.x)                       \
        _Pragma("unroll") for (int u = 0; u < kUnroll; ++u)                                       \
            if (base + u * T_ < (D).n)

// Edge fluxes of the unfused step (mpdata.py:189-199), three per vertex item: edge
// (i, c, j) has its origin at vertex (i, j) (E->V slot 0, connectivity.py:38-42), so one
// item loads the origin's pd pair once plus the three other ends c0 (i, j+1), c1
// (i+1, j+1), c2 (i+1, j) and writes the three colours -- 4 instead of 6 pd loads per
// three fluxes.  O1280 (2560x2576x137): 13.3 vs 17.1 ms and 51 vs 74 GB of DRAM reads
// against the one-edge-per-item form (ncu, tools/prof_unfused_o1280.py).
template <int OP>
__global__ void __launch_bounds__(256) flux3_pairs_kernel(FieldIx Fp, FieldIx Fe, PointDec D,
                                                          const double *__restrict__ pd,
                                                          const double *__restrict__ vn,
                                                          double *__restrict__ flux, int flags) {
    TSG_ITEMS(base, u, D, 1) {
        const Pt e = decompose((uint32_t)(base + u * T_), D);
        const int k = 2 * e.k;
        const double2 po = ld2(pd + Fp.at(e.i, 0, e.j) + k);
        const double2 p0 = ld2(pd + Fp.at(e.i, 0, e.j + 1) + k);      // c0 (0,+1)
        const double2 p1 = ld2(pd + Fp.at(e.i + 1, 0, e.j + 1) + k);  // c1 (+1,+1)
        const double2 p2 = ld2(pd + Fp.at(e.i + 1, 0, e.j) + k);      // c2 (+1,0)
        const double2 v0 = ld2(vn + Fe.at(e.i, 0, e.j) + k);
        const double2 v1 = ld2(vn + Fe.at(e.i, 1, e.j) + k);
        const double2 v2 = ld2(vn + Fe.at(e.i, 2, e.j) + k);
        const Img m = images(Fe, e.i, e.j, flags);
        put2(flux + Fe.at(e.i, 0, e.j), m, k, make_double2(edge_flux<OP>(po.x, p0.x, v0.x), edge_flux<OP>(po.y, p0.y, v0.y)));
        put2(flux + Fe.at(e.i, 1, e.j), m, k, make_double2(edge_flux<OP>(po.x, p1.x, v1.x), edge_flux<OP>(po.y, p1.y, v1.y)));
        put2(flux + Fe.at(e.i, 2, e.j), m, k, make_double2(edge_flux<OP>(po.x, p2.x, v2.x), edge_flux<OP>(po.y, p2.y, v2.y)));
    }
}

// interface pairs (2p, 2p+1) over 0..K; the partner of the last interface is padding (0)
__global__ void __launch_bounds__(256) fluz_pairs_kernel(FieldIx Fp, FieldIx Fw, PointDec D, int K,
                                                         double pivbz, const double *__restrict__ pd,
                                                         const double *__restrict__ wn,
                                                         double *__restrict__ fluz, int flags) {
    TSG_ITEMS(base, u, D, 2) {
        const Pt e = decompose((uint32_t)(base + u * T_), D);
        const double *P = pd + Fp.at(e.i, 0, e.j), *W = wn + Fw.at(e.i, 0, e.j);
        double f[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = 2 * e.k + h;
            if (k == 0) f[h] = mul(pivbz, fluz_interior(W[1], P[0], P[1]));
            else if (k == K) f[h] = mul(pivbz, fluz_interior(W[K - 1], P[K - 2], P[K - 1]));
            else if (k > K) f[h] = 0.0;
            else f[h] = fluz_interior(W[k], P[k - 1], P[k]);
        }
        put2(fluz + Fw.at(e.i, 0, e.j), images(Fw, e.i, e.j, flags), 2 * e.k, make_double2(f[0], f[1]));
    }
}

__global__ void __launch_bounds__(256) div_pairs_kernel(FieldIx Fe, FieldIx Fw, FieldIx Fs, FieldIx Fd,
                                                        FieldIx Fv, PointDec D,
                                                        const double *__restrict__ flux,
                                                        const double *__restrict__ fluz,
                                                        const double *__restrict__ signs,
                                                        const double *__restrict__ dual,
                                                        double *__restrict__ divvd, int flags) {
    constexpr int REL = TSG_VERTICES * 3 + TSG_EDGES;
    TSG_ITEMS(base, u, D, 4) {
        const Pt e = decompose((uint32_t)(base + u * T_), D);
        const int k = 2 * e.k;
        const double *S = signs + Fs.at(e.i, 0, e.j);
        const double *Z = fluz + Fw.at(e.i, 0, e.j);
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int s = 0; s < 6; ++s) {
            const int8_t *o = c_offsets[REL][0][s];
            const double2 f = ld2(flux + Fe.at(e.i + o[0], o[1], e.j + o[2]) + k);
            const double sg = __ldg(S + s);
            acc.x = add(mul(sg, f.x), acc.x);
            acc.y = add(mul(sg, f.y), acc.y);
        }
        const double2 z01 = ld2(Z + k);
        const double z2 = Z[k + 2];
        acc.x = add(acc.x, sub(z01.y, z01.x));
        acc.y = add(acc.y, sub(z2, z01.y));
        const double du = __ldg(dual + Fd.at(e.i, 0, e.j));
        put2(divvd + Fv.at(e.i, 0, e.j), images(Fv, e.i, e.j, flags), k,
             make_double2(dvd(acc.x, du), dvd(acc.y, du)));
    }
}

__global__ void __launch_bounds__(256) advance_pairs_kernel(FieldIx Fv, PointDec D, double dt,
                                                            const double *__restrict__ pd,
                                                            const double *__restrict__ divvd,
                                                            const double *__restrict__ rho,
                                                            double *__restrict__ pd_out, int flags) {
    TSG_ITEMS(base, u, D, 8) {
        const Pt e = decompose((uint32_t)(base + u * T_), D);
        const int64_t q = Fv.at(e.i, 0, e.j) + 2 * e.k;
        const double2 d = ld2(divvd + q), r = ld2(rho + q), p = ld2(pd + q);
        put2(pd_out + Fv.at(e.i, 0, e.j), images(Fv, e.i, e.j, flags), 2 * e.k,
             make_double2(sub(p.x, dvd(mul(dt, d.x), r.x)), sub(p.y, dvd(mul(dt, d.y), r.y))));
    }
}
#undef TSG_ITEMS

// -- indirect (table-driven) MPDATA over flat arrays (reference.py:93-116) -------------

#define TSG_FLAT_ROWS(r, n)                                                          \
    for (int64_t r = (int64_t)blockIdx.x * kWarps + threadIdx.y; r < (n);          \
         r += (int64_t)gridDim.x * kWarps)

template <int OP>
__global__ void __launch_bounds__(256) iflux_kernel(const int64_t *__restrict__ e2v, int64_t ne,
                                                    int K, const double *__restrict__ pd,
                                                    const double *__restrict__ vn,
                                                    double *__restrict__ flux) {
    TSG_FLAT_ROWS(e, ne) {
        const double *po = pd + __ldg(e2v + 2 * e) * K, *pp = pd + __ldg(e2v + 2 * e + 1) * K;
        const double *v = vn + e * K;
        double *o = flux + e * K;
        for (int k = threadIdx.x; k < K; k += 32) o[k] = edge_flux<OP>(po[k], pp[k], v[k]);
    }
}

__global__ void __launch_bounds__(256) ifluz_kernel(int64_t nv, int K, double pivbz,
                                                    const double *__restrict__ pd,
                                                    const double *__restrict__ wn,
                                                    double *__restrict__ fluz) {
    TSG_FLAT_ROWS(v, nv) {
        const double *P = pd + v * K, *W = wn + v * (K + 1);
        double *o = fluz + v * (K + 1);
        for (int k = threadIdx.x; k <= K; k += 32) {
            double f;
            if (k == 0) f = mul(pivbz, fluz_interior(W[1], P[0], P[1]));
            else if (k == K) f = mul(pivbz, fluz_interior(W[K - 1], P[K - 2], P[K - 1]));
            else f = fluz_interior(W[k], P[k - 1], P[k]);
            o[k] = f;
        }
    }
}

// The reference's flat stages one by one (reference.py:18-90, 119-134), for callers of
// its per-stage functions: the divergence over a table of any width, the explicit update,
// and the table-driven cell divergence.  Same operation order as the fused kernels.
__global__ void __launch_bounds__(256) idiv_kernel(const int64_t *__restrict__ v2e, int W, int64_t nv, int K,
                                                   const double *__restrict__ signs,
                                                   const double *__restrict__ dual,
                                                   const double *__restrict__ flux,
                                                   const double *__restrict__ fluz,
                                                   double *__restrict__ div) {
    TSG_FLAT_ROWS(v, nv) {
        const int64_t *row = v2e + v * W;
        const double *sg = signs + v * W, *Z = fluz + v * (K + 1);
        const double du = __ldg(dual + v);
        for (int k = threadIdx.x; k < K; k += 32) {
            double acc = 0.0;
            for (int s = 0; s < W; ++s) acc = add(mul(__ldg(sg + s), flux[__ldg(row + s) * K + k]), acc);
            acc = add(acc, sub(Z[k + 1], Z[k]));
            div[v * K + k] = dvd(acc, du);
        }
    }
}

__global__ void __launch_bounds__(256) advance_flat_kernel(int64_t n, double dt, const double *__restrict__ pd,
                                                           const double *__restrict__ div,
                                                           const double *__restrict__ rho,
                                                           double *__restrict__ out) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        double slope = mul(dt, div[q]);
        slope = dvd(slope, rho[q]);
        out[q] = sub(pd[q], slope);
    }
}

__global__ void __launch_bounds__(256) icell_div_kernel(const int64_t *__restrict__ c2e, int W, int64_t nc, int K,
                                                        const double *__restrict__ vn,
                                                        const double *__restrict__ length,
                                                        const double *__restrict__ area,
                                                        double *__restrict__ out) {
    TSG_FLAT_ROWS(c, nc) {
        const int64_t *row = c2e + c * W;
        const double ar = __ldg(area + c);
        for (int k = threadIdx.x; k < K; k += 32) {
            double acc = 0.0;
            for (int s = 0; s < W; ++s) {
                const int64_t e = __ldg(row + s);
                acc = add(mul(vn[e * K + k], __ldg(length + e)), acc);
            }
            out[c * K + k] = dvd(acc, ar);
        }
    }
}

__global__ void __launch_bounds__(256) idiv_advance_kernel(
    const int64_t *__restrict__ v2e, int64_t nv, int K, double dt, const double *__restrict__ signs,
    const double *__restrict__ dual, const double *__restrict__ flux,
    const double *__restrict__ fluz, const double *__restrict__ pd, const double *__restrict__ rho,
    double *__restrict__ div, double *__restrict__ pd_out) {
    TSG_FLAT_ROWS(v, nv) {
        const double *f[6];
        double sg[6];
#pragma unroll
        for (int s = 0; s < 6; ++s) {
            f[s] = flux + __ldg(v2e + v * 6 + s) * K;
            sg[s] = __ldg(signs + v * 6 + s);
        }
        const double *Z = fluz + v * (K + 1);
        const double du = __ldg(dual + v);
        const int64_t e = v * K;
        for (int k = threadIdx.x; k < K; k += 32) {
            double acc = 0.0;
#pragma unroll
            for (int s = 0; s < 6; ++s) acc = add(mul(sg[s], f[s][k]), acc);
            acc = add(acc, sub(Z[k + 1], Z[k]));
            const double d = dvd(acc, du);
            div[e + k] = d;
            double slope = mul(dt, d);
            slope = dvd(slope, rho[e + k]);
            pd_out[e + k] = sub(pd[e + k], slope);
        }
    }
}

// Level-pair item forms of the table-driven step (even level counts: 16-byte aligned flat
// rows): one thread per (row, level pair), kUnroll items in flight per thread.
#define TSG_FLAT_ITEMS(it, u, n)                                                              \
    for (uint32_t base_ = blockIdx.x * blockDim.x + threadIdx.x, T_ = gridDim.x * blockDim.x;  \
         base_ < (n); base_ += kUnroll * T_)                                                    \
        _Pragma("unroll") for (int u = 0; u < kUnroll; ++u)                                    \
            for (uint32_t it = base_ + u * T_; it < (n); it = (n))

template <int OP>
__global__ void __launch_bounds__(256) iflux_pairs_kernel(const int64_t *__restrict__ e2v, uint32_t n,
                                                          FastDiv np, int K, const double *__restrict__ pd,
                                                          const double *__restrict__ vn,
                                                          double *__restrict__ flux) {
    TSG_FLAT_ITEMS(it, u, n) {
        const uint32_t e = np.div(it);
        const int k = 2 * (it - e * np.d);
        const double2 po = ld2(pd + __ldg(e2v + 2 * (int64_t)e) * K + k);
        const double2 pp = ld2(pd + __ldg(e2v + 2 * (int64_t)e + 1) * K + k);
        const double2 v = ld2(vn + (int64_t)e * K + k);
        st2(flux + (int64_t)e * K + k,
            make_double2(edge_flux<OP>(po.x, pp.x, v.x), edge_flux<OP>(po.y, pp.y, v.y)));
    }
}

// The divergence + update stage with the next item's six table entries fetched while the
// current item's flux rows are in flight (one item per thread, as the Table-1 gather
// above: the table load and the gather it feeds are dependent loads).  279x256x80 step
// 155.3 -> 149.0 us, 1024x1024x80 2112 -> 1993 us (tools/indirect_step_variants.py,
// TSG_IPIPE A/B build, bitwise unchanged); the same for the two-row edge flux gather
// lost (157.4 / 2126 us), so that stage keeps four items per thread.
// ADV = false: the divergence alone (the reference's flux_divergence, reference.py:63-79,
// for callers of the per-stage functions); pd / rho / pd_out are then unused.
template <bool ADV>
__global__ void __launch_bounds__(256) idiv_advance_pipe_kernel(
    const int64_t *__restrict__ v2e, uint32_t n, FastDiv np, int K, double dt,
    const double *__restrict__ signs, const double *__restrict__ dual, const double *__restrict__ flux,
    const double *__restrict__ fluz, const double *__restrict__ pd, const double *__restrict__ rho,
    double *__restrict__ div, double *__restrict__ pd_out) {
    const uint32_t T = gridDim.x * blockDim.x;
    uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t v = 0;
    int64_t nb[6];
    auto fetch = [&](uint32_t i) {
        v = np.div(i);
#pragma unroll
        for (int s = 0; s < 6; ++s) nb[s] = __ldg(v2e + (int64_t)v * 6 + s);
    };
    if (it < n) fetch(it);
    for (; it < n; it += T) {
        const int k = 2 * (it - v * np.d);
        const uint32_t vc = v;
        double2 f[6];
#pragma unroll
        for (int s = 0; s < 6; ++s) f[s] = ld2(flux + nb[s] * K + k);
        if (it + T < n) fetch(it + T);
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int s = 0; s < 6; ++s) {
            const double sg = __ldg(signs + (int64_t)vc * 6 + s);
            acc.x = add(mul(sg, f[s].x), acc.x);
            acc.y = add(mul(sg, f[s].y), acc.y);
        }
        const double *Z = fluz + (int64_t)vc * (K + 1) + k;  // odd row width: scalar loads
        const double z0 = Z[0], z1 = Z[1], z2 = Z[2];
        acc.x = add(acc.x, sub(z1, z0));
        acc.y = add(acc.y, sub(z2, z1));
        const double du = __ldg(dual + vc);
        const double2 d = make_double2(dvd(acc.x, du), dvd(acc.y, du));
        const int64_t qq = (int64_t)vc * K + k;
        st2(div + qq, d);
        if constexpr (ADV) {
            const double2 r = ld2(rho + qq), p = ld2(pd + qq);
            st2(pd_out + qq, make_double2(sub(p.x, dvd(mul(dt, d.x), r.x)), sub(p.y, dvd(mul(dt, d.y), r.y))));
        }
    }
}

// The table-driven cell divergence (reference.cell_divergence, reference.py:119-134) in
// level-pair items, pipelined like the Table-1 gather: the table row of the item after
// next and the edge lengths of the next item (they depend on its table row, fetched one
// iteration earlier) are in flight while the current item's vn pairs are.
#ifndef TSG_CDIV_DEPTH  // A/B builds only
#define TSG_CDIV_DEPTH 2
#endif
__global__ void __launch_bounds__(256) icell_div_pipe_kernel(const int64_t *__restrict__ c2e, uint32_t n,
                                                             FastDiv np, int K, const double *__restrict__ vn,
                                                             const double *__restrict__ length,
                                                             const double *__restrict__ area,
                                                             double *__restrict__ out) {
    const uint32_t T = gridDim.x * blockDim.x;
    uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t c = 0, c1 = 0;
    int64_t nb[3], nb1[3];
    double ln[3], ar = 1.0;
    auto rows = [&](uint32_t i, uint32_t &cc, int64_t *q) {
        cc = np.div(i);
#pragma unroll
        for (int s = 0; s < 3; ++s) q[s] = __ldg(c2e + (int64_t)cc * 3 + s);
    };
    auto weights = [&](uint32_t cc, const int64_t *q) {
#pragma unroll
        for (int s = 0; s < 3; ++s) ln[s] = __ldg(length + q[s]);
        ar = __ldg(area + cc);
    };
    if (it < n) {
        rows(it, c, nb);
        weights(c, nb);
        if (TSG_CDIV_DEPTH == 2 && it + T < n) rows(it + T, c1, nb1);
    }
    for (; it < n; it += T) {
        const int k = 2 * (it - c * np.d);
        const uint32_t cc = c;
        double2 v[3];
        double l[3];
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            v[s] = ld2(vn + nb[s] * K + k);
            l[s] = ln[s];
        }
        const double a = ar;
        if (it + T < n) {
            if (TSG_CDIV_DEPTH == 2) {
                c = c1;
#pragma unroll
                for (int s = 0; s < 3; ++s) nb[s] = nb1[s];
                weights(c, nb);
                if (it + 2 * T < n) rows(it + 2 * T, c1, nb1);
            } else {
                rows(it + T, c, nb);
                weights(c, nb);
            }
        }
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            acc.x = add(mul(v[s].x, l[s]), acc.x);
            acc.y = add(mul(v[s].y, l[s]), acc.y);
        }
        st2(out + (int64_t)cc * K + k, make_double2(dvd(acc.x, a), dvd(acc.y, a)));
    }
}

// The explicit update over value pairs (16-byte loads and stores)
__global__ void __launch_bounds__(256) advance_flat2_kernel(int64_t n2, double dt, const double *__restrict__ pd,
                                                            const double *__restrict__ div,
                                                            const double *__restrict__ rho,
                                                            double *__restrict__ out) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n2; q += (int64_t)gridDim.x * blockDim.x) {
        const double2 d = ld2(div + 2 * q), r = ld2(rho + 2 * q), p = ld2(pd + 2 * q);
        st2(out + 2 * q, make_double2(sub(p.x, dvd(mul(dt, d.x), r.x)), sub(p.y, dvd(mul(dt, d.y), r.y))));
    }
}

// interfaces in pairs over 0..K of a K+1-wide row (odd width: the last item is a single)
__global__ void __launch_bounds__(256) ifluz_pairs_kernel(uint32_t n, FastDiv np, int K, double pivbz,
                                                          const double *__restrict__ pd,
                                                          const double *__restrict__ wn,
                                                          double *__restrict__ fluz) {
    TSG_FLAT_ITEMS(it, u, n) {
        const uint32_t v = np.div(it);
        const int k0 = 2 * (it - v * np.d);
        const double *P = pd + (int64_t)v * K, *W = wn + (int64_t)v * (K + 1);
        double *o = fluz + (int64_t)v * (K + 1);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = k0 + h;
            if (k > K) break;
            double f;
            if (k == 0) f = mul(pivbz, fluz_interior(W[1], P[0], P[1]));
            else if (k == K) f = mul(pivbz, fluz_interior(W[K - 1], P[K - 2], P[K - 1]));
            else f = fluz_interior(W[k], P[k - 1], P[k]);
            o[k] = f;
        }
    }
}

#undef TSG_FLAT_ITEMS

// Point items (one thread per (row, level), kUnroll per thread per pass) for odd level
// counts, whose flat rows are not 16-byte aligned (the cfg5 depth, K = 137): scalar loads,
// a warp on 32 consecutive levels of a row (table entries broadcast).  Same operation
// order as the level-pair forms.  n < 2^32 - 2^24 (point_limit()); 64-bit pass arithmetic.
#define TSG_POINT_ITEMS(q, u, n)                                                                 \
    const bool ch_ = (uint64_t)kUnroll * gridDim.x * blockDim.x >= (n);                         \
    for (uint64_t base_ = (uint64_t)blockIdx.x * blockDim.x * (ch_ ? kUnroll : 1) + threadIdx.x, \
                  T_ = ch_ ? blockDim.x : (uint64_t)gridDim.x * blockDim.x;                      \
         base_ < (n); base_ += (uint64_t)kUnroll * gridDim.x * blockDim.x)                       \
        _Pragma("unroll") for (int u = 0; u < kUnroll; ++u)                                       \
            if (const uint64_t q64_ = base_ + u * T_; q64_ < (n))                                   \
                if (const uint32_t q = (uint32_t)q64_; true)

template <int OP>
__global__ void __launch_bounds__(256) iflux_points_kernel(const int64_t *__restrict__ e2v, uint32_t n,
                                                           FastDiv nk, const double *__restrict__ pd,
                                                           const double *__restrict__ vn,
                                                           double *__restrict__ flux) {
    TSG_POINT_ITEMS(q, u, n) {
        const uint32_t e = nk.div(q);
        const int k = (int)(q - e * nk.d);
        const int64_t o = __ldg(e2v + 2 * (int64_t)e), p = __ldg(e2v + 2 * (int64_t)e + 1);
        flux[q] = edge_flux<OP>(pd[o * nk.d + k], pd[p * nk.d + k], vn[q]);
    }
}

// Table-1 gather (reference.neighbor_sum(_scaled), reference.py:137-157) at odd level
// counts: pairs of the flat [row, level] output (16-byte stores; a pair may straddle two
// rows, whose table entries are then both read), scalar neighbour gathers, the next
// pair's table entries fetched while this pair's gathers are in flight (the even-level
// pipeline's scheme; one pair per thread per iteration on a resident grid).
template <int W, bool SCALE>
__global__ void __launch_bounds__(256) reduce_indirect_flatpairs_kernel(const int64_t *__restrict__ table,
                                                                        uint32_t n, FastDiv nk,
                                                                        const double *__restrict__ src,
                                                                        const double *__restrict__ scale,
                                                                        double *__restrict__ dst) {
    const uint32_t n2 = (n + 1) / 2, T = gridDim.x * blockDim.x;
    const int K = (int)nk.d;
    int64_t nb0[W], nb1[W];
    uint32_t r0 = 0;
    int k0 = 0;
    bool next = false;
    double sc0 = 1.0, sc1 = 1.0;
    auto fetch = [&](uint32_t m) {
        const uint32_t q0 = 2 * m;
        r0 = nk.div(q0);
        k0 = (int)(q0 - r0 * nk.d);
        next = k0 + 1 == K && q0 + 1 < n;
#pragma unroll
        for (int s = 0; s < W; ++s) nb0[s] = __ldg(table + (int64_t)r0 * W + s);
#pragma unroll
        for (int s = 0; s < W; ++s) nb1[s] = next ? __ldg(table + (int64_t)(r0 + 1) * W + s) : nb0[s];
        if (SCALE) {
            sc0 = __ldg(scale + r0);
            sc1 = next ? __ldg(scale + r0 + 1) : sc0;
        }
    };
    uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m < n2) fetch(m);
    for (; m < n2; m += T) {
        const uint32_t q0 = 2 * m;
        const bool two = q0 + 1 < n, nx = next;
        const double s0 = sc0, s1 = sc1;
        const int kc = k0, k1 = nx ? 0 : k0 + 1;
        double v0[W], v1[W];
#pragma unroll
        for (int s = 0; s < W; ++s) {
            v0[s] = src[nb0[s] * K + kc];
            v1[s] = two ? src[nb1[s] * K + k1] : 0.0;
        }
        if (m + T < n2) fetch(m + T);
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int s = 0; s < W; ++s) {
            a0 = add(v0[s], a0);
            a1 = add(v1[s], a1);
        }
        if (SCALE) {
            a0 = mul(a0, s0);
            a1 = mul(a1, s1);
        }
        if (two) st2(dst + q0, make_double2(a0, a1));
        else dst[q0] = a0;
    }
}

// The same over pairs of the flat [edge, level] array (16-byte vn loads and flux stores
// whatever the row alignment; a pair may straddle two edges' rows); the pd gathers stay
// scalar.
template <int OP>
__global__ void __launch_bounds__(256) iflux_flatpairs_kernel(const int64_t *__restrict__ e2v, uint32_t n,
                                                              FastDiv nk, const double *__restrict__ pd,
                                                              const double *__restrict__ vn,
                                                              double *__restrict__ flux) {
    const uint32_t n2 = (n + 1) / 2;
    const int K = (int)nk.d;
    TSG_POINT_ITEMS(m, u, n2) {
        const uint32_t q0 = 2 * m;
        const uint32_t e0 = nk.div(q0);
        const int k0 = (int)(q0 - e0 * nk.d);
        const int64_t o0 = __ldg(e2v + 2 * (int64_t)e0), p0 = __ldg(e2v + 2 * (int64_t)e0 + 1);
        if (q0 + 1 < n) {
            const bool next = k0 + 1 == K;  // the pair's second value opens the next edge's row
            const int k1 = next ? 0 : k0 + 1;
            const int64_t o1 = next ? __ldg(e2v + 2 * (int64_t)e0 + 2) : o0;
            const int64_t p1 = next ? __ldg(e2v + 2 * (int64_t)e0 + 3) : p0;
            const double2 v = ld2(vn + q0);
            st2(flux + q0, make_double2(edge_flux<OP>(pd[o0 * K + k0], pd[p0 * K + k0], v.x),
                                        edge_flux<OP>(pd[o1 * K + k1], pd[p1 * K + k1], v.y)));
        } else {
            flux[q0] = edge_flux<OP>(pd[o0 * K + k0], pd[p0 * K + k0], vn[q0]);
        }
    }
}

// ADV = false: the divergence alone (reference.py:63-79)
template <bool ADV>
__global__ void __launch_bounds__(256) idiv_advance_points_kernel(
    const int64_t *__restrict__ v2e, uint32_t n, FastDiv nk, double dt, const double *__restrict__ signs,
    const double *__restrict__ dual, const double *__restrict__ flux, const double *__restrict__ fluz,
    const double *__restrict__ pd, const double *__restrict__ rho, double *__restrict__ div,
    double *__restrict__ pd_out) {
    const int K = (int)nk.d;
    TSG_POINT_ITEMS(q, u, n) {
        const uint32_t v = nk.div(q);
        const int k = (int)(q - v * nk.d);
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < 6; ++s)
            acc = add(mul(__ldg(signs + (int64_t)v * 6 + s), flux[__ldg(v2e + (int64_t)v * 6 + s) * K + k]), acc);
        const double *Z = fluz + (int64_t)v * (K + 1) + k;
        acc = add(acc, sub(Z[1], Z[0]));
        const double d = dvd(acc, __ldg(dual + v));
        div[q] = d;
        if constexpr (ADV) pd_out[q] = sub(pd[q], dvd(mul(dt, d), rho[q]));
    }
}

__global__ void __launch_bounds__(256) icell_div_points_kernel(const int64_t *__restrict__ c2e, uint32_t n,
                                                               FastDiv nk, const double *__restrict__ vn,
                                                               const double *__restrict__ length,
                                                               const double *__restrict__ area,
                                                               double *__restrict__ out) {
    const int K = (int)nk.d;
    TSG_POINT_ITEMS(q, u, n) {
        const uint32_t c = nk.div(q);
        const int k = (int)(q - c * nk.d);
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const int64_t e = __ldg(c2e + (int64_t)c * 3 + s);
            acc = add(mul(vn[e * K + k], __ldg(length + e)), acc);
        }
        out[q] = dvd(acc, __ldg(area + c));
    }
}
#undef TSG_POINT_ITEMS

}  // namespace tsg

using namespace tsg;

static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

extern "C" int tsg_neighbor_reduce(const tsg_grid *g, int from_loc, int to_loc, int inner,
                                   const double *src, const double *scale, double *dst,
                                   tsg_stream s) {
    if (!g) return fail(TSG_EVALUE, "grid is NULL");
    if (!valid_loc(from_loc) || !valid_loc(to_loc))
        return fail(TSG_EVALUE, "no structured relation %d -> %d", from_loc, to_loc);
    if (inner < 1) return fail(TSG_EVALUE, "inner must be >= 1");
    if (!src || !dst) return fail(TSG_EVALUE, "tsg_neighbor_reduce: NULL array");
    FieldIx Fs(g->rows, g->cols, colors_of(to_loc), inner);
    FieldIx Fd(g->rows, g->cols, colors_of(from_loc), inner);
    FieldIx Fsc(g->rows, g->cols, colors_of(from_loc), 1);
    cudaStream_t st = (cudaStream_t)s;
    const int rel = from_loc * 3 + to_loc;
    // long level runs: the TMA-staged tile kernel (reduce_tma.cu); short ones: element lines
    if (inner >= 16 && (reinterpret_cast<uintptr_t>(src) % 16) == 0 &&
        (reinterpret_cast<uintptr_t>(dst) % 16) == 0)
        return reduce_tma(g, rel, inner, src, scale, dst, st);
    const int64_t lines = (int64_t)g->rows * Fd.colors;
#define TSG_REDUCE_CASE(R)                                                                        \
    case R:                                                                                      \
        if (scale)                                                                               \
            launch_lines(reduce_kernel<R, true>, g->cols, lines, g->num_sms, st, Fs, Fd, Fsc,     \
                         inner, src, scale, dst, g->flags);                                      \
        else                                                                                     \
            launch_lines(reduce_kernel<R, false>, g->cols, lines, g->num_sms, st, Fs, Fd, Fsc,    \
                         inner, src, scale, dst, g->flags);                                      \
        break;
    switch (rel) {
        TSG_REDUCE_CASE(0) TSG_REDUCE_CASE(1) TSG_REDUCE_CASE(2) TSG_REDUCE_CASE(3)
        TSG_REDUCE_CASE(4) TSG_REDUCE_CASE(5) TSG_REDUCE_CASE(6) TSG_REDUCE_CASE(7)
        TSG_REDUCE_CASE(8)
    }
#undef TSG_REDUCE_CASE
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_neighbor_reduce_indirect(const int64_t *table, int64_t nrows, int width,
                                            int nlev, const double *src, const double *scale,
                                            double *dst, tsg_stream s) {
    if (!table || !src || !dst) return fail(TSG_EVALUE, "tsg_neighbor_reduce_indirect: NULL array");
    if (nrows < 0 || width < 1 || nlev < 1)
        return fail(TSG_EVALUE, "bad table shape (%lld, %d) / levels %d", (long long)nrows, width, nlev);
    if (nrows == 0) return TSG_OK;
    const int sms = sm_count();
    cudaStream_t st = (cudaStream_t)s;
    const int64_t nitems = nrows * (int64_t)(nlev / 2);
    const bool aligned = (reinterpret_cast<uintptr_t>(src) % 16) == 0 &&
                         (reinterpret_cast<uintptr_t>(dst) % 16) == 0;
    if ((nlev & 1) == 0 && aligned && nitems < (1LL << 31) && (width == 2 || width == 3 || width == 4 || width == 6)) {
        const FastDiv np((uint32_t)(nlev / 2));
        auto go = [&](auto kernel) {
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0);
            int64_t blocks = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
            const int64_t need = (nitems + 256 * kUnroll - 1) / (256 * kUnroll);
            if (blocks > need) blocks = need;
            kernel<<<(unsigned)blocks, 256, 0, st>>>(table, (uint32_t)nitems, np, nlev, src, scale, dst);
        };
        if (scale) {
            switch (width) {
                case 2: go(reduce_indirect_pipe_kernel<2, true, 1>); break;
                case 3: go(reduce_indirect_pipe_kernel<3, true, 1>); break;
                case 4: go(reduce_indirect_pipe_kernel<4, true, 1>); break;
                default: go(reduce_indirect_pipe_kernel<6, true, 1>); break;
            }
        } else {
            switch (width) {
                case 2: go(reduce_indirect_pipe_kernel<2, false, 1>); break;
                case 3: go(reduce_indirect_pipe_kernel<3, false, 1>); break;
                case 4: go(reduce_indirect_pipe_kernel<4, false, 1>); break;
                default: go(reduce_indirect_pipe_kernel<6, false, 1>); break;
            }
        }
        TSG_CHECK_LAUNCH();
        return TSG_OK;
    }
    if ((reinterpret_cast<uintptr_t>(dst) % 16) == 0 && nrows * (int64_t)nlev < point_limit() &&
        (width == 2 || width == 3 || width == 4 || width == 6)) {  // odd level counts
        const uint32_t n = (uint32_t)(nrows * nlev);
        auto go = [&](auto kernel) {
            kernel<<<item_grid((const void *)kernel, (n + 1) / 2, 1, sms, true), 256, 0, st>>>(
                table, n, FastDiv((uint32_t)nlev), src, scale, dst);
        };
        if (scale) {
            switch (width) {
                case 2: go(reduce_indirect_flatpairs_kernel<2, true>); break;
                case 3: go(reduce_indirect_flatpairs_kernel<3, true>); break;
                case 4: go(reduce_indirect_flatpairs_kernel<4, true>); break;
                default: go(reduce_indirect_flatpairs_kernel<6, true>); break;
            }
        } else {
            switch (width) {
                case 2: go(reduce_indirect_flatpairs_kernel<2, false>); break;
                case 3: go(reduce_indirect_flatpairs_kernel<3, false>); break;
                case 4: go(reduce_indirect_flatpairs_kernel<4, false>); break;
                default: go(reduce_indirect_flatpairs_kernel<6, false>); break;
            }
        }
        TSG_CHECK_LAUNCH();
        return TSG_OK;
    }
    switch (width) {
        case 2: launch_rows(reduce_indirect_kernel<2>, nrows, sms, st, table, nrows, width, nlev, src, scale, dst); break;
        case 3: launch_rows(reduce_indirect_kernel<3>, nrows, sms, st, table, nrows, width, nlev, src, scale, dst); break;
        case 4: launch_rows(reduce_indirect_kernel<4>, nrows, sms, st, table, nrows, width, nlev, src, scale, dst); break;
        case 6: launch_rows(reduce_indirect_kernel<6>, nrows, sms, st, table, nrows, width, nlev, src, scale, dst); break;
        default: launch_rows(reduce_indirect_kernel<0>, nrows, sms, st, table, nrows, width, nlev, src, scale, dst);
    }
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_cell_divergence(const tsg_grid *g, int weighted, const double *vn,
                                   const double *length, const double *area,
                                   const double *weights, double *out, tsg_stream s) {
    if (!g) return fail(TSG_EVALUE, "grid is NULL");
    if (!vn || !out || (weighted ? !weights : (!length || !area)))
        return fail(TSG_EVALUE, "tsg_cell_divergence: NULL array");
    int K = g->levels;
    FieldIx Fvn(g->rows, g->cols, 3, K), Fl(g->rows, g->cols, 3, 1), Fa(g->rows, g->cols, 2, 1),
        Fw(g->rows, g->cols, 2, 3), Fo(g->rows, g->cols, 2, K);
    if (K >= 16 && (reinterpret_cast<uintptr_t>(vn) % 16) == 0 &&
        (reinterpret_cast<uintptr_t>(out) % 16) == 0)
        return cell_divergence_tma(g, weighted, vn, length, area, weights, out, (cudaStream_t)s);
    if (weighted)
        launch_lines(cell_div_kernel<true>, g->cols, 2LL * g->rows, g->num_sms, (cudaStream_t)s, Fvn,
                     Fl, Fa, Fw, Fo, K, vn, length, area, weights, out, g->flags);
    else
        launch_lines(cell_div_kernel<false>, g->cols, 2LL * g->rows, g->num_sms, (cudaStream_t)s, Fvn,
                     Fl, Fa, Fw, Fo, K, vn, length, area, weights, out, g->flags);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

static int check_step_args(int K, int flux_op) {
    if (K < 2) return fail(TSG_EVALUE, "the transport step needs at least 2 levels, got %d", K);
    if (flux_op != TSG_UPWIND && flux_op != TSG_CENTRED)
        return fail(TSG_EVALUE, "flux operator must be one of ['centred', 'upwind'], got %d", flux_op);
    return TSG_OK;
}

extern "C" int tsg_mpdata_step_unfused(const tsg_grid *g, const double *pd, const double *vn,
                                       const double *wn, const double *rho, const double *signs,
                                       const double *dual, double *flux, double *fluz,
                                       double *divvd, double *pd_out, double dt, double pivbz,
                                       int flux_op, tsg_stream s) {
    if (!g) return fail(TSG_EVALUE, "grid is NULL");
    int K = g->levels;
    if (int rc = check_step_args(K, flux_op)) return rc;
    if (!pd || !vn || !wn || !rho || !signs || !dual || !flux || !fluz || !divvd || !pd_out)
        return fail(TSG_EVALUE, "tsg_mpdata_step_unfused: NULL array");
    cudaStream_t st = (cudaStream_t)s;
    FieldIx Fv(g->rows, g->cols, 1, K), Fe(g->rows, g->cols, 3, K), Fw(g->rows, g->cols, 1, K + 1),
        Fs(g->rows, g->cols, 1, 6), Fd(g->rows, g->cols, 1, 1);
    const int C = g->cols, sms = g->num_sms;
    // level-pair items; an odd level count's last pair ends in the padding of every field
    // (even pitch).  Each stage runs over row bands of at most point_limit() items (one
    // band up to ~62 M vertices at 137 levels) before the next stage starts.
    const int np = (K + 1) / 2;
    auto stage = [&](auto kernel, int pairs, auto launch) {
        for_point_bands(g->rows, C, 1, pairs, [&](const PointDec &D) {
            launch(item_grid((const void *)kernel, D.n, kUnroll, sms), D);
        });
    };
    if (flux_op == TSG_UPWIND)
        stage(flux3_pairs_kernel<TSG_UPWIND>, np, [&](unsigned b, const PointDec &D) {
            flux3_pairs_kernel<TSG_UPWIND><<<b, 256, 0, st>>>(Fv, Fe, D, pd, vn, flux, g->flags);
        });
    else
        stage(flux3_pairs_kernel<TSG_CENTRED>, np, [&](unsigned b, const PointDec &D) {
            flux3_pairs_kernel<TSG_CENTRED><<<b, 256, 0, st>>>(Fv, Fe, D, pd, vn, flux, g->flags);
        });
    stage(fluz_pairs_kernel, K / 2 + 1, [&](unsigned b, const PointDec &D) {
        fluz_pairs_kernel<<<b, 256, 0, st>>>(Fv, Fw, D, K, pivbz, pd, wn, fluz, g->flags);
    });
    stage(div_pairs_kernel, np, [&](unsigned b, const PointDec &D) {
        div_pairs_kernel<<<b, 256, 0, st>>>(Fe, Fw, Fs, Fd, Fv, D, flux, fluz, signs, dual, divvd, g->flags);
    });
    stage(advance_pairs_kernel, np, [&](unsigned b, const PointDec &D) {
        advance_pairs_kernel<<<b, 256, 0, st>>>(Fv, D, dt, pd, divvd, rho, pd_out, g->flags);
    });
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

// odd level counts / unaligned rows: flat pairs when vn and flux are 16-byte aligned
static void launch_iflux_points(int flux_op, const int64_t *e2v, uint32_t nE, int nlev, const double *pd,
                                const double *vn, double *flux, int sms, cudaStream_t st) {
    const bool pairs = (reinterpret_cast<uintptr_t>(vn) % 16) == 0 && (reinterpret_cast<uintptr_t>(flux) % 16) == 0;
    auto go = [&](auto kernel, uint32_t items) {
        kernel<<<item_grid((const void *)kernel, items, kUnroll, sms), 256, 0, st>>>(e2v, nE, FastDiv(nlev), pd, vn,
                                                                                     flux);
    };
    if (pairs) {
        if (flux_op == TSG_UPWIND) go(iflux_flatpairs_kernel<TSG_UPWIND>, (nE + 1) / 2);
        else go(iflux_flatpairs_kernel<TSG_CENTRED>, (nE + 1) / 2);
    } else {
        if (flux_op == TSG_UPWIND) go(iflux_points_kernel<TSG_UPWIND>, nE);
        else go(iflux_points_kernel<TSG_CENTRED>, nE);
    }
}

extern "C" int tsg_transport_indirect(const int64_t *e2v, const int64_t *v2e, const double *signs,
                                      const double *dual, const double *pd, const double *vn,
                                      const double *wn, const double *rho, int64_t nv, int64_t ne,
                                      int nlev, double dt, double pivbz, int flux_op, double *flux,
                                      double *fluz, double *div, double *pd_out, tsg_stream s) {
    if (int rc = check_step_args(nlev, flux_op)) return rc;
    if (!e2v || !v2e || !signs || !dual || !pd || !vn || !wn || !rho || !flux || !fluz || !div ||
        !pd_out)
        return fail(TSG_EVALUE, "tsg_transport_indirect: NULL array");
    if (nv < 1 || ne < 1) return fail(TSG_EVALUE, "empty mesh (nv=%lld, ne=%lld)", (long long)nv, (long long)ne);
    cudaStream_t st = (cudaStream_t)s;
    const int sms = sm_count();
    auto a16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) % 16) == 0; };
    if ((nlev & 1) == 0 && ne * (nlev / 2) < (1LL << 31) && nv * (nlev / 2 + 1) < (1LL << 31) &&
        a16(pd) && a16(vn) && a16(rho) && a16(flux) && a16(div) && a16(pd_out)) {
        const int np = nlev / 2;
        const uint32_t nE = (uint32_t)(ne * np), nV = (uint32_t)(nv * np), nZ = (uint32_t)(nv * (np + 1));
        auto blocks = [&](const void *kernel, uint32_t n, int per_thread) {
            return item_grid(kernel, n, per_thread, sms, per_thread == 1);
        };
        if (flux_op == TSG_UPWIND)
            iflux_pairs_kernel<TSG_UPWIND><<<blocks((const void *)iflux_pairs_kernel<TSG_UPWIND>, nE, kUnroll), 256, 0,
                                             st>>>(e2v, nE, FastDiv(np), nlev, pd, vn, flux);
        else
            iflux_pairs_kernel<TSG_CENTRED><<<blocks((const void *)iflux_pairs_kernel<TSG_CENTRED>, nE, kUnroll), 256,
                                              0, st>>>(e2v, nE, FastDiv(np), nlev, pd, vn, flux);
        ifluz_pairs_kernel<<<blocks((const void *)ifluz_pairs_kernel, nZ, kUnroll), 256, 0, st>>>(
            nZ, FastDiv(np + 1), nlev, pivbz, pd, wn, fluz);
        const unsigned bV = blocks((const void *)idiv_advance_pipe_kernel<true>, nV, 1);
        idiv_advance_pipe_kernel<true><<<bV, 256, 0, st>>>(v2e, nV, FastDiv(np), nlev, dt, signs, dual, flux, fluz, pd,
                                                     rho, div, pd_out);
        TSG_CHECK_LAUNCH();
        return TSG_OK;
    }
    if (ne * (int64_t)nlev < point_limit() && nv * (int64_t)(nlev / 2 + 1) < (1LL << 31)) {
        // odd level counts (rows not 16-byte aligned): point items, any alignment
        const uint32_t nE = (uint32_t)(ne * nlev), nV = (uint32_t)(nv * nlev);
        const uint32_t nZ = (uint32_t)(nv * (nlev / 2 + 1));
        launch_iflux_points(flux_op, e2v, nE, nlev, pd, vn, flux, sms, st);
        ifluz_pairs_kernel<<<item_grid((const void *)ifluz_pairs_kernel, nZ, kUnroll, sms), 256, 0, st>>>(
            nZ, FastDiv(nlev / 2 + 1), nlev, pivbz, pd, wn, fluz);
        idiv_advance_points_kernel<true><<<item_grid((const void *)idiv_advance_points_kernel<true>, nV, kUnroll, sms),
                                           256, 0, st>>>(v2e, nV, FastDiv(nlev), dt, signs, dual, flux, fluz, pd, rho,
                                                         div, pd_out);
        TSG_CHECK_LAUNCH();
        return TSG_OK;
    }
    if (flux_op == TSG_UPWIND)
        launch_rows(iflux_kernel<TSG_UPWIND>, ne, sms, st, e2v, ne, nlev, pd, vn, flux);
    else
        launch_rows(iflux_kernel<TSG_CENTRED>, ne, sms, st, e2v, ne, nlev, pd, vn, flux);
    launch_rows(ifluz_kernel, nv, sms, st, nv, nlev, pivbz, pd, wn, fluz);
    launch_rows(idiv_advance_kernel, nv, sms, st, v2e, nv, nlev, dt, signs, dual, flux, fluz, pd, rho,
                div, pd_out);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

// -- the reference's flat stages one by one (reference.py:18-90, 119-134) ---------------

extern "C" int tsg_flat_flux(const int64_t *e2v, const double *pd, const double *vn, int64_t ne, int nlev,
                             int flux_op, double *flux, tsg_stream s) {
    if (!e2v || !pd || !vn || !flux) return fail(TSG_EVALUE, "tsg_flat_flux: NULL array");
    if (flux_op != TSG_UPWIND && flux_op != TSG_CENTRED) return fail(TSG_EVALUE, "unknown flux operator %d", flux_op);
    if (ne < 0 || nlev < 1) return fail(TSG_EVALUE, "bad shape (ne=%lld, levels %d)", (long long)ne, nlev);
    if (ne == 0) return TSG_OK;
    cudaStream_t st = (cudaStream_t)s;
    const int sms = sm_count();
    auto a16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) % 16) == 0; };
    if ((nlev & 1) == 0 && ne * (nlev / 2) < (1LL << 31) && a16(pd) && a16(vn) && a16(flux)) {
        const int np = nlev / 2;
        const uint32_t nE = (uint32_t)(ne * np);
        if (flux_op == TSG_UPWIND)
            iflux_pairs_kernel<TSG_UPWIND><<<item_grid((const void *)iflux_pairs_kernel<TSG_UPWIND>, nE, kUnroll,
                                                           sms), 256, 0, st>>>(e2v, nE, FastDiv(np), nlev, pd, vn, flux);
        else
            iflux_pairs_kernel<TSG_CENTRED><<<item_grid((const void *)iflux_pairs_kernel<TSG_CENTRED>, nE, kUnroll,
                                                            sms), 256, 0, st>>>(e2v, nE, FastDiv(np), nlev, pd, vn, flux);
    } else if (ne * (int64_t)nlev < point_limit()) {
        const uint32_t nE = (uint32_t)(ne * nlev);
        launch_iflux_points(flux_op, e2v, nE, nlev, pd, vn, flux, sms, st);
    } else if (flux_op == TSG_UPWIND) {
        launch_rows(iflux_kernel<TSG_UPWIND>, ne, sms, st, e2v, ne, nlev, pd, vn, flux);
    } else {
        launch_rows(iflux_kernel<TSG_CENTRED>, ne, sms, st, e2v, ne, nlev, pd, vn, flux);
    }
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_flat_fluz(const double *pd, const double *wn, int64_t nv, int nlev, double pivbz, double *fluz,
                             tsg_stream s) {
    if (!pd || !wn || !fluz) return fail(TSG_EVALUE, "tsg_flat_fluz: NULL array");
    if (nlev < 2) return fail(TSG_EVALUE, "need at least 2 levels, got %d", nlev);
    if (nv < 0) return fail(TSG_EVALUE, "bad vertex count %lld", (long long)nv);
    if (nv == 0) return TSG_OK;
    const int np = nlev / 2 + 1;  // interface pairs covering 0..nlev
    if (nv * np < (1LL << 31)) {
        const uint32_t n = (uint32_t)(nv * np);
        ifluz_pairs_kernel<<<item_grid((const void *)ifluz_pairs_kernel, n, kUnroll, sm_count()), 256, 0,
                             (cudaStream_t)s>>>(n, FastDiv(np), nlev, pivbz, pd, wn, fluz);
    } else {
        launch_rows(ifluz_kernel, nv, sm_count(), (cudaStream_t)s, nv, nlev, pivbz, pd, wn, fluz);
    }
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_flat_divergence(const int64_t *v2e, int width, const double *signs, const double *dual,
                                   const double *flux, const double *fluz, int64_t nv, int nlev, double *div,
                                   tsg_stream s) {
    if (!v2e || !signs || !dual || !flux || !fluz || !div) return fail(TSG_EVALUE, "tsg_flat_divergence: NULL array");
    if (nv < 0 || width < 0 || nlev < 1)
        return fail(TSG_EVALUE, "bad shape (nv=%lld, width %d, levels %d)", (long long)nv, width, nlev);
    if (nv == 0) return TSG_OK;
    auto a16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) % 16) == 0; };
    if (width == 6 && (nlev & 1) == 0 && nv * (nlev / 2) < (1LL << 31) && a16(flux) && a16(div)) {
        const uint32_t n = (uint32_t)(nv * (nlev / 2));
        idiv_advance_pipe_kernel<false><<<item_grid((const void *)idiv_advance_pipe_kernel<false>, n, 1, sm_count(),
                                                    true), 256, 0, (cudaStream_t)s>>>(
            v2e, n, FastDiv(nlev / 2), nlev, 0.0, signs, dual, flux, fluz, nullptr, nullptr, div, nullptr);
    } else if (width == 6 && nv * (int64_t)nlev < point_limit()) {
        const uint32_t n = (uint32_t)(nv * nlev);
        idiv_advance_points_kernel<false><<<item_grid((const void *)idiv_advance_points_kernel<false>, n, kUnroll,
                                                      sm_count()), 256, 0, (cudaStream_t)s>>>(
            v2e, n, FastDiv(nlev), 0.0, signs, dual, flux, fluz, nullptr, nullptr, div, nullptr);
    } else {
        launch_rows(idiv_kernel, nv, sm_count(), (cudaStream_t)s, v2e, width, nv, nlev, signs, dual, flux, fluz,
                    div);
    }
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_flat_advance(const double *pd, const double *div, const double *rho, int64_t n, double dt,
                                double *pd_out, tsg_stream s) {
    if (!pd || !div || !rho || !pd_out) return fail(TSG_EVALUE, "tsg_flat_advance: NULL array");
    if (n < 0) return fail(TSG_EVALUE, "bad value count %lld", (long long)n);
    if (n == 0) return TSG_OK;
    auto a16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) % 16) == 0; };
    if ((n & 1) == 0 && a16(pd) && a16(div) && a16(rho) && a16(pd_out)) {
        advance_flat2_kernel<<<item_grid((const void *)advance_flat2_kernel, n / 2, 1, sm_count()), 256, 0,
                               (cudaStream_t)s>>>(n / 2, dt, pd, div, rho, pd_out);
    } else {
        const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
        advance_flat_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)s>>>(n, dt, pd, div, rho, pd_out);
    }
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_flat_cell_divergence(const int64_t *c2e, int width, const double *vn, const double *length,
                                        const double *area, int64_t nc, int nlev, double *out, tsg_stream s) {
    if (!c2e || !vn || !length || !area || !out) return fail(TSG_EVALUE, "tsg_flat_cell_divergence: NULL array");
    if (nc < 0 || width < 0 || nlev < 1)
        return fail(TSG_EVALUE, "bad shape (nc=%lld, width %d, levels %d)", (long long)nc, width, nlev);
    if (nc == 0) return TSG_OK;
    auto a16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) % 16) == 0; };
    if (width == 3 && (nlev & 1) == 0 && nc * (nlev / 2) < (1LL << 31) && a16(vn) && a16(out)) {
        const uint32_t n = (uint32_t)(nc * (nlev / 2));
        icell_div_pipe_kernel<<<item_grid((const void *)icell_div_pipe_kernel, n, 1, sm_count(), true), 256, 0,
                                (cudaStream_t)s>>>(c2e, n, FastDiv(nlev / 2), nlev, vn, length, area, out);
    } else if (width == 3 && nc * (int64_t)nlev < point_limit()) {
        const uint32_t n = (uint32_t)(nc * nlev);
        icell_div_points_kernel<<<item_grid((const void *)icell_div_points_kernel, n, kUnroll, sm_count()), 256, 0,
                                  (cudaStream_t)s>>>(c2e, n, FastDiv(nlev), vn, length, area, out);
    } else {
        launch_rows(icell_div_kernel, nc, sm_count(), (cudaStream_t)s, c2e, width, nc, nlev, vn, length, area,
                    out);
    }
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}
