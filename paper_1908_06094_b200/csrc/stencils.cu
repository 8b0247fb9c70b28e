// Neighbour-reduction stencils and the materialising (unfused / indirect) MPDATA steps.
//
// These kernels are HBM-bound streaming sweeps: one thread per (element, level) with the
// level axis fastest, so every neighbour read is a contiguous run of a neighbouring
// element's level column (coalesced; neighbour reuse is served by L1/L2).  Grids are a
// multiple of the SM count with grid-stride loops.
#include "tsg_common.cuh"
#include "tsg_offsets.cuh"

namespace tsg {

static inline int grid_for(int64_t work, int threads, int num_sms) {
    int64_t blocks = (work + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms * 16;
    if (blocks > cap) blocks = cap;
    return (int)(blocks < 1 ? 1 : blocks);
}

#define GRID_STRIDE(t, n)                                                     \
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (n); \
         t += (int64_t)gridDim.x * blockDim.x)

// t -> (i, c, j, k) over [rows][colors][cols][nk]
struct Pt {
    int i, c, j, k;
};
__device__ __forceinline__ Pt decompose(int64_t t, int nk, int cols, int colors) {
    Pt p;
    int64_t id = t / nk;
    p.k = (int)(t - id * nk);
    p.j = (int)(id % cols);
    int64_t rest = id / cols;
    p.c = (int)(rest % colors);
    p.i = (int)(rest / colors);
    return p;
}

// -- structured reduce over any relation (stencil.py:404-408 with the sum fold) -------

__global__ void reduce_kernel(FieldIx Fs, FieldIx Fd, FieldIx Fsc, int rel, int nk,
                              const double *__restrict__ src, const double *__restrict__ scale,
                              double *__restrict__ dst, int flags) {
    const int width = c_rel_width[rel];
    const int64_t n = (int64_t)Fd.rows * Fd.colors * Fd.cols * nk;
    GRID_STRIDE(t, n) {
        Pt p = decompose(t, nk, Fd.cols, Fd.colors);
        double acc = 0.0;
        for (int s = 0; s < width; ++s) {
            const int8_t *o = c_offsets[rel][p.c][s];
            acc = add(src[Fs.at(p.i + o[0], o[1], p.j + o[2]) + p.k], acc);
        }
        if (scale) acc = mul(acc, scale[Fsc.at(p.i, p.c, p.j)]);
        store_img(dst, Fd, p.i, p.c, p.j, p.k, acc, flags);
    }
}

// -- table-driven reduce over flat arrays (kernels.py:83-104, reference.py:137-157) -----

__global__ void reduce_indirect_kernel(const int64_t *__restrict__ table, int64_t nrows,
                                       int width, int nlev, const double *__restrict__ src,
                                       const double *__restrict__ scale,
                                       double *__restrict__ dst) {
    const int64_t n = nrows * nlev;
    GRID_STRIDE(t, n) {
        int64_t r = t / nlev;
        int k = (int)(t - r * nlev);
        double acc = 0.0;
        for (int s = 0; s < width; ++s) acc = add(src[__ldg(table + r * width + s) * nlev + k], acc);
        if (scale) acc = mul(acc, scale[r]);
        dst[t] = acc;
    }
}

// -- cell divergence (mpdata.py:361-416, reference.py:119-134) --------------------------

__global__ void cell_div_kernel(FieldIx Fvn, FieldIx Fl, FieldIx Fa, FieldIx Fw, FieldIx Fo,
                                int nk, int weighted, const double *__restrict__ vn,
                                const double *__restrict__ length,
                                const double *__restrict__ area,
                                const double *__restrict__ weights, double *__restrict__ out,
                                int flags) {
    const int rel = TSG_CELLS * 3 + TSG_EDGES;
    const int64_t n = (int64_t)Fo.rows * 2 * Fo.cols * nk;
    GRID_STRIDE(t, n) {
        Pt p = decompose(t, nk, Fo.cols, 2);
        double acc = 0.0;
        for (int s = 0; s < 3; ++s) {
            const int8_t *o = c_offsets[rel][p.c][s];
            int ei = p.i + o[0], ec = o[1], ej = p.j + o[2];
            double v = vn[Fvn.at(ei, ec, ej) + p.k];
            double w = weighted ? weights[Fw.at(p.i, p.c, p.j) + s] : length[Fl.at(ei, ec, ej)];
            acc = add(mul(v, w), acc);
        }
        if (!weighted) acc = dvd(acc, area[Fa.at(p.i, p.c, p.j)]);
        store_img(out, Fo, p.i, p.c, p.j, p.k, acc, flags);
    }
}

// -- unfused MPDATA (run_naive analogue, executors.py:213-245) --------------------------

template <int OP>
__global__ void flux_kernel(FieldIx Fp, FieldIx Fe, int K, const double *__restrict__ pd,
                            const double *__restrict__ vn, double *__restrict__ flux, int flags) {
    const int64_t n = (int64_t)Fe.rows * 3 * Fe.cols * K;
    GRID_STRIDE(t, n) {
        Pt p = decompose(t, K, Fe.cols, 3);
        // E->V slot 1 (connectivity.py:38-42): c0 (0,+1), c1 (+1,+1), c2 (+1,0)
        int oi = p.c == 0 ? 0 : 1, oj = p.c == 2 ? 0 : 1;
        double po = pd[Fp.at(p.i, 0, p.j) + p.k];
        double pp = pd[Fp.at(p.i + oi, 0, p.j + oj) + p.k];
        double v = vn[Fe.at(p.i, p.c, p.j) + p.k];
        store_img(flux, Fe, p.i, p.c, p.j, p.k, edge_flux<OP>(po, pp, v), flags);
    }
}

__global__ void fluz_kernel(FieldIx Fp, FieldIx Fw, int K, double pivbz,
                            const double *__restrict__ pd, const double *__restrict__ wn,
                            double *__restrict__ fluz, int flags) {
    const int64_t n = (int64_t)Fp.rows * Fp.cols * (K + 1);
    GRID_STRIDE(t, n) {
        Pt p = decompose(t, K + 1, Fp.cols, 1);
        const double *P = pd + Fp.at(p.i, 0, p.j);
        const double *W = wn + Fw.at(p.i, 0, p.j);
        double f;
        if (p.k == 0) f = mul(pivbz, fluz_interior(W[1], P[0], P[1]));
        else if (p.k == K) f = mul(pivbz, fluz_interior(W[K - 1], P[K - 2], P[K - 1]));
        else f = fluz_interior(W[p.k], P[p.k - 1], P[p.k]);
        store_img(fluz, Fw, p.i, 0, p.j, p.k, f, flags);
    }
}

__global__ void div_kernel(FieldIx Fe, FieldIx Fw, FieldIx Fs, FieldIx Fd, FieldIx Fv, int K,
                           const double *__restrict__ flux, const double *__restrict__ fluz,
                           const double *__restrict__ signs, const double *__restrict__ dual,
                           double *__restrict__ divvd, int flags) {
    const int rel = TSG_VERTICES * 3 + TSG_EDGES;
    const int64_t n = (int64_t)Fv.rows * Fv.cols * K;
    GRID_STRIDE(t, n) {
        Pt p = decompose(t, K, Fv.cols, 1);
        const double *S = signs + Fs.at(p.i, 0, p.j);
        double acc = 0.0;
        for (int s = 0; s < 6; ++s) {
            const int8_t *o = c_offsets[rel][0][s];
            acc = add(mul(S[s], flux[Fe.at(p.i + o[0], o[1], p.j + o[2]) + p.k]), acc);
        }
        const double *Z = fluz + Fw.at(p.i, 0, p.j);
        acc = add(acc, sub(Z[p.k + 1], Z[p.k]));
        store_img(divvd, Fv, p.i, 0, p.j, p.k, dvd(acc, dual[Fd.at(p.i, 0, p.j)]), flags);
    }
}

__global__ void advance_kernel(FieldIx Fv, int K, double dt, const double *__restrict__ pd,
                               const double *__restrict__ divvd, const double *__restrict__ rho,
                               double *__restrict__ pd_out, int flags) {
    const int64_t n = (int64_t)Fv.rows * Fv.cols * K;
    GRID_STRIDE(t, n) {
        Pt p = decompose(t, K, Fv.cols, 1);
        int64_t o = Fv.at(p.i, 0, p.j) + p.k;
        double slope = mul(dt, divvd[o]);
        slope = dvd(slope, rho[o]);
        store_img(pd_out, Fv, p.i, 0, p.j, p.k, sub(pd[o], slope), flags);
    }
}

// -- indirect (table-driven) MPDATA over flat arrays (reference.py:93-116) -------------

template <int OP>
__global__ void iflux_kernel(const int64_t *__restrict__ e2v, int64_t ne, int K,
                             const double *__restrict__ pd, const double *__restrict__ vn,
                             double *__restrict__ flux) {
    GRID_STRIDE(t, ne * K) {
        int64_t e = t / K;
        int k = (int)(t - e * K);
        double po = pd[__ldg(e2v + 2 * e) * K + k], pp = pd[__ldg(e2v + 2 * e + 1) * K + k];
        flux[t] = edge_flux<OP>(po, pp, vn[t]);
    }
}

__global__ void ifluz_kernel(int64_t nv, int K, double pivbz, const double *__restrict__ pd,
                             const double *__restrict__ wn, double *__restrict__ fluz) {
    GRID_STRIDE(t, nv * (K + 1)) {
        int64_t v = t / (K + 1);
        int k = (int)(t - v * (K + 1));
        const double *P = pd + v * K, *W = wn + v * (K + 1);
        double f;
        if (k == 0) f = mul(pivbz, fluz_interior(W[1], P[0], P[1]));
        else if (k == K) f = mul(pivbz, fluz_interior(W[K - 1], P[K - 2], P[K - 1]));
        else f = fluz_interior(W[k], P[k - 1], P[k]);
        fluz[t] = f;
    }
}

__global__ void idiv_advance_kernel(const int64_t *__restrict__ v2e, int64_t nv, int K, double dt,
                                    const double *__restrict__ signs,
                                    const double *__restrict__ dual,
                                    const double *__restrict__ flux,
                                    const double *__restrict__ fluz,
                                    const double *__restrict__ pd, const double *__restrict__ rho,
                                    double *__restrict__ div, double *__restrict__ pd_out) {
    GRID_STRIDE(t, nv * K) {
        int64_t v = t / K;
        int k = (int)(t - v * K);
        double acc = 0.0;
        for (int s = 0; s < 6; ++s)
            acc = add(mul(__ldg(signs + v * 6 + s), flux[__ldg(v2e + v * 6 + s) * K + k]), acc);
        const double *Z = fluz + v * (K + 1);
        acc = add(acc, sub(Z[k + 1], Z[k]));
        double d = dvd(acc, __ldg(dual + v));
        div[t] = d;
        double slope = mul(dt, d);
        slope = dvd(slope, rho[t]);
        pd_out[t] = sub(pd[t], slope);
    }
}

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
    int64_t n = (int64_t)g->rows * Fd.colors * g->cols * inner;
    reduce_kernel<<<grid_for(n, 256, g->num_sms), 256, 0, (cudaStream_t)s>>>(
        Fs, Fd, Fsc, from_loc * 3 + to_loc, inner, src, scale, dst, g->flags);
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
    reduce_indirect_kernel<<<grid_for(nrows * nlev, 256, sm_count()), 256, 0, (cudaStream_t)s>>>(
        table, nrows, width, nlev, src, scale, dst);
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
    int64_t n = (int64_t)g->rows * 2 * g->cols * K;
    cell_div_kernel<<<grid_for(n, 256, g->num_sms), 256, 0, (cudaStream_t)s>>>(
        Fvn, Fl, Fa, Fw, Fo, K, weighted, vn, length, area, weights, out, g->flags);
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
    const int T = 256, sms = g->num_sms;
    int64_t nE = (int64_t)g->rows * 3 * g->cols * K, nV = (int64_t)g->rows * g->cols * K;
    if (flux_op == TSG_UPWIND)
        flux_kernel<TSG_UPWIND><<<grid_for(nE, T, sms), T, 0, st>>>(Fv, Fe, K, pd, vn, flux, g->flags);
    else
        flux_kernel<TSG_CENTRED><<<grid_for(nE, T, sms), T, 0, st>>>(Fv, Fe, K, pd, vn, flux, g->flags);
    fluz_kernel<<<grid_for(nV + g->rows * (int64_t)g->cols, T, sms), T, 0, st>>>(Fv, Fw, K, pivbz,
                                                                               pd, wn, fluz, g->flags);
    div_kernel<<<grid_for(nV, T, sms), T, 0, st>>>(Fe, Fw, Fs, Fd, Fv, K, flux, fluz, signs, dual,
                                                  divvd, g->flags);
    advance_kernel<<<grid_for(nV, T, sms), T, 0, st>>>(Fv, K, dt, pd, divvd, rho, pd_out, g->flags);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
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
    const int T = 256, sms = sm_count();
    if (flux_op == TSG_UPWIND)
        iflux_kernel<TSG_UPWIND><<<grid_for(ne * nlev, T, sms), T, 0, st>>>(e2v, ne, nlev, pd, vn, flux);
    else
        iflux_kernel<TSG_CENTRED><<<grid_for(ne * nlev, T, sms), T, 0, st>>>(e2v, ne, nlev, pd, vn, flux);
    ifluz_kernel<<<grid_for(nv * (nlev + 1), T, sms), T, 0, st>>>(nv, nlev, pivbz, pd, wn, fluz);
    idiv_advance_kernel<<<grid_for(nv * nlev, T, sms), T, 0, st>>>(v2e, nv, nlev, dt, signs, dual,
                                                                  flux, fluz, pd, rho, div, pd_out);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}
