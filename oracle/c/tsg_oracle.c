/* Plain-C restatement of the reference flat transport step -- TEST/BASELINE ONLY.
 *
 * Restates /root/reference/pkg/src/tristencil/reference.py:
 *   upwind_flux      :18-26    centred_flux   :29-35
 *   upwind_fluz      :38-60    flux_divergence:63-79
 *   advance_density  :82-90    transport_step :93-116
 *   neighbor_sum(_scaled) :137-157
 * Same per-element operation order as the reference (and as oracle/tsg_oracle.py);
 * compiled with -ffp-contract=off so no multiply-add is fused.  Elements are
 * distributed over OpenMP threads; each element's arithmetic is independent, so
 * results do not depend on the thread count.
 *
 * Arrays are flat [element, level] row-major; neighbour tables are int64
 * [n_from, width] in any numbering, exactly like the reference's flat oracle.
 * Used by tests (bitwise cross-check with the numpy restatement) and as the
 * multi-core CPU baseline in bench.py.  Never linked into the product.
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* numpy.maximum / numpy.minimum with a zero second operand:
 * NaN in the first operand propagates; ties return the second operand. */
static inline double np_max0(double a) { return (a > 0.0 || a != a) ? a : 0.0; }
static inline double np_min0(double a) { return (a < 0.0 || a != a) ? a : 0.0; }

int tsgo_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void tsgo_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int tsgo_transport_step(const int64_t *e2v, const int64_t *v2e, const double *signs,
                        const double *dual, const double *pd, const double *vn,
                        const double *wn, const double *rho, int64_t nv, int64_t ne,
                        int nlev, double dt, double pivbz, int flux_op, double *flux,
                        double *fluz, double *div, double *pd_out) {
    const int64_t K = nlev, KW = nlev + 1;
    if (nlev < 2) return 1;
    /* reference.py:18-35 */
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < ne; ++e) {
        const double *p1 = pd + e2v[2 * e] * K, *p2 = pd + e2v[2 * e + 1] * K;
        const double *v = vn + e * K;
        double *f = flux + e * K;
        if (flux_op == 0) {
            for (int64_t k = 0; k < K; ++k) {
                double zpos = np_max0(v[k]), zneg = np_min0(v[k]);
                double a = p1[k] * zpos;
                double b = p2[k] * zneg;
                f[k] = a + b;
            }
        } else {
            for (int64_t k = 0; k < K; ++k) {
                double h = 0.5 * v[k];
                double s = p1[k] + p2[k];
                f[k] = h * s;
            }
        }
    }
    /* reference.py:38-60 */
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < nv; ++n) {
        const double *w = wn + n * KW, *p = pd + n * K;
        double *fz = fluz + n * KW;
        for (int64_t k = 1; k < K; ++k) {
            double a = np_max0(w[k]) * p[k - 1];
            double b = np_min0(w[k]) * p[k];
            fz[k] = a + b;
        }
        fz[0] = pivbz * fz[1];
        fz[K] = pivbz * fz[K - 1];
    }
    /* reference.py:63-79 and :82-90 */
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < nv; ++n) {
        const double *fz = fluz + n * KW, *p = pd + n * K, *r = rho + n * K;
        double *d = div + n * K, *o = pd_out + n * K;
        for (int64_t k = 0; k < K; ++k) {
            double acc = 0.0;
            for (int s = 0; s < 6; ++s) {
                double t = signs[n * 6 + s] * flux[v2e[n * 6 + s] * K + k];
                acc = t + acc;
            }
            double dz = fz[k + 1] - fz[k];
            acc = acc + dz;
            d[k] = acc / dual[n];
            double slope = dt * d[k];
            slope = slope / r[k];
            o[k] = p[k] - slope;
        }
    }
    return 0;
}

/* reference.py:137-157: out[r] = ((0 + a[t0]) + a[t1]) + ... (* fac[r]) */
int tsgo_neighbor_sum(const int64_t *table, int64_t nrows, int width, const double *a,
                      int nlev, const double *fac, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; ++r) {
        for (int64_t k = 0; k < nlev; ++k) {
            double acc = 0.0;
            for (int s = 0; s < width; ++s) acc = a[table[r * width + s] * nlev + k] + acc;
            out[r * nlev + k] = fac ? acc * fac[r] : acc;
        }
    }
    return 0;
}
