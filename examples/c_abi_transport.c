/* A transport step through the C ABI alone (include/tsg.h + libtsg.so + the CUDA runtime),
 * the way a non-Python caller integrates: no PyTorch, no Python.
 *
 * It builds the neighbour tables and orientation signs of a periodic rows x cols patch on
 * the device, fills flat [element, level] inputs with a host PRNG, and advances them two
 * ways that must agree bitwise:
 *   1. tsg_transport_indirect -- reference.transport_step (reference.py:93-116) over flat
 *      arrays and neighbour tables (any numbering; canonical here);
 *   2. the structured fast path: tsg_grid_create -> tsg_pack (flat -> the parallelogram
 *      layout) -> tsg_mpdata_step (the fused kernel) -> tsg_unpack.
 * Then it runs a 5-step persistent loop (tsg_mpdata_run) and checks it against five
 * chained tsg_transport_indirect calls.  Prints "OK" and exits 0 when everything matches.
 *
 *   gcc -O2 -I include examples/c_abi_transport.c -L paper_1908_06094_b200 -ltsg \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -o c_abi_transport
 *   ./c_abi_transport [rows cols levels]
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "tsg.h"

#define CK(call)                                                                          \
    do {                                                                                  \
        int rc_ = (call);                                                                 \
        if (rc_) {                                                                        \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, tsg_last_error());        \
            exit(1);                                                                      \
        }                                                                                 \
    } while (0)
#define CU(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            fprintf(stderr, "%s failed: %s\n", #call, cudaGetErrorString(e_));            \
            exit(1);                                                                      \
        }                                                                                 \
    } while (0)

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static double uniform(double lo, double hi) {  /* splitmix64 */
    uint64_t z = (rng_state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return lo + (hi - lo) * (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

static void *dev(size_t bytes) {
    void *p = NULL;
    CU(cudaMalloc(&p, bytes));
    return p;
}

static double *dev_fill(size_t n, double lo, double hi) {
    double *h = (double *)malloc(n * sizeof(double));
    for (size_t i = 0; i < n; ++i) h[i] = uniform(lo, hi);
    double *d = (double *)dev(n * sizeof(double));
    CU(cudaMemcpy(d, h, n * sizeof(double), cudaMemcpyHostToDevice));
    free(h);
    return d;
}

static int same(const double *a, const double *b, size_t n) {
    double *ha = (double *)malloc(n * sizeof(double)), *hb = (double *)malloc(n * sizeof(double));
    CU(cudaMemcpy(ha, a, n * sizeof(double), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(hb, b, n * sizeof(double), cudaMemcpyDeviceToHost));
    int ok = memcmp(ha, hb, n * sizeof(double)) == 0;
    free(ha);
    free(hb);
    return ok;
}

int main(int argc, char **argv) {
    const int rows = argc > 3 ? atoi(argv[1]) : 37, cols = argc > 3 ? atoi(argv[2]) : 45;
    const int K = argc > 3 ? atoi(argv[3]) : 24;
    const double dt = 0.1, pivbz = 0.8;
    const int64_t nv = (int64_t)rows * cols, ne = 3 * nv;
    if (tsg_abi_version() < 1) return 1;

    /* neighbour tables and orientation signs, on the device */
    int64_t *e2v = (int64_t *)dev(ne * 2 * sizeof(int64_t)), *v2e = (int64_t *)dev(nv * 6 * sizeof(int64_t));
    double *signs = (double *)dev(nv * 6 * sizeof(double));
    CK(tsg_build_neighbor_table(rows, cols, TSG_EDGES, TSG_VERTICES, NULL, NULL, e2v, NULL));
    CK(tsg_build_neighbor_table(rows, cols, TSG_VERTICES, TSG_EDGES, NULL, NULL, v2e, NULL));
    CK(tsg_edge_signs(rows, cols, signs, NULL));

    /* flat inputs (canonical numbering) */
    double *pd = dev_fill(nv * K, 0.5, 1.5), *vn = dev_fill(ne * K, -0.5, 0.5);
    double *wn = dev_fill(nv * (K + 1), -0.5, 0.5), *rho = dev_fill(nv * K, 0.5, 1.5);
    double *dual = dev_fill(nv, 0.5, 1.5);
    double *flux = (double *)dev(ne * K * 8), *fluz = (double *)dev(nv * (K + 1) * 8);
    double *div = (double *)dev(nv * K * 8), *out_flat = (double *)dev(nv * K * 8);

    /* 1. the flat oracle call on the GPU */
    CK(tsg_transport_indirect(e2v, v2e, signs, dual, pd, vn, wn, rho, nv, ne, K, dt, pivbz, TSG_UPWIND,
                              flux, fluz, div, out_flat, NULL));

    /* 2. the structured fast path */
    tsg_grid *g = NULL;
    CK(tsg_grid_create(rows, cols, K, TSG_PERIODIC_ROWS | TSG_PERIODIC_COLS, &g));
    double *f_pd = (double *)dev(tsg_field_elems(g, TSG_VERTICES, K) * 8);
    double *f_out = (double *)dev(tsg_field_elems(g, TSG_VERTICES, K) * 8);
    double *f_vn = (double *)dev(tsg_field_elems(g, TSG_EDGES, K) * 8);
    double *f_wn = (double *)dev(tsg_field_elems(g, TSG_VERTICES, K + 1) * 8);
    double *f_rho = (double *)dev(tsg_field_elems(g, TSG_VERTICES, K) * 8);
    double *f_signs = (double *)dev(tsg_field_elems(g, TSG_VERTICES, 6) * 8);
    double *f_dual = (double *)dev(tsg_field_elems(g, TSG_VERTICES, 1) * 8);
    CK(tsg_pack(g, TSG_VERTICES, K, pd, NULL, f_pd, NULL));
    CK(tsg_pack(g, TSG_EDGES, K, vn, NULL, f_vn, NULL));
    CK(tsg_pack(g, TSG_VERTICES, K + 1, wn, NULL, f_wn, NULL));
    CK(tsg_pack(g, TSG_VERTICES, K, rho, NULL, f_rho, NULL));
    CK(tsg_pack(g, TSG_VERTICES, 6, signs, NULL, f_signs, NULL));
    CK(tsg_pack(g, TSG_VERTICES, 1, dual, NULL, f_dual, NULL));
    CK(tsg_mpdata_step(g, f_pd, f_vn, f_wn, f_rho, f_signs, f_dual, f_out, dt, pivbz, TSG_UPWIND, NULL));
    double *out_fused = (double *)dev(nv * K * 8);
    CK(tsg_unpack(g, TSG_VERTICES, K, f_out, NULL, out_fused, NULL));
    CU(cudaDeviceSynchronize());
    if (!same(out_flat, out_fused, (size_t)(nv * K))) {
        fprintf(stderr, "structured step differs from the flat step\n");
        return 2;
    }

    /* 3. a 5-step persistent loop against five chained flat steps */
    double *cur = (double *)dev(nv * K * 8), *nxt = (double *)dev(nv * K * 8);
    CU(cudaMemcpy(cur, pd, nv * K * 8, cudaMemcpyDeviceToDevice));
    for (int s = 0; s < 5; ++s) {
        CK(tsg_transport_indirect(e2v, v2e, signs, dual, cur, vn, wn, rho, nv, ne, K, dt, pivbz, TSG_UPWIND,
                                  flux, fluz, div, nxt, NULL));
        double *t = cur;
        cur = nxt;
        nxt = t;
    }
    CK(tsg_pack(g, TSG_VERTICES, K, pd, NULL, f_pd, NULL));
    CK(tsg_mpdata_run(g, f_pd, f_out, f_vn, f_wn, f_rho, f_signs, f_dual, dt, pivbz, TSG_UPWIND, 5, NULL));
    /* after an odd number of steps the newest density is in the second buffer */
    CK(tsg_unpack(g, TSG_VERTICES, K, f_out, NULL, out_fused, NULL));
    CU(cudaDeviceSynchronize());
    if (!same(cur, out_fused, (size_t)(nv * K))) {
        fprintf(stderr, "5-step persistent loop differs from five flat steps\n");
        return 3;
    }
    int werr = 0;
    CK(tsg_fused_wait_error(g, &werr));
    CK(tsg_grid_destroy(g));
    printf("OK %dx%dx%d: flat step == structured step, 5-step loop == 5 flat steps (bitwise)\n", rows, cols, K);
    return werr;
}
