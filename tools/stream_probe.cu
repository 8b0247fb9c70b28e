// Practical HBM ceiling for the fused MPDATA step's byte mix (not part of the product).
//
// Streams exactly the step's algorithmic traffic -- read pd, rho (V*K), wn (V*(K+1)),
// vn (3*V*K), write pd_out (V*K), fp64 -- with ideal coalesced 16-byte accesses and no
// stencil, and times it with CUDA events after a read-only L2 flush, the same protocol
// bench.py uses.  The result is the bandwidth a perfect one-pass kernel of this size
// could reach, next to the copy figure MEASURED_PEAKS.json holds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_probe tools/stream_probe.cu
//   tools/stream_probe [V] [K]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); std::exit(1); } } while (0)

__global__ void step_mix(const double2 *__restrict__ pd, const double2 *__restrict__ rho,
                         const double2 *__restrict__ wn, const double2 *__restrict__ vn,
                         double2 *__restrict__ out, long n2) {
    // n2 = V*K/2 pairs; vn has 3*n2 pairs, wn ~n2 pairs
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n2; q += (long)gridDim.x * blockDim.x) {
        double2 a = pd[q], r = rho[q], w = wn[q];
        double2 v0 = vn[q], v1 = vn[q + n2], v2 = vn[q + 2 * n2];
        out[q] = make_double2(a.x + r.x + w.x + v0.x + v1.x + v2.x, a.y + r.y + w.y + v0.y + v1.y + v2.y);
    }
}

__global__ void copy2(const double2 *__restrict__ a, double2 *__restrict__ b, long n2) {
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n2; q += (long)gridDim.x * blockDim.x)
        b[q] = a[q];
}

__global__ void read_sum(const double2 *__restrict__ a, long n2, double *sink) {
    double s = 0;
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n2; q += (long)gridDim.x * blockDim.x) {
        double2 v = a[q];
        s += v.x + v.y;
    }
    if (s == 12345.678) *sink = s;
}


// The fused kernel's unit order and access granularity with plain loads (no TMA, no halo):
// unit = 4x16 vertex tile x 16-level chunk, a thread owns a level pair.  PITCH layout:
// f[row][col][pitch] (a vertex's levels contiguous, what the product uses); BLOCKED:
// f[chunk][row][col][16] (a tile row's 16-level runs contiguous).
template <bool BLOCKED>
__global__ void tile_pattern(const double *__restrict__ pd, const double *__restrict__ rho,
                             const double *__restrict__ wn, const double *__restrict__ vn,
                             double *__restrict__ out, int H, int W, int K, long units) {
    const int chunks = K / 16, tiles_j = W / 16;
    const long ub = units * blockIdx.x / gridDim.x, ue = units * (blockIdx.x + 1) / gridDim.x;
    const int t = threadIdx.x % 512, vl = t / 8, kq = (t % 8) * 2;
    const long plane = (long)H * W * K;  // one field
    for (long u = ub + threadIdx.x / 512; u < ue; u += blockDim.x / 512) {
        const int chunk = (int)(u % chunks);
        const long tile = u / chunks;
        const int i = (int)(tile / tiles_j) * 4 + vl / 16, j = (int)(tile % tiles_j) * 16 + vl % 16;
        if (i >= H) continue;
        long o = BLOCKED ? (((long)chunk * H + i) * W + j) * 16 + kq : ((long)i * W + j) * K + chunk * 16 + kq;
        const double2 a = *(const double2 *)(pd + o), r = *(const double2 *)(rho + o), w = *(const double2 *)(wn + o);
        const double2 v0 = *(const double2 *)(vn + o), v1 = *(const double2 *)(vn + o + plane),
                      v2 = *(const double2 *)(vn + o + 2 * plane);
        *(double2 *)(out + o) = make_double2(a.x + r.x + w.x + v0.x + v1.x + v2.x, a.y + r.y + w.y + v0.y + v1.y + v2.y);
    }
}

int main(int argc, char **argv) {
    long V = argc > 1 ? atol(argv[1]) : 71424;
    long K = argc > 2 ? atol(argv[2]) : 80;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    long n = V * K, n2 = n / 2;
    double *pd, *rho, *wn, *vn, *out, *flush, *sink;
    CK(cudaMalloc(&pd, n * 8)); CK(cudaMalloc(&rho, n * 8)); CK(cudaMalloc(&wn, (n + V) * 8));
    CK(cudaMalloc(&vn, 3 * n * 8)); CK(cudaMalloc(&out, n * 8));
    long nf = 256L << 20;
    CK(cudaMalloc(&flush, nf)); CK(cudaMalloc(&sink, 8));
    CK(cudaMemset(pd, 0, n * 8)); CK(cudaMemset(rho, 0, n * 8)); CK(cudaMemset(wn, 0, (n + V) * 8));
    CK(cudaMemset(vn, 0, 3 * n * 8)); CK(cudaMemset(flush, 0, nf));
    const double bytes = 8.0 * (6 * n + n);  // 6 reads (pd, rho, wn, 3 vn) + 1 write
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    std::printf("V=%ld K=%ld  algorithmic bytes %.0f  SMs %d\n", V, K, bytes, sms);
    for (int per_sm : {2, 4, 8, 16}) {
        for (int threads : {256, 512, 1024}) {
            if (per_sm * threads > 2048) continue;
            int grid = sms * per_sm;
            std::vector<float> t;
            for (int rep = 0; rep < 60; ++rep) {
                read_sum<<<sms * 4, 512>>>((const double2 *)flush, nf / 16, sink);
                CK(cudaEventRecord(e0));
                step_mix<<<grid, threads>>>((const double2 *)pd, (const double2 *)rho, (const double2 *)wn,
                                            (const double2 *)vn, (double2 *)out, n2);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                if (rep >= 10) t.push_back(ms);
            }
            std::sort(t.begin(), t.end());
            double med = t[t.size() / 2];
            std::printf("step_mix grid %4d x %4d: median %.1f us  %.0f GB/s\n", grid, threads, med * 1e3,
                        bytes / (med * 1e-3) / 1e9);
        }
    }

    // the fused kernel's unit order and access granularity, pitch vs level-blocked layout
    {
        const int W = 256, H = (int)(V / W), Kq = (int)K / 16 * 16;
        const long units = (long)((H + 3) / 4) * (W / 16) * (Kq / 16);
        for (int blocked = 0; blocked < 2; ++blocked)
            for (int threads : {512, 1024}) {
                std::vector<float> t;
                for (int rep = 0; rep < 60; ++rep) {
                    read_sum<<<sms * 4, 512>>>((const double2 *)flush, nf / 16, sink);
                    CK(cudaEventRecord(e0));
                    if (blocked) tile_pattern<true><<<sms * (2048 / threads), threads>>>(pd, rho, wn, vn, out, H, W, Kq, units);
                    else tile_pattern<false><<<sms * (2048 / threads), threads>>>(pd, rho, wn, vn, out, H, W, Kq, units);
                    CK(cudaEventRecord(e1));
                    CK(cudaEventSynchronize(e1));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, e0, e1));
                    if (rep >= 10) t.push_back(ms);
                }
                std::sort(t.begin(), t.end());
                double med = t[t.size() / 2];
                const double b = 8.0 * 7 * (double)H * W * Kq;
                std::printf("tile_pattern %s x %4d: median %.1f us  %.0f GB/s\n", blocked ? "blocked" : "pitch  ",
                            threads, med * 1e3, b / (med * 1e-3) / 1e9);
            }
    }
    // the copy the peaks file uses, at this size and at 1 GiB
    for (long cb : {(long)(bytes / 2), 1L << 30}) {
        double *a, *b;
        CK(cudaMalloc(&a, cb)); CK(cudaMalloc(&b, cb)); CK(cudaMemset(a, 0, cb));
        std::vector<float> t;
        for (int rep = 0; rep < 40; ++rep) {
            read_sum<<<sms * 4, 512>>>((const double2 *)flush, nf / 16, sink);
            CK(cudaEventRecord(e0));
            copy2<<<sms * 4, 512>>>((const double2 *)a, (double2 *)b, cb / 16);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (rep >= 5) t.push_back(ms);
        }
        std::sort(t.begin(), t.end());
        double med = t[t.size() / 2];
        std::printf("copy %ld MB each way: median %.1f us  %.0f GB/s (read+write)\n", cb >> 20, med * 1e3,
                    2.0 * cb / (med * 1e-3) / 1e9);
        CK(cudaFree(a)); CK(cudaFree(b));
    }
    return 0;
}
