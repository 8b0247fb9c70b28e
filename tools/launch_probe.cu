// Fixed per-launch cost of a persistent one-CTA-per-SM kernel (not part of the product).
//
// Times, with CUDA events after an L2 flush (the bench protocol), an EMPTY kernel launched
// like the fused step (148 x 544 threads, 202,112 B dynamic shared memory) and variants:
// no dynamic shared memory, back to back without a flush in between, and after a flush
// kernel whose shared-memory carveout already matches.  The difference between the fused
// kernel's CTA span (tsg_debug_trace) and its event time is this fixed cost.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_probe tools/launch_probe.cu
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); std::exit(1); } } while (0)

__global__ void empty_kernel(int *sink) {
    extern __shared__ int s[];
    if (threadIdx.x == 100000) sink[0] = s[0];
}

__global__ void flush_kernel(const double2 *__restrict__ a, long n2, double *sink) {
    double s = 0;
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n2; q += (long)gridDim.x * blockDim.x) {
        double2 v = a[q];
        s += v.x + v.y;
    }
    if (s == 12345.678) *sink = s;
}

__global__ void flush_kernel_carve(const double2 *__restrict__ a, long n2, double *sink) {
    double s = 0;
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n2; q += (long)gridDim.x * blockDim.x) {
        double2 v = a[q];
        s += v.x + v.y;
    }
    if (s == 12345.678) *sink = s;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const long n2 = 256L * 1024 * 1024 / 16;
    double2 *buf;
    double *dsink;
    int *isink;
    CK(cudaMalloc(&buf, n2 * 16));
    CK(cudaMemset(buf, 0, n2 * 16));
    CK(cudaMalloc(&dsink, 8));
    CK(cudaMalloc(&isink, 4));
    const int smem = 202112;
    CK(cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(flush_kernel_carve, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto run = [&](const char *name, int flush, int dsmem, int threads, int grid = 0, int reps = 1) {
        std::vector<float> t;
        if (!grid) grid = sms;
        for (int r = 0; r < 60; ++r) {
            if (flush == 1) flush_kernel<<<sms * 4, 512>>>(buf, n2, dsink);
            if (flush == 2) flush_kernel_carve<<<sms * 4, 512>>>(buf, n2, dsink);
            if (flush == 3) empty_kernel<<<grid, threads, dsmem>>>(isink);
            CK(cudaEventRecord(e0));
            for (int q = 0; q < reps; ++q) empty_kernel<<<grid, threads, dsmem>>>(isink);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (r >= 10) t.push_back(ms * 1e3f);
        }
        std::sort(t.begin(), t.end());
        std::printf("%-64s median %6.2f us  min %6.2f  max %6.2f\n", name, t[t.size() / 2], t[0], t.back());
    };
    run("empty, 544 thr, 202112 B smem, after flush", 1, smem, 544);
    run("empty, 544 thr, 0 B smem, after flush", 1, 0, 544);
    run("empty, 544 thr, 202112 B smem, after carveout-100 flush", 2, smem, 544);
    run("empty, 544 thr, 202112 B smem, after the same empty kernel", 3, smem, 544);
    run("empty, 544 thr, 202112 B smem, idle stream", 0, smem, 544);
    run("empty, 544 thr, 0 B smem, idle stream", 0, 0, 544);
    run("empty, 1 CTA x 32 thr, after flush", 1, 0, 32, 1);
    run("empty, 1 CTA x 32 thr, idle stream", 0, 0, 32, 1);
    run("2 x empty, 544 thr, 202112 B smem, after flush", 1, smem, 544, 0, 2);
    run("10 x empty, 544 thr, 202112 B smem, after flush", 1, smem, 544, 0, 10);
    run("10 x empty, 1 CTA x 32 thr, after flush", 1, 0, 32, 1, 10);
    {  // the events' own cost: nothing between them
        std::vector<float> t;
        for (int r = 0; r < 60; ++r) {
            flush_kernel<<<sms * 4, 512>>>(buf, n2, dsink);
            CK(cudaEventRecord(e0));
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (r >= 10) t.push_back(ms * 1e3f);
        }
        std::sort(t.begin(), t.end());
        std::printf("%-64s median %6.2f us  min %6.2f  max %6.2f\n", "no kernel between the events, after flush", t[t.size() / 2], t[0], t.back());
    }
    return 0;
}
