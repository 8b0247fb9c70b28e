// Cross-GPU plumbing for the fused halo exchange of the row-strip decomposition.
//
// One process per GPU.  Each rank exports its two density buffers with CUDA IPC; its ring
// neighbours map them (NVLink peer mappings on an NVSwitch box) and the step kernel's
// epilogue stores boundary rows straight into the neighbour's halo row
// (tsg_mpdata_step_rows_peer).  A per-step fence orders the exchange: after its boundary
// rows a rank releases a step counter into both neighbours' flag words; before the next
// step's boundary rows it acquires its own two flag words.
#include <string.h>

#include "tsg_common.cuh"

namespace tsg {

__global__ void signal_kernel(int64_t *flag_up, int64_t *flag_down, int64_t value) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    __threadfence_system();  // the step's peer stores are visible before the flag
    if (flag_up) asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(flag_up), "l"(value) : "memory");
    if (flag_down) asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(flag_down), "l"(value) : "memory");
}

__device__ __forceinline__ int64_t load_acquire(const int64_t *p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void wait_kernel(const int64_t *flags, int64_t value, uint64_t timeout_ns, int *err) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const uint64_t t0 = global_ns();
    unsigned backoff = 32;
    while (load_acquire(flags) < value || load_acquire(flags + 1) < value) {
        if (global_ns() - t0 > timeout_ns) {
            if (err) atomicExch(err, 1);
            return;
        }
        __nanosleep(backoff);
        if (backoff < 4096) backoff *= 2;
    }
}

}  // namespace tsg

using namespace tsg;

extern "C" int tsg_malloc(int64_t bytes, void **out) {
    if (!out || bytes < 0) return fail(TSG_EVALUE, "tsg_malloc: bad arguments");
    *out = nullptr;
    TSG_CHECK_CUDA(cudaMalloc(out, bytes > 0 ? (size_t)bytes : 16));
    TSG_CHECK_CUDA(cudaMemset(*out, 0, bytes > 0 ? (size_t)bytes : 16));
    return TSG_OK;
}

extern "C" int tsg_free(void *ptr) {
    if (ptr) TSG_CHECK_CUDA(cudaFree(ptr));
    return TSG_OK;
}

extern "C" int tsg_ipc_handle(void *ptr, unsigned char *handle64) {
    if (!ptr || !handle64) return fail(TSG_EVALUE, "tsg_ipc_handle: NULL argument");
    cudaIpcMemHandle_t h;
    TSG_CHECK_CUDA(cudaIpcGetMemHandle(&h, ptr));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    memcpy(handle64, &h, 64);
    return TSG_OK;
}

extern "C" int tsg_ipc_open(const unsigned char *handle64, void **out) {
    if (!handle64 || !out) return fail(TSG_EVALUE, "tsg_ipc_open: NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    TSG_CHECK_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
    return TSG_OK;
}

extern "C" int tsg_ipc_close(void *ptr) {
    if (ptr) TSG_CHECK_CUDA(cudaIpcCloseMemHandle(ptr));
    return TSG_OK;
}

extern "C" int tsg_signal_peers(int64_t *flag_up, int64_t *flag_down, int64_t value, tsg_stream s) {
    signal_kernel<<<1, 32, 0, (cudaStream_t)s>>>(flag_up, flag_down, value);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}

extern "C" int tsg_wait_flags(const int64_t *my_flags, int64_t value, int timeout_ms, int *error_word,
                              tsg_stream s) {
    if (!my_flags) return fail(TSG_EVALUE, "tsg_wait_flags: NULL flags");
    if (timeout_ms <= 0) return fail(TSG_EVALUE, "timeout must be positive");
    wait_kernel<<<1, 32, 0, (cudaStream_t)s>>>(my_flags, value, (uint64_t)timeout_ms * 1000000ULL,
                                                error_word);
    TSG_CHECK_LAUNCH();
    return TSG_OK;
}
