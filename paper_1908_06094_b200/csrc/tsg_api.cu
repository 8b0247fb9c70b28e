// libtsg: error state and grid handle (the device-side PatchSpec, topology.py:44-83).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <new>

#include "tsg_common.cuh"

namespace tsg {

static thread_local char g_err[1024] = "";

int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

void clear_error() { g_err[0] = '\0'; }

constexpr int64_t kPointLimit = (1LL << 32) - (1LL << 24);
static std::atomic<int64_t> g_point_limit{kPointLimit};
int64_t point_limit() { return g_point_limit.load(std::memory_order_relaxed); }

}  // namespace tsg

extern "C" int tsg_set_point_limit(int64_t n) {
    if (n < 0 || n > tsg::kPointLimit) return tsg::fail(TSG_EVALUE, "point limit %lld out of range", (long long)n);
    tsg::g_point_limit.store(n ? n : tsg::kPointLimit, std::memory_order_relaxed);
    return TSG_OK;
}

extern "C" const char *tsg_last_error(void) { return tsg::g_err; }

extern "C" int tsg_abi_version(void) { return TSG_ABI_VERSION; }

extern "C" int64_t tsg_inner_pitch(int inner) { return tsg::pitch_of(inner); }

extern "C" int tsg_grid_create(int rows, int cols, int levels, int flags, tsg_grid **out) {
    if (!out) return tsg::fail(TSG_EVALUE, "tsg_grid_create: out is NULL");
    *out = nullptr;
    // topology.py:58-75
    if (rows < 2 || cols < 2)
        return tsg::fail(TSG_EVALUE, "rows and cols must each be >= 2, got %dx%d", rows, cols);
    if (levels < 1) return tsg::fail(TSG_EVALUE, "levels must be >= 1, got %d", levels);
    if (flags & ~(TSG_PERIODIC_ROWS | TSG_PERIODIC_COLS))
        return tsg::fail(TSG_EVALUE, "unknown grid flags 0x%x", flags);
    int dev = 0;
    TSG_CHECK_CUDA(cudaGetDevice(&dev));
    int sms = 0;
    TSG_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    tsg_grid *g = new (std::nothrow) tsg_grid;
    if (!g) return tsg::fail(TSG_ESTATE, "out of host memory");
    g->rows = rows;
    g->cols = cols;
    g->levels = levels;
    g->flags = flags;
    g->row0 = 0;
    g->global_rows = rows;
    g->device = dev;
    g->num_sms = sms;
    g->graph = nullptr;
    g->launches = nullptr;
    g->dyn_ws = nullptr;
    g->dyn_tiles = 0;
    if (int rc = tsg::create_dyn_workspace(g)) {
        delete g;
        return rc;
    }
    *out = g;
    tsg::clear_error();
    return TSG_OK;
}

extern "C" int tsg_grid_set_origin(tsg_grid *g, int row0, int global_rows) {
    if (!g) return tsg::fail(TSG_EVALUE, "grid is NULL");
    if (row0 < 0 || global_rows < g->rows || row0 + g->rows > global_rows)
        return tsg::fail(TSG_EVALUE, "strip rows [%d, %d) outside a %d-row patch", row0,
                         row0 + g->rows, global_rows);
    g->row0 = row0;
    g->global_rows = global_rows;
    return TSG_OK;
}

extern "C" int tsg_grid_destroy(tsg_grid *g) {
    if (g) {
        tsg::destroy_graph_cache(g);
        tsg::destroy_launch_cache(g);
        tsg::destroy_dyn_workspace(g);
    }
    delete g;
    return TSG_OK;
}

extern "C" int64_t tsg_field_elems(const tsg_grid *g, int loc, int inner) {
    if (!g || !tsg::valid_loc(loc) || inner < 1) return -1;
    return tsg::FieldIx(g->rows, g->cols, tsg::colors_of(loc), inner).elems();
}
